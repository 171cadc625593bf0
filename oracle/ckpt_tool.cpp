// ckpt_tool.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never measured).
//
// Writes a small WSVD checkpoint directory with the REFERENCE's own writer
// (wsvd::ckpt::save, src/checkpoint.cpp:168-247), linked from the unmodified
// reference sources by oracle/Makefile.  The fixture it produces
// (tests/golden/ckpt_e64/, committed) pins our checkpoint reader
// (paper_2604_02570_b200/csrc/checkpoint.cpp) on machines without the
// reference tree.
//
//   ckpt_tool <out_dir> [weight_bits=8]
//   ckpt_tool dump <dir> <layer> <head> <role q|k|v>   (ckpt::load, then prints
//       rank, the fp64 factors and the quantised factors of that head as text:
//       the cross-check of our reader against the reference's loader)
//
// Contents follow the reference pipeline's artefacts: dense toy-model weights
// (toy::init_weights, toymodel.cpp:75-95), per-head truncated SVD factors
// with ragged ranks (factorize::per_head_svd, factorize.cpp:37-49), and
// quantised factors in the QAT export format (quant.cpp:344-358):
// Q(S1 . A . S2^T), Q(S2 . B) with S1 = hadamard(E) and S2 = cayley(theta),
// per-column clip-grid scales (quant::quantize_weight).  (QAT itself only
// changes the values, not the format.)
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "wsvd/checkpoint.hpp"
#include "wsvd/factorize.hpp"
#include "wsvd/linalg.hpp"
#include "wsvd/quant.hpp"
#include "wsvd/rng.hpp"
#include "wsvd/toymodel.hpp"

using namespace wsvd;

static int dump(int argc, char** argv) {
    if (argc < 6) return 2;
    const ckpt::Checkpoint c = ckpt::load(argv[2]);
    const std::size_t li = std::strtoul(argv[3], nullptr, 10), h = std::strtoul(argv[4], nullptr, 10);
    const char role = argv[5][0];
    const decode::HeadProjection& hp = c.factors.at(li).heads.at(h);
    const ckpt::HeadQuant& hq = c.quantized.at(li).heads.at(h);
    const factorize::HeadFactors& f = role == 'q' ? hp.q : role == 'k' ? hp.k : hp.v;
    const quant::QuantizedFactors& q = role == 'q' ? hq.q : role == 'k' ? hq.k : hq.v;
    std::printf("rank %zu bits %d\n", f.rank, c.weight_bits);
    auto mat = [](const char* tag, const Matrix& m) {
        std::printf("%s %zu %zu", tag, m.rows(), m.cols());
        for (std::size_t i = 0; i < m.rows(); ++i)
            for (std::size_t j = 0; j < m.cols(); ++j) std::printf(" %.17g", m(i, j));
        std::printf("\n");
    };
    auto imat = [](const char* tag, const quant::WeightQuant& w) {
        std::printf("%s %zu %zu", tag, w.q.rows, w.q.cols);
        for (std::size_t i = 0; i < w.q.rows * w.q.cols; ++i) std::printf(" %d", static_cast<int>(w.q.data[i]));
        std::printf("\n%s_scales %zu", tag, w.scales.size());
        for (double v : w.scales) std::printf(" %.17g", v);
        std::printf("\n");
    };
    mat("a", f.a);
    mat("b", f.b);
    imat("qa", q.a);
    imat("qb", q.b);
    mat("w_o", c.dense.layers.at(li).w_o);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "dump") {
        try {
            return dump(argc, argv);
        } catch (const std::exception& e) {
            std::fprintf(stderr, "ckpt_tool: %s\n", e.what());
            return 1;
        }
    }
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <out_dir> [weight_bits]\n", argv[0]);
        return 2;
    }
    const int bits = argc > 2 ? std::atoi(argv[2]) : 8;
    try {
        toy::ModelConfig cfg;
        cfg.embed_dim = 64;
        cfg.head_dim = 16;
        cfg.n_heads = 4;
        cfg.n_layers = 2;
        cfg.seed = 11;
        cfg.validate();
        ckpt::Checkpoint c;
        c.stage = ckpt::Stage::Quantized;
        c.config = cfg;
        c.dense = toy::init_weights(cfg);
        c.weight_bits = bits;
        c.activation_bits = 8;
        const Matrix s1 = hadamard(cfg.embed_dim);
        Rng rng = Rng::stream(cfg.seed, 77);
        const std::size_t ranks[4][3] = {{8, 6, 5}, {3, 8, 7}, {4, 4, 4}, {8, 2, 6}};
        for (std::size_t li = 0; li < cfg.n_layers; ++li) {
            decode::LayerFactors lf;
            lf.embed_dim = cfg.embed_dim;
            lf.head_dim = cfg.head_dim;
            ckpt::LayerQuant lq;
            const toy::LayerWeights& w = c.dense.layers[li];
            for (std::size_t h = 0; h < cfg.n_heads; ++h) {
                decode::HeadProjection hp;
                ckpt::HeadQuant hq;
                const factorize::Role roles[3] = {factorize::Role::Q, factorize::Role::K, factorize::Role::V};
                const Matrix* full[3] = {&w.w_q, &w.w_k, &w.w_v};
                for (int role = 0; role < 3; ++role) {
                    const std::size_t r = ranks[h][role];
                    factorize::HeadFactors f =
                        factorize::per_head_svd(*full[role], li, roles[role], h, cfg.head_dim, r);
                    // a seeded latent rotation S2 = cayley(theta), theta skew
                    Matrix theta(r, r);
                    for (std::size_t i = 0; i < r; ++i)
                        for (std::size_t j = i + 1; j < r; ++j) {
                            const double v = 0.3 * rng.normal();
                            theta(i, j) = v;
                            theta(j, i) = -v;
                        }
                    const Matrix s2 = cayley(SkewParam(theta));
                    quant::RotationPair rp{s1, s2};
                    const factorize::HeadFactors rf = quant::insert_rotations(f, rp);
                    quant::QuantSpec spec;
                    spec.weight_bits = bits;
                    quant::QuantizedFactors qf;
                    qf.a = quant::quantize_weight(rf.a, spec);
                    qf.b = quant::quantize_weight(rf.b, spec);
                    qf.s2_skew = theta;
                    qf.rank = r;
                    qf.layer = li;
                    qf.head = h;
                    qf.role = roles[role];
                    qf.weight_bits = bits;
                    if (role == 0) {
                        hp.q = f;
                        hq.q = qf;
                    } else if (role == 1) {
                        hp.k = f;
                        hq.k = qf;
                    } else {
                        hp.v = f;
                        hq.v = qf;
                    }
                }
                lf.heads.push_back(std::move(hp));
                lq.heads.push_back(std::move(hq));
            }
            c.factors.push_back(std::move(lf));
            c.quantized.push_back(std::move(lq));
        }
        ckpt::save(argv[1], c);
        std::printf("wrote %s (E=%zu H=%zu heads=%zu layers=%zu, W%d)\n", argv[1], cfg.embed_dim, cfg.head_dim,
                    cfg.n_heads, cfg.n_layers, bits);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ckpt_tool: %s\n", e.what());
        return 1;
    }
}
