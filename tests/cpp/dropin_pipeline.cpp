// dropin_pipeline.cpp -- one driver, built twice by oracle/Makefile (target
// dropin): against the reference's own decode.hpp + decode.cpp
// (pipeline_ref, CPU fp64) and against this repo's drop-in decode.hpp +
// host_decode.cpp + libwsvd_b200.so (pipeline_gpu, B200).  Every other object
// -- matrix, rng, factorize, toymodel, pipeline, ... -- is the reference's,
// compiled from /root/reference/proj/src unmodified.  tests/test_gpu_dropin.py
// runs both and compares the records: traffic tallies exactly, values within
// the fp32-storage tolerance.
//
// Records (text, hex floats): "name rows cols" then rows*cols values.
//   c3/<seed>/tile<t>   acceptance criterion 3 (tests/acceptance_main.cpp:212-240):
//                       fused_decode_step over a random ragged-rank layer, every tiling
//   c3/<seed>/counter   its TrafficCounter (21 tallies)
//   full/<seed>/...     the full-rank part (acceptance_main.cpp:242-274):
//                       per_head_svd factors vs append_token_dense + flash / eager
//   shared/...          append_token_shared + shared_decode_step (both schedules)
//   factored/...        pipe::decode_factored over a 2-layer toy model (pipeline.cpp:304-339)
//   dense/...           pipe::decode_dense on the same model (pipeline.cpp:341-375)
#include <array>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "wsvd/decode.hpp"
#include "wsvd/errors.hpp"
#include "wsvd/factorize.hpp"
#include "wsvd/matrix.hpp"
#include "wsvd/pipeline.hpp"
#include "wsvd/rng.hpp"
#include "wsvd/toymodel.hpp"

using namespace wsvd;

namespace {

FILE* g_out = nullptr;

void record(const std::string& name, const Matrix& m) {
    std::fprintf(g_out, "%s %zu %zu\n", name.c_str(), m.rows(), m.cols());
    for (double v : m.data()) std::fprintf(g_out, "%a\n", v);
}

void record(const std::string& name, const decode::TrafficCounter& c) {
    Matrix m(3, decode::kStreamCount);
    for (std::size_t s = 0; s < decode::kStreamCount; ++s) {
        const decode::StreamTally& t = c[static_cast<decode::Stream>(s)];
        m(0, s) = static_cast<double>(t.loads);
        m(1, s) = static_cast<double>(t.stores);
        m(2, s) = static_cast<double>(t.flops);
    }
    record(name, m);
}

factorize::HeadFactors random_head(Rng& rng, std::size_t E, std::size_t H, std::size_t r, std::size_t head,
                                   factorize::Role role) {
    factorize::HeadFactors hf;
    hf.a = rng.normal_matrix(E, r, 1.0 / std::sqrt(static_cast<double>(E)));
    hf.b = rng.normal_matrix(r, H, 1.0 / std::sqrt(static_cast<double>(r)));
    hf.rank = r;
    hf.head = head;
    hf.role = role;
    return hf;
}

// acceptance criterion 3, first half: ragged ranks, every tiling
void criterion3(std::uint64_t seed) {
    Rng rng(2000 + seed);
    const std::size_t E = std::size_t{16} << (seed % 3), nh = seed % 2 == 0 ? 2 : 4, H = E / nh;
    const std::size_t len = 5 + (seed * 7) % 36;
    decode::LayerFactors f;
    f.embed_dim = E;
    f.head_dim = H;
    for (std::size_t h = 0; h < nh; ++h) {
        const std::size_t rq = 1 + rng.index(H), rk = 1 + rng.index(H), rv = 1 + rng.index(H);
        decode::HeadProjection p;
        p.q = random_head(rng, E, H, rq, h, factorize::Role::Q);
        p.k = random_head(rng, E, H, rk, h, factorize::Role::K);
        p.v = random_head(rng, E, H, rv, h, factorize::Role::V);
        f.heads.push_back(std::move(p));
    }
    decode::LatentCache cache(f);
    Matrix q(0, 0);
    decode::TrafficCounter ca;
    for (std::size_t t = 0; t < len; ++t) {
        const Matrix x = rng.normal_matrix(1, E);
        q = decode::append_token(cache, f, x.row(0), &ca);
    }
    const std::string tag = "c3/" + std::to_string(seed);
    record(tag + "/append_counter", ca);
    record(tag + "/q", q);
    for (std::size_t h = 0; h < nh; ++h) record(tag + "/latent_k" + std::to_string(h), cache.latent_k(h));
    for (std::size_t tile : {std::size_t{1}, std::size_t{7}, std::size_t{16}, len}) {
        decode::TrafficCounter c;
        const Matrix out = decode::fused_decode_step(cache, f, q, decode::TileConfig{tile}, c);
        record(tag + "/tile" + std::to_string(tile), out);
        if (tile == 7) record(tag + "/counter", c);
    }
}

// acceptance criterion 3, second half: full-rank factors vs the dense cache
void full_rank(std::uint64_t seed) {
    Rng rng(2100 + seed);
    const std::size_t E = 32, H = 8, nh = 4, len = 19;
    decode::DenseProjections dense;
    const double s = 1.0 / std::sqrt(static_cast<double>(E));
    dense.w_q = rng.normal_matrix(E, E, s);
    dense.w_k = rng.normal_matrix(E, E, s);
    dense.w_v = rng.normal_matrix(E, E, s);
    dense.head_dim = H;
    decode::LayerFactors f;
    f.embed_dim = E;
    f.head_dim = H;
    for (std::size_t h = 0; h < nh; ++h) {
        decode::HeadProjection p;
        p.q = factorize::per_head_svd(dense.w_q, 0, factorize::Role::Q, h, H, H);
        p.k = factorize::per_head_svd(dense.w_k, 0, factorize::Role::K, h, H, H);
        p.v = factorize::per_head_svd(dense.w_v, 0, factorize::Role::V, h, H, H);
        f.heads.push_back(std::move(p));
    }
    decode::LatentCache latent(f);
    decode::FullKvCache full(nh, H);
    Matrix qf(0, 0), qd(0, 0);
    decode::TrafficCounter cdense;
    for (std::size_t t = 0; t < len; ++t) {
        const Matrix x = rng.normal_matrix(1, E);
        qf = decode::append_token(latent, f, x.row(0));
        qd = decode::append_token_dense(full, dense, x.row(0), &cdense);
    }
    const std::string tag = "full/" + std::to_string(seed);
    decode::TrafficCounter cf, cfl, ce;
    record(tag + "/fused", decode::fused_decode_step(latent, f, qf, decode::TileConfig{8}, cf));
    record(tag + "/flash", decode::flash_decode_step(full, qd, decode::TileConfig{8}, cfl));
    record(tag + "/eager", decode::eager_decode_step(full, qd, ce));
    record(tag + "/keys0", full.keys(0));
    record(tag + "/append_dense_counter", cdense);
    record(tag + "/flash_counter", cfl);
    record(tag + "/eager_counter", ce);
}

void shared_latent() {
    Rng rng(77);
    const std::size_t E = 32, H = 8, nh = 4, R = 12, len = 23;
    decode::SharedFactors f;
    f.a_k = rng.normal_matrix(E, R, 0.2);
    f.a_v = rng.normal_matrix(E, R, 0.2);
    f.b_k = rng.normal_matrix(R, E, 0.3);
    f.b_v = rng.normal_matrix(R, E, 0.3);
    f.head_dim = H;
    f.n_heads = nh;
    decode::SharedLatentCache cache{Matrix(0, R), Matrix(0, R)};
    decode::TrafficCounter ca;
    for (std::size_t t = 0; t < len; ++t) {
        const Matrix x = rng.normal_matrix(1, E);
        decode::append_token_shared(cache, f, x.row(0), &ca);
    }
    const Matrix q = rng.normal_matrix(nh, H);
    decode::TrafficCounter cs, cm;
    record("shared/c_k", cache.c_k);
    record("shared/streamed", decode::shared_decode_step(cache, f, q, decode::TileConfig{5}, cs, false));
    record("shared/materialized", decode::shared_decode_step(cache, f, q, decode::TileConfig{5}, cm, true));
    record("shared/append_counter", ca);
    record("shared/streamed_counter", cs);
    record("shared/materialized_counter", cm);
}

// pipe::decode_factored / decode_dense over a small toy model (2 layers,
// ragged per-head ranks from truncated SVDs of the trained-shape weights)
void pipeline_decode() {
    toy::ModelConfig cfg;
    cfg.embed_dim = 64;
    cfg.head_dim = 16;
    cfg.n_heads = 4;
    cfg.n_layers = 2;
    cfg.seed = 5;
    cfg.validate();
    const toy::AttentionWeights w = toy::init_weights(cfg);
    std::vector<decode::LayerFactors> factors;
    for (std::size_t l = 0; l < cfg.n_layers; ++l) {
        decode::LayerFactors lf;
        lf.embed_dim = cfg.embed_dim;
        lf.head_dim = cfg.head_dim;
        for (std::size_t h = 0; h < cfg.n_heads; ++h) {
            decode::HeadProjection p;
            const std::size_t r = 6 + 2 * ((h + l) % 4);  // 6..12, ragged
            p.q = factorize::per_head_svd(w.layers[l].w_q, l, factorize::Role::Q, h, cfg.head_dim, r);
            p.k = factorize::per_head_svd(w.layers[l].w_k, l, factorize::Role::K, h, cfg.head_dim, r + 2);
            p.v = factorize::per_head_svd(w.layers[l].w_v, l, factorize::Role::V, h, cfg.head_dim, r);
            lf.heads.push_back(std::move(p));
        }
        factors.push_back(std::move(lf));
    }
    Rng rng(99);
    const Matrix x = rng.normal_matrix(7, cfg.embed_dim);
    decode::TrafficCounter cf, cd;
    record("factored/out", pipe::decode_factored(cfg, w, factors, x, decode::TileConfig{8}, cf));
    record("factored/counter", cf);
    record("dense/out", pipe::decode_dense(cfg, w, x, decode::TileConfig{8}, cd));
    record("dense/counter", cd);
}

// the reference's error classes reach the caller from both implementations
void errors() {
    Matrix flags(1, 4);
    decode::LayerFactors f;
    f.embed_dim = 8;
    f.head_dim = 4;
    Rng rng(1);
    decode::HeadProjection p;
    p.q = random_head(rng, 8, 4, 2, 0, factorize::Role::Q);
    p.k = random_head(rng, 8, 4, 2, 0, factorize::Role::K);
    p.v = random_head(rng, 8, 4, 2, 0, factorize::Role::V);
    f.heads.push_back(p);
    decode::LatentCache cache(f);
    decode::TrafficCounter c;
    try {
        decode::fused_decode_step(cache, f, Matrix(1, 4), decode::TileConfig{4}, c);
    } catch (const ShapeError&) {
        flags(0, 0) = 1;  // empty cache
    }
    const Matrix x = rng.normal_matrix(1, 8);
    const Matrix q = decode::append_token(cache, f, x.row(0));
    try {
        decode::fused_decode_step(cache, f, q, decode::TileConfig{0}, c);
    } catch (const ConfigError&) {
        flags(0, 1) = 1;  // tile 0
    }
    try {
        decode::fused_decode_step(cache, f, Matrix(2, 4), decode::TileConfig{4}, c);
    } catch (const ShapeError&) {
        flags(0, 2) = 1;  // query shape
    }
    try {
        decode::append_token(cache, f, std::vector<double>(5, 0.0));
    } catch (const ShapeError&) {
        flags(0, 3) = 1;  // token width
    }
    record("errors/flags", flags);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s OUT_FILE\n", argv[0]);
        return 2;
    }
    g_out = std::fopen(argv[1], "w");
    if (!g_out) return 2;
    try {
        for (std::uint64_t seed = 0; seed < 32; ++seed) criterion3(seed);
        for (std::uint64_t seed = 0; seed < 8; ++seed) full_rank(seed);
        shared_latent();
        pipeline_decode();
        errors();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        std::fclose(g_out);
        return 1;
    }
    std::fclose(g_out);
    std::printf("ok\n");
    return 0;
}
