// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" harness around the UNMODIFIED reference library
// (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libwsvdref.so).  It lets the Python tests and bench.py's
// reference arm drive the reference's own wsvd::decode / wsvd::quant / Rng
// objects on padded arrays.  Nothing here re-implements reference logic; it
// only marshals arrays into reference types and calls the reference API:
//   decode::append_token        src/decode.cpp:127-153
//   decode::fused_decode_step   src/decode.cpp:155-206
//   quant::quantize_weight      src/quant.cpp:99-119
//   quant::quantize_activation  src/quant.cpp:131-150
//   linalg::hadamard            src/linalg.cpp:219-243
//   Rng                         src/rng.cpp
//   parallel_for                include/wsvd/parallel.hpp:17-47
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "wsvd/decode.hpp"
#include "wsvd/errors.hpp"
#include "wsvd/linalg.hpp"
#include "wsvd/matrix.hpp"
#include "wsvd/parallel.hpp"
#include "wsvd/quant.hpp"
#include "wsvd/rng.hpp"

using namespace wsvd;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ShapeError*>(&e)) return -1;
    if (dynamic_cast<const ConfigError*>(&e)) return -2;
    if (dynamic_cast<const NumericError*>(&e)) return -3;
    return -9;
}

// padded layout (see oracle/wsvd_oracle.h): A[h][role][E][rmax], B[h][role][rmax][H]
decode::LayerFactors make_layer(std::size_t E, std::size_t H, std::size_t nh, std::size_t rmax,
                                const int32_t* ranks, const double* A, const double* B) {
    decode::LayerFactors f;
    f.embed_dim = E;
    f.head_dim = H;
    for (std::size_t h = 0; h < nh; ++h) {
        decode::HeadProjection p;
        factorize::HeadFactors* roles[3] = {&p.q, &p.k, &p.v};
        const factorize::Role rr[3] = {factorize::Role::Q, factorize::Role::K, factorize::Role::V};
        for (int role = 0; role < 3; ++role) {
            const std::size_t r = static_cast<std::size_t>(ranks[h * 3 + role]);
            const double* a = A + (h * 3 + role) * E * rmax;
            const double* b = B + (h * 3 + role) * rmax * H;
            factorize::HeadFactors& hf = *roles[role];
            hf.a = Matrix(E, r);
            for (std::size_t i = 0; i < E; ++i)
                for (std::size_t j = 0; j < r; ++j) hf.a(i, j) = a[i * rmax + j];
            hf.b = Matrix(r, H);
            for (std::size_t i = 0; i < r; ++i)
                for (std::size_t j = 0; j < H; ++j) hf.b(i, j) = b[i * H + j];
            hf.rank = r;
            hf.head = h;
            hf.role = rr[role];
        }
        f.heads.push_back(std::move(p));
    }
    return f;
}

void export_counter(const decode::TrafficCounter& c, uint64_t* out21) {
    if (!out21) return;
    for (std::size_t s = 0; s < decode::kStreamCount; ++s) {
        const auto& t = c[static_cast<decode::Stream>(s)];
        out21[s] = t.loads;
        out21[7 + s] = t.stores;
        out21[14 + s] = t.flops;
    }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Appends `n_tok` tokens (tokens [n_tok][E]) through decode::append_token,
// returns the padded caches ck/cv [nh][n_tok][rmax] and the q block of the
// last token, then runs decode::fused_decode_step with that q.
int ref_append_then_decode(std::size_t E, std::size_t H, std::size_t nh, std::size_t rmax,
                           const int32_t* ranks, const double* A, const double* B,
                           std::size_t n_tok, const double* tokens, std::size_t tile,
                           double* ck, double* cv, double* q_last, double* out,
                           uint64_t* append_counter21, uint64_t* decode_counter21) {
    try {
        const decode::LayerFactors f = make_layer(E, H, nh, rmax, ranks, A, B);
        decode::LatentCache cache(f);
        decode::TrafficCounter ac;
        Matrix q(0, 0);
        for (std::size_t t = 0; t < n_tok; ++t) {
            q = decode::append_token(cache, f, std::span<const double>(tokens + t * E, E), &ac);
        }
        export_counter(ac, append_counter21);
        for (std::size_t h = 0; h < nh; ++h) {
            const Matrix& k = cache.latent_k(h);
            const Matrix& v = cache.latent_v(h);
            for (std::size_t t = 0; t < n_tok; ++t)
                for (std::size_t j = 0; j < rmax; ++j) {
                    ck[(h * n_tok + t) * rmax + j] = j < k.cols() ? k(t, j) : 0.0;
                    cv[(h * n_tok + t) * rmax + j] = j < v.cols() ? v(t, j) : 0.0;
                }
        }
        if (q_last && q.rows()) std::memcpy(q_last, q.data().data(), nh * H * sizeof(double));
        decode::TrafficCounter dc;
        Matrix o = decode::fused_decode_step(cache, f, q, decode::TileConfig{tile}, dc);
        std::memcpy(out, o.data().data(), nh * H * sizeof(double));
        export_counter(dc, decode_counter21);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// fused_decode_step over caller-provided latents ck/cv [nh][len][rmax]
// (pushed through LatentCache::push) and q [nh][H].
int ref_fused_decode(std::size_t E, std::size_t H, std::size_t nh, std::size_t rmax,
                     const int32_t* ranks, const double* A, const double* B, std::size_t len,
                     const double* ck, const double* cv, const double* q, std::size_t tile,
                     double* out, uint64_t* counter21) {
    try {
        const decode::LayerFactors f = make_layer(E, H, nh, rmax, ranks, A, B);
        decode::LatentCache cache(f);
        for (std::size_t t = 0; t < len; ++t) {
            for (std::size_t h = 0; h < nh; ++h) {
                const std::size_t rk = f.heads[h].k.rank, rv = f.heads[h].v.rank;
                cache.push(h, std::span<const double>(ck + (h * len + t) * rmax, rk),
                           std::span<const double>(cv + (h * len + t) * rmax, rv));
            }
            cache.bump_length();
        }
        Matrix qm(nh, H);
        std::memcpy(qm.data().data(), q, nh * H * sizeof(double));
        decode::TrafficCounter c;
        Matrix o = decode::fused_decode_step(cache, f, qm, decode::TileConfig{tile}, c);
        std::memcpy(out, o.data().data(), nh * H * sizeof(double));
        export_counter(c, counter21);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_traffic_match_fused(const uint64_t* counter21, uint64_t seq_len, uint64_t n_heads,
                            uint64_t head_dim, uint64_t rank_k) {
    try {
        decode::TrafficCounter c;
        for (std::size_t s = 0; s < decode::kStreamCount; ++s) {
            const auto st = static_cast<decode::Stream>(s);
            c.add_loads(st, counter21[s]);
            c.add_stores(st, counter21[7 + s]);
            c.add_flops(st, counter21[14 + s]);
        }
        return decode::traffic_report(decode::Mode::Fused, c, seq_len, n_heads, head_dim, rank_k,
                                      0)
                       .match
                   ? 1
                   : 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_rng_normals(uint64_t seed, uint64_t stream, int use_stream, std::size_t n,
                     double stddev, double* out) {
    Rng rng = use_stream ? Rng::stream(seed, stream) : Rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = stddev * rng.normal();
}

void ref_rng_u64s(uint64_t seed, std::size_t n, uint64_t* out) {
    Rng rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

void ref_rng_indices(uint64_t seed, uint64_t bound, std::size_t n, uint64_t* out) {
    Rng rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.index(bound);
}

double ref_quantize_weight(const double* w, std::size_t rows, std::size_t cols, int bits,
                           int8_t* q, double* scales) {
    try {
        Matrix m(rows, cols, std::vector<double>(w, w + rows * cols));
        quant::QuantSpec spec;
        spec.weight_bits = bits;
        quant::WeightQuant wq = quant::quantize_weight(m, spec);
        std::memcpy(q, wq.q.data.data(), rows * cols);
        std::memcpy(scales, wq.scales.data(), cols * sizeof(double));
        return wq.clip;
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

int ref_quantize_activation(const double* x, std::size_t rows, std::size_t cols, int bits,
                            int8_t* q, double* scales) {
    try {
        Matrix m(rows, cols, std::vector<double>(x, x + rows * cols));
        quant::ActivationQuant aq = quant::quantize_activation(m, bits);
        std::memcpy(q, aq.q.data.data(), rows * cols);
        std::memcpy(scales, aq.scales.data(), rows * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_hadamard(std::size_t dim, double* out) {
    try {
        Matrix h = hadamard(dim);
        std::memcpy(out, h.data().data(), dim * dim * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------------------
// CPU baseline (bench.py --impl reference / cpu_baseline kind "reference").
// One single-head LayerFactors + LatentCache per (sequence, head), as
// SURVEY.md section 8(d) prescribes; factors follow the decode-bench recipe
// (tools/wsvd_main.cpp:360-391: Rng::stream(seed, 5), A ~ N(0, 1/E),
// B ~ N(0, 1/r), order q.a q.b k.a k.b v.a v.b per head).  The prefill pushes
// N(0,1) latent rows (the distribution of x.A for x ~ N(0,1)); it is setup,
// not timed.  One step = append_token of a fresh token + fused_decode_step,
// for every (sequence, head), spread over `threads` with parallel_for.
struct RefBaseline {
    std::size_t E, H, nh, r, B, tile;
    std::vector<decode::LayerFactors> heads;          // nh single-head layers
    std::vector<std::unique_ptr<decode::LatentCache>> caches; // B * nh
    std::vector<double> x;                            // B x E current tokens
    Rng tok_rng{0};
};

void* ref_baseline_create(std::size_t E, std::size_t H, std::size_t nh, std::size_t r,
                          std::size_t B, std::size_t L, std::size_t tile, uint64_t seed,
                          int threads) {
    try {
        auto* s = new RefBaseline{E, H, nh, r, B, tile, {}, {}, {}, Rng(seed)};
        Rng rng = Rng::stream(seed, 5);
        const double a_std = 1.0 / std::sqrt(static_cast<double>(E));
        const double b_std = 1.0 / std::sqrt(static_cast<double>(r));
        for (std::size_t h = 0; h < nh; ++h) {
            decode::LayerFactors f;
            f.embed_dim = E;
            f.head_dim = H;
            decode::HeadProjection p;
            for (factorize::HeadFactors* hf : {&p.q, &p.k, &p.v}) {
                hf->a = rng.normal_matrix(E, r, a_std);
                hf->b = rng.normal_matrix(r, H, b_std);
                hf->rank = r;
                hf->head = 0;
            }
            p.q.role = factorize::Role::Q;
            p.k.role = factorize::Role::K;
            p.v.role = factorize::Role::V;
            f.heads.push_back(std::move(p));
            s->heads.push_back(std::move(f));
        }
        s->caches.resize(B * nh);
        const std::size_t prefill = L > 0 ? L - 1 : 0;
        parallel_for(B * nh, static_cast<std::size_t>(threads > 0 ? threads : 1),
                     [&](std::size_t i) {
                         const std::size_t h = i % nh;
                         auto c = std::make_unique<decode::LatentCache>(s->heads[h]);
                         Rng lr = Rng::stream(seed, 1000 + i);
                         std::vector<double> ck(r), cv(r);
                         for (std::size_t t = 0; t < prefill; ++t) {
                             for (double& v : ck) v = lr.normal();
                             for (double& v : cv) v = lr.normal();
                             c->push(0, ck, cv);
                             c->bump_length();
                         }
                         s->caches[i] = std::move(c);
                     });
        s->x.resize(B * E);
        s->tok_rng = Rng::stream(seed, 999);
        return s;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Runs one decode step for all (sequence, head) pairs; returns wall ms.
double ref_baseline_step(void* handle, int threads) {
    auto* s = static_cast<RefBaseline*>(handle);
    for (double& v : s->x) v = s->tok_rng.normal();
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(s->B * s->nh, static_cast<std::size_t>(threads > 0 ? threads : 1),
                 [&](std::size_t i) {
                     const std::size_t b = i / s->nh, h = i % s->nh;
                     decode::LatentCache& c = *s->caches[i];
                     const Matrix q = decode::append_token(
                         c, s->heads[h], std::span<const double>(s->x.data() + b * s->E, s->E));
                     decode::TrafficCounter counter;
                     const Matrix o = decode::fused_decode_step(c, s->heads[h], q,
                                                                decode::TileConfig{s->tile},
                                                                counter);
                     (void)o;
                 });
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

void ref_baseline_destroy(void* handle) { delete static_cast<RefBaseline*>(handle); }

} // extern "C"
