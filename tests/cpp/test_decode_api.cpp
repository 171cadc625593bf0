// test_decode_api.cpp -- the reference's decode unit tests (tests/test_decode.cpp)
// written against the C++ drop-in (include/wsvd/decode.hpp) and checked
// against the CPU oracle (oracle/wsvd_oracle.h, test infrastructure).
// Built and run by tests/test_gpu_cpp.py on a B200.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../../oracle/wsvd_oracle.h"
#include "wsvd/decode.hpp"
#include "wsvd/errors.hpp"

using namespace wsvd;
using namespace wsvd::decode;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(cond)) {                                                       \
            ++g_fail;                                                        \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                    \
    } while (0)

template <typename Ex>
static bool throws(const std::function<void()>& fn) {
    try {
        fn();
    } catch (const Ex&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// random layer in both representations (test_decode.cpp:25-46 draw order)
struct TestLayer {
    LayerFactors f;
    std::size_t E, H, nh, rmax;
    std::vector<int32_t> ranks;
    std::vector<double> A, B;  // oracle padded layout
    orc_layer c() const { return orc_layer{E, H, nh, rmax, ranks.data(), A.data(), B.data()}; }
};

static Matrix normal_matrix(orc_rng& r, std::size_t rows, std::size_t cols, double sd) {
    Matrix m(rows, cols);
    orc_rng_normal_fill(&r, m.data().data(), m.size(), sd);
    return m;
}

static TestLayer random_layer(orc_rng& rng, std::size_t E, std::size_t H, const std::vector<std::array<int, 3>>& ranks) {
    TestLayer t;
    t.E = E;
    t.H = H;
    t.nh = ranks.size();
    t.rmax = 0;
    for (auto& r : ranks)
        for (int v : r) t.rmax = std::max<std::size_t>(t.rmax, v);
    t.A.assign(t.nh * 3 * E * t.rmax, 0.0);
    t.B.assign(t.nh * 3 * t.rmax * H, 0.0);
    t.f.embed_dim = E;
    t.f.head_dim = H;
    for (std::size_t h = 0; h < t.nh; ++h) {
        HeadProjection p;
        factorize::HeadFactors* roles[3] = {&p.q, &p.k, &p.v};
        for (int role = 0; role < 3; ++role) {
            const std::size_t r = ranks[h][role];
            t.ranks.push_back(static_cast<int32_t>(r));
            roles[role]->a = normal_matrix(rng, E, r, 1.0 / std::sqrt(double(E)));
            roles[role]->b = normal_matrix(rng, r, H, 1.0 / std::sqrt(double(r)));
            roles[role]->rank = r;
            roles[role]->head = h;
            roles[role]->role = static_cast<factorize::Role>(role);
            for (std::size_t i = 0; i < E; ++i)
                for (std::size_t j = 0; j < r; ++j)
                    t.A[((h * 3 + role) * E + i) * t.rmax + j] = roles[role]->a(i, j);
            for (std::size_t i = 0; i < r; ++i)
                for (std::size_t j = 0; j < H; ++j) t.B[((h * 3 + role) * t.rmax + i) * H + j] = roles[role]->b(i, j);
        }
        t.f.heads.push_back(std::move(p));
    }
    return t;
}

// max over head rows of max|a-b| / max|b|
static double rel_rows(const Matrix& a, const std::vector<double>& b, std::size_t H) {
    double worst = 0.0;
    for (std::size_t r = 0; r < a.rows(); ++r) {
        double num = 0.0, den = 1e-30;
        for (std::size_t j = 0; j < H; ++j) {
            num = std::max(num, std::abs(a(r, j) - b[r * H + j]));
            den = std::max(den, std::abs(b[r * H + j]));
        }
        worst = std::max(worst, num / den);
    }
    return worst;
}

static void test_fused_matches_reconstruct_then_attend() {
    const std::size_t cfgs[][4] = {{16, 4, 2, 13}, {32, 8, 4, 9}, {24, 4, 3, 31}, {32, 8, 2, 1}};
    uint64_t seed = 310;
    for (auto& cfg : cfgs) {
        orc_rng rng;
        orc_rng_seed(&rng, seed++);
        std::vector<std::array<int, 3>> ranks;
        for (std::size_t h = 0; h < cfg[2]; ++h)
            ranks.push_back({1 + int(orc_rng_index(&rng, cfg[1])), 1 + int(orc_rng_index(&rng, cfg[1])),
                             1 + int(orc_rng_index(&rng, cfg[1]))});
        TestLayer t = random_layer(rng, cfg[0], cfg[1], ranks);
        LatentCache cache(t.f);
        Matrix tokens = normal_matrix(rng, cfg[3], cfg[0], 1.0);
        Matrix q;
        std::vector<double> ck(t.nh * cfg[3] * t.rmax), cv(ck.size()), qo(t.nh * t.H);
        orc_layer ol = t.c();
        for (std::size_t i = 0; i < cfg[3]; ++i) {
            q = append_token(cache, t.f, tokens.row(i));
            orc_append_token(&ol, ck.data(), cv.data(), cfg[3], i, tokens.row(i).data(), qo.data(), nullptr);
        }
        TrafficCounter c;
        Matrix out = fused_decode_step(cache, t.f, q, TileConfig{5}, c);
        std::vector<double> ref(t.nh * t.H);
        orc_reconstruct_then_attend(&ol, ck.data(), cv.data(), cfg[3], cfg[3], qo.data(), ref.data());
        CHECK(rel_rows(q, qo, t.H) <= 1e-3);
        CHECK(rel_rows(out, ref, t.H) <= 1e-3);
    }
}

static void test_counters_and_report() {
    orc_rng rng;
    orc_rng_seed(&rng, 330);
    const std::size_t L = 17;
    TestLayer t = random_layer(rng, 24, 6, {{2, 3, 4}, {5, 1, 2}, {3, 6, 5}});
    LatentCache cache(t.f);
    TrafficCounter ca;
    Matrix q;
    for (std::size_t i = 0; i < L; ++i) {
        Matrix x = normal_matrix(rng, 1, 24, 1.0);
        q = append_token(cache, t.f, x.row(0), &ca);
    }
    TrafficCounter cd;
    fused_decode_step(cache, t.f, q, TileConfig{4}, cd);
    uint64_t k_loads = 0, k_flops = 0, v_loads = 0, b_loads = 0, out_flops = 0, q_flops = 0;
    for (std::size_t h = 0; h < 3; ++h) {
        const auto& p = t.f.heads[h];
        k_loads += L * p.k.rank;
        k_flops += L * p.k.rank * 6;
        v_loads += L * p.v.rank;
        b_loads += (p.k.rank + p.v.rank) * 6;
        out_flops += p.v.rank * 6;
        q_flops += L * (24 * p.q.rank + p.q.rank * 6);
    }
    CHECK(cd[Stream::LatentK].loads == k_loads);
    CHECK(cd[Stream::LatentK].flops == k_flops);
    CHECK(cd[Stream::LatentV].loads == v_loads);
    CHECK(cd[Stream::WeightsB].loads == b_loads);
    CHECK(cd[Stream::Output].flops == out_flops);
    CHECK(cd[Stream::Output].stores == 3 * 6);
    CHECK(cd[Stream::Query].stores == 0);
    CHECK(ca[Stream::Query].flops == q_flops);
    CHECK(ca[Stream::Query].loads == L * 24);
    TestLayer u = random_layer(rng, 32, 8, {{3, 3, 3}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}});
    LatentCache c2(u.f);
    for (std::size_t i = 0; i < 19; ++i) q = append_token(c2, u.f, normal_matrix(rng, 1, 32, 1.0).row(0));
    TrafficCounter c;
    fused_decode_step(c2, u.f, q, TileConfig{4}, c);
    CHECK(traffic_report(Mode::Fused, c, 19, 4, 8, 3, 0).match);
    CHECK(!traffic_report(Mode::Fused, c, 20, 4, 8, 3, 0).match);
    CHECK(mode_from_name(mode_name(Mode::SharedLatent)) == Mode::SharedLatent);
    CHECK(std::string(stream_name(Stream::WeightsB)) == "weights_b");
}

static void test_cache_rows_and_single_token() {
    orc_rng rng;
    orc_rng_seed(&rng, 332);
    TestLayer t = random_layer(rng, 16, 4, {{3, 3, 3}, {3, 3, 3}});
    LatentCache cache(t.f);
    Matrix tokens = normal_matrix(rng, 5, 16, 1.0);
    for (std::size_t i = 0; i < 5; ++i) append_token(cache, t.f, tokens.row(i));
    CHECK(cache.length() == 5);
    for (std::size_t h = 0; h < 2; ++h) {
        Matrix k = cache.latent_k(h);
        CHECK(k.rows() == 5 && k.cols() == 3);
        double worst = 0.0;
        for (std::size_t i = 0; i < 5; ++i)
            for (std::size_t j = 0; j < 3; ++j) {
                double e = 0.0;
                for (std::size_t d = 0; d < 16; ++d) e += tokens(i, d) * t.f.heads[h].k.a(d, j);
                worst = std::max(worst, std::abs(k(i, j) - e));
            }
        CHECK(worst <= 1e-5);
    }
}

static void test_batched_sequences() {
    orc_rng rng;
    orc_rng_seed(&rng, 340);
    const std::size_t Bn = 3, L = 40;
    TestLayer t = random_layer(rng, 64, 16, {{8, 8, 8}, {8, 8, 8}, {8, 8, 8}, {8, 8, 8}});
    DeviceOptions opt;
    opt.batch = Bn;
    opt.capacity = 64;
    LatentCache cache(t.f, opt);
    orc_layer ol = t.c();
    std::vector<std::vector<double>> ck(Bn, std::vector<double>(t.nh * L * t.rmax)), cv = ck;
    std::vector<double> qo(Bn * t.nh * t.H);
    Matrix q;
    for (std::size_t i = 0; i < L; ++i) {
        Matrix x = normal_matrix(rng, Bn, 64, 1.0);
        q = append_token(cache, t.f, x);
        for (std::size_t b = 0; b < Bn; ++b)
            orc_append_token(&ol, ck[b].data(), cv[b].data(), L, i, x.row(b).data(), qo.data() + b * t.nh * t.H, nullptr);
    }
    CHECK(rel_rows(q, qo, t.H) <= 1e-3);
    TrafficCounter c;
    Matrix out = fused_decode_step(cache, t.f, q, TileConfig{32}, c);
    CHECK(out.rows() == Bn * t.nh);
    std::vector<double> ref(Bn * t.nh * t.H);
    for (std::size_t b = 0; b < Bn; ++b)
        orc_fused_decode_step(&ol, ck[b].data(), cv[b].data(), L, L, qo.data() + b * t.nh * t.H, 32,
                              ref.data() + b * t.nh * t.H, nullptr);
    CHECK(rel_rows(out, ref, t.H) <= 1e-3);
    CHECK(c[Stream::LatentK].loads == Bn * t.nh * L * 8);
}

static void test_errors() {
    orc_rng rng;
    orc_rng_seed(&rng, 360);
    TestLayer t = random_layer(rng, 16, 4, {{2, 2, 2}, {2, 2, 2}});
    LatentCache cache(t.f);
    Matrix q(2, 4);
    TrafficCounter c;
    CHECK(throws<ShapeError>([&] { fused_decode_step(cache, t.f, q, TileConfig{}, c); }));
    for (int i = 0; i < 3; ++i) append_token(cache, t.f, normal_matrix(rng, 1, 16, 1.0).row(0));
    CHECK(throws<ConfigError>([&] { fused_decode_step(cache, t.f, q, TileConfig{0}, c); }));
    Matrix bad(2, 5);
    CHECK(throws<ShapeError>([&] { fused_decode_step(cache, t.f, bad, TileConfig{}, c); }));
    TestLayer other = random_layer(rng, 16, 4, {{2, 2, 2}, {2, 2, 2}, {2, 2, 2}});
    CHECK(throws<ShapeError>([&] { fused_decode_step(cache, other.f, q, TileConfig{}, c); }));
    CHECK(throws<ShapeError>([&] { LatentCache empty{LayerFactors{}}; }));
    std::vector<double> short_token(7, 0.0);
    CHECK(throws<ShapeError>([&] { append_token(cache, t.f, short_token); }));
    CHECK(throws<Error>([&] { append_token(cache, t.f, short_token); }));
}

int main() {
    test_fused_matches_reconstruct_then_attend();
    test_counters_and_report();
    test_cache_rows_and_single_token();
    test_batched_sequences();
    test_errors();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
