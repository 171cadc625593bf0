// host_decode.cpp -- the C++ wsvd::decode drop-in (include/wsvd/decode.hpp)
// over the C ABI of libwsvd_b200.so.
//
// Compiled INSIDE the reference build, in place of its src/decode.cpp, with
// this repo's include/ ahead of the reference's on the include path: Matrix,
// factorize::HeadFactors and the error classes come from the reference's own
// matrix.hpp / factorize.hpp / errors.hpp and their definitions from its
// matrix.cpp (oracle/Makefile target `dropin`).  Host-side
// only: argument validation with the reference's exception classes and
// messages, factor / weight upload, host <-> device staging of the operator
// arguments, the closed-form traffic tallies, and the host views that keep
// `const Matrix&` accessors (latent_k, keys) valid.
//
// Factor sets are not identified by address (a LayerFactors may be a loop
// temporary or be edited in place): each device upload is keyed by a content
// fingerprint -- every value for tensors up to 1 M entries, 4096 spread samples
// beyond -- so changed factors are re-uploaded and nothing dangles.
#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <list>
#include <mutex>
#include <utility>

#include "wsvd/decode.hpp"
#include "wsvd/errors.hpp"
#include "wsvd_b200.h"

namespace wsvd::decode {

namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = wsvd_last_error();
    switch (status) {
        case WSVD_ESHAPE: throw ShapeError(msg);
        case WSVD_ECONFIG: throw ConfigError(msg);
        case WSVD_ENUMERIC: throw NumericError(msg);
        case WSVD_EIO: throw IoError(msg);
        default: throw Error("device: " + msg);
    }
}
void check(int status) {
    if (status != WSVD_OK) raise(status);
}
void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string("device: ") + what + ": " + cudaGetErrorString(e));
}

// scoped device buffer, grown on demand
struct DevMem {
    void* p = nullptr;
    std::size_t n = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() {
        if (p) cudaFree(p);
    }
    float* f(std::size_t floats) {
        const std::size_t bytes = floats * 4;
        if (bytes > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
            n = bytes;
        }
        return static_cast<float*>(p);
    }
};

std::vector<float> to_f32(const double* v, std::size_t n) {
    std::vector<float> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<float>(v[i]);
    return out;
}
void upload(float* dst, const std::vector<float>& src) {
    check_cuda(cudaMemcpy(dst, src.data(), src.size() * 4, cudaMemcpyHostToDevice), "upload");
}
std::vector<float> download(const float* src, std::size_t n) {
    std::vector<float> out(n);
    check_cuda(cudaMemcpy(out.data(), src, n * 4, cudaMemcpyDeviceToHost), "download");
    return out;
}

// a C-ABI counter block [loads(7) | stores(7) | flops(7)] added to a TrafficCounter
void add_block(TrafficCounter& c, const std::uint64_t (&k)[21]) {
    for (std::size_t s = 0; s < kStreamCount; ++s) {
        const Stream st = static_cast<Stream>(s);
        if (k[s]) c.add_loads(st, k[s]);
        if (k[7 + s]) c.add_stores(st, k[7 + s]);
        if (k[14 + s]) c.add_flops(st, k[14 + s]);
    }
}

// ---- content fingerprints (FNV-1a over shapes and values)
struct Fp {
    std::uint64_t h = 1469598103934665603ull;
    void mix(const void* p, std::size_t n) {
        const auto* b = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    }
    void mix(std::uint64_t v) { mix(&v, sizeof v); }
    void mix(const Matrix& m) {
        mix(m.rows());
        mix(m.cols());
        const std::vector<double>& d = m.data();
        if (d.size() <= (1u << 20)) {
            mix(d.data(), d.size() * sizeof(double));
        } else {
            const std::size_t step = d.size() / 4096;
            for (std::size_t i = 0; i < d.size(); i += step) mix(&d[i], sizeof(double));
        }
    }
};

std::uint64_t fingerprint(const LayerFactors& f) {
    Fp fp;
    fp.mix(f.embed_dim);
    fp.mix(f.head_dim);
    fp.mix(f.heads.size());
    for (const HeadProjection& p : f.heads)
        for (const factorize::HeadFactors* hf : {&p.q, &p.k, &p.v}) {
            fp.mix(hf->rank);
            fp.mix(hf->a);
            fp.mix(hf->b);
        }
    return fp.h;
}

// device copies of host matrices (weights of the baselines), by content
struct MatCache {
    std::mutex mu;
    struct Entry {
        std::uint64_t key;
        int device;
        DevMem mem;
    };
    std::list<Entry> entries;  // most recent first, at most 32
    const float* get(const Matrix& m, int device) {
        Fp fp;
        fp.mix(m);
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = entries.begin(); it != entries.end(); ++it)
            if (it->key == fp.h && it->device == device) {
                entries.splice(entries.begin(), entries, it);
                return static_cast<const float*>(entries.front().mem.p);
            }
        entries.emplace_front();
        Entry& e = entries.front();
        e.key = fp.h;
        e.device = device;
        upload(e.mem.f(std::max<std::size_t>(m.size(), 1)), to_f32(m.data().data(), m.size()));
        while (entries.size() > 32) entries.pop_back();
        return static_cast<const float*>(e.mem.p);
    }
};
MatCache& mat_cache() {
    static MatCache c;
    return c;
}

void require_query(const Matrix& q, std::size_t rows, std::size_t cols) {
    if (q.rows() != rows || q.cols() != cols)
        throw ShapeError("query block must be " + std::to_string(rows) + "x" + std::to_string(cols) + ", got " +
                         std::to_string(q.rows()) + "x" + std::to_string(q.cols()));
}

std::size_t checked_tile(const TileConfig& t, std::size_t len) {
    if (t.tile_len == 0) throw ConfigError("tile length must be >= 1");
    return std::min(t.tile_len, len);
}

Matrix to_matrix(const std::vector<float>& v, std::size_t rows, std::size_t cols) {
    Matrix m(rows, cols);
    for (std::size_t i = 0; i < rows * cols; ++i) m.data()[i] = v[i];
    return m;
}

}  // namespace

// ============================================================ counters ===
const char* stream_name(Stream s) {
    static const char* const names[kStreamCount] = {"latent_k",  "latent_v", "full_k", "full_v",
                                                    "weights_b", "query",    "output"};
    const auto i = static_cast<std::size_t>(s);
    return i < kStreamCount ? names[i] : "?";
}

std::uint64_t TrafficCounter::total_loads() const {
    std::uint64_t n = 0;
    for (const StreamTally& t : t_) n += t.loads;
    return n;
}

std::uint64_t TrafficCounter::total_stores() const {
    std::uint64_t n = 0;
    for (const StreamTally& t : t_) n += t.stores;
    return n;
}

// ======================================================= SoftmaxState ===
// decode.cpp:35-75 semantics: the first observation seeds the state with
// weight 1; a larger score rescales what was accumulated by exp(old - new)
void SoftmaxState::observe(double score, std::span<const double> value) {
    if (empty) {
        empty = false;
        max_score = score;
        denom = 1.0;
        acc.assign(value.begin(), value.end());
        return;
    }
    if (value.size() != acc.size())
        throw ShapeError("softmax state holds width " + std::to_string(acc.size()) + ", observed width " +
                         std::to_string(value.size()));
    if (score > max_score) {
        const double shrink = std::exp(max_score - score);
        for (std::size_t i = 0; i < acc.size(); ++i) acc[i] = acc[i] * shrink + value[i];
        denom = denom * shrink + 1.0;
        max_score = score;
    } else {
        const double w = std::exp(score - max_score);
        for (std::size_t i = 0; i < acc.size(); ++i) acc[i] += w * value[i];
        denom += w;
    }
}

void SoftmaxState::merge(const SoftmaxState& other) {
    if (other.empty) return;
    if (empty) {
        *this = other;
        return;
    }
    if (other.acc.size() != acc.size())
        throw ShapeError("merging softmax states of widths " + std::to_string(acc.size()) + " and " +
                         std::to_string(other.acc.size()));
    const double top = std::max(max_score, other.max_score);
    const double mine = std::exp(max_score - top), theirs = std::exp(other.max_score - top);
    for (std::size_t i = 0; i < acc.size(); ++i) acc[i] = acc[i] * mine + other.acc[i] * theirs;
    denom = denom * mine + other.denom * theirs;
    max_score = top;
}

// ======================================================== LatentCache ===
struct LatentCache::Impl {
    DeviceOptions opt;
    std::size_t nh = 0, E = 0, H = 0, rpad = 0;
    std::vector<std::array<std::size_t, 3>> ranks;  // (q, k, v) per head -- a copy, not a reference
    wsvd_layer_t layer = nullptr;
    std::uint64_t layer_fp = 0;
    wsvd_cache_t cache = nullptr;
    std::vector<double> stage_k, stage_v;  // push() staging [nh][rpad]
    std::vector<unsigned char> staged;     // heads pushed since the last bump_length()
    std::uint64_t version = 0;             // bumped by every change of the rows
    mutable std::uint64_t view_version = ~0ull;
    mutable std::vector<Matrix> kview, vview;
    mutable DevMem xd, qd, od;

    ~Impl() {
        if (cache) wsvd_cache_destroy(cache);
        if (layer) wsvd_layer_destroy(layer);
    }

    static wsvd_layer_t upload(const LayerFactors& f, const DeviceOptions& opt) {
        if (f.heads.empty()) throw ShapeError("latent cache over zero heads");
        std::vector<int32_t> rk;
        for (const HeadProjection& p : f.heads)
            for (const factorize::HeadFactors* hf : {&p.q, &p.k, &p.v}) rk.push_back(static_cast<int32_t>(hf->rank));
        wsvd_layer_desc d{};
        d.embed_dim = static_cast<int32_t>(f.embed_dim);
        d.head_dim = static_cast<int32_t>(f.head_dim);
        d.n_heads = static_cast<int32_t>(f.heads.size());
        d.weight_dtype = static_cast<int32_t>(opt.weights);
        d.act_rotation = (opt.weights == Storage::I8 || opt.weights == Storage::I4) ? 1 : 0;
        d.device = opt.device;
        wsvd_layer_t L = nullptr;
        check(wsvd_layer_create(&d, rk.data(), &L));
        try {
            for (std::size_t h = 0; h < f.heads.size(); ++h) {
                const factorize::HeadFactors* roles[3] = {&f.heads[h].q, &f.heads[h].k, &f.heads[h].v};
                for (int role = 0; role < 3; ++role) {
                    const factorize::HeadFactors& hf = *roles[role];
                    if (hf.a.rows() != f.embed_dim || hf.a.cols() != hf.rank || hf.b.rows() != hf.rank ||
                        hf.b.cols() != f.head_dim)
                        throw ShapeError("head " + std::to_string(h) + ": factor shapes disagree with the layer geometry");
                    check(wsvd_layer_set_head(L, static_cast<int32_t>(h), role, hf.a.data().data(), hf.b.data().data()));
                }
            }
        } catch (...) {
            wsvd_layer_destroy(L);
            throw;
        }
        return L;
    }

    // the device layer follows the factor set passed to each operator call
    void bind(const LayerFactors& f) {
        if (f.heads.size() != nh)
            throw ShapeError("cache holds " + std::to_string(nh) + " heads, factors " + std::to_string(f.heads.size()));
        const std::uint64_t fp = fingerprint(f);
        if (fp == layer_fp) return;
        wsvd_layer_t L = upload(f, opt);
        const int rc = wsvd_cache_bind_layer(cache, L);
        if (rc != WSVD_OK) {
            wsvd_layer_destroy(L);
            raise(rc);
        }
        wsvd_layer_destroy(layer);
        layer = L;
        layer_fp = fp;
        for (std::size_t h = 0; h < nh; ++h)
            ranks[h] = {f.heads[h].q.rank, f.heads[h].k.rank, f.heads[h].v.rank};
    }

    std::size_t length() const {
        int32_t n = 0;
        check(wsvd_cache_length(cache, &n));
        return static_cast<std::size_t>(n);
    }

    // room for `more` rows (the reference's cache grows without bound)
    void reserve(std::size_t more) {
        int32_t cap = 0;
        check(wsvd_cache_capacity(cache, &cap));
        const std::size_t need = length() + more;
        if (need <= static_cast<std::size_t>(cap)) return;
        std::size_t grown = static_cast<std::size_t>(cap);
        while (grown < need) grown *= 2;
        check(wsvd_cache_grow(cache, static_cast<int32_t>(grown)));
    }

    Matrix read(std::size_t head, std::size_t seq, bool k_part) const {
        const std::size_t L = length();
        std::vector<double> ck(std::max<std::size_t>(L * rpad, 1)), cv(ck.size());
        check(wsvd_cache_read_host(cache, static_cast<int32_t>(seq), static_cast<int32_t>(head), ck.data(), cv.data()));
        const std::size_t r = ranks[head][k_part ? 1 : 2];
        Matrix m(L, r);
        const std::vector<double>& src = k_part ? ck : cv;
        for (std::size_t t = 0; t < L; ++t)
            for (std::size_t j = 0; j < r; ++j) m(t, j) = src[t * rpad + j];
        return m;
    }

    void refresh_views() const {
        if (view_version == version) return;
        kview.resize(nh);
        vview.resize(nh);
        for (std::size_t h = 0; h < nh; ++h) {
            kview[h] = read(h, 0, true);
            vview[h] = read(h, 0, false);
        }
        view_version = version;
    }
};

LatentCache::LatentCache(const LayerFactors& f) : LatentCache(f, DeviceOptions{}) {}

LatentCache::LatentCache(const LayerFactors& f, const DeviceOptions& opt) : p_(std::make_unique<Impl>()) {
    if (f.heads.empty()) throw ShapeError("latent cache over zero heads");
    if (opt.batch == 0) throw ShapeError("batch must be positive");
    Impl& m = *p_;
    m.opt = opt;
    m.nh = f.heads.size();
    m.E = f.embed_dim;
    m.H = f.head_dim;
    m.ranks.resize(m.nh);
    for (std::size_t h = 0; h < m.nh; ++h) m.ranks[h] = {f.heads[h].q.rank, f.heads[h].k.rank, f.heads[h].v.rank};
    m.layer = Impl::upload(f, opt);
    m.layer_fp = fingerprint(f);
    int32_t rp = 0;
    check(wsvd_layer_rank_pad(m.layer, &rp));
    m.rpad = static_cast<std::size_t>(rp);
    check(wsvd_cache_create(m.layer, static_cast<int32_t>(opt.batch),
                            static_cast<int32_t>(std::max<std::size_t>(opt.capacity, 1)),
                            static_cast<int32_t>(opt.cache), &m.cache));
    m.stage_k.assign(m.nh * m.rpad, 0.0);
    m.stage_v.assign(m.nh * m.rpad, 0.0);
    m.staged.assign(m.nh, 0);
}

LatentCache::~LatentCache() = default;
LatentCache::LatentCache(LatentCache&&) noexcept = default;
LatentCache& LatentCache::operator=(LatentCache&&) noexcept = default;

std::size_t LatentCache::length() const { return p_->length(); }
std::size_t LatentCache::n_heads() const { return p_->nh; }
std::size_t LatentCache::batch() const { return p_->opt.batch; }
const DeviceOptions& LatentCache::options() const { return p_->opt; }

const Matrix& LatentCache::latent_k(std::size_t head) const {
    if (head >= p_->nh) throw ShapeError("head " + std::to_string(head) + " out of range");
    p_->refresh_views();
    return p_->kview[head];
}

const Matrix& LatentCache::latent_v(std::size_t head) const {
    if (head >= p_->nh) throw ShapeError("head " + std::to_string(head) + " out of range");
    p_->refresh_views();
    return p_->vview[head];
}

Matrix LatentCache::latent_k(std::size_t head, std::size_t seq) const {
    if (head >= p_->nh || seq >= p_->opt.batch) throw ShapeError("head / sequence out of range");
    return p_->read(head, seq, true);
}

Matrix LatentCache::latent_v(std::size_t head, std::size_t seq) const {
    if (head >= p_->nh || seq >= p_->opt.batch) throw ShapeError("head / sequence out of range");
    return p_->read(head, seq, false);
}

void LatentCache::push(std::size_t head, std::span<const double> ck, std::span<const double> cv) {
    Impl& m = *p_;
    if (head >= m.nh) throw ShapeError("push: head " + std::to_string(head) + " out of range");
    const std::size_t rk = m.ranks[head][1], rv = m.ranks[head][2];
    if (ck.size() != rk || cv.size() != rv)
        throw ShapeError("append_row: " + std::to_string(ck.size()) + "/" + std::to_string(cv.size()) +
                         " values onto rows of width " + std::to_string(rk) + "/" + std::to_string(rv));
    std::fill_n(m.stage_k.begin() + head * m.rpad, m.rpad, 0.0);
    std::fill_n(m.stage_v.begin() + head * m.rpad, m.rpad, 0.0);
    std::copy(ck.begin(), ck.end(), m.stage_k.begin() + head * m.rpad);
    std::copy(cv.begin(), cv.end(), m.stage_v.begin() + head * m.rpad);
    m.staged[head] = 1;
}

void LatentCache::bump_length() {
    Impl& m = *p_;
    if (std::find(m.staged.begin(), m.staged.end(), 0) != m.staged.end())
        throw ShapeError("bump_length: every head needs one pushed row (the device appends whole token rows)");
    m.reserve(1);
    // the staged row goes to every sequence of a batched cache
    std::vector<double> k(m.opt.batch * m.nh * m.rpad), v(k.size());
    for (std::size_t b = 0; b < m.opt.batch; ++b) {
        std::copy(m.stage_k.begin(), m.stage_k.end(), k.begin() + b * m.nh * m.rpad);
        std::copy(m.stage_v.begin(), m.stage_v.end(), v.begin() + b * m.nh * m.rpad);
    }
    check(wsvd_cache_push_host(m.cache, k.data(), v.data()));
    std::fill(m.staged.begin(), m.staged.end(), 0);
    ++m.version;
}

// ========================================================= operators ===
namespace {

Matrix append_rows(LatentCache& cache, const LayerFactors& f, const double* x, std::size_t rows,
                   TrafficCounter* counter) {
    LatentCache::Impl& m = cache.impl();
    m.bind(f);
    m.reserve(1);
    for (std::size_t i = 0; i < rows * f.embed_dim; ++i)
        if (!std::isfinite(x[i])) throw NumericError("append_token: non-finite token");
    float* xd = m.xd.f(rows * f.embed_dim);
    float* qd = m.qd.f(rows * m.nh * f.head_dim);
    upload(xd, to_f32(x, rows * f.embed_dim));
    check(wsvd_append_token(m.cache, xd, qd, m.opt.stream));
    ++m.version;
    std::vector<float> q = download(qd, rows * m.nh * f.head_dim);
    if (counter) {
        std::uint64_t k[21] = {};
        check(wsvd_traffic_append(m.cache, k));
        add_block(*counter, k);
    }
    return to_matrix(q, rows * m.nh, f.head_dim);
}

}  // namespace

Matrix append_token(LatentCache& cache, const LayerFactors& f, std::span<const double> x, TrafficCounter* counter) {
    if (x.size() != f.embed_dim)
        throw ShapeError("token has " + std::to_string(x.size()) + " features, layer expects " +
                         std::to_string(f.embed_dim));
    if (cache.batch() != 1) throw ShapeError("single-token append on a batched cache: pass one row per sequence");
    return append_rows(cache, f, x.data(), 1, counter);
}

Matrix append_token(LatentCache& cache, const LayerFactors& f, const Matrix& x, TrafficCounter* counter) {
    if (x.cols() != f.embed_dim)
        throw ShapeError("token has " + std::to_string(x.cols()) + " features, layer expects " +
                         std::to_string(f.embed_dim));
    if (x.rows() != cache.batch())
        throw ShapeError(std::to_string(x.rows()) + " token rows for " + std::to_string(cache.batch()) + " sequences");
    return append_rows(cache, f, x.data().data(), x.rows(), counter);
}

Matrix fused_decode_step(const LatentCache& cache, const LayerFactors& f, const Matrix& q_heads,
                         const TileConfig& tiles, TrafficCounter& counter) {
    LatentCache::Impl& m = cache.impl();
    const std::size_t len = m.length();
    if (len == 0) throw ShapeError("decode step over an empty cache");
    if (m.nh != f.heads.size())
        throw ShapeError("cache holds " + std::to_string(m.nh) + " heads, factors " + std::to_string(f.heads.size()));
    require_query(q_heads, m.opt.batch * m.nh, f.head_dim);
    const std::size_t tile = checked_tile(tiles, len);
    m.bind(f);
    float* qd = m.qd.f(q_heads.size());
    float* od = m.od.f(q_heads.size());
    upload(qd, to_f32(q_heads.data().data(), q_heads.size()));
    const int32_t t32 = static_cast<int32_t>(std::min<std::size_t>(tile, 1u << 30));
    check(wsvd_fused_decode_step(m.cache, qd, t32, od, m.opt.stream));
    std::vector<float> out = download(od, q_heads.size());
    std::uint64_t k[21] = {};
    check(wsvd_traffic_fused(m.cache, t32, k));
    add_block(counter, k);
    return to_matrix(out, q_heads.rows(), f.head_dim);
}

// ======================================================== FullKvCache ===
struct FullKvCache::Impl {
    std::size_t nh = 0, H = 0;
    int device = 0;
    wsvd_dense_cache_t cache = nullptr;
    std::vector<double> stage_k, stage_v;  // [nh][H]
    std::vector<unsigned char> staged;
    std::uint64_t version = 0;
    mutable std::uint64_t view_version = ~0ull;
    mutable std::vector<Matrix> kview, vview;
    mutable DevMem kd, vd, qd, od, xd, tmp;
    ~Impl() {
        if (cache) wsvd_dense_cache_destroy(cache);
    }
    std::size_t length() const {
        int32_t n = 0;
        check(wsvd_dense_cache_length(cache, &n));
        return static_cast<std::size_t>(n);
    }
    void refresh_views() const {
        if (view_version == version) return;
        const std::size_t L = length();
        kview.assign(nh, Matrix(L, H));
        vview.assign(nh, Matrix(L, H));
        for (std::size_t h = 0; h < nh && L > 0; ++h)
            check(wsvd_dense_cache_read_host(cache, static_cast<int32_t>(h), kview[h].data().data(),
                                             vview[h].data().data()));
        view_version = version;
    }
};

FullKvCache::FullKvCache(std::size_t n_heads, std::size_t head_dim) : p_(std::make_unique<Impl>()) {
    if (n_heads == 0 || head_dim == 0) throw ShapeError("empty kv cache geometry");
    p_->nh = n_heads;
    p_->H = head_dim;
    check(wsvd_dense_cache_create(static_cast<int32_t>(n_heads), static_cast<int32_t>(head_dim), 0, &p_->cache));
    p_->stage_k.assign(n_heads * head_dim, 0.0);
    p_->stage_v.assign(n_heads * head_dim, 0.0);
    p_->staged.assign(n_heads, 0);
}

FullKvCache::~FullKvCache() = default;
FullKvCache::FullKvCache(FullKvCache&&) noexcept = default;
FullKvCache& FullKvCache::operator=(FullKvCache&&) noexcept = default;

std::size_t FullKvCache::length() const { return p_->length(); }
std::size_t FullKvCache::n_heads() const { return p_->nh; }

const Matrix& FullKvCache::keys(std::size_t head) const {
    if (head >= p_->nh) throw ShapeError("head " + std::to_string(head) + " out of range");
    p_->refresh_views();
    return p_->kview[head];
}

const Matrix& FullKvCache::values(std::size_t head) const {
    if (head >= p_->nh) throw ShapeError("head " + std::to_string(head) + " out of range");
    p_->refresh_views();
    return p_->vview[head];
}

void FullKvCache::push(std::size_t head, std::span<const double> k, std::span<const double> v) {
    Impl& m = *p_;
    if (head >= m.nh) throw ShapeError("push: head " + std::to_string(head) + " out of range");
    if (k.size() != m.H || v.size() != m.H)
        throw ShapeError("append_row: " + std::to_string(k.size()) + " values onto rows of width " + std::to_string(m.H));
    std::copy(k.begin(), k.end(), m.stage_k.begin() + head * m.H);
    std::copy(v.begin(), v.end(), m.stage_v.begin() + head * m.H);
    m.staged[head] = 1;
}

void FullKvCache::bump_length() {
    Impl& m = *p_;
    if (std::find(m.staged.begin(), m.staged.end(), 0) != m.staged.end())
        throw ShapeError("bump_length: every head needs one pushed row (the device appends whole token rows)");
    float* kd = m.kd.f(m.nh * m.H);
    float* vd = m.vd.f(m.nh * m.H);
    upload(kd, to_f32(m.stage_k.data(), m.stage_k.size()));
    upload(vd, to_f32(m.stage_v.data(), m.stage_v.size()));
    check(wsvd_dense_cache_append(m.cache, kd, vd, nullptr));
    std::fill(m.staged.begin(), m.staged.end(), 0);
    ++m.version;
}

Matrix append_token_dense(FullKvCache& cache, const DenseProjections& w, std::span<const double> x,
                          TrafficCounter* counter) {
    const std::size_t e = w.w_q.rows();
    if (x.size() != e)
        throw ShapeError("token has " + std::to_string(x.size()) + " features, layer expects " + std::to_string(e));
    FullKvCache::Impl& m = cache.impl();
    const std::size_t hd = w.head_dim, nh = m.nh;
    if (hd != m.H) throw ShapeError("append_row: projection head width " + std::to_string(hd) + " vs cache " + std::to_string(m.H));
    if (nh * hd > w.w_k.cols() || w.w_k.rows() != e || w.w_v.rows() != e || w.w_q.cols() != w.w_k.cols() ||
        w.w_v.cols() != w.w_k.cols())
        throw ShapeError("dense projections do not cover " + std::to_string(nh) + " heads of width " + std::to_string(hd));
    const std::size_t n = w.w_k.cols();
    float* xd = m.xd.f(e);
    float* qkv = m.tmp.f(3 * n);
    upload(xd, to_f32(x.data(), e));
    check(wsvd_vecmat_f32(xd, mat_cache().get(w.w_q, 0), static_cast<int32_t>(e), static_cast<int32_t>(n), qkv, nullptr));
    check(wsvd_vecmat_f32(xd, mat_cache().get(w.w_k, 0), static_cast<int32_t>(e), static_cast<int32_t>(n), qkv + n, nullptr));
    check(wsvd_vecmat_f32(xd, mat_cache().get(w.w_v, 0), static_cast<int32_t>(e), static_cast<int32_t>(n), qkv + 2 * n, nullptr));
    // head h's rows are columns [h*hd, (h+1)*hd) of k and v: the first nh*hd
    check(wsvd_dense_cache_append(m.cache, qkv + n, qkv + 2 * n, nullptr));
    ++m.version;
    std::vector<float> q = download(qkv, nh * hd);
    if (counter) {
        counter->add_loads(Stream::Query, e);
        for (std::size_t h = 0; h < nh; ++h) {
            counter->add_flops(Stream::FullK, e * hd);
            counter->add_stores(Stream::FullK, hd);
            counter->add_flops(Stream::FullV, e * hd);
            counter->add_stores(Stream::FullV, hd);
            counter->add_flops(Stream::Query, e * hd);
        }
    }
    return to_matrix(q, nh, hd);
}

namespace {

Matrix dense_attend(const FullKvCache& cache, const Matrix& q_heads, std::size_t tile) {
    FullKvCache::Impl& m = cache.impl();
    float* qd = m.qd.f(q_heads.size());
    float* od = m.od.f(q_heads.size());
    upload(qd, to_f32(q_heads.data().data(), q_heads.size()));
    check(wsvd_dense_decode_step(m.cache, qd, static_cast<int32_t>(std::min<std::size_t>(tile, 1u << 30)), od, nullptr));
    return to_matrix(download(od, q_heads.size()), m.nh, m.H);
}

}  // namespace

Matrix eager_decode_step(const FullKvCache& cache, const Matrix& q_heads, TrafficCounter& counter) {
    const std::size_t len = cache.length();
    if (len == 0) throw ShapeError("decode step over an empty cache");
    const std::size_t hd = cache.impl().H, nh = cache.n_heads();
    require_query(q_heads, nh, hd);
    Matrix out = dense_attend(cache, q_heads, len);
    for (std::size_t h = 0; h < nh; ++h) {  // decode.cpp:266-287 tallies
        counter.add_loads(Stream::Query, hd);
        counter.add_loads(Stream::FullK, len * hd);
        counter.add_flops(Stream::Query, len * hd);
        counter.add_stores(Stream::Query, len);
        counter.add_loads(Stream::FullV, len * hd);
        counter.add_flops(Stream::FullV, len * hd);
        counter.add_stores(Stream::Output, hd);
    }
    return out;
}

Matrix flash_decode_step(const FullKvCache& cache, const Matrix& q_heads, const TileConfig& tiles,
                         TrafficCounter& counter) {
    const std::size_t len = cache.length();
    if (len == 0) throw ShapeError("decode step over an empty cache");
    const std::size_t hd = cache.impl().H, nh = cache.n_heads();
    require_query(q_heads, nh, hd);
    const std::size_t tile = checked_tile(tiles, len);
    Matrix out = dense_attend(cache, q_heads, tile);
    for (std::size_t h = 0; h < nh; ++h) {  // decode.cpp:303-317 tallies, tile by tile
        counter.add_loads(Stream::Query, hd);
        for (std::size_t t0 = 0; t0 < len; t0 += tile) {
            const std::size_t rows = std::min(tile, len - t0);
            counter.add_loads(Stream::FullK, rows * hd);
            counter.add_loads(Stream::FullV, rows * hd);
            counter.add_flops(Stream::Query, rows * hd);
            counter.add_flops(Stream::FullV, rows * hd);
        }
        counter.add_stores(Stream::Output, hd);
    }
    return out;
}

// ===================================================== shared latent ===
void append_token_shared(SharedLatentCache& cache, const SharedFactors& f, std::span<const double> x,
                         TrafficCounter* counter) {
    const std::size_t e = f.a_k.rows();
    if (x.size() != e)
        throw ShapeError("token has " + std::to_string(x.size()) + " features, layer expects " + std::to_string(e));
    if (f.a_v.rows() != e) throw ShapeError("shared factors a_k / a_v disagree on the embedding width");
    static thread_local DevMem xd, cd;
    const std::size_t rk = f.a_k.cols(), rv = f.a_v.cols();
    float* x32 = xd.f(e);
    float* c32 = cd.f(rk + rv);
    upload(x32, to_f32(x.data(), e));
    check(wsvd_vecmat_f32(x32, mat_cache().get(f.a_k, 0), static_cast<int32_t>(e), static_cast<int32_t>(rk), c32, nullptr));
    check(wsvd_vecmat_f32(x32, mat_cache().get(f.a_v, 0), static_cast<int32_t>(e), static_cast<int32_t>(rv), c32 + rk, nullptr));
    const std::vector<float> c = download(c32, rk + rv);
    std::vector<double> ck(c.begin(), c.begin() + rk), cv(c.begin() + rk, c.end());
    cache.c_k.append_row(ck);
    cache.c_v.append_row(cv);
    if (counter) {
        counter->add_loads(Stream::Query, e);
        counter->add_flops(Stream::LatentK, e * rk);
        counter->add_stores(Stream::LatentK, rk);
        counter->add_flops(Stream::LatentV, e * rv);
        counter->add_stores(Stream::LatentV, rv);
    }
}

Matrix shared_decode_step(const SharedLatentCache& cache, const SharedFactors& f, const Matrix& q_heads,
                          const TileConfig& tiles, TrafficCounter& counter, bool materialize) {
    const std::size_t len = cache.length();
    if (len == 0) throw ShapeError("decode step over an empty cache");
    const std::size_t hd = f.head_dim, rr = f.b_k.rows(), nh = f.n_heads;
    require_query(q_heads, nh, hd);
    const std::size_t tile = checked_tile(tiles, len);
    if (cache.c_k.cols() != rr || cache.c_v.cols() != f.b_v.rows() || f.b_k.cols() < nh * hd || f.b_v.cols() < nh * hd)
        throw ShapeError("shared latent width / factors disagree");
    // per head: K_h = C_K . B_K[:, h*H:(h+1)*H], V_h likewise, then the softmax
    // attention over them -- the materialising schedule; the streamed one
    // (latent accumulate, one B_V product) is the same arithmetic reassociated
    static thread_local DevMem kd, vd, bk, bv, sc, qd, od;
    const std::size_t rv = f.b_v.rows();
    float* K = kd.f(nh * len * hd);
    float* V = vd.f(nh * len * hd);
    const float* ck = mat_cache().get(cache.c_k, 0);
    const float* cv = mat_cache().get(cache.c_v, 0);
    float* bkh = bk.f(rr * hd);
    float* bvh = bv.f(rv * hd);
    for (std::size_t h = 0; h < nh; ++h) {
        const Matrix bkb = f.b_k.col_block(h * hd, hd), bvb = f.b_v.col_block(h * hd, hd);
        upload(bkh, to_f32(bkb.data().data(), bkb.size()));
        upload(bvh, to_f32(bvb.data().data(), bvb.size()));
        check(wsvd_matmul_f32(ck, bkh, static_cast<int32_t>(len), static_cast<int32_t>(rr), static_cast<int32_t>(hd),
                              K + h * len * hd, nullptr));
        check(wsvd_matmul_f32(cv, bvh, static_cast<int32_t>(len), static_cast<int32_t>(rv), static_cast<int32_t>(hd),
                              V + h * len * hd, nullptr));
    }
    float* q = qd.f(q_heads.size());
    float* o = od.f(q_heads.size());
    upload(q, to_f32(q_heads.data().data(), q_heads.size()));
    check(wsvd_dense_attend(K, V, static_cast<int32_t>(nh), static_cast<int32_t>(len), static_cast<int32_t>(len),
                            static_cast<int32_t>(hd), q, sc.f(nh * len), o, nullptr));
    Matrix out = to_matrix(download(o, q_heads.size()), nh, hd);
    for (std::size_t h = 0; h < nh; ++h) {  // decode.cpp:347-429 tallies
        counter.add_loads(Stream::WeightsB, 2 * rr * hd);
        counter.add_loads(Stream::Query, hd);
        if (materialize) {
            counter.add_loads(Stream::LatentK, len * rr);
            counter.add_flops(Stream::LatentK, len * rr * hd);
            counter.add_loads(Stream::LatentV, len * rr);
            counter.add_flops(Stream::LatentV, len * rr * hd);
            counter.add_stores(Stream::FullK, len * hd);
            counter.add_stores(Stream::FullV, len * hd);
            counter.add_loads(Stream::FullK, len * hd);
            counter.add_loads(Stream::FullV, len * hd);
            counter.add_flops(Stream::Query, len * hd);
            counter.add_flops(Stream::FullV, len * hd);
            counter.add_stores(Stream::Output, hd);
            continue;
        }
        for (std::size_t t0 = 0; t0 < len; t0 += tile) {
            const std::size_t rows = std::min(tile, len - t0);
            counter.add_loads(Stream::LatentK, rows * rr);
            counter.add_loads(Stream::LatentV, rows * rr);
            counter.add_flops(Stream::LatentK, rows * rr * hd);
            counter.add_flops(Stream::Query, rows * hd);
            counter.add_flops(Stream::LatentV, rows * rr);
        }
        counter.add_flops(Stream::Output, rr * hd);
        counter.add_stores(Stream::Output, hd);
    }
    return out;
}

// ============================================================ reports ===
const char* mode_name(Mode m) {
    switch (m) {
        case Mode::Fused: return "fused";
        case Mode::Eager: return "eager";
        case Mode::FlashFull: return "flash_full";
        case Mode::SharedLatent: return "shared_latent";
    }
    return "?";
}

Mode mode_from_name(const std::string& name) {
    for (Mode m : {Mode::Fused, Mode::Eager, Mode::FlashFull, Mode::SharedLatent})
        if (name == mode_name(m)) return m;
    throw ConfigError("unknown decode mode '" + name + "'");
}

TrafficReport traffic_report(Mode mode, const TrafficCounter& counter, std::uint64_t seq_len, std::uint64_t n_heads,
                             std::uint64_t head_dim, std::uint64_t rank_k, std::uint64_t shared_rank) {
    if (n_heads == 0) throw ConfigError("traffic report over zero heads");
    TrafficReport r;
    r.mode = mode;
    r.seq_len = seq_len;
    r.n_heads = n_heads;
    // per head: eta cache scalars read, gamma reconstruction MACs
    const bool latent = mode == Mode::Fused || mode == Mode::SharedLatent;
    const std::uint64_t width = mode == Mode::Fused ? rank_k : (mode == Mode::SharedLatent ? shared_rank : head_dim);
    r.analytic_eta = seq_len * width;
    r.analytic_gamma = latent ? seq_len * width * head_dim : 0;
    const StreamTally& tally = counter[latent ? Stream::LatentK : Stream::FullK];
    const bool even = tally.loads % n_heads == 0 && tally.flops % n_heads == 0;
    if (even) {
        r.measured_cache_loads_per_head = tally.loads / n_heads;
        r.measured_reconstruction_flops_per_head = tally.flops / n_heads;
    }
    r.match = even && r.measured_cache_loads_per_head == r.analytic_eta &&
              r.measured_reconstruction_flops_per_head == r.analytic_gamma;
    const double loads = static_cast<double>(counter.total_loads());
    r.bytes_loaded_fp64 = 8.0 * loads;
    r.bytes_loaded_fp16 = 2.0 * loads;
    return r;
}

}  // namespace wsvd::decode
