// host_decode.cpp -- the C++ wsvd::decode drop-in (include/wsvd/decode.hpp)
// implemented over the C ABI (include/wsvd_b200.h).  Host-side only: shape /
// config validation with the reference's exception classes, factor upload,
// host<->device staging of the operator arguments, counters.
#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <utility>

#include "wsvd/decode.hpp"

namespace wsvd {

void throw_status(int status) {
    if (status == WSVD_OK) return;
    const std::string msg = wsvd_last_error();
    switch (status) {
        case WSVD_ESHAPE: throw ShapeError(msg);
        case WSVD_ECONFIG: throw ConfigError(msg);
        case WSVD_ENUMERIC: throw NumericError(msg);
        case WSVD_EIO: throw IoError(msg);
        case WSVD_ECUDA:
        case WSVD_ENCCL: throw DeviceError(msg);
        default: throw Error(msg);
    }
}

Matrix::Matrix(std::size_t rows, std::size_t cols, std::vector<double> values)
    : r_(rows), c_(cols), v_(std::move(values)) {
    if (v_.size() != r_ * c_)
        throw ShapeError("matrix init: " + std::to_string(v_.size()) + " values for " + std::to_string(r_) +
                         "x" + std::to_string(c_));
}

void Matrix::append_row(std::span<const double> values) {
    if (r_ == 0 && c_ == 0) c_ = values.size();
    if (values.size() != c_)
        throw ShapeError("append_row: " + std::to_string(values.size()) + " values onto a " + std::to_string(r_) +
                         "x" + std::to_string(c_) + " matrix");
    v_.insert(v_.end(), values.begin(), values.end());
    ++r_;
}

double dot(std::span<const double> a, std::span<const double> b) {
    if (a.size() != b.size()) throw ShapeError("dot: lengths differ");
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

double max_abs_diff(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw ShapeError("max_abs_diff: shapes differ");
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.data()[i] - b.data()[i]));
    return m;
}

}  // namespace wsvd

namespace wsvd::decode {

namespace {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// scoped device buffer
struct DevMem {
    void* p = nullptr;
    std::size_t n = 0;
    void ensure(std::size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
        n = bytes;
    }
    ~DevMem() {
        if (p) cudaFree(p);
    }
};

struct LayerHandle {
    wsvd_layer_t h = nullptr;
    ~LayerHandle() {
        if (h) wsvd_layer_destroy(h);
    }
};

std::unique_ptr<LayerHandle> upload(const LayerFactors& f, const DeviceOptions& opt) {
    if (f.heads.empty()) throw ShapeError("latent cache over zero heads");
    std::vector<int32_t> ranks;
    for (const HeadProjection& p : f.heads)
        for (const factorize::HeadFactors* hf : {&p.q, &p.k, &p.v}) ranks.push_back(static_cast<int32_t>(hf->rank));
    wsvd_layer_desc d{};
    d.embed_dim = static_cast<int32_t>(f.embed_dim);
    d.head_dim = static_cast<int32_t>(f.head_dim);
    d.n_heads = static_cast<int32_t>(f.heads.size());
    d.head_offset = 0;
    d.weight_dtype = static_cast<int32_t>(opt.weights);
    d.act_rotation = (opt.weights == Storage::I8 || opt.weights == Storage::I4) ? 1 : 0;
    d.device = opt.device;
    auto L = std::make_unique<LayerHandle>();
    throw_status(wsvd_layer_create(&d, ranks.data(), &L->h));
    for (std::size_t h = 0; h < f.heads.size(); ++h) {
        const factorize::HeadFactors* roles[3] = {&f.heads[h].q, &f.heads[h].k, &f.heads[h].v};
        for (int role = 0; role < 3; ++role) {
            const factorize::HeadFactors& hf = *roles[role];
            if (hf.a.rows() != f.embed_dim || hf.a.cols() != hf.rank || hf.b.rows() != hf.rank ||
                hf.b.cols() != f.head_dim)
                throw ShapeError("head " + std::to_string(h) + ": factor shapes disagree with the layer geometry");
            throw_status(wsvd_layer_set_head(L->h, static_cast<int32_t>(h), role, hf.a.data().data(),
                                             hf.b.data().data()));
        }
    }
    return L;
}

}  // namespace

const char* stream_name(Stream s) {
    static const char* names[] = {"latent_k", "latent_v", "full_k", "full_v", "weights_b", "query", "output"};
    return names[static_cast<std::size_t>(s)];
}

std::uint64_t TrafficCounter::total_loads() const {
    std::uint64_t t = 0;
    for (std::size_t i = 0; i < 7; ++i) t += c_[i];
    return t;
}

std::uint64_t TrafficCounter::total_stores() const {
    std::uint64_t t = 0;
    for (std::size_t i = 7; i < 14; ++i) t += c_[i];
    return t;
}

struct LatentCache::Impl {
    DeviceOptions opt;
    const LayerFactors* home = nullptr;
    std::map<const LayerFactors*, std::unique_ptr<LayerHandle>> layers;  // uploads by factor object
    wsvd_layer_t bound = nullptr;
    wsvd_cache_t cache = nullptr;
    std::size_t nh = 0, E = 0, H = 0, rpad = 0;
    std::vector<double> stage_k, stage_v;  // push() staging [batch][nh][rpad]
    mutable DevMem x, q, out;
    ~Impl() {
        if (cache) wsvd_cache_destroy(cache);
    }
    void bind(const LayerFactors& f) {
        if (f.heads.size() != nh)
            throw ShapeError("cache holds " + std::to_string(nh) + " heads, factors " + std::to_string(f.heads.size()));
        auto it = layers.find(&f);
        if (it == layers.end()) it = layers.emplace(&f, upload(f, opt)).first;
        if (it->second->h != bound) {
            throw_status(wsvd_cache_bind_layer(cache, it->second->h));
            bound = it->second->h;
        }
    }
};

LatentCache::LatentCache(const LayerFactors& f, const DeviceOptions& opt) : p_(std::make_unique<Impl>()) {
    p_->opt = opt;
    p_->home = &f;
    auto L = upload(f, opt);
    p_->bound = L->h;
    p_->nh = f.heads.size();
    p_->E = f.embed_dim;
    p_->H = f.head_dim;
    int32_t rp = 0;
    throw_status(wsvd_layer_rank_pad(L->h, &rp));
    p_->rpad = static_cast<std::size_t>(rp);
    throw_status(wsvd_cache_create(L->h, static_cast<int32_t>(opt.batch), static_cast<int32_t>(opt.capacity),
                                   static_cast<int32_t>(opt.cache), &p_->cache));
    p_->layers.emplace(&f, std::move(L));
    p_->stage_k.assign(opt.batch * p_->nh * p_->rpad, 0.0);
    p_->stage_v.assign(opt.batch * p_->nh * p_->rpad, 0.0);
}

LatentCache::~LatentCache() = default;
LatentCache::LatentCache(LatentCache&&) noexcept = default;
LatentCache& LatentCache::operator=(LatentCache&&) noexcept = default;

std::size_t LatentCache::length() const {
    int32_t n = 0;
    throw_status(wsvd_cache_length(p_->cache, &n));
    return static_cast<std::size_t>(n);
}
std::size_t LatentCache::n_heads() const { return p_->nh; }
std::size_t LatentCache::batch() const { return p_->opt.batch; }
wsvd_cache_t LatentCache::handle() const { return p_->cache; }
const DeviceOptions& LatentCache::options() const { return p_->opt; }

wsvd_layer_t LatentCache::layer_for(const LayerFactors& f) const {
    p_->bind(f);
    return p_->bound;
}

static Matrix read_latents(const LatentCache& c, std::size_t head, std::size_t seq, std::size_t rank, bool k_part,
                           std::size_t rpad) {
    const std::size_t L = c.length();
    std::vector<double> ck(L * rpad), cv(L * rpad);
    throw_status(wsvd_cache_read_host(c.handle(), static_cast<int32_t>(seq), static_cast<int32_t>(head), ck.data(),
                                      cv.data()));
    Matrix m(L, rank);
    const std::vector<double>& src = k_part ? ck : cv;
    for (std::size_t t = 0; t < L; ++t)
        for (std::size_t j = 0; j < rank; ++j) m(t, j) = src[t * rpad + j];
    return m;
}

Matrix LatentCache::latent_k(std::size_t head, std::size_t seq) const {
    const auto& f = *p_->home;
    return read_latents(*this, head, seq, f.heads.at(head).k.rank, true, p_->rpad);
}

Matrix LatentCache::latent_v(std::size_t head, std::size_t seq) const {
    const auto& f = *p_->home;
    return read_latents(*this, head, seq, f.heads.at(head).v.rank, false, p_->rpad);
}

void LatentCache::push(std::size_t head, std::span<const double> ck, std::span<const double> cv) {
    if (head >= p_->nh) throw ShapeError("push: head out of range");
    const auto& hp = p_->home->heads[head];
    if (ck.size() != hp.k.rank || cv.size() != hp.v.rank) throw ShapeError("push: row width differs from the rank");
    for (std::size_t b = 0; b < p_->opt.batch; ++b) {
        std::copy(ck.begin(), ck.end(), p_->stage_k.begin() + (b * p_->nh + head) * p_->rpad);
        std::copy(cv.begin(), cv.end(), p_->stage_v.begin() + (b * p_->nh + head) * p_->rpad);
    }
}

void LatentCache::bump_length() {
    throw_status(wsvd_cache_push_host(p_->cache, p_->stage_k.data(), p_->stage_v.data()));
    std::fill(p_->stage_k.begin(), p_->stage_k.end(), 0.0);
    std::fill(p_->stage_v.begin(), p_->stage_v.end(), 0.0);
}

static Matrix append_impl(LatentCache& cache, const LayerFactors& f, const double* x, std::size_t rows,
                          TrafficCounter* counter) {
    const std::size_t E = f.embed_dim, nh = f.heads.size(), H = f.head_dim;
    wsvd_cache_t h = cache.handle();
    cache.layer_for(f);  // binds (and validates the head count)
    std::vector<float> xf(rows * E);
    for (std::size_t i = 0; i < xf.size(); ++i) {
        if (!std::isfinite(x[i])) throw NumericError("append_token: non-finite token");
        xf[i] = static_cast<float>(x[i]);
    }
    DevMem xd, qd;
    xd.ensure(xf.size() * 4);
    qd.ensure(rows * nh * H * 4);
    check_cuda(cudaMemcpy(xd.p, xf.data(), xf.size() * 4, cudaMemcpyHostToDevice), "copy token");
    throw_status(wsvd_append_token(h, static_cast<const float*>(xd.p), static_cast<float*>(qd.p), cache.options().stream));
    std::vector<float> qf(rows * nh * H);
    check_cuda(cudaMemcpy(qf.data(), qd.p, qf.size() * 4, cudaMemcpyDeviceToHost), "copy query");
    if (counter) throw_status(wsvd_traffic_append(h, counter->raw()));
    Matrix q(rows * nh, H);
    for (std::size_t i = 0; i < qf.size(); ++i) q.data()[i] = qf[i];
    return q;
}

Matrix append_token(LatentCache& cache, const LayerFactors& f, std::span<const double> x, TrafficCounter* counter) {
    if (x.size() != f.embed_dim)
        throw ShapeError("token has " + std::to_string(x.size()) + " features, layer expects " +
                         std::to_string(f.embed_dim));
    if (cache.batch() != 1) throw ShapeError("single-token append on a batched cache: pass one row per sequence");
    return append_impl(cache, f, x.data(), 1, counter);
}

Matrix append_token(LatentCache& cache, const LayerFactors& f, const Matrix& x, TrafficCounter* counter) {
    if (x.cols() != f.embed_dim)
        throw ShapeError("token has " + std::to_string(x.cols()) + " features, layer expects " +
                         std::to_string(f.embed_dim));
    if (x.rows() != cache.batch())
        throw ShapeError(std::to_string(x.rows()) + " token rows for " + std::to_string(cache.batch()) + " sequences");
    return append_impl(cache, f, x.data().data(), x.rows(), counter);
}

Matrix fused_decode_step(const LatentCache& cache, const LayerFactors& f, const Matrix& q_heads,
                         const TileConfig& tiles, TrafficCounter& counter) {
    if (cache.length() == 0) throw ShapeError("decode step over an empty cache");
    const std::size_t nh = f.heads.size(), H = f.head_dim;
    if (cache.n_heads() != nh)
        throw ShapeError("cache holds " + std::to_string(cache.n_heads()) + " heads, factors " + std::to_string(nh));
    if (q_heads.rows() != cache.batch() * nh || q_heads.cols() != H)
        throw ShapeError("query block must be " + std::to_string(cache.batch() * nh) + "x" + std::to_string(H) +
                         ", got " + std::to_string(q_heads.rows()) + "x" + std::to_string(q_heads.cols()));
    if (tiles.tile_len == 0) throw ConfigError("tile length must be >= 1");
    cache.layer_for(f);
    std::vector<float> qf(q_heads.size());
    for (std::size_t i = 0; i < qf.size(); ++i) qf[i] = static_cast<float>(q_heads.data()[i]);
    DevMem qd, od;
    qd.ensure(qf.size() * 4);
    od.ensure(qf.size() * 4);
    check_cuda(cudaMemcpy(qd.p, qf.data(), qf.size() * 4, cudaMemcpyHostToDevice), "copy query");
    const int32_t tile = static_cast<int32_t>(std::min<std::size_t>(tiles.tile_len, 1u << 30));
    throw_status(wsvd_fused_decode_step(cache.handle(), static_cast<const float*>(qd.p), tile,
                                        static_cast<float*>(od.p), cache.options().stream));
    std::vector<float> of(qf.size());
    check_cuda(cudaMemcpy(of.data(), od.p, of.size() * 4, cudaMemcpyDeviceToHost), "copy output");
    throw_status(wsvd_traffic_fused(cache.handle(), tile, counter.raw()));
    Matrix out(q_heads.rows(), H);
    for (std::size_t i = 0; i < of.size(); ++i) out.data()[i] = of[i];
    return out;
}

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
    TrafficReport rep;
    rep.mode = mode;
    rep.seq_len = seq_len;
    rep.n_heads = n_heads;
    const std::uint64_t width = mode == Mode::Fused ? rank_k : mode == Mode::SharedLatent ? shared_rank : head_dim;
    rep.analytic_eta = seq_len * width;
    rep.analytic_gamma = (mode == Mode::Fused || mode == Mode::SharedLatent) ? seq_len * width * head_dim : 0;
    const bool latent = mode == Mode::Fused || mode == Mode::SharedLatent;
    const StreamTally st = counter[latent ? Stream::LatentK : Stream::FullK];
    const bool divisible = st.loads % n_heads == 0 && st.flops % n_heads == 0;
    rep.measured_cache_loads_per_head = divisible ? st.loads / n_heads : 0;
    rep.measured_reconstruction_flops_per_head = divisible ? st.flops / n_heads : 0;
    rep.match = divisible && rep.measured_cache_loads_per_head == rep.analytic_eta &&
                rep.measured_reconstruction_flops_per_head == rep.analytic_gamma;
    rep.bytes_loaded_fp64 = 8.0 * static_cast<double>(counter.total_loads());
    rep.bytes_loaded_fp16 = 2.0 * static_cast<double>(counter.total_loads());
    return rep;
}

}  // namespace wsvd::decode
