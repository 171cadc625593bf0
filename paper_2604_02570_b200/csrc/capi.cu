// capi.cu -- the extern "C" boundary (include/wsvd_b200.h): device-resident
// layers and latent caches, operator launches, CUDA-graph replay, NCCL.
//
// Host-side responsibilities that the reference keeps inside its operators:
//   * shape / config validation with the reference's error classes
//     (decode.cpp:117-123, 129-131, 158-163, 112-115 -> WSVD_ESHAPE/ECONFIG);
//   * the TrafficCounter closed forms (decode.cpp:132-149, 176-203);
//   * factor preparation: rounding to bf16/fp32, or the reference weight
//     quantiser (quant.cpp:99-119) after the S1 rotation (quant.cpp:182-189).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wsvd_b200.h"
#include "kernels.h"

using namespace wsvd_k;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return set_err(WSVD_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// host copy of cache_swz (common.cuh): the 16-byte XOR swizzle of cache rows
uint32_t wsvd_dev_swz(uint32_t a) { return a ^ (((a >> 7) & 7u) << 4); }

// W-tiles (gemm.cu): rows [nrows][row_bytes] -> [nrows/16][row_bytes/ksb][16][ksb],
// the 16-byte units of odd rows XOR 4.  nrows must be a multiple of 16.
void pack_wtiles(const uint8_t* rows, int nrows, int row_bytes, int ksb, uint8_t* out) {
    const int splits = row_bytes / ksb, units = ksb / 16;
    for (int r = 0; r < nrows; ++r) {
        const int tile = r / 16, rr = r % 16;
        for (int s = 0; s < splits; ++s)
            for (int u = 0; u < units; ++u) {
                const size_t dst = ((static_cast<size_t>(tile) * splits + s) * 16 + rr) * ksb +
                                   static_cast<size_t>(u ^ ((rr & 1) << 2)) * 16;
                std::memcpy(out + dst, rows + static_cast<size_t>(r) * row_bytes + static_cast<size_t>(s) * ksb + u * 16, 16);
            }
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t bytes) {
        if (p) cudaFree(p);
        p = nullptr;
        n = bytes;
        if (bytes == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
        return e;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

uint16_t f32_to_bf16_bits(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// Reference weight quantiser (quant.cpp:40-119): per-column symmetric RTN,
// clip ratio from the grid 0.50..1.00 (first minimum wins), llround, clamp
// to +-qmax, zero columns get scale 1.  w is row-major rows x cols.
double quantize_weight_ref(const std::vector<double>& w, size_t rows, size_t cols, int bits,
                           std::vector<int8_t>& q, std::vector<double>& scales) {
    const long long lim = (1LL << (bits - 1)) - 1;
    const double qd = static_cast<double>(lim);
    std::vector<double> maxabs(cols, 0.0), s(cols);
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) maxabs[j] = std::max(maxabs[j], std::abs(w[i * cols + j]));
    double best_clip = 0.5, best_err = -1.0;
    for (int g = 10; g <= 20; ++g) {
        const double clip = static_cast<double>(g) / 20.0;
        for (size_t j = 0; j < cols; ++j) s[j] = maxabs[j] == 0.0 ? 1.0 : clip * maxabs[j] / qd;
        double err = 0.0;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                const long long qi = std::clamp(std::llround(w[i * cols + j] / s[j]), -lim, lim);
                const double d = w[i * cols + j] - static_cast<double>(qi) * s[j];
                err += d * d;
            }
        if (best_err < 0.0 || err < best_err) {
            best_err = err;
            best_clip = clip;
        }
    }
    scales.assign(cols, 0.0);
    q.assign(rows * cols, 0);
    for (size_t j = 0; j < cols; ++j) scales[j] = maxabs[j] == 0.0 ? 1.0 : best_clip * maxabs[j] / qd;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j)
            q[i * cols + j] = static_cast<int8_t>(
                std::clamp(std::llround(w[i * cols + j] / scales[j]), -lim, lim));
    return best_clip;
}

// S1 = blockdiag(H_blk / sqrt(blk)) applied to the columns of a (E x r): fp64 FWHT.
void rotate_columns(std::vector<double>& a, size_t E, size_t r, size_t blk) {
    const double scale = 1.0 / std::sqrt(static_cast<double>(blk));
    std::vector<double> col(E);
    for (size_t j = 0; j < r; ++j) {
        for (size_t i = 0; i < E; ++i) col[i] = a[i * r + j];
        for (size_t b0 = 0; b0 < E; b0 += blk)
            for (size_t len = 1; len < blk; len <<= 1)
                for (size_t i = b0; i < b0 + blk; i += 2 * len)
                    for (size_t k = i; k < i + len; ++k) {
                        const double x = col[k], y = col[k + len];
                        col[k] = x + y;
                        col[k + len] = x - y;
                    }
        for (size_t i = 0; i < E; ++i) a[i * r + j] = col[i] * scale;
    }
}

size_t rot_block(size_t E) {
    if (E && !(E & (E - 1))) return E;
    if (E % 128 == 0) return 128;
    return 0;
}

int sm100_devices() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
    }
    return good;
}

// ------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    const char* (*errStr)(int) = nullptr;
    bool ok = false;
};

struct NcclId {
    char b[128];
};
using CommInitFn = int (*)(void**, int, NcclId, int);

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
        api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
        api.allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
            dlsym(h, "ncclAllReduce"));
        api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
        api.errStr = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.getUniqueId && api.allReduce && api.commDestroy && dlsym(h, "ncclCommInitRank");
    });
    return api;
}

}  // namespace

// ============================================================== handles ===
struct wsvd_layer_s {
    wsvd_layer_desc d{};
    int R = 0, Kp = 0, Nrows = 0;
    int bdtype = F32;                 // storage of B factors
    std::vector<int32_t> ranks;       // [nh][3]
    std::vector<uint8_t> have;        // [nh][3] uploaded
    DevBuf A;                         // [Nrows][Kp] (or Kp/2 for I4)
    DevBuf a_scale;                   // [Nrows] fp32
    DevBuf B[3];                      // [nh][R][H] per role
    DevBuf b_scale[3];                // [nh][H] per role
    int rot_blk = 0;
    float rot_scale = 1.f;
    // O-projection
    int e_out = 0, o_dtype = BF16, oKp = 0;
    int ks = 512, oks = 1024;         // K split of the projection / O-projection W-tiles
    DevBuf Wo;                        // [e_out][oKp] rows of W'_o = B_V . W_o (K = nh*R)
    std::vector<double> b_host[3];    // [nh][R][H] device B values per role (for host folds)
    DevBuf mqk;                       // [nh][R][R] qt_scale * B_Q . B_K^T (fp32)
    bool mqk_ready = false;
    DevBuf bkt;                       // [nh] B_K^T tiles for the tcgen05 attention (attn_tc.cu)
    DevBuf Atc;                       // bf16 A in K-chunk-major layout for the tcgen05 token GEMM
    unsigned atc_gen = ~0u;           // the generation Atc was built from
    bool bkt_ready = false;
    unsigned gen = 0;                 // bumped by every upload: captured step graphs go stale
};

struct GraphKey {
    const float* x = nullptr;
    float* y = nullptr;
    cudaStream_t s = nullptr;
};

struct wsvd_cache_s {
    wsvd_layer_s* L = nullptr;
    int B = 0, cap = 0, cap_alloc = 0, cdtype = BF16, row_bytes = 0;
    int len = 0;                      // host mirror of *d_len
    DevBuf data, scales, ctrl;        // ctrl: [0]=d_len, [1]=done
    DevBuf qt, q_tmp, attn_ws, attn_cnt, vlat;
    DevBuf P, xq, sx, xb;             // projection workspace (xb: bf16 token rows of the tcgen05 GEMM)
    int P_M = 0, P_splits = 0;        // rows / K splits of the last projection
    DevBuf oP, y_tmp;                 // O-proj partials
    DevBuf x_dev, y_dev;              // staging for the host-buffer step
    DevBuf trace;                     // fused-step phase timeline (WSVD_STEP_TRACE)
    DevBuf xo;                        // fused step: bf16 X rows of the O-projection
    DevBuf Pt;                        // fused step: tagged projection partials
    DevBuf xtag;                      // fused chain: tagged bf16 tokens between layers
    DevBuf fws;                       // fused step: per-CTA segment states
    DevBuf pP, pxo, pws;              // two-group chain (step2.cu): partials, O-proj rows, segment states
    DevBuf dbg;                       // test hook: int8 score accumulators [B*nh][cap_alloc][2]
    bool dbg_on = false;
    int attn_mode = 0;                // WSVD_ATTN_ABSORBED or WSVD_ATTN_EXPLICIT_TC
    DevBuf qfull;                     // [B][nh][H] query of the last append (explicit mode)
    int chunk = 512, max_chunks = 1, grid = 148;
    int fmax_chunks = 1;              // split-KV chunks of the fused step kernel
    int pair_ok = -1;                 // the fused step can run as resident CTA pairs (-1: not probed)
    int sms = 148;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaStream_t gstream = nullptr;
    bool gpending = false;
    GraphKey gkey;
    unsigned ggen = 0;                // layer generation and attention mode the graph captured
    int gmode = -1;
    // host-buffer step (wsvd_layer_step_host): mapped-pointer cache of the last buffers
    GraphKey hkey;
    bool hzc = false;
    const float* hx = nullptr;
    float* hy = nullptr;
    ~wsvd_cache_s() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        if (gstream) cudaStreamDestroy(gstream);
    }
    int* d_len() const { return ctrl.as<int>(); }
    int* d_done() const { return ctrl.as<int>() + 1; }
};

struct wsvd_ffn_s {
    int E = 0, F = 0, device = 0, sms = 148;
    int Kp1 = 0, Kp2 = 0;  // padded K of the two GEMMs (E, F)
    bool tc = false;       // E, F multiples of 64: tcgen05 GEMMs over plain row-major bf16 weights
    DevBuf W1, W2;         // tc: ff1^T [F][E], ff2^T [E][F] bf16; else W-tiles (rows n = output unit)
    DevBuf P, Hd, Xb;      // split partials; hidden activations; the bf16 input rows (tc)
};

struct wsvd_comm_s {
    void* comm = nullptr;
    int nranks = 1, rank = 0;
};

namespace {

int check_layer(wsvd_layer_t l) {
    if (!l) return set_err(WSVD_ECONFIG, "null layer handle");
    for (size_t i = 0; i < l->have.size(); ++i)
        if (!l->have[i])
            return set_err(WSVD_ECONFIG, "factors of head " + std::to_string(i / 3) + " role " +
                                             std::to_string(i % 3) + " were never uploaded");
    return WSVD_OK;
}

// projection of M token rows (fp32 x [M][E]) into the partial workspace
// Many token rows (prefill; steps at B >= 64) with bf16 weights: the dense
// projection on tcgen05 (gemm_tc.cu) over a K-chunk-major copy of A, its K
// splits left as partials for the append epilogue to sum in split order.
int run_projection_tc(wsvd_cache_s* c, const float* x, int M, cudaStream_t s, int* splits_out) {
    wsvd_layer_s* L = c->L;
    if (L->atc_gen != L->gen || !L->Atc.p) {
        CUDA_TRY(L->Atc.alloc(static_cast<size_t>(L->Nrows) * L->Kp * 2));
        CUDA_TRY(launch_wtiles_to_chunks(L->A.p, L->Nrows, L->Kp, L->ks, L->Atc.p, s));
        L->atc_gen = L->gen;
    }
    const int nt = L->Nrows / 64;
    const int splits = std::max(1, std::min(L->Kp / 64, c->sms / nt));
    const size_t need = static_cast<size_t>(splits) * M * L->Nrows * 4;
    if (c->P.n < need) CUDA_TRY(c->P.alloc(need));
    if (c->xb.n < static_cast<size_t>(128) * L->Kp * 2) CUDA_TRY(c->xb.alloc(static_cast<size_t>(128) * L->Kp * 2));
    for (int m0 = 0; m0 < M; m0 += 128) {
        const int mc = std::min(128, M - m0);
        CUDA_TRY(launch_f32_to_bf16(x + static_cast<size_t>(m0) * L->Kp, c->xb.p, static_cast<size_t>(mc) * L->Kp, s));
        TcGemmArgs g{c->xb.p, L->Atc.p, c->P.as<float>() + static_cast<size_t>(m0) * L->Nrows, mc, L->Nrows, L->Kp,
                     L->Nrows, splits, 0, 0, 0, 0, M};
        CUDA_TRY(launch_tc_gemm(g, s));
    }
    *splits_out = splits;
    c->P_M = M;
    c->P_splits = splits;
    return WSVD_OK;
}

int run_projection(wsvd_cache_s* c, const float* x, int M, cudaStream_t s, int* splits_out) {
    wsvd_layer_s* L = c->L;
    const int wd = L->d.weight_dtype;
    static const bool no_tc = getenv("WSVD_PROJ_SKINNY") != nullptr;  // A/B switch
    if (!no_tc && wd == BF16 && M >= 64 && L->Kp == L->d.embed_dim && L->Kp % 64 == 0 &&
        tc_gemm_supported(std::min(M, 128), L->Nrows, L->Kp))
        return run_projection_tc(c, x, M, s, splits_out);
    static const bool f32_rows = getenv("WSVD_F32_ROWS") != nullptr;  // A/B switch: the register GEMV
    const int ks = (wd == F32 && !f32_rows && f32_tma_path(M, L->Kp, L->Kp)) ? L->Kp
                   : (wd == F32 && f32_rows_path(M, L->Kp, 512)) ? 512 : L->ks;
    if (!gemm_fits(wd, M, ks))
        return set_err(WSVD_ECONFIG, std::to_string(M) + " token rows do not fit the projection kernel");
    const int splits = L->Kp / ks;
    const size_t need = static_cast<size_t>(splits) * M * L->Nrows * 4;
    if (c->P.n < need) CUDA_TRY(c->P.alloc(need));
    GemmArgs g{};
    g.W = L->A.p;
    g.P = c->P.p;
    g.M = M;
    g.N = L->Nrows;
    g.K = L->d.embed_dim;
    g.Kp = L->Kp;
    g.KS = ks;
    g.ldx = L->d.embed_dim;
    g.wdtype = wd;
    g.grid = c->sms;
    if (wd == I8 || wd == I4) {
        if (c->xq.n < static_cast<size_t>(M) * L->Kp) CUDA_TRY(c->xq.alloc(static_cast<size_t>(M) * L->Kp));
        if (c->sx.n < static_cast<size_t>(M) * 4) CUDA_TRY(c->sx.alloc(static_cast<size_t>(M) * 4));
        CUDA_TRY(launch_act_quant(x, M, L->d.embed_dim, L->Kp, L->d.act_rotation, L->rot_blk,
                                  L->rot_scale, c->xq.as<int8_t>(), c->sx.as<float>(), s));
        g.X = c->xq.p;
    } else {
        g.X = x;
    }
    CUDA_TRY(launch_gemm(g, s));
    *splits_out = splits;
    c->P_M = M;
    c->P_splits = splits;
    return WSVD_OK;
}

// M_QK[h] = qt_scale * B_Q[h] . B_K[h]^T (R x R, fp64 -> fp32) from the device's B values
int ensure_mqk(wsvd_layer_s* L) {
    if (L->mqk_ready) return WSVD_OK;
    const int nh = L->d.n_heads, R = L->R, H = L->d.head_dim;
    const double scale = 1.4426950408889634 / std::sqrt(static_cast<double>(H));
    std::vector<float> m(static_cast<size_t>(nh) * R * R);
    for (int h = 0; h < nh; ++h)
        for (int j = 0; j < R; ++j)
            for (int i = 0; i < R; ++i) {
                const double* bq = L->b_host[0].data() + (static_cast<size_t>(h) * R + j) * H;
                const double* bk = L->b_host[1].data() + (static_cast<size_t>(h) * R + i) * H;
                double acc = 0.0;
                for (int d = 0; d < H; ++d) acc += bq[d] * bk[d];
                m[(static_cast<size_t>(h) * R + j) * R + i] = static_cast<float>(acc * scale);
            }
    if (!L->mqk.p) CUDA_TRY(L->mqk.alloc(m.size() * 4));
    CUDA_TRY(cudaMemcpy(L->mqk.p, m.data(), m.size() * 4, cudaMemcpyHostToDevice));
    L->mqk_ready = true;
    return WSVD_OK;
}

// B_K^T of every head in the tcgen05 B-operand layout (attn_tc.cu), from the
// device's bf16 B_K values
int ensure_bkt(wsvd_layer_s* L) {
    if (L->bkt_ready) return WSVD_OK;
    const int nh = L->d.n_heads, R = L->R, H = L->d.head_dim;
    const size_t per = static_cast<size_t>(attn_tc_btile_bytes());
    std::vector<uint8_t> t(per * nh, 0);
    for (int h = 0; h < nh; ++h)
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < H; ++d) {
                const uint16_t v = f32_to_bf16_bits(static_cast<float>(L->b_host[1][(static_cast<size_t>(h) * R + r) * H + d]));
                std::memcpy(t.data() + h * per + attn_tc_btile_offset(d, r), &v, 2);
            }
    if (!L->bkt.p) CUDA_TRY(L->bkt.alloc(t.size()));
    CUDA_TRY(cudaMemcpy(L->bkt.p, t.data(), t.size(), cudaMemcpyHostToDevice));
    L->bkt_ready = true;
    return WSVD_OK;
}

int run_append(wsvd_cache_s* c, const float* x, int T, float* q_out, float* qt, int commit, cudaStream_t s) {
    wsvd_layer_s* L = c->L;
    const int M = T * c->B;
    if (qt && !q_out) {
        const int rc0 = ensure_mqk(L);
        if (rc0) return rc0;
    }
    int splits = 0;
    int rc = run_projection(c, x, M, s, &splits);
    if (rc) return rc;
    AppendArgs a{};
    a.P = c->P.p;
    a.splits = splits;
    a.M = M;
    a.Nrows = L->Nrows;
    a.wdtype = L->d.weight_dtype;
    a.a_scale = L->a_scale.as<float>();
    a.sx = c->sx.as<float>();
    a.T = T;
    a.B = c->B;
    a.nh = L->d.n_heads;
    a.R = L->R;
    a.H = L->d.head_dim;
    a.cache = c->data.as<uint8_t>();
    a.cscale = c->scales.as<__half2>();
    a.cdtype = c->cdtype;
    a.cap = c->cap_alloc;
    a.row_bytes = c->row_bytes;
    a.d_len = c->d_len();
    a.done = c->d_done();
    a.bq = L->B[0].p;
    a.bk = L->B[1].p;
    a.bq_scale = L->b_scale[0].as<float>();
    a.bk_scale = L->b_scale[1].as<float>();
    a.bdtype = L->bdtype;
    a.q_out = q_out;
    a.qt = qt;
    a.qt_scale = 1.4426950408889634f / std::sqrt(static_cast<float>(L->d.head_dim));
    a.mqk = L->mqk.as<float>();
    a.commit = commit;
    CUDA_TRY(launch_append_epilogue(a, s));
    return WSVD_OK;
}

// out: per-head outputs (B_V applied) or null; vlat: latent outputs or null;
// len_add: rows appended by this step but not yet committed to *d_len
// Cluster size of the layer step's attention (latent outputs): few (sequence,
// head) pairs get clusters of C CTAs, one unit each, C chunks per pair merged
// through DSMEM in the kernel (no combine launch); 1 = not used.
int attn_cluster_for(const wsvd_cache_s* c) {
    static const bool no_cl = getenv("WSVD_ATTN_NOCLUSTER") != nullptr;  // A/B switch
    static const bool no_fin = getenv("WSVD_ATTN_COMBINE") != nullptr;
    const wsvd_layer_s* L = c->L;
    if (no_cl || no_fin || c->chunk != 0 || c->attn_mode == WSVD_ATTN_EXPLICIT_TC) return 1;
    const int pairs = c->B * L->d.n_heads;
    for (int C = 8; C >= 2; C /= 2)
        if (pairs * C <= c->grid)
            return (C <= c->max_chunks && attn_cluster_ok(c->cdtype, L->R, C)) ? C : 1;
    return 1;
}

int run_attention(wsvd_cache_s* c, float* out, float* vlat, int len_add, cudaStream_t s,
                  const float* q = nullptr) {
    wsvd_layer_s* L = c->L;
    AttnArgs a{};
    a.cache = c->data.as<uint8_t>();
    a.cscale = c->scales.as<__half2>();
    a.qt = c->qt.as<float>();
    a.bv = L->B[2].p;
    a.bv_scale = L->b_scale[2].as<float>();
    a.bdtype = L->bdtype;
    a.out = out;
    a.vlat = vlat;
    a.ws = c->attn_ws.as<float>();
    a.counters = c->attn_cnt.as<int>();
    a.d_len = c->d_len();
    a.len_add = len_add;
    a.B = c->B;
    a.nh = L->d.n_heads;
    a.H = L->d.head_dim;
    a.R = L->R;
    a.cap = c->cap_alloc;
    a.chunk = c->chunk;
    a.max_chunks = c->max_chunks;
    a.cdtype = c->cdtype;
    a.row_bytes = c->row_bytes;
    a.grid = c->grid;
    a.dbg_scores = c->dbg_on ? c->dbg.as<int>() : nullptr;
    static const bool no_fin = getenv("WSVD_ATTN_COMBINE") != nullptr;
    a.no_finalize = no_fin ? 1 : 0;
    // Few (sequence, head) pairs (e.g. one sequence): clusters of C CTAs, one
    // unit each, C chunks per pair merged through DSMEM inside the kernel
    // instead of the combine launch (layer step: latent outputs only)
    a.cluster = 1;
    if (out == nullptr && vlat != nullptr) {
        const int cl = attn_cluster_for(c);
        if (cl > 1) {
            a.cluster = cl;
            a.max_chunks = cl;  // <= the cache's max_chunks: every (sequence, head) ws slot exists
            a.grid = c->B * L->d.n_heads * cl;
        }
    }
    if (c->attn_mode == WSVD_ATTN_EXPLICIT_TC) {
        // explicit key reconstruction on tcgen05 (attn_tc.cu), then the combine
        int rc = ensure_bkt(L);
        if (rc) return rc;
        a.bkt = L->bkt.as<uint8_t>();
        a.q = q ? q : c->qfull.as<float>();
        a.grid = c->sms;
        CUDA_TRY(launch_decode_attn_tc(a, s));
        CUDA_TRY(launch_attn_combine(a, 8, s));
        return WSVD_OK;
    }
    CUDA_TRY(launch_decode_attn(a, s));
    return WSVD_OK;
}

// y = vlat . (B_V W_o): the V-path up-projection folded into the output
// projection (SPEC section 3.4, "B_Vh is fused into the output projection").
// bf16 W'_o: the fp32 latents enter the tensor cores as hi + lo bf16 token
// tiles (xsplit), 64 sequences per GEMM launch.
int run_oproj(wsvd_cache_s* c, const float* vlat, float* y, int* commit_len, cudaStream_t s) {
    wsvd_layer_s* L = c->L;
    if (!L->Wo.p) return set_err(WSVD_ECONFIG, "layer has no O-projection (wsvd_layer_set_oproj)");
    const int K = L->d.n_heads * L->R;
    const bool split = L->o_dtype == BF16;
    const int mchunk = split ? 64 : c->B;
    const int ks = L->oks;
    if (!gemm_fits(L->o_dtype, split ? 2 * std::min(c->B, mchunk) : c->B, ks))
        return set_err(WSVD_ECONFIG, "batch of " + std::to_string(c->B) + " does not fit the O-projection kernel");
    const int splits = L->oKp / ks;
    const size_t need = static_cast<size_t>(splits) * c->B * L->e_out * 4;
    if (c->oP.n < need) CUDA_TRY(c->oP.alloc(need));
    for (int m0 = 0; m0 < c->B; m0 += mchunk) {
        const int M = std::min(mchunk, c->B - m0);
        GemmArgs g{};
        g.W = L->Wo.p;
        g.X = vlat + static_cast<size_t>(m0) * K;
        float* yc = y + static_cast<size_t>(m0) * L->e_out;
        float* pc = c->oP.as<float>() + static_cast<size_t>(splits) * m0 * L->e_out;  // [splits][M][N] per chunk
        g.P = splits == 1 ? static_cast<void*>(yc) : static_cast<void*>(pc);
        g.commit_len = m0 == 0 ? commit_len : nullptr;
        g.M = M;
        g.N = L->e_out;
        g.K = K;
        g.Kp = L->oKp;
        g.KS = ks;
        g.ldx = K;
        g.wdtype = L->o_dtype;
        g.grid = c->sms;
        g.xsplit = split ? 1 : 0;
        CUDA_TRY(launch_gemm(g, s));
        if (splits > 1) CUDA_TRY(launch_reduce_partials(pc, splits, M, L->e_out, yc, s));
    }
    return WSVD_OK;
}

bool fused_step_ok(wsvd_cache_s* c) {
    static const bool off = getenv("WSVD_STEP_MULTI") != nullptr;  // A/B switch: multi-kernel step
    const wsvd_layer_s* L = c->L;
    if (off || c->attn_mode != WSVD_ATTN_ABSORBED) return false;
    if (c->cdtype != BF16 || L->d.weight_dtype != BF16 || L->o_dtype != BF16 || !L->Wo.p) return false;
    if (L->ks != step_item_k() || L->oks != step_item_k()) return false;
    // the chunk count never exceeds max_chunks (adaptive) or the capacity split (fixed chunk)
    const int mc = c->chunk > 0 ? c->max_chunks : c->fmax_chunks;
    // one CTA per SM must be resident (grid barriers): probed once per batch tile
    static int occ[3] = {-1, -1, -1};
    const int mt = (c->B + 15) / 16;
    if (mt >= 1 && mt <= 2 && occ[mt] < 0) occ[mt] = step_resident_ctas_per_sm(c->B);
    if (mt >= 1 && mt <= 2 && occ[mt] < 1) return false;
    (void)mc;
    return step_supported(L->R, c->B, L->d.n_heads, L->Kp, L->oKp, round_up(L->e_out, 16) / 16, c->sms);
}

// The fused step's grid barriers need all of its CTAs (one per SM) resident
// at once, so two fused steps must never run concurrently on one device (each
// would hold some SMs and wait for the other's).  Steps on one stream are
// ordered anyway; when a fused step is issued on a different stream than the
// device's previous one, the new stream first waits for everything issued on
// the old one.  Nothing is recorded in the steady state (one stream), so the
// PDL overlap of back-to-back steps is untouched.
struct FusedOrder {
    std::mutex mu;
    cudaStream_t last = nullptr;
    bool any = false;
    cudaEvent_t ev = nullptr;
};

int fused_serialize(int device, cudaStream_t s) {
    static FusedOrder order[64];
    if (device < 0 || device >= 64) return WSVD_OK;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return WSVD_OK;  // inside a caller's graph: the graph's own edges order it
    }
    FusedOrder& o = order[device];
    std::lock_guard<std::mutex> lk(o.mu);
    if (o.any && o.last != s) {
        if (!o.ev) CUDA_TRY(cudaEventCreateWithFlags(&o.ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(o.ev, o.last));
        CUDA_TRY(cudaStreamWaitEvent(s, o.ev, 0));
    }
    o.last = s;
    o.any = true;
    return WSVD_OK;
}

// The whole step as one persistent kernel (step.cu), for a chain of n layers
// (n = 1: one layer step).  Layer l's token is ys[l - 1] (l > 0); the launch's
// control block, workspaces and trace are the first cache's.  x_host / y_host:
// x (layer 0) / ys[n - 1] are mapped pinned host memory.
int run_chain_fused(wsvd_cache_s* const* cs, int n, const float* x, float* const* ys, cudaStream_t s,
                    bool x_host = false, bool y_host = false) {
    wsvd_cache_s* c = cs[0];
    wsvd_layer_s* L = c->L;
    if (n < 1 || n > kStepMaxLayers) return set_err(WSVD_ECONFIG, "a fused chain holds 1 .. " + std::to_string(kStepMaxLayers) + " layers");
    StepArgs a{};
    for (int l = 0; l < n; ++l) {
        int rc = ensure_mqk(cs[l]->L);
        if (rc) return rc;
        StepLayer& Ly = a.layer[l];
        Ly.A = cs[l]->L->A.as<uint8_t>();
        Ly.mqk = cs[l]->L->mqk.as<float>();
        Ly.cache = cs[l]->data.as<uint8_t>();
        Ly.counters = cs[l]->attn_cnt.as<int>();
        Ly.Wo = cs[l]->L->Wo.as<uint8_t>();
        Ly.d_len = cs[l]->d_len();
        Ly.y = ys[l];
        Ly.cap = cs[l]->cap_alloc;
    }
    a.nlayers = n;
    const int splits = L->Kp / L->ks;
    a.x = x;
    a.x_host = x_host ? 1 : 0;
    a.y_host = y_host ? 1 : 0;
    if (x_host) {
        const size_t xb = static_cast<size_t>(c->B) * L->d.embed_dim * 4;
        if (c->x_dev.n < xb) CUDA_TRY(c->x_dev.alloc(xb));
        a.xd = c->x_dev.as<float>();
    }
    const size_t needt = static_cast<size_t>(splits) * c->B * L->Nrows * 8;
    if (c->Pt.n < needt) CUDA_TRY(c->Pt.alloc(needt));  // zeroed: tag 0 is never a layer step's
    a.Pt = c->Pt.as<unsigned long long>();
    // ctrl: [0] len [1] done [2] fused launches [4] grid barrier [5] barrier generations [16..32) x-fetch counters
    a.bar = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 4);
    a.bgen = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 5);
    a.epoch = c->ctrl.as<int>() + 2;
    a.xcnt = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 16);
    a.p1gen = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 3);
    a.yflag = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 256);  // one 128-byte line per CTA
    static const int g1 = std::getenv("WSVD_STEP_G1") ? std::atoi(std::getenv("WSVD_STEP_G1")) : 0;
    static const int g3 = std::getenv("WSVD_STEP_G3") ? std::atoi(std::getenv("WSVD_STEP_G3")) : 0;
    a.g1 = g1;
    a.g3 = g3;
    static const int short_seg = std::getenv("WSVD_STEP_SHORTSEG") ? std::atoi(std::getenv("WSVD_STEP_SHORTSEG")) : 2048;
    a.short_seg = short_seg;
    const size_t xob = 2 * step_xo_bytes(c->B, L->oKp);  // one per layer parity (chained layers overlap)
    if (c->xo.n < xob) CUDA_TRY(c->xo.alloc(xob));       // zeroed: rows past the batch stay 0
    a.xo = c->xo.as<uint8_t>();
    const size_t wsb = step_ws_bytes(c->sms);
    if (c->fws.n < wsb) CUDA_TRY(c->fws.alloc(wsb));
    a.ws = c->fws.as<float>();
    a.B = c->B;
    a.nh = L->d.n_heads;
    a.E = L->d.embed_dim;
    a.Kp = L->Kp;
    a.Nrows = L->Nrows;
    a.e_out = L->e_out;
    a.oKp = L->oKp;
    a.otiles = round_up(L->e_out, 16) / 16;
    a.grid = c->sms;
    // CTA pairs: the region a pair shares meets through DSMEM (WSVD_STEP_NOCLUSTER=1: through L2)
    static const bool no_cluster = getenv("WSVD_STEP_NOCLUSTER") != nullptr;
    if (c->pair_ok < 0) c->pair_ok = step_pair_clusters_ok(c->B, c->sms);
    a.cluster = (!no_cluster && c->pair_ok == 1) ? 2 : 1;
    // without pairs, two K splits of the O-projection meet in y by red.add onto
    // zeros each CTA writes after its projection: a y aliasing x needs every
    // CTA's token consumed first -- the grid barrier
    if (a.cluster != 2 && L->oKp / L->oks == 2 && a.g1 == 0) a.g1 = 1;
    // chained layers with pair O-projections: the next layer's token also as
    // tagged bf16 pairs (its projection validates each word: no flag round trip)
    static const bool no_xtag = getenv("WSVD_STEP_NOXTAG") != nullptr;  // A/B switch
    a.xtagged = (!no_xtag && n > 1 && a.cluster == 2 && L->oKp / L->oks == 2 && a.E % L->ks == 0 && a.g3 == 0) ? 1 : 0;
    if (a.xtagged) {
        const size_t xtb = 2 * static_cast<size_t>(c->B) * a.E / 2 * 8;
        if (c->xtag.n < xtb) CUDA_TRY(c->xtag.alloc(xtb));
        a.xtag = c->xtag.as<unsigned long long>();
    }
    // L2 prefetch of the first cache stages before the grid-dependency wait, at
    // the host mirror's length (unknown inside a caller's graph capture)
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap_st) != cudaSuccess) cudaGetLastError();
    a.pos_hint = cap_st == cudaStreamCaptureStatusNone ? c->len : -1;
    static const int pre = getenv("WSVD_STEP_PRE") ? atoi(getenv("WSVD_STEP_PRE")) : 0;  // A/B: stages (measured: 0 best)
    a.pre_stages = std::max(0, pre);
    static const bool p3_tma = getenv("WSVD_STEP_P3TMA") && std::string(getenv("WSVD_STEP_P3TMA")) == "1";
    a.p3_tma = p3_tma ? 1 : 0;
    static const bool x_first = !(getenv("WSVD_STEP_XFIRST") && std::string(getenv("WSVD_STEP_XFIRST")) == "0");
    a.x_first = x_first ? 1 : 0;
    static const int l2n = getenv("WSVD_STEP_L2NEXT") ? atoi(getenv("WSVD_STEP_L2NEXT")) : 1;  // A/B switch
    a.l2_next = l2n;
    // the next layer's first stages per CTA into L2 once this CTA's O-projection
    // is done (every attention stream has ended: HBM is idle until the next
    // layer's starts): 4 measured best (54.1 -> 53.4 us per layer; 8+ no gain)
    static const int cpre = getenv("WSVD_CHAIN_PRE") ? atoi(getenv("WSVD_CHAIN_PRE")) : 4;  // A/B switch
    a.chain_pre = cpre;
    static const bool trace = getenv("WSVD_STEP_TRACE") != nullptr;  // phase timeline (debug_copy 4)
    static const int trace_layer = getenv("WSVD_STEP_TRACE_LAYER") ? atoi(getenv("WSVD_STEP_TRACE_LAYER")) : -1;
    if (trace && !c->trace.p) CUDA_TRY(c->trace.alloc(static_cast<size_t>(c->sms) * 32 * 8));
    a.trace = trace ? c->trace.as<uint64_t>() : nullptr;
    a.trace_layer = trace_layer >= 0 && trace_layer < n ? trace_layer : n - 1;  // default: the last layer
    int rc = fused_serialize(L->d.device, s);
    if (rc) return rc;
    CUDA_TRY(launch_layer_step(a, s));
    c->P_M = 0;  // (the fused step's partials are tagged, in Pt: nothing for debug_copy)
    return WSVD_OK;
}

// The chain as two batch groups half a layer apart (step2.cu); workspaces and
// control words (ctrl[6..9]: per group barrier count and generations) are the
// first cache's.
bool chain_pipe_ok(wsvd_cache_s* const* cs, int n) {
    // opt-in (WSVD_CHAIN_PIPE=1): measured slower than the one-group chain on
    // B200 -- the hidden phases run at loaded latencies
    static const bool on = getenv("WSVD_CHAIN_PIPE") && std::string(getenv("WSVD_CHAIN_PIPE")) == "1";
    if (!on || n < 1 || n > kStepMaxLayers) return false;
    const wsvd_cache_s* c = cs[0];
    const wsvd_layer_s* L = c->L;
    if (!pipe_supported(L->R, c->B, L->d.n_heads, L->Kp, L->oKp, round_up(L->e_out, 16) / 16, c->sms)) return false;
    static int occ = -1;
    if (occ < 0) occ = pipe_resident_ctas_per_sm();
    return occ >= 1;
}

int run_chain_pipe(wsvd_cache_s* const* cs, int n, const float* x, float* const* ys, cudaStream_t s) {
    wsvd_cache_s* c = cs[0];
    wsvd_layer_s* L = c->L;
    PipeArgs a{};
    for (int l = 0; l < n; ++l) {
        int rc = ensure_mqk(cs[l]->L);
        if (rc) return rc;
        StepLayer& Ly = a.layer[l];
        Ly.A = cs[l]->L->A.as<uint8_t>();
        Ly.mqk = cs[l]->L->mqk.as<float>();
        Ly.cache = cs[l]->data.as<uint8_t>();
        Ly.counters = cs[l]->attn_cnt.as<int>();
        Ly.Wo = cs[l]->L->Wo.as<uint8_t>();
        Ly.d_len = cs[l]->d_len();
        Ly.y = ys[l];
        Ly.cap = cs[l]->cap_alloc;
    }
    a.nlayers = n;
    a.x = x;
    const size_t pb = pipe_p_bytes(L->Kp, L->Nrows), xb = pipe_xo_bytes(L->oKp), wb = pipe_ws_bytes(c->sms);
    if (c->pP.n < 2 * pb) CUDA_TRY(c->pP.alloc(2 * pb));
    if (c->pxo.n < 2 * xb) CUDA_TRY(c->pxo.alloc(2 * xb));  // zeroed: rows past a group's batch stay 0
    if (c->pws.n < 2 * wb) CUDA_TRY(c->pws.alloc(2 * wb));
    for (int g = 0; g < 2; ++g) {
        a.bar[g] = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 6 + 2 * g);
        a.bgen[g] = reinterpret_cast<unsigned*>(c->ctrl.as<int>() + 7 + 2 * g);
        a.P[g] = reinterpret_cast<float*>(c->pP.as<uint8_t>() + g * pb);
        a.xo[g] = c->pxo.as<uint8_t>() + g * xb;
        a.ws[g] = reinterpret_cast<float*>(c->pws.as<uint8_t>() + g * wb);
    }
    a.B = c->B;
    a.nh = L->d.n_heads;
    a.E = L->d.embed_dim;
    a.Kp = L->Kp;
    a.Nrows = L->Nrows;
    a.e_out = L->e_out;
    a.oKp = L->oKp;
    a.otiles = round_up(L->e_out, 16) / 16;
    a.grid = c->sms;
    static const bool no_cluster = getenv("WSVD_STEP_NOCLUSTER") != nullptr;
    static int pair = -1;
    if (pair < 0) pair = pipe_pair_clusters_ok(c->sms);
    a.cluster = (!no_cluster && pair == 1) ? 2 : 1;
    static const bool trace = getenv("WSVD_STEP_TRACE") != nullptr;
    static const int trace_layer = getenv("WSVD_STEP_TRACE_LAYER") ? atoi(getenv("WSVD_STEP_TRACE_LAYER")) : -1;
    static const int trace_group = getenv("WSVD_STEP_TRACE_GROUP") ? atoi(getenv("WSVD_STEP_TRACE_GROUP")) : 0;
    if (trace && !c->trace.p) CUDA_TRY(c->trace.alloc(static_cast<size_t>(c->sms) * 32 * 8));
    a.trace = trace ? c->trace.as<uint64_t>() : nullptr;
    a.trace_layer = trace_layer >= 0 && trace_layer < n ? trace_layer : n - 1;
    a.trace_group = trace_group & 1;
    int rc = fused_serialize(L->d.device, s);
    if (rc) return rc;
    static int* dbg_host = nullptr;
    static int* dbg_dev = nullptr;
    if (!dbg_host && getenv("WSVD_PIPE_DEBUG")) {
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&dbg_host), 4 * 4096, cudaHostAllocMapped));
        std::memset(dbg_host, 0, 4 * 4096);
        CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dbg_dev), dbg_host, 0));
        pipe_set_debug(dbg_dev);
    }
    CUDA_TRY(launch_chain_pipe(a, s));
    if (dbg_host) {
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess || dbg_host[0] > 0) {
            fprintf(stderr, "[pipe debug] %s, %d stuck waits (cta thread tag parity):\n", cudaGetErrorString(e), dbg_host[0]);
            for (int k = 0; k < std::min(dbg_host[0], 1000); ++k)
                fprintf(stderr, "  %d %d %d %d\n", dbg_host[1 + 4 * k], dbg_host[2 + 4 * k], dbg_host[3 + 4 * k], dbg_host[4 + 4 * k]);
            fflush(stderr);
        }
    }
    return WSVD_OK;
}

int run_step_fused(wsvd_cache_s* c, const float* x, float* y, cudaStream_t s, bool x_host = false) {
    wsvd_cache_s* cs[1] = {c};
    float* ys[1] = {y};
    return run_chain_fused(cs, 1, x, ys, s, x_host, x_host);
}

// append (row written, length not yet committed) -> attention over len + 1
// -> combine -> folded O-projection, whose first thread commits the length
int layer_step_impl(wsvd_cache_s* c, const float* x, float* attn_out, float* y, cudaStream_t s) {
    if (attn_out == nullptr && fused_step_ok(c)) return run_step_fused(c, x, y, s);
    const bool tc = c->attn_mode == WSVD_ATTN_EXPLICIT_TC;
    int rc = tc ? run_append(c, x, 1, c->qfull.as<float>(), nullptr, 0, s)
                : run_append(c, x, 1, nullptr, c->qt.as<float>(), 0, s);
    if (rc) return rc;
    rc = run_attention(c, attn_out, c->vlat.as<float>(), 1, s);
    if (rc) return rc;
    return run_oproj(c, c->vlat.as<float>(), y, c->d_len(), s);
}

}  // namespace

// ================================================================= C ABI ===
extern "C" {

const char* wsvd_last_error(void) { return g_err.c_str(); }
int wsvd_abi_version(void) { return WSVD_ABI_VERSION; }

// error slot shared with the checkpoint reader (checkpoint.cpp); not in the header
void wsvd_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

int wsvd_device_count(int32_t* n) {
    if (!n) return set_err(WSVD_ECONFIG, "null output");
    *n = sm100_devices();
    return WSVD_OK;
}

int wsvd_layer_create(const wsvd_layer_desc* desc, const int32_t* ranks, wsvd_layer_t* out) {
    if (!desc || !ranks || !out) return set_err(WSVD_ECONFIG, "null argument");
    const wsvd_layer_desc& d = *desc;
    if (d.n_heads <= 0) return set_err(WSVD_ESHAPE, "latent cache over zero heads");
    if (d.embed_dim <= 0 || d.head_dim <= 0) return set_err(WSVD_ESHAPE, "empty layer geometry");
    if (d.weight_dtype < WSVD_F32 || d.weight_dtype > WSVD_I4)
        return set_err(WSVD_ECONFIG, "unknown weight dtype " + std::to_string(d.weight_dtype));
    if (d.act_rotation && d.weight_dtype != WSVD_I8 && d.weight_dtype != WSVD_I4)
        return set_err(WSVD_ECONFIG, "act_rotation applies to I8/I4 weights only");
    if (sm100_devices() == 0) return set_err(WSVD_ECUDA, "no sm_100 (B200) device visible");
    int rmax = 0;
    for (int i = 0; i < d.n_heads * 3; ++i) {
        if (ranks[i] <= 0 || ranks[i] > d.head_dim)
            return set_err(WSVD_ESHAPE, "rank " + std::to_string(ranks[i]) + " outside [1, head_dim]");
        rmax = std::max(rmax, static_cast<int>(ranks[i]));
    }
    // every head is zero-padded to one common width, a multiple of 16 (the
    // MMA k-step); the reference accepts any rank <= H (factorize.cpp:72-164),
    // the kernels any padded width up to 128 (= the LLaVA head dim)
    const int R = round_up(rmax, 16);
    if (R > 128)
        return set_err(WSVD_ECONFIG, "padded rank " + std::to_string(R) + " unsupported (max 128)");
    CUDA_TRY(cudaSetDevice(d.device));
    auto* L = new wsvd_layer_s();
    L->d = d;
    L->R = R;
    L->Kp = round_up(d.embed_dim, 256);
    L->ks = (L->Kp % 512 == 0 && d.weight_dtype != WSVD_F32) ? 512 : 256;
    L->Nrows = d.n_heads * 3 * R;
    L->ranks.assign(ranks, ranks + d.n_heads * 3);
    L->have.assign(d.n_heads * 3, 0);
    for (auto& bh : L->b_host) bh.assign(static_cast<size_t>(d.n_heads) * R * d.head_dim, 0.0);
    L->bdtype = (d.weight_dtype == WSVD_I4) ? I8 : d.weight_dtype;
    if (d.act_rotation) {
        const size_t blk = rot_block(static_cast<size_t>(d.embed_dim));
        if (!blk) {
            delete L;
            return set_err(WSVD_ESHAPE, "hadamard: embed_dim must be a power of two or a multiple of 128");
        }
        L->rot_blk = static_cast<int>(blk);
        L->rot_scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(blk)));
    }
    const size_t row_bytes = (d.weight_dtype == WSVD_I4) ? L->Kp / 2
                             : static_cast<size_t>(L->Kp) * (d.weight_dtype == WSVD_F32 ? 4 : d.weight_dtype == WSVD_BF16 ? 2 : 1);
    const size_t bel = (L->bdtype == F32) ? 4 : (L->bdtype == BF16 ? 2 : 1);
    cudaError_t e = L->A.alloc(static_cast<size_t>(L->Nrows) * row_bytes);
    if (e == cudaSuccess) e = L->a_scale.alloc(static_cast<size_t>(L->Nrows) * 4);
    for (int r = 0; r < 3 && e == cudaSuccess; ++r) {
        e = L->B[r].alloc(static_cast<size_t>(d.n_heads) * R * d.head_dim * bel);
        if (e == cudaSuccess) e = L->b_scale[r].alloc(static_cast<size_t>(d.n_heads) * d.head_dim * 4);
    }
    if (e != cudaSuccess) {
        delete L;
        return set_err(WSVD_ECUDA, std::string("layer allocation: ") + cudaGetErrorString(e));
    }
    *out = L;
    return WSVD_OK;
}

int wsvd_layer_destroy(wsvd_layer_t layer) {
    delete layer;
    return WSVD_OK;
}

int wsvd_layer_rank_pad(wsvd_layer_t layer, int32_t* rpad) {
    if (!layer || !rpad) return set_err(WSVD_ECONFIG, "null argument");
    *rpad = layer->R;
    return WSVD_OK;
}

static int upload_head(wsvd_layer_t L, int head, int role, const std::vector<int8_t>* aq,
                       const std::vector<double>* as, const std::vector<double>* af,
                       const std::vector<int8_t>* bq, const std::vector<double>* bs,
                       const std::vector<double>* bf) {
    const int E = L->d.embed_dim, H = L->d.head_dim, R = L->R;
    const int r = L->ranks[head * 3 + role];
    const int wd = L->d.weight_dtype;
    CUDA_TRY(cudaSetDevice(L->d.device));
    // ---- A: rows n = (head*3+role)*R + i, each the i-th column of a (E values)
    const size_t n0 = static_cast<size_t>(head * 3 + role) * R;
    const size_t rb = (wd == WSVD_I4) ? L->Kp / 2 : static_cast<size_t>(L->Kp) * (wd == WSVD_F32 ? 4 : wd == WSVD_BF16 ? 2 : 1);
    std::vector<uint8_t> rows(static_cast<size_t>(R) * rb, 0);
    std::vector<float> ascale(R, 1.f);
    for (int i = 0; i < r; ++i) {
        uint8_t* dst = rows.data() + static_cast<size_t>(i) * rb;
        for (int k = 0; k < E; ++k) {
            const size_t src = static_cast<size_t>(k) * r + i;
            if (wd == WSVD_F32) {
                reinterpret_cast<float*>(dst)[k] = static_cast<float>((*af)[src]);
            } else if (wd == WSVD_BF16) {
                reinterpret_cast<uint16_t*>(dst)[k] = f32_to_bf16_bits(static_cast<float>((*af)[src]));
            } else if (wd == WSVD_I8) {
                reinterpret_cast<int8_t*>(dst)[k] = (*aq)[src];
            } else {
                const int v = (*aq)[src];
                if (v < -7 || v > 7) return set_err(WSVD_ENUMERIC, "int4 weight outside [-7, 7]");
                uint8_t& byte = dst[k >> 1];
                byte = static_cast<uint8_t>((k & 1) ? ((byte & 0x0f) | ((v & 0xf) << 4)) : ((byte & 0xf0) | (v & 0xf)));
            }
        }
        if (as) ascale[i] = static_cast<float>((*as)[i]);
    }
    if (wd != WSVD_F32) {
        // W-tiles: this head-role's R rows are R/16 whole tiles at byte offset n0 * rb
        std::vector<uint8_t> tiled(rows.size());
        pack_wtiles(rows.data(), R, static_cast<int>(rb), wd == WSVD_I4 ? L->ks / 2 : L->ks * (wd == WSVD_BF16 ? 2 : 1),
                    tiled.data());
        rows.swap(tiled);
    }
    CUDA_TRY(cudaMemcpy(L->A.as<uint8_t>() + n0 * rb, rows.data(), rows.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->a_scale.as<float>() + n0, ascale.data(), R * 4, cudaMemcpyHostToDevice));
    // ---- B: [head][R][H]
    const size_t bel = (L->bdtype == F32) ? 4 : (L->bdtype == BF16 ? 2 : 1);
    std::vector<uint8_t> bh(static_cast<size_t>(R) * H * bel, 0);
    std::vector<float> bsc(H, 1.f);
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < H; ++j) {
            const size_t src = static_cast<size_t>(i) * H + j;
            const size_t o = static_cast<size_t>(i) * H + j;
            if (L->bdtype == F32) reinterpret_cast<float*>(bh.data())[o] = static_cast<float>((*bf)[src]);
            else if (L->bdtype == BF16) reinterpret_cast<uint16_t*>(bh.data())[o] = f32_to_bf16_bits(static_cast<float>((*bf)[src]));
            else reinterpret_cast<int8_t*>(bh.data())[o] = (*bq)[src];
        }
    if (bs)
        for (int j = 0; j < H; ++j) bsc[j] = static_cast<float>((*bs)[j]);
    {
        // host copy of the device's B values, for the host-side folds
        // (B_Q . B_K^T for the absorbed query, B_V . W_o for the O-projection)
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < H; ++j) {
                const size_t o = static_cast<size_t>(i) * H + j;
                double v = 0.0;
                if (L->bdtype == F32) v = reinterpret_cast<const float*>(bh.data())[o];
                else if (L->bdtype == BF16) {
                    const uint32_t u = static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(bh.data())[o]) << 16;
                    float f;
                    std::memcpy(&f, &u, 4);
                    v = f;
                } else {
                    v = static_cast<double>(reinterpret_cast<const int8_t*>(bh.data())[o]) * static_cast<double>(bsc[j]);
                }
                L->b_host[role][(static_cast<size_t>(head) * R + i) * H + j] = v;
            }
    }
    L->mqk_ready = false;
    L->bkt_ready = false;
    L->gen += 1;
    if (role == 2 && L->Wo.p) {
        // W'_o = B_V . W_o was folded from the previous V factors: drop it, so
        // a layer step fails with ECONFIG until wsvd_layer_set_oproj refolds
        L->Wo.alloc(0);
        L->e_out = 0;
    }
    CUDA_TRY(cudaMemcpy(L->B[role].as<uint8_t>() + static_cast<size_t>(head) * R * H * bel, bh.data(), bh.size(),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->b_scale[role].as<float>() + static_cast<size_t>(head) * H, bsc.data(), H * 4,
                        cudaMemcpyHostToDevice));
    L->have[head * 3 + role] = 1;
    return WSVD_OK;
}

int wsvd_layer_set_head(wsvd_layer_t L, int32_t head, int32_t role, const double* a, const double* b) {
    if (!L || !a || !b) return set_err(WSVD_ECONFIG, "null argument");
    if (head < 0 || head >= L->d.n_heads) return set_err(WSVD_ESHAPE, "head index out of range");
    if (role < 0 || role > 2) return set_err(WSVD_ECONFIG, "role must be 0 (q), 1 (k) or 2 (v)");
    const size_t E = L->d.embed_dim, H = L->d.head_dim;
    const size_t r = L->ranks[head * 3 + role];
    for (size_t i = 0; i < E * r; ++i)
        if (!std::isfinite(a[i])) return set_err(WSVD_ENUMERIC, "non-finite entry in factor a");
    for (size_t i = 0; i < r * H; ++i)
        if (!std::isfinite(b[i])) return set_err(WSVD_ENUMERIC, "non-finite entry in factor b");
    std::vector<double> af(a, a + E * r), bf(b, b + r * H);
    const int wd = L->d.weight_dtype;
    if (wd == WSVD_F32 || wd == WSVD_BF16) return upload_head(L, head, role, nullptr, nullptr, &af, nullptr, nullptr, &bf);
    if (L->d.act_rotation) rotate_columns(af, E, r, L->rot_blk);
    const int bits = (wd == WSVD_I8) ? 8 : 4;
    std::vector<int8_t> aq, bq;
    std::vector<double> as, bs;
    quantize_weight_ref(af, E, r, bits, aq, as);
    quantize_weight_ref(bf, r, H, bits, bq, bs);
    return upload_head(L, head, role, &aq, &as, nullptr, &bq, &bs, nullptr);
}

int wsvd_layer_set_head_quantized(wsvd_layer_t L, int32_t head, int32_t role, const int8_t* a_q,
                                  const double* a_scales, const int8_t* b_q, const double* b_scales) {
    if (!L || !a_q || !a_scales || !b_q || !b_scales) return set_err(WSVD_ECONFIG, "null argument");
    if (L->d.weight_dtype != WSVD_I8 && L->d.weight_dtype != WSVD_I4)
        return set_err(WSVD_ECONFIG, "quantised upload needs an I8 or I4 layer");
    if (head < 0 || head >= L->d.n_heads) return set_err(WSVD_ESHAPE, "head index out of range");
    if (role < 0 || role > 2) return set_err(WSVD_ECONFIG, "role must be 0 (q), 1 (k) or 2 (v)");
    const size_t E = L->d.embed_dim, H = L->d.head_dim;
    const size_t r = L->ranks[head * 3 + role];
    std::vector<int8_t> aq(a_q, a_q + E * r), bq(b_q, b_q + r * H);
    std::vector<double> as(a_scales, a_scales + r), bs(b_scales, b_scales + H);
    for (double s : as)
        if (!(s > 0.0)) return set_err(WSVD_ENUMERIC, "quantization scales must be positive");
    for (double s : bs)
        if (!(s > 0.0)) return set_err(WSVD_ENUMERIC, "quantization scales must be positive");
    return upload_head(L, head, role, &aq, &as, nullptr, &bq, &bs, nullptr);
}

int wsvd_layer_set_oproj(wsvd_layer_t L, const double* w, int32_t e_out, int32_t dtype) {
    if (!L || !w) return set_err(WSVD_ECONFIG, "null argument");
    L->gen += 1;
    if (e_out <= 0) return set_err(WSVD_ESHAPE, "e_out must be positive");
    if (dtype != WSVD_F32 && dtype != WSVD_BF16) return set_err(WSVD_ECONFIG, "O-projection dtype must be F32 or BF16");
    if (!L->have[2]) return set_err(WSVD_ECONFIG, "upload the V factors before the O-projection");
    for (size_t i = 0; i < L->have.size(); i += 3)
        if (!L->have[i + 2]) return set_err(WSVD_ECONFIG, "upload the V factors before the O-projection");
    CUDA_TRY(cudaSetDevice(L->d.device));
    // W'_o = blockdiag_h(B_Vh) . W_o  ((n_heads*R) x e_out): the latent attention
    // output is projected straight to the model width (SPEC section 3.4)
    const int nh = L->d.n_heads, H = L->d.head_dim, R = L->R;
    const int K = nh * R;
    L->e_out = e_out;
    L->o_dtype = dtype;
    L->oKp = round_up(K, 256);
    // 512-wide K splits (16 KB W-tile items, the fused step's weight-ring slot)
    L->oks = (L->oKp % 512 == 0) ? 512 : 256;
    if (dtype == WSVD_F32) L->oks = std::min(L->oKp, 1024);
    const int e_pad = round_up(e_out, 16);  // whole W-tiles
    const size_t el = dtype == WSVD_F32 ? 4 : 2;
    std::vector<double> fold(static_cast<size_t>(K) * e_out, 0.0);
    for (int h = 0; h < nh; ++h)
        for (int i = 0; i < R; ++i) {
            double* dst = fold.data() + (static_cast<size_t>(h) * R + i) * e_out;
            for (int j = 0; j < H; ++j) {
                const double bv = L->b_host[2][(static_cast<size_t>(h) * R + i) * H + j];
                if (bv == 0.0) continue;
                const double* src = w + (static_cast<size_t>(h) * H + j) * e_out;
                for (int e = 0; e < e_out; ++e) dst[e] += bv * src[e];
            }
        }
    std::vector<uint8_t> rows(static_cast<size_t>(e_pad) * L->oKp * el, 0);
    for (int e = 0; e < e_out; ++e)
        for (int k = 0; k < K; ++k) {
            const double v = fold[static_cast<size_t>(k) * e_out + e];
            const size_t o = static_cast<size_t>(e) * L->oKp + k;
            if (dtype == WSVD_F32) reinterpret_cast<float*>(rows.data())[o] = static_cast<float>(v);
            else reinterpret_cast<uint16_t*>(rows.data())[o] = f32_to_bf16_bits(static_cast<float>(v));
        }
    if (dtype == WSVD_BF16) {
        std::vector<uint8_t> tiled(rows.size());
        pack_wtiles(rows.data(), e_pad, L->oKp * 2, L->oks * 2, tiled.data());
        rows.swap(tiled);
    }
    CUDA_TRY(L->Wo.alloc(rows.size()));
    CUDA_TRY(cudaMemcpy(L->Wo.p, rows.data(), rows.size(), cudaMemcpyHostToDevice));
    return WSVD_OK;
}

int wsvd_cache_create(wsvd_layer_t L, int32_t batch, int32_t capacity, int32_t cache_dtype, wsvd_cache_t* out) {
    if (!L || !out) return set_err(WSVD_ECONFIG, "null argument");
    if (batch <= 0 || capacity <= 0) return set_err(WSVD_ESHAPE, "batch and capacity must be positive");
    if (cache_dtype != WSVD_F32 && cache_dtype != WSVD_BF16 && cache_dtype != WSVD_I8)
        return set_err(WSVD_ECONFIG, "cache dtype must be F32, BF16 or I8");
    if (attn_smem_bytes(cache_dtype, L->R) <= 0) return set_err(WSVD_ECONFIG, "unsupported rank for this cache dtype");
    CUDA_TRY(cudaSetDevice(L->d.device));
    auto* c = new wsvd_cache_s();
    c->L = L;
    c->B = batch;
    c->cap = capacity;
    c->cap_alloc = round_up(capacity, 128);
    c->cdtype = cache_dtype;
    const int eb = cache_dtype == WSVD_F32 ? 4 : (cache_dtype == WSVD_BF16 ? 2 : 1);
    c->row_bytes = 2 * L->R * eb;
    const int nh = L->d.n_heads, H = L->d.head_dim;
    cudaDeviceProp p;
    CUDA_TRY(cudaGetDeviceProperties(&p, L->d.device));
    c->sms = p.multiProcessorCount;
    c->grid = c->sms * attn_occupancy(cache_dtype, L->R);
    // split-KV: each (sequence, head) is cut into up to max_chunks equal chunks
    // per launch (attn.cu chunking()).  Fewer pairs than CTAs: about one unit
    // per CTA (B1 ctx2K fp32: attention + combine 12.3 us against 26.9 at four
    // units per CTA).  Otherwise the fewest chunks whose units spread over the
    // persistent grid at >= 90 % balance (units / (grid * rounds)): B16 x 32
    // heads -> 2 chunks (1 chunk leaves 3.46 units per CTA on 4 rounds; the
    // 32-layer B128 stack measured 13.1 ms at 2 against 13.3+ at 1);
    // B32 / B64 int8 configs -> 1
    c->chunk = 0;
    {
        const int pairs = batch * nh;
        int nchk = 1;
        if (pairs < c->grid) {
            nchk = (c->grid + pairs - 1) / pairs;
        } else {
            while (nchk < 8) {
                const long u = static_cast<long>(pairs) * nchk;
                const long rounds = (u + c->grid - 1) / c->grid;
                if (u * 10 >= rounds * c->grid * 9) break;
                ++nchk;
            }
        }
        if (const char* env = getenv("WSVD_ATTN_UNITS"))  // A/B: target units per CTA
            nchk = (std::max(1, atoi(env)) * c->grid + pairs - 1) / pairs;
        c->max_chunks = std::max(1, std::min(64, nchk));
    }
    if (const char* env = getenv("WSVD_ATTN_CHUNK")) {  // fixed chunk length (tests)
        c->chunk = std::max(32, round_up(atoi(env), 32));
        c->max_chunks = (c->cap_alloc + c->chunk - 1) / c->chunk;
    }
    // the fused step streams up to step_max_units() units per CTA
    {
        const int mu = step_max_units();
        int fu = mu;
        if (const char* env = getenv("WSVD_STEP_UNITS")) fu = std::max(1, std::min(mu, atoi(env)));
        const int pairs = batch * nh;
        c->fmax_chunks = std::max(1, (fu * c->sms + pairs - 1) / pairs);
        while (c->fmax_chunks > 1 && (pairs * c->fmax_chunks + c->sms - 1) / c->sms > mu) --c->fmax_chunks;
    }
    const size_t rows = static_cast<size_t>(batch) * nh * c->cap_alloc;
    // + 128 KB: the attention rings copy a slot's first stage whole, which may run past the last row
    cudaError_t e = c->data.alloc(rows * c->row_bytes + (128u << 10));
    if (e == cudaSuccess && cache_dtype == WSVD_I8) e = c->scales.alloc(rows * 4 + (16u << 10));  // + a stage of scales
    if (e == cudaSuccess) e = c->ctrl.alloc(1024 + 160 * 128);  // [0] len [1] done [2] step epoch [3] layer steps
        // [4,5] barrier [16..32) x-fetch counters [256 + 32 c] y flags
    if (e == cudaSuccess) e = c->qt.alloc(static_cast<size_t>(batch) * nh * L->R * 4);
    if (e == cudaSuccess)
        e = c->attn_ws.alloc(static_cast<size_t>(batch) * nh *
                             std::max(c->max_chunks * attn_parts_per_chunk() * (L->R + 2), c->fmax_chunks * (L->R + 4)) * 4);
    if (e == cudaSuccess) e = c->attn_cnt.alloc(static_cast<size_t>(batch) * nh * 4);
    if (e == cudaSuccess) e = c->vlat.alloc(static_cast<size_t>(batch) * nh * L->R * 4);
    if (e == cudaSuccess) e = c->qfull.alloc(static_cast<size_t>(batch) * nh * L->d.head_dim * 4);
    if (const char* env = getenv("WSVD_ATTN_MODE"))  // default for new caches (A/B runs)
        if (std::string(env) == "tc" && attn_tc_supported(cache_dtype, L->R, L->d.head_dim, L->bdtype))
            c->attn_mode = WSVD_ATTN_EXPLICIT_TC;
    (void)H;
    if (e != cudaSuccess) {
        delete c;
        return set_err(WSVD_ECUDA, std::string("cache allocation: ") + cudaGetErrorString(e));
    }
    *out = c;
    return WSVD_OK;
}

int wsvd_cache_grow(wsvd_cache_t c, int32_t capacity) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    if (capacity <= c->cap) return WSVD_OK;
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    const int cap_alloc = round_up(capacity, 128);
    const size_t regions = static_cast<size_t>(c->B) * c->L->d.n_heads;
    const size_t old_pitch = static_cast<size_t>(c->cap_alloc) * c->row_bytes;
    const size_t new_pitch = static_cast<size_t>(cap_alloc) * c->row_bytes;
    DevBuf nd, ns;
    CUDA_TRY(nd.alloc(regions * new_pitch + (128u << 10)));
    if (c->len > 0) {
        // whole 1 KB swizzle blocks of the used rows: the 16-byte XOR swizzle
        // permutes units inside 128-byte lines, relative to the region start
        const size_t used = std::min((static_cast<size_t>(c->len) * c->row_bytes + 1023) / 1024 * 1024, old_pitch);
        CUDA_TRY(cudaMemcpy2D(nd.p, new_pitch, c->data.p, old_pitch, used, regions, cudaMemcpyDeviceToDevice));
    }
    if (c->cdtype == WSVD_I8) {
        CUDA_TRY(ns.alloc(regions * cap_alloc * 4 + (16u << 10)));
        if (c->len > 0)
            CUDA_TRY(cudaMemcpy2D(ns.p, static_cast<size_t>(cap_alloc) * 4, c->scales.p, static_cast<size_t>(c->cap_alloc) * 4,
                                  static_cast<size_t>(c->len) * 4, regions, cudaMemcpyDeviceToDevice));
    }
    std::swap(c->data.p, nd.p);
    std::swap(c->data.n, nd.n);
    if (c->cdtype == WSVD_I8) {
        std::swap(c->scales.p, ns.p);
        std::swap(c->scales.n, ns.n);
    }
    c->cap = capacity;
    c->cap_alloc = cap_alloc;
    // captured step graphs hold the old buffers
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    if (c->graph) {
        cudaGraphDestroy(c->graph);
        c->graph = nullptr;
    }
    c->gpending = false;
    c->gkey = GraphKey{};
    return WSVD_OK;
}

int wsvd_cache_capacity(wsvd_cache_t c, int32_t* capacity) {
    if (!c || !capacity) return set_err(WSVD_ECONFIG, "null argument");
    *capacity = c->cap;
    return WSVD_OK;
}

int wsvd_cache_destroy(wsvd_cache_t c) {
    delete c;
    return WSVD_OK;
}

int wsvd_cache_reset(wsvd_cache_t c) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemset(c->ctrl.p, 0, c->ctrl.n));
    c->len = 0;
    return WSVD_OK;
}

int wsvd_cache_bind_layer(wsvd_cache_t c, wsvd_layer_t L) {
    if (!c || !L) return set_err(WSVD_ECONFIG, "null argument");
    const wsvd_layer_s* o = c->L;
    if (L->d.n_heads != o->d.n_heads)
        return set_err(WSVD_ESHAPE, "cache holds " + std::to_string(o->d.n_heads) + " heads, factors " +
                                        std::to_string(L->d.n_heads));
    if (L->R != o->R || L->d.embed_dim != o->d.embed_dim || L->d.head_dim != o->d.head_dim ||
        L->d.device != o->d.device)
        return set_err(WSVD_ESHAPE, "factor geometry differs from the cache's layer");
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    if (c->graph) {
        cudaGraphDestroy(c->graph);
        c->graph = nullptr;
    }
    c->gpending = false;
    c->gkey = GraphKey{};
    c->hkey = GraphKey{};
    c->L = L;
    return WSVD_OK;
}

int wsvd_cache_length(wsvd_cache_t c, int32_t* len) {
    if (!c || !len) return set_err(WSVD_ECONFIG, "null argument");
    *len = c->len;
    return WSVD_OK;
}

int wsvd_cache_sync_length(wsvd_cache_t c, int32_t* len) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    int32_t d = 0;
    CUDA_TRY(cudaMemcpy(&d, c->d_len(), 4, cudaMemcpyDeviceToHost));
    if (d < 0 || d > c->cap) return set_err(WSVD_ESHAPE, "device length out of range");
    c->len = d;
    if (len) *len = d;
    return WSVD_OK;
}

int wsvd_cache_fill_synthetic(wsvd_cache_t c, int32_t length, uint64_t seed, float scale) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    if (length < 0 || length > c->cap) return set_err(WSVD_ESHAPE, "synthetic length exceeds the capacity");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    const int regions = c->B * c->L->d.n_heads;
    if (length > 0)
        CUDA_TRY(launch_fill_synthetic(c->data.as<uint8_t>(), c->scales.as<__half2>(), regions, c->cap_alloc, length,
                                       c->L->R, c->cdtype, c->row_bytes, static_cast<uint32_t>(seed ^ (seed >> 32)),
                                       scale, nullptr));
    CUDA_TRY(cudaMemcpy(c->d_len(), &length, 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaDeviceSynchronize());
    c->len = length;
    return WSVD_OK;
}

int wsvd_cache_set_attention_mode(wsvd_cache_t c, int32_t mode) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    if (mode == WSVD_ATTN_ABSORBED) {
        c->attn_mode = mode;
        return WSVD_OK;
    }
    if (mode != WSVD_ATTN_EXPLICIT_TC) return set_err(WSVD_ECONFIG, "unknown attention mode");
    const wsvd_layer_s* L = c->L;
    if (!attn_tc_supported(c->cdtype, L->R, L->d.head_dim, L->bdtype))
        return set_err(WSVD_ECONFIG, "explicit tcgen05 attention needs a bf16 cache, bf16 factors, rank 32 and head dim 128");
    c->attn_mode = mode;
    return WSVD_OK;
}

int wsvd_cache_attention_mode(wsvd_cache_t c, int32_t* mode) {
    if (!c || !mode) return set_err(WSVD_ECONFIG, "null argument");
    *mode = c->attn_mode;
    return WSVD_OK;
}

int wsvd_cache_step_info(wsvd_cache_t c, int32_t* fused, int32_t* launches) {
    if (!c || !fused || !launches) return set_err(WSVD_ECONFIG, "null argument");
    const wsvd_layer_s* L = c->L;
    if (fused_step_ok(c)) {
        *fused = 1;
        *launches = 1;
        return WSVD_OK;
    }
    const int wd = L->d.weight_dtype;
    int n = 3;                                               // projection, epilogue, attention
    static const bool no_fin = getenv("WSVD_ATTN_COMBINE") != nullptr;
    const bool merged = c->attn_mode != WSVD_ATTN_EXPLICIT_TC && c->chunk == 0 && !no_fin &&
                        (c->max_chunks == 1 || attn_cluster_for(c) > 1);
    if (!merged) n += 1;                                     // the split-KV combine
    if (wd == WSVD_I8 || wd == WSVD_I4) n += 1;              // activation quantiser
    const int ochunks = L->o_dtype == BF16 ? (c->B + 63) / 64 : 1;  // run_oproj: 64 sequences per GEMM
    n += ochunks;                                            // O-projection GEMM
    if (L->oKp > 0 && L->oKp / L->oks > 1) n += ochunks;     // its split reduction
    *fused = 0;
    *launches = n;
    return WSVD_OK;
}

int wsvd_cache_row_bytes(wsvd_cache_t c, int32_t* rb) {
    if (!c || !rb) return set_err(WSVD_ECONFIG, "null argument");
    *rb = c->row_bytes;
    return WSVD_OK;
}

int wsvd_cache_push_host(wsvd_cache_t c, const double* ck, const double* cv) {
    if (!c || !ck || !cv) return set_err(WSVD_ECONFIG, "null argument");
    if (c->len >= c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    wsvd_layer_s* L = c->L;
    const int nh = L->d.n_heads, R = L->R;
    if (c->cdtype == WSVD_I8) return set_err(WSVD_ECONFIG, "push_host supports F32/BF16 caches");
    CUDA_TRY(cudaSetDevice(L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    const int n = c->B * nh;
    std::vector<uint8_t> rows(static_cast<size_t>(n) * c->row_bytes);
    for (int b = 0; b < c->B; ++b)
        for (int h = 0; h < nh; ++h) {
            const int rk = L->ranks[h * 3 + 1], rv = L->ranks[h * 3 + 2];
            uint8_t* row = rows.data() + (static_cast<size_t>(b) * nh + h) * c->row_bytes;
            for (int i = 0; i < 2 * R; ++i) {
                const bool kpart = i < R;
                const int j = kpart ? i : i - R;
                double v = 0.0;
                if (kpart && j < rk) v = ck[(static_cast<size_t>(b) * nh + h) * R + j];
                if (!kpart && j < rv) v = cv[(static_cast<size_t>(b) * nh + h) * R + j];
                if (c->cdtype == WSVD_F32) reinterpret_cast<float*>(row)[i] = static_cast<float>(v);
                else reinterpret_cast<uint16_t*>(row)[i] = f32_to_bf16_bits(static_cast<float>(v));
            }
        }
    DevBuf tmp;
    CUDA_TRY(tmp.alloc(rows.size()));
    CUDA_TRY(cudaMemcpy(tmp.p, rows.data(), rows.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(launch_push_rows(tmp.as<uint8_t>(), n, c->data.as<uint8_t>(), c->cap_alloc, c->row_bytes, c->len, nullptr));
    CUDA_TRY(cudaDeviceSynchronize());
    c->len += 1;
    CUDA_TRY(cudaMemcpy(c->d_len(), &c->len, 4, cudaMemcpyHostToDevice));
    return WSVD_OK;
}

int wsvd_cache_read_raw(wsvd_cache_t c, int32_t b, int32_t h, void* rows_host, uint16_t* scales_host) {
    if (!c || !rows_host) return set_err(WSVD_ECONFIG, "null argument");
    if (b < 0 || b >= c->B || h < 0 || h >= c->L->d.n_heads) return set_err(WSVD_ESHAPE, "sequence/head out of range");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    const size_t bh = static_cast<size_t>(b) * c->L->d.n_heads + h;
    if (c->len > 0) {
        // copy the covering 1 KB swizzle blocks, then undo the 16-byte XOR swizzle
        const size_t used = static_cast<size_t>(c->len) * c->row_bytes;
        const size_t span = std::min((used + 1023) / 1024 * 1024, static_cast<size_t>(c->cap_alloc) * c->row_bytes);
        std::vector<uint8_t> raw(span);
        CUDA_TRY(cudaMemcpy(raw.data(), c->data.as<uint8_t>() + bh * c->cap_alloc * c->row_bytes, span,
                            cudaMemcpyDeviceToHost));
        uint8_t* out = static_cast<uint8_t*>(rows_host);
        for (size_t u = 0; u < used / 16; ++u)
            std::memcpy(out + u * 16, raw.data() + wsvd_dev_swz(static_cast<uint32_t>(u * 16)), 16);
        if (scales_host && c->cdtype == WSVD_I8)
            CUDA_TRY(cudaMemcpy(scales_host, c->scales.as<uint8_t>() + bh * c->cap_alloc * 4,
                                static_cast<size_t>(c->len) * 4, cudaMemcpyDeviceToHost));
    }
    return WSVD_OK;
}

static float half_bits_to_float(uint16_t h) {
    const uint32_t sign = (static_cast<uint32_t>(h) & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ff;
    float v;
    if (e == 0) {
        v = static_cast<float>(m) * 5.9604644775390625e-08f;
        return sign ? -v : v;
    }
    uint32_t u = (e == 31) ? (sign | 0x7f800000u | (m << 13)) : (sign | ((e - 15 + 127) << 23) | (m << 13));
    std::memcpy(&v, &u, 4);
    return v;
}

int wsvd_cache_read_host(wsvd_cache_t c, int32_t b, int32_t h, double* ck, double* cv) {
    if (!c || !ck || !cv) return set_err(WSVD_ECONFIG, "null argument");
    const int R = c->L->R;
    std::vector<uint8_t> rows(static_cast<size_t>(c->len) * c->row_bytes);
    std::vector<uint16_t> sc(static_cast<size_t>(c->len) * 2);
    int rc = wsvd_cache_read_raw(c, b, h, rows.data(), sc.data());
    if (rc) return rc;
    for (int t = 0; t < c->len; ++t) {
        const uint8_t* r = rows.data() + static_cast<size_t>(t) * c->row_bytes;
        for (int i = 0; i < 2 * R; ++i) {
            double v;
            if (c->cdtype == WSVD_F32) v = reinterpret_cast<const float*>(r)[i];
            else if (c->cdtype == WSVD_BF16) {
                uint32_t u = static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(r)[i]) << 16;
                float f;
                std::memcpy(&f, &u, 4);
                v = f;
            } else {
                const float s = half_bits_to_float(sc[t * 2 + (i < R ? 0 : 1)]);
                v = static_cast<double>(reinterpret_cast<const int8_t*>(r)[i]) * static_cast<double>(s);
            }
            if (i < R) ck[static_cast<size_t>(t) * R + i] = v;
            else cv[static_cast<size_t>(t) * R + i - R] = v;
        }
    }
    return WSVD_OK;
}

int wsvd_append_token(wsvd_cache_t c, const float* x, float* q_out, void* stream) {
    if (!c || !x) return set_err(WSVD_ECONFIG, "null argument");
    int rc = check_layer(c->L);
    if (rc) return rc;
    if (c->len + 1 > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (c->attn_mode == WSVD_ATTN_EXPLICIT_TC) {
        // the explicit kernel attends with q itself (kept for wsvd_decode_attention)
        rc = run_append(c, x, 1, c->qfull.as<float>(), nullptr, 1, s);
        if (rc) return rc;
        if (q_out)
            CUDA_TRY(cudaMemcpyAsync(q_out, c->qfull.p, static_cast<size_t>(c->B) * c->L->d.n_heads * c->L->d.head_dim * 4,
                                     cudaMemcpyDeviceToDevice, s));
    } else {
        rc = run_append(c, x, 1, q_out, c->qt.as<float>(), 1, s);
        if (rc) return rc;
    }
    c->len += 1;
    return WSVD_OK;
}

int wsvd_prefill(wsvd_cache_t c, const float* x, int32_t T, void* stream) {
    if (!c || !x) return set_err(WSVD_ECONFIG, "null argument");
    if (T <= 0) return set_err(WSVD_ESHAPE, "prefill of zero tokens");
    int rc = check_layer(c->L);
    if (rc) return rc;
    if (c->len + T > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    const int E = c->L->d.embed_dim;
    const int tc = std::max(1, 128 / c->B);  // <= 128 token rows per projection
    for (int t0 = 0; t0 < T; t0 += tc) {
        const int n = std::min(tc, T - t0);
        rc = run_append(c, x + static_cast<size_t>(t0) * c->B * E, n, nullptr, nullptr, 1, static_cast<cudaStream_t>(stream));
        if (rc) return rc;
        c->len += n;
    }
    return WSVD_OK;
}

int wsvd_fused_decode_step(wsvd_cache_t c, const float* q, int32_t tile_len, float* out, void* stream) {
    if (!c || !q || !out) return set_err(WSVD_ECONFIG, "null argument");
    if (c->len == 0) return set_err(WSVD_ESHAPE, "decode step over an empty cache");
    if (tile_len <= 0) return set_err(WSVD_ECONFIG, "tile length must be >= 1");
    int rc = check_layer(c->L);
    if (rc) return rc;
    wsvd_layer_s* L = c->L;
    CUDA_TRY(cudaSetDevice(L->d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (c->attn_mode == WSVD_ATTN_EXPLICIT_TC) return run_attention(c, out, nullptr, 0, s, q);
    CUDA_TRY(launch_absorb_query(q, c->B, L->d.n_heads, L->R, L->d.head_dim, L->B[1].p, L->b_scale[1].as<float>(),
                                 L->bdtype, 1.4426950408889634f / std::sqrt(static_cast<float>(L->d.head_dim)),
                                 c->qt.as<float>(), s));
    return run_attention(c, out, nullptr, 0, s);
}

int wsvd_decode_attention(wsvd_cache_t c, float* out, void* stream) {
    if (!c || !out) return set_err(WSVD_ECONFIG, "null argument");
    if (c->len == 0) return set_err(WSVD_ESHAPE, "decode step over an empty cache");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    return run_attention(c, out, nullptr, 0, static_cast<cudaStream_t>(stream));
}

int wsvd_layer_step(wsvd_cache_t c, const float* x, float* attn_out, float* y, void* stream) {
    if (!c || !x || !y) return set_err(WSVD_ECONFIG, "null argument");
    int rc = check_layer(c->L);
    if (rc) return rc;
    if (!c->L->Wo.p) return set_err(WSVD_ECONFIG, "layer has no O-projection folded from its current V factors (wsvd_layer_set_oproj)");
    if (c->len + 1 > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    rc = layer_step_impl(c, x, attn_out, y, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
    c->len += 1;
    return WSVD_OK;
}

int wsvd_layer_step_graph(wsvd_cache_t c, const float* x, float* y, void* stream) {
    if (!c || !x || !y) return set_err(WSVD_ECONFIG, "null argument");
    int rc = check_layer(c->L);
    if (rc) return rc;
    if (!c->L->Wo.p) return set_err(WSVD_ECONFIG, "layer has no O-projection folded from its current V factors (wsvd_layer_set_oproj)");
    if (c->len + 1 > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    CUDA_TRY(cudaSetDevice(c->L->d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (fused_step_ok(c)) {
        // one persistent kernel per step: a plain (PDL) launch is already as
        // cheap as a graph replay, and x / y may change from step to step
        rc = run_step_fused(c, x, y, s);
        if (rc) return rc;
        c->len += 1;
        return WSVD_OK;
    }
    const bool same = c->gkey.x == x && c->gkey.y == y && c->gkey.s == s &&
                      c->ggen == c->L->gen && c->gmode == c->attn_mode;
    if (c->gexec && same) {
        // replay on the caller's stream (the graph was captured on it); the
        // owned stream only stands in for the legacy default stream
        CUDA_TRY(cudaGraphLaunch(c->gexec, s ? s : c->gstream));
        c->len += 1;
        return WSVD_OK;
    }
    if (!same || !c->gpending) {
        // first call with these buffers: run eagerly (sizes workspaces, sets
        // kernel attributes); the next call captures and replays.  (Replaying
        // one graph for every (x, y) through staging copies measured slower
        // than these PDL-chained eager launches: 92.8 vs 88.7 us at config 3.)
        if (c->gexec) cudaGraphExecDestroy(c->gexec);
        if (c->graph) cudaGraphDestroy(c->graph);
        c->gexec = nullptr;
        c->graph = nullptr;
        rc = layer_step_impl(c, x, nullptr, y, s);
        if (rc) return rc;
        c->gkey = {x, y, s};
        c->ggen = c->L->gen;
        c->gmode = c->attn_mode;
        c->gpending = true;
        c->len += 1;
        return WSVD_OK;
    }
    // capture (the legacy stream cannot be captured: use an owned blocking stream)
    cudaStream_t cs = s;
    if (cs == nullptr) {
        if (!c->gstream) CUDA_TRY(cudaStreamCreateWithFlags(&c->gstream, cudaStreamDefault));
        cs = c->gstream;
    }
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    rc = layer_step_impl(c, x, nullptr, y, cs);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return set_err(WSVD_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    c->graph = g;
    CUDA_TRY(cudaGraphInstantiate(&c->gexec, g, 0));
    c->gpending = false;
    CUDA_TRY(cudaGraphLaunch(c->gexec, cs));
    c->len += 1;
    return WSVD_OK;
}

int wsvd_layer_step_host(wsvd_cache_t c, const float* x_host, float* y_host, void* stream) {
    if (!c || !x_host || !y_host) return set_err(WSVD_ECONFIG, "null argument");
    wsvd_layer_s* L = c->L;
    if (!L->Wo.p) return set_err(WSVD_ECONFIG, "layer has no O-projection (wsvd_layer_set_oproj)");
    int rc = check_layer(L);
    if (rc) return rc;
    if (c->len + 1 > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
    CUDA_TRY(cudaSetDevice(L->d.device));
    const size_t xb = static_cast<size_t>(c->B) * L->d.embed_dim * 4;
    const size_t yb = static_cast<size_t>(c->B) * L->e_out * 4;
    if (c->x_dev.n < xb) CUDA_TRY(c->x_dev.alloc(xb));
    if (c->y_dev.n < yb) CUDA_TRY(c->y_dev.alloc(yb));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // A/B switch: WSVD_HOST_ZEROCOPY=0 moves x / y with the copy engine
    static const bool no_zc = getenv("WSVD_HOST_ZEROCOPY") && std::string(getenv("WSVD_HOST_ZEROCOPY")) == "0";
    if (!fused_step_ok(c) || no_zc) {
        CUDA_TRY(cudaMemcpyAsync(c->x_dev.p, x_host, xb, cudaMemcpyHostToDevice, s));
        rc = wsvd_layer_step_graph(c, c->x_dev.as<float>(), c->y_dev.as<float>(), stream);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(y_host, c->y_dev.p, yb, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return WSVD_OK;
    }
    // fused step with pinned (mapped) host buffers: the kernel itself moves the
    // bytes -- x is fetched once over the bus by the projection CTAs, y is
    // written with plain stores from the O-projection epilogue -- so the step
    // is one launch and one synchronise, with no copy engine round trips
    if (!(c->hkey.x == x_host && c->hkey.y == y_host)) {
        cudaPointerAttributes ax{}, ay{};
        const bool okx = cudaPointerGetAttributes(&ax, x_host) == cudaSuccess;
        const bool oky = cudaPointerGetAttributes(&ay, y_host) == cudaSuccess;
        cudaGetLastError();
        c->hzc = okx && oky && ax.type == cudaMemoryTypeHost && ay.type == cudaMemoryTypeHost && ax.devicePointer &&
                 ay.devicePointer;
        c->hx = c->hzc ? static_cast<const float*>(ax.devicePointer) : nullptr;
        c->hy = c->hzc ? static_cast<float*>(ay.devicePointer) : nullptr;
        c->hkey = {x_host, y_host, s};
    }
    if (c->hzc) {
        rc = run_step_fused(c, c->hx, c->hy, s, true);
    } else {  // pageable host memory: copy engine
        CUDA_TRY(cudaMemcpyAsync(c->x_dev.p, x_host, xb, cudaMemcpyHostToDevice, s));
        rc = run_step_fused(c, c->x_dev.as<float>(), c->y_dev.as<float>(), s);
        if (rc == WSVD_OK) CUDA_TRY(cudaMemcpyAsync(y_host, c->y_dev.p, yb, cudaMemcpyDeviceToHost, s));
    }
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(s));
    c->len += 1;
    return WSVD_OK;
}

// ---------------------------------------------------------------- chains --
// pipe::decode_factored's layer loop (pipeline.cpp:318-336), attention blocks
// chained: one persistent launch when every layer runs the fused step.
static int chain_check(wsvd_cache_t const* cs, int32_t n, bool& fused) {
    if (!cs || n < 1) return set_err(WSVD_ECONFIG, "a chain needs at least one cache");
    fused = n <= kStepMaxLayers;
    const wsvd_cache_s* c0 = cs[0];
    if (!c0) return set_err(WSVD_ECONFIG, "null cache handle");
    for (int l = 0; l < n; ++l) {
        wsvd_cache_s* c = cs[l];
        if (!c) return set_err(WSVD_ECONFIG, "null cache handle");
        for (int k = 0; k < l; ++k)
            if (cs[k] == c) return set_err(WSVD_ECONFIG, "a cache appears twice in the chain");
        int rc = check_layer(c->L);
        if (rc) return rc;
        const wsvd_layer_s* L = c->L;
        const wsvd_layer_s* L0 = c0->L;
        if (!L->Wo.p) return set_err(WSVD_ECONFIG, "layer has no O-projection folded from its current V factors (wsvd_layer_set_oproj)");
        if (L->e_out != L->d.embed_dim) return set_err(WSVD_ESHAPE, "a chained layer must project back to embed_dim");
        if (c->B != c0->B || L->d.embed_dim != L0->d.embed_dim || L->d.n_heads != L0->d.n_heads ||
            L->d.head_dim != L0->d.head_dim || L->R != L0->R || L->d.device != L0->d.device)
            return set_err(WSVD_ESHAPE, "chained caches differ in geometry (batch, heads, embed_dim, rank, device)");
        if (c->len + 1 > c->cap) return set_err(WSVD_ESHAPE, "latent cache is full (capacity " + std::to_string(c->cap) + ")");
        if (!fused_step_ok(c) || L->Kp != L0->Kp || L->oKp != L0->oKp || L->Nrows != L0->Nrows || c->sms != c0->sms)
            fused = false;
    }
    return WSVD_OK;
}

int wsvd_chain_step(wsvd_cache_t const* cs, int32_t n, const float* x, float* const* ys, void* stream) {
    if (!x || !ys) return set_err(WSVD_ECONFIG, "null argument");
    bool fused = false;
    int rc = chain_check(cs, n, fused);
    if (rc) return rc;
    for (int l = 0; l < n; ++l)
        if (!ys[l]) return set_err(WSVD_ECONFIG, "null layer output");
    CUDA_TRY(cudaSetDevice(cs[0]->L->d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (fused) {
        rc = chain_pipe_ok(cs, n) ? run_chain_pipe(cs, n, x, ys, s) : run_chain_fused(cs, n, x, ys, s);
        if (rc) return rc;
        for (int l = 0; l < n; ++l) cs[l]->len += 1;
        return WSVD_OK;
    }
    for (int l = 0; l < n; ++l) {
        rc = wsvd_layer_step(cs[l], l == 0 ? x : ys[l - 1], nullptr, ys[l], stream);
        if (rc) return rc;
    }
    return WSVD_OK;
}

int wsvd_chain_step_host(wsvd_cache_t const* cs, int32_t n, const float* x_host, float* y_host, void* stream) {
    if (!x_host || !y_host) return set_err(WSVD_ECONFIG, "null argument");
    bool fused = false;
    int rc = chain_check(cs, n, fused);
    if (rc) return rc;
    wsvd_cache_s* c0 = cs[0];
    CUDA_TRY(cudaSetDevice(c0->L->d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t xb = static_cast<size_t>(c0->B) * c0->L->d.embed_dim * 4;
    std::vector<float*> ys(n);
    for (int l = 0; l < n; ++l) {
        if (cs[l]->y_dev.n < xb) CUDA_TRY(cs[l]->y_dev.alloc(xb));
        ys[l] = cs[l]->y_dev.as<float>();
    }
    if (c0->x_dev.n < xb) CUDA_TRY(c0->x_dev.alloc(xb));
    // mapped pinned buffers: the kernel fetches x and stores the last y itself
    // (one launch + one synchronise, as wsvd_layer_step_host)
    static const bool no_zc = getenv("WSVD_HOST_ZEROCOPY") && std::string(getenv("WSVD_HOST_ZEROCOPY")) == "0";
    if (fused && !no_zc && !chain_pipe_ok(cs, n) && !(c0->hkey.x == x_host && c0->hkey.y == y_host)) {
        cudaPointerAttributes ax{}, ay{};
        const bool okx = cudaPointerGetAttributes(&ax, x_host) == cudaSuccess;
        const bool oky = cudaPointerGetAttributes(&ay, y_host) == cudaSuccess;
        cudaGetLastError();
        c0->hzc = okx && oky && ax.type == cudaMemoryTypeHost && ay.type == cudaMemoryTypeHost && ax.devicePointer &&
                  ay.devicePointer;
        c0->hx = c0->hzc ? static_cast<const float*>(ax.devicePointer) : nullptr;
        c0->hy = c0->hzc ? static_cast<float*>(ay.devicePointer) : nullptr;
        c0->hkey = {x_host, y_host, s};
    }
    if (fused && !no_zc && c0->hzc && !chain_pipe_ok(cs, n)) {
        ys[n - 1] = c0->hy;
        rc = run_chain_fused(cs, n, c0->hx, ys.data(), s, true, true);
        if (rc) return rc;
        for (int l = 0; l < n; ++l) cs[l]->len += 1;
    } else {
        CUDA_TRY(cudaMemcpyAsync(c0->x_dev.p, x_host, xb, cudaMemcpyHostToDevice, s));
        rc = wsvd_chain_step(cs, n, c0->x_dev.as<float>(), ys.data(), stream);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(y_host, ys[n - 1], xb, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    return WSVD_OK;
}

// ----------------------------------------------------------- feed-forward --
// pipe::decode_factored's toy FFN (pipeline.cpp:330-334) on the skinny GEMM
int wsvd_ffn_create(int32_t E, int32_t F, const float* ff1, const float* ff2, int32_t device, wsvd_ffn_t* out) {
    if (!ff1 || !ff2 || !out) return set_err(WSVD_ECONFIG, "null argument");
    if (E <= 0 || F <= 0) return set_err(WSVD_ESHAPE, "empty feed-forward");
    if (sm100_devices() == 0) return set_err(WSVD_ECUDA, "no sm_100 (B200) device visible");
    CUDA_TRY(cudaSetDevice(device));
    auto* f = new wsvd_ffn_s();
    f->E = E;
    f->F = F;
    f->device = device;
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    f->sms = prop.multiProcessorCount;
    f->Kp1 = round_up(E, 512);
    f->Kp2 = round_up(F, 512);
    // W-tiles of a [N][K] row matrix (row n = output unit, K = input): W1 rows are
    // ff1's columns, W2 rows ff2's columns
    auto pack = [&](const float* w, int K, int N, int Kp, DevBuf& dst) -> int {
        const int np = round_up(N, 16);
        std::vector<uint8_t> rows(static_cast<size_t>(np) * Kp * 2, 0), tiled(rows.size());
        uint16_t* rr = reinterpret_cast<uint16_t*>(rows.data());
        for (int n0 = 0; n0 < N; n0 += 64)  // blocked transpose: both sides stay in cache
            for (int k0 = 0; k0 < K; k0 += 64)
                for (int k = k0; k < std::min(K, k0 + 64); ++k)
                    for (int n = n0; n < std::min(N, n0 + 64); ++n)
                        rr[static_cast<size_t>(n) * Kp + k] = f32_to_bf16_bits(w[static_cast<size_t>(k) * N + n]);
        pack_wtiles(rows.data(), np, Kp * 2, 512 * 2, tiled.data());
        CUDA_TRY(dst.alloc(tiled.size()));
        CUDA_TRY(cudaMemcpy(dst.p, tiled.data(), tiled.size(), cudaMemcpyHostToDevice));
        return WSVD_OK;
    };
    // K-chunk-major bf16 [K/64][N][64] (the tcgen05 GEMM's TMA layout: every
    // 256-row box of a 64-wide K chunk is one contiguous 32 KB block)
    auto plain = [&](const float* w, int K, int N, DevBuf& dst) -> int {
        std::vector<uint16_t> rows(static_cast<size_t>(N) * K);
        for (int k0 = 0; k0 < K; k0 += 64)
            for (int k = k0; k < std::min(K, k0 + 64); ++k)
                for (int n = 0; n < N; ++n)
                    rows[(static_cast<size_t>(k0 / 64) * N + n) * 64 + (k - k0)] =
                        f32_to_bf16_bits(w[static_cast<size_t>(k) * N + n]);
        CUDA_TRY(dst.alloc(rows.size() * 2));
        CUDA_TRY(cudaMemcpy(dst.p, rows.data(), rows.size() * 2, cudaMemcpyHostToDevice));
        return WSVD_OK;
    };
    static const bool no_tc = getenv("WSVD_FFN_SKINNY") != nullptr;  // A/B switch: the mma.sync skinny GEMM
    f->tc = !no_tc && tc_gemm_supported(1, F, E) && tc_gemm_supported(1, E, F);
    int rc = f->tc ? plain(ff1, E, F, f->W1) : pack(ff1, E, F, f->Kp1, f->W1);
    if (rc == WSVD_OK) rc = f->tc ? plain(ff2, F, E, f->W2) : pack(ff2, F, E, f->Kp2, f->W2);
    if (rc) {
        delete f;
        return rc;
    }
    *out = f;
    return WSVD_OK;
}

int wsvd_ffn_destroy(wsvd_ffn_t f) {
    delete f;
    return WSVD_OK;
}

int wsvd_ffn_forward(wsvd_ffn_t f, const float* o, int32_t M, float* out, void* stream) {
    if (!f || !o || !out) return set_err(WSVD_ECONFIG, "null argument");
    if (M <= 0) return set_err(WSVD_ESHAPE, "feed-forward over zero rows");
    if (!f->tc && !gemm_fits(BF16, M, 512)) return set_err(WSVD_ECONFIG, std::to_string(M) + " rows do not fit the GEMM kernel");
    CUDA_TRY(cudaSetDevice(f->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (f->tc) {
        // tcgen05: hidden = bf16(tanh(bf16(o) . ff1)) in the GEMM epilogue; out
        // = hidden . ff2 over K splits when its N tiles leave SMs idle (summed by
        // the reduction kernel in split order)
        const int ch = std::min(M, 128);
        const int nt2 = f->E / 64;
        const int sp2 = std::max(1, std::min(f->F / 64, f->sms / nt2));
        if (f->Xb.n < static_cast<size_t>(ch) * f->E * 2) CUDA_TRY(f->Xb.alloc(static_cast<size_t>(ch) * f->E * 2));
        if (f->Hd.n < static_cast<size_t>(ch) * f->F * 2) CUDA_TRY(f->Hd.alloc(static_cast<size_t>(ch) * f->F * 2));
        if (f->P.n < static_cast<size_t>(sp2) * ch * f->E * 4) CUDA_TRY(f->P.alloc(static_cast<size_t>(sp2) * ch * f->E * 4));
        for (int m0 = 0; m0 < M; m0 += 128) {
            const int mc = std::min(128, M - m0);
            CUDA_TRY(launch_f32_to_bf16(o + static_cast<size_t>(m0) * f->E, f->Xb.p, static_cast<size_t>(mc) * f->E, s));
            TcGemmArgs g1{f->Xb.p, f->W1.p, f->Hd.p, mc, f->F, f->E, f->F, 1, 1, 1, 0, 0};
            CUDA_TRY(launch_tc_gemm(g1, s));
            float* dst = out + static_cast<size_t>(m0) * f->E;
            TcGemmArgs g2{f->Hd.p, f->W2.p, sp2 == 1 ? static_cast<void*>(dst) : f->P.p, mc, f->E, f->F, f->E, sp2, 0, 0, 0, 0};
            CUDA_TRY(launch_tc_gemm(g2, s));
            if (sp2 > 1) CUDA_TRY(launch_reduce_partials(f->P.as<float>(), sp2, mc, f->E, dst, s, 0, 0));
        }
        return WSVD_OK;
    }
    const int s1 = f->Kp1 / 512, s2 = f->Kp2 / 512;
    const size_t need = std::max(static_cast<size_t>(s1) * M * f->F, static_cast<size_t>(s2) * M * f->E) * 4;
    if (f->P.n < need) CUDA_TRY(f->P.alloc(need));
    if (f->Hd.n < static_cast<size_t>(M) * f->F * 4) CUDA_TRY(f->Hd.alloc(static_cast<size_t>(M) * f->F * 4));
    auto gemm = [&](const void* W, const float* X, int N, int K, int Kp) -> cudaError_t {
        GemmArgs g{};
        g.W = W;
        g.X = X;
        g.P = f->P.p;
        g.M = M;
        g.N = N;
        g.K = K;
        g.Kp = Kp;
        g.KS = 512;
        g.ldx = K;
        g.wdtype = BF16;
        g.grid = f->sms;
        return launch_gemm(g, s);
    };
    // hidden = tanh(o . ff1)  (pipeline.cpp:330-333), out = hidden . ff2 (:334)
    CUDA_TRY(gemm(f->W1.p, o, f->F, f->E, f->Kp1));
    CUDA_TRY(launch_reduce_partials(f->P.as<float>(), s1, M, f->F, f->Hd.as<float>(), s, 1));
    CUDA_TRY(gemm(f->W2.p, f->Hd.as<float>(), f->E, f->F, f->Kp2));
    CUDA_TRY(launch_reduce_partials(f->P.as<float>(), s2, M, f->E, out, s, 0));
    return WSVD_OK;
}

int wsvd_cache_debug_copy(wsvd_cache_t c, int32_t what, void* host, int64_t* bytes) {
    if (!c || !host || !bytes) return set_err(WSVD_ECONFIG, "null argument");
    wsvd_layer_s* L = c->L;
    CUDA_TRY(cudaSetDevice(L->d.device));
    CUDA_TRY(cudaDeviceSynchronize());
    const int M = c->P_M;
    if (what == 0 || what == 1) {
        const DevBuf& b = what == 0 ? c->xq : c->sx;
        const size_t n = what == 0 ? static_cast<size_t>(M) * L->Kp : static_cast<size_t>(M) * 4;
        if (!b.p || n > b.n) return set_err(WSVD_ECONFIG, "no quantised activations (not an I8/I4 layer?)");
        if (*bytes < static_cast<int64_t>(n)) return set_err(WSVD_ESHAPE, "host buffer too small");
        CUDA_TRY(cudaMemcpy(host, b.p, n, cudaMemcpyDeviceToHost));
        *bytes = static_cast<int64_t>(n);
        return WSVD_OK;
    }
    if (what == 2) {
        const size_t per = static_cast<size_t>(M) * L->Nrows;
        if (*bytes < static_cast<int64_t>(per * 4)) return set_err(WSVD_ESHAPE, "host buffer too small");
        std::vector<uint8_t> all(per * 4 * c->P_splits);
        CUDA_TRY(cudaMemcpy(all.data(), c->P.p, all.size(), cudaMemcpyDeviceToHost));
        const bool ints = L->d.weight_dtype == WSVD_I8 || L->d.weight_dtype == WSVD_I4;
        for (size_t i = 0; i < per; ++i) {
            if (ints) {
                int32_t s = 0;
                for (int k = 0; k < c->P_splits; ++k) s += reinterpret_cast<const int32_t*>(all.data())[k * per + i];
                static_cast<int32_t*>(host)[i] = s;
            } else {
                float s = 0.f;
                for (int k = 0; k < c->P_splits; ++k) s += reinterpret_cast<const float*>(all.data())[k * per + i];
                static_cast<float*>(host)[i] = s;
            }
        }
        *bytes = static_cast<int64_t>(per * 4);
        return WSVD_OK;
    }
    if (what == 3) {
        const size_t n = static_cast<size_t>(c->B) * L->d.n_heads * L->R * 4;
        if (*bytes < static_cast<int64_t>(n)) return set_err(WSVD_ESHAPE, "host buffer too small");
        CUDA_TRY(cudaMemcpy(host, c->qt.p, n, cudaMemcpyDeviceToHost));
        *bytes = static_cast<int64_t>(n);
        return WSVD_OK;
    }
    if (what == 5) {
        if (!c->dbg_on) return set_err(WSVD_ECONFIG, "score capture is off (wsvd_cache_set_debug)");
        const size_t per = static_cast<size_t>(c->cap_alloc) * 2 * 4;
        const size_t n = static_cast<size_t>(c->B) * L->d.n_heads * per;
        if (*bytes < static_cast<int64_t>(n)) return set_err(WSVD_ESHAPE, "host buffer too small");
        CUDA_TRY(cudaMemcpy(host, c->dbg.p, n, cudaMemcpyDeviceToHost));
        *bytes = static_cast<int64_t>(n);
        return WSVD_OK;
    }
    if (what == 4) {
        if (!c->trace.p) return set_err(WSVD_ECONFIG, "no step trace (set WSVD_STEP_TRACE)");
        if (*bytes < static_cast<int64_t>(c->trace.n)) return set_err(WSVD_ESHAPE, "host buffer too small");
        CUDA_TRY(cudaMemcpy(host, c->trace.p, c->trace.n, cudaMemcpyDeviceToHost));
        *bytes = static_cast<int64_t>(c->trace.n);
        return WSVD_OK;
    }
    return set_err(WSVD_ECONFIG, "unknown debug buffer");
}

int wsvd_cache_set_debug(wsvd_cache_t c, int32_t flags) {
    if (!c) return set_err(WSVD_ECONFIG, "null cache");
    c->dbg_on = (flags & 1) != 0 && c->cdtype == WSVD_I8;
    if (c->dbg_on) {
        const size_t need = static_cast<size_t>(c->B) * c->L->d.n_heads * c->cap_alloc * 2 * 4;
        if (c->dbg.n < need) CUDA_TRY(c->dbg.alloc(need));
    }
    return WSVD_OK;
}

int wsvd_quantize_weight(const double* w, int64_t rows, int64_t cols, int32_t bits, int8_t* q,
                         double* scales, double* clip) {
    if (!w || !q || !scales) return set_err(WSVD_ECONFIG, "null argument");
    if (bits != 4 && bits != 8) return set_err(WSVD_ECONFIG, "bit width must be 4 or 8");
    if (rows <= 0 || cols <= 0) return set_err(WSVD_ESHAPE, "empty matrix");
    for (int64_t i = 0; i < rows * cols; ++i)
        if (!std::isfinite(w[i])) return set_err(WSVD_ENUMERIC, "quantize input: non-finite entry");
    std::vector<double> wv(w, w + rows * cols), s;
    std::vector<int8_t> qv;
    const double c = quantize_weight_ref(wv, static_cast<size_t>(rows), static_cast<size_t>(cols), bits, qv, s);
    std::memcpy(q, qv.data(), qv.size());
    std::memcpy(scales, s.data(), s.size() * sizeof(double));
    if (clip) *clip = c;
    return WSVD_OK;
}

int wsvd_traffic_append(wsvd_cache_t c, uint64_t* k) {
    if (!c || !k) return set_err(WSVD_ECONFIG, "null argument");
    wsvd_layer_s* L = c->L;
    const uint64_t E = L->d.embed_dim, H = L->d.head_dim, Bn = c->B;
    k[WSVD_STREAM_QUERY] += Bn * E;  // decode.cpp:132
    for (int h = 0; h < L->d.n_heads; ++h) {
        const uint64_t rq = L->ranks[h * 3], rk = L->ranks[h * 3 + 1], rv = L->ranks[h * 3 + 2];
        k[14 + WSVD_STREAM_LATENT_K] += Bn * E * rk;
        k[7 + WSVD_STREAM_LATENT_K] += Bn * rk;
        k[14 + WSVD_STREAM_LATENT_V] += Bn * E * rv;
        k[7 + WSVD_STREAM_LATENT_V] += Bn * rv;
        k[14 + WSVD_STREAM_QUERY] += Bn * (E * rq + rq * H);
    }
    return WSVD_OK;
}

int wsvd_traffic_fused(wsvd_cache_t c, int32_t tile_len, uint64_t* k) {
    if (!c || !k) return set_err(WSVD_ECONFIG, "null argument");
    if (c->len == 0) return set_err(WSVD_ESHAPE, "decode step over an empty cache");
    if (tile_len <= 0) return set_err(WSVD_ECONFIG, "tile length must be >= 1");
    wsvd_layer_s* L = c->L;
    const uint64_t H = L->d.head_dim, Bn = c->B, len = c->len;
    for (int h = 0; h < L->d.n_heads; ++h) {
        const uint64_t rk = L->ranks[h * 3 + 1], rv = L->ranks[h * 3 + 2];
        k[WSVD_STREAM_WEIGHTS_B] += Bn * (rk * H + rv * H);      // decode.cpp:176
        k[WSVD_STREAM_QUERY] += Bn * H;                          // decode.cpp:177
        k[WSVD_STREAM_LATENT_K] += Bn * len * rk;                // decode.cpp:184
        k[WSVD_STREAM_LATENT_V] += Bn * len * rv;                // decode.cpp:185
        k[14 + WSVD_STREAM_LATENT_K] += Bn * len * rk * H;       // decode.cpp:189
        k[14 + WSVD_STREAM_QUERY] += Bn * len * H;               // decode.cpp:191
        k[14 + WSVD_STREAM_LATENT_V] += Bn * len * rv;           // decode.cpp:193
        k[14 + WSVD_STREAM_OUTPUT] += Bn * rv * H;               // decode.cpp:201
        k[7 + WSVD_STREAM_OUTPUT] += Bn * H;                     // decode.cpp:202
    }
    return WSVD_OK;
}

int wsvd_nccl_unique_id(uint8_t id[128]) {
    NcclApi& n = nccl();
    if (!n.ok) return set_err(WSVD_ENCCL, "libnccl.so.2 not loadable");
    const int r = n.getUniqueId(id);
    if (r) return set_err(WSVD_ENCCL, std::string("ncclGetUniqueId: ") + (n.errStr ? n.errStr(r) : "?"));
    return WSVD_OK;
}

int wsvd_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, wsvd_comm_t* out) {
    if (!id || !out) return set_err(WSVD_ECONFIG, "null argument");
    NcclApi& n = nccl();
    if (!n.ok) return set_err(WSVD_ENCCL, "libnccl.so.2 not loadable");
    CUDA_TRY(cudaSetDevice(device));
    auto init = reinterpret_cast<CommInitFn>(dlsym(n.h, "ncclCommInitRank"));
    NcclId nid;
    std::memcpy(nid.b, id, 128);
    void* comm = nullptr;
    const int r = init(&comm, nranks, nid, rank);
    if (r) return set_err(WSVD_ENCCL, std::string("ncclCommInitRank: ") + (n.errStr ? n.errStr(r) : "?"));
    auto* c = new wsvd_comm_s();
    c->comm = comm;
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return WSVD_OK;
}

int wsvd_comm_destroy(wsvd_comm_t c) {
    if (!c) return WSVD_OK;
    NcclApi& n = nccl();
    if (n.ok && c->comm) n.commDestroy(c->comm);
    delete c;
    return WSVD_OK;
}

int wsvd_allreduce_sum_f32(wsvd_comm_t c, float* buf, int64_t count, void* stream) {
    if (!c || !buf) return set_err(WSVD_ECONFIG, "null argument");
    NcclApi& n = nccl();
    if (!n.ok) return set_err(WSVD_ENCCL, "libnccl.so.2 not loadable");
    const int r = n.allReduce(buf, buf, static_cast<size_t>(count), /*ncclFloat32*/ 7, /*ncclSum*/ 0, c->comm,
                              static_cast<cudaStream_t>(stream));
    if (r) return set_err(WSVD_ENCCL, std::string("ncclAllReduce: ") + (n.errStr ? n.errStr(r) : "?"));
    return WSVD_OK;
}

}  // extern "C"
