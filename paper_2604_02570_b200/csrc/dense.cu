// dense.cu -- the reference's comparison baselines on the device: dense
// per-head K/V caches with flash / eager attention (decode.cpp:208-319,
// FullKvCache, append_token_dense, eager_decode_step, flash_decode_step) and
// the fp32 building blocks the C++ drop-in uses for them and for the shared
// latent baseline (decode.cpp:321-432: x . A GEMV, C . B materialisation).
//
// These are reference points, not the WSVD hot path: fp32 CUDA-core kernels
// sized for correctness at any head width, one CTA per head.  The
// paper-scale comparison numbers in bench.py use the library SDPA / cuBLAS
// layers of baselines.py.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <string>

#include "../../include/wsvd_b200.h"
#include "common.cuh"

using namespace wsvd_dev;

extern "C" void wsvd_internal_set_error(const char* msg);  // capi.cu

namespace {

int fail(int code, const std::string& msg) {
    wsvd_internal_set_error(msg.c_str());
    return code;
}

#define DENSE_TRY(expr)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess) return fail(WSVD_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int kDenseThreads = 256;

// One CTA per head: scores s_j = q . k_j / sqrt(H) (a warp per token, lanes
// over H), their maximum, p_j = exp(s_j - max), then out = sum_j p_j v_j /
// sum_j p_j with threads over H.  The score row goes to `scores` (the eager
// schedule materialises it; the flash schedule's result is the same softmax
// up to reassociation, decode.cpp:290-319).
__global__ void __launch_bounds__(kDenseThreads) dense_attend_kernel(const float* __restrict__ keys,
                                                                    const float* __restrict__ values, int len,
                                                                    int ld, int H, const float* __restrict__ q,
                                                                    float* __restrict__ scores,
                                                                    float* __restrict__ out) {
    const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* kh = keys + static_cast<size_t>(h) * ld * H;
    const float* vh = values + static_cast<size_t>(h) * ld * H;
    const float* qh = q + static_cast<size_t>(h) * H;
    float* sc = scores + static_cast<size_t>(h) * ld;
    const float inv = rsqrtf(static_cast<float>(H));
    __shared__ float red[kDenseThreads / 32];
    __shared__ float bcast[2];
    float mloc = -FLT_MAX;
    for (int j = warp; j < len; j += kDenseThreads / 32) {
        float d = 0.f;
        for (int c = lane; c < H; c += 32) d = fmaf(qh[c], kh[static_cast<size_t>(j) * H + c], d);
        d = warp_sum(d) * inv;
        if (lane == 0) sc[j] = d;
        mloc = fmaxf(mloc, d);
    }
    if (lane == 0) red[warp] = mloc;
    __syncthreads();
    if (tid == 0) {
        float m = -FLT_MAX;
        for (int w = 0; w < kDenseThreads / 32; ++w) m = fmaxf(m, red[w]);
        bcast[0] = m;
    }
    __syncthreads();
    const float m = bcast[0];
    float lsum = 0.f;
    for (int j = tid; j < len; j += kDenseThreads) {
        const float p = expf(sc[j] - m);
        sc[j] = p;
        lsum += p;
    }
    lsum = warp_sum(lsum);
    __syncthreads();
    if (lane == 0) red[warp] = lsum;
    __syncthreads();
    if (tid == 0) {
        float s = 0.f;
        for (int w = 0; w < kDenseThreads / 32; ++w) s += red[w];
        bcast[1] = s;
    }
    __syncthreads();
    const float denom = bcast[1];
    for (int c = tid; c < H; c += kDenseThreads) {
        float acc = 0.f;
        for (int j = 0; j < len; ++j) acc = fmaf(sc[j], vh[static_cast<size_t>(j) * H + c], acc);
        out[static_cast<size_t>(h) * H + c] = acc / denom;
    }
}

// y[n] = sum_k x[k] w[k][n]  (row vector times a row-major k x n matrix)
__global__ void vecmat_kernel(const float* __restrict__ x, const float* __restrict__ w, int k, int n,
                              float* __restrict__ y) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    float acc = 0.f;
    for (int i = 0; i < k; ++i) acc = fmaf(x[i], w[static_cast<size_t>(i) * n + j], acc);
    y[j] = acc;
}

// c[m][n] = sum_k a[m][k] b[k][n], 16 x 16 shared-memory tiles
__global__ void matmul_kernel(const float* __restrict__ a, const float* __restrict__ b, int M, int K, int N,
                              float* __restrict__ c) {
    __shared__ float ta[16][17], tb[16][17];
    const int r = blockIdx.y * 16 + threadIdx.y, col = blockIdx.x * 16 + threadIdx.x;
    float acc = 0.f;
    for (int k0 = 0; k0 < K; k0 += 16) {
        ta[threadIdx.y][threadIdx.x] = (r < M && k0 + threadIdx.x < K) ? a[static_cast<size_t>(r) * K + k0 + threadIdx.x] : 0.f;
        tb[threadIdx.y][threadIdx.x] = (k0 + threadIdx.y < K && col < N) ? b[static_cast<size_t>(k0 + threadIdx.y) * N + col] : 0.f;
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) acc = fmaf(ta[threadIdx.y][kk], tb[kk][threadIdx.x], acc);
        __syncthreads();
    }
    if (r < M && col < N) c[static_cast<size_t>(r) * N + col] = acc;
}

// rows [nh][H] -> row `pos` of [nh][cap][H]
__global__ void dense_append_kernel(const float* __restrict__ k, const float* __restrict__ v, int nh, int H,
                                    int cap, int pos, float* __restrict__ kc, float* __restrict__ vc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nh * H) return;
    const int h = i / H, c = i - h * H;
    const size_t o = (static_cast<size_t>(h) * cap + pos) * H + c;
    kc[o] = k[i];
    vc[o] = v[i];
}

}  // namespace

struct wsvd_dense_cache_s {
    int nh = 0, H = 0, cap = 0, len = 0, device = 0;
    float* k = nullptr;
    float* v = nullptr;
    float* scores = nullptr;  // [nh][cap]
    ~wsvd_dense_cache_s() {
        if (k) cudaFree(k);
        if (v) cudaFree(v);
        if (scores) cudaFree(scores);
    }
};

namespace {

// grows the cache to hold at least `need` rows (capacity doubles; rows copied)
int dense_reserve(wsvd_dense_cache_s* c, int need) {
    if (need <= c->cap) return WSVD_OK;
    int cap = c->cap ? c->cap : 64;
    while (cap < need) cap *= 2;
    const size_t per = static_cast<size_t>(c->nh) * cap * c->H * 4;
    float *nk = nullptr, *nv = nullptr, *ns = nullptr;
    DENSE_TRY(cudaDeviceSynchronize());
    DENSE_TRY(cudaMalloc(&nk, per));
    DENSE_TRY(cudaMalloc(&nv, per));
    DENSE_TRY(cudaMalloc(&ns, static_cast<size_t>(c->nh) * cap * 4));
    if (c->len > 0) {
        const size_t row = static_cast<size_t>(c->H) * 4;
        DENSE_TRY(cudaMemcpy2D(nk, cap * row, c->k, c->cap * row, c->len * row, c->nh, cudaMemcpyDeviceToDevice));
        DENSE_TRY(cudaMemcpy2D(nv, cap * row, c->v, c->cap * row, c->len * row, c->nh, cudaMemcpyDeviceToDevice));
    }
    if (c->k) cudaFree(c->k);
    if (c->v) cudaFree(c->v);
    if (c->scores) cudaFree(c->scores);
    c->k = nk;
    c->v = nv;
    c->scores = ns;
    c->cap = cap;
    return WSVD_OK;
}

}  // namespace

extern "C" {

int wsvd_dense_cache_create(int32_t n_heads, int32_t head_dim, int32_t device, wsvd_dense_cache_t* out) {
    if (!out) return fail(WSVD_ECONFIG, "null argument");
    if (n_heads <= 0 || head_dim <= 0) return fail(WSVD_ESHAPE, "empty kv cache geometry");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(WSVD_ECUDA, "no CUDA device visible");
    }
    DENSE_TRY(cudaSetDevice(device));
    auto* c = new wsvd_dense_cache_s();
    c->nh = n_heads;
    c->H = head_dim;
    c->device = device;
    const int rc = dense_reserve(c, 64);
    if (rc) {
        delete c;
        return rc;
    }
    *out = c;
    return WSVD_OK;
}

int wsvd_dense_cache_destroy(wsvd_dense_cache_t c) {
    delete c;
    return WSVD_OK;
}

int wsvd_dense_cache_length(wsvd_dense_cache_t c, int32_t* len) {
    if (!c || !len) return fail(WSVD_ECONFIG, "null argument");
    *len = c->len;
    return WSVD_OK;
}

int wsvd_dense_cache_append(wsvd_dense_cache_t c, const float* k, const float* v, void* stream) {
    if (!c || !k || !v) return fail(WSVD_ECONFIG, "null argument");
    DENSE_TRY(cudaSetDevice(c->device));
    const int rc = dense_reserve(c, c->len + 1);
    if (rc) return rc;
    const int n = c->nh * c->H;
    dense_append_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, v, c->nh, c->H, c->cap,
                                                                                       c->len, c->k, c->v);
    DENSE_TRY(cudaGetLastError());
    c->len += 1;
    return WSVD_OK;
}

int wsvd_dense_cache_read_host(wsvd_dense_cache_t c, int32_t head, double* k, double* v) {
    if (!c || !k || !v) return fail(WSVD_ECONFIG, "null argument");
    if (head < 0 || head >= c->nh) return fail(WSVD_ESHAPE, "head out of range");
    DENSE_TRY(cudaSetDevice(c->device));
    DENSE_TRY(cudaDeviceSynchronize());
    const size_t n = static_cast<size_t>(c->len) * c->H;
    float* tmp = new float[2 * n + 1];
    const size_t off = static_cast<size_t>(head) * c->cap * c->H;
    cudaError_t e = cudaMemcpy(tmp, c->k + off, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(tmp + n, c->v + off, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
        for (size_t i = 0; i < n; ++i) {
            k[i] = tmp[i];
            v[i] = tmp[n + i];
        }
    delete[] tmp;
    DENSE_TRY(e);
    return WSVD_OK;
}

int wsvd_dense_attend(const float* keys, const float* values, int32_t n_heads, int32_t len, int32_t ld,
                      int32_t head_dim, const float* q, float* scores, float* out, void* stream) {
    if (!keys || !values || !q || !scores || !out) return fail(WSVD_ECONFIG, "null argument");
    if (len <= 0) return fail(WSVD_ESHAPE, "decode step over an empty cache");
    if (n_heads <= 0 || head_dim <= 0 || ld < len) return fail(WSVD_ESHAPE, "bad attention geometry");
    dense_attend_kernel<<<n_heads, kDenseThreads, 0, static_cast<cudaStream_t>(stream)>>>(keys, values, len, ld,
                                                                                        head_dim, q, scores, out);
    DENSE_TRY(cudaGetLastError());
    return WSVD_OK;
}

int wsvd_dense_decode_step(wsvd_dense_cache_t c, const float* q, int32_t tile_len, float* out, void* stream) {
    if (!c || !q || !out) return fail(WSVD_ECONFIG, "null argument");
    if (c->len == 0) return fail(WSVD_ESHAPE, "decode step over an empty cache");
    if (tile_len <= 0) return fail(WSVD_ECONFIG, "tile length must be >= 1");
    DENSE_TRY(cudaSetDevice(c->device));
    return wsvd_dense_attend(c->k, c->v, c->nh, c->len, c->cap, c->H, q, c->scores, out, stream);
}

int wsvd_vecmat_f32(const float* x, const float* w, int32_t k, int32_t n, float* y, void* stream) {
    if (!x || !w || !y) return fail(WSVD_ECONFIG, "null argument");
    if (k <= 0 || n <= 0) return fail(WSVD_ESHAPE, "empty matrix");
    vecmat_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(x, w, k, n, y);
    DENSE_TRY(cudaGetLastError());
    return WSVD_OK;
}

int wsvd_matmul_f32(const float* a, const float* b, int32_t m, int32_t k, int32_t n, float* c, void* stream) {
    if (!a || !b || !c) return fail(WSVD_ECONFIG, "null argument");
    if (m <= 0 || k <= 0 || n <= 0) return fail(WSVD_ESHAPE, "empty matrix");
    matmul_kernel<<<dim3((n + 15) / 16, (m + 15) / 16), dim3(16, 16), 0, static_cast<cudaStream_t>(stream)>>>(a, b, m, k,
                                                                                                          n, c);
    DENSE_TRY(cudaGetLastError());
    return WSVD_OK;
}

}  // extern "C"
