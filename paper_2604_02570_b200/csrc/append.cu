// append.cu -- token-side kernels of the decode step.
//
//   act_quant        W8A8 / W4A8 activation path (SURVEY.md Appendix A steps
//                    1-2): x_hat = x . S1^T by an in-place fp32 FWHT, then the
//                    per-token quantiser of quant.cpp:131-150 with the same
//                    fp32 operation order as the oracle (bit-exact).
//   append_epilogue  finishes append_token (decode.cpp:127-153): sums the
//                    projection's K-split partials, dequantises (int modes),
//                    writes the K/V latent rows at the cache tail (bf16 / f32 /
//                    int8 + fp16 row scale), up-projects the query latent
//                    q_h = c_Q . B_Q and absorbs it into the key side,
//                    qt = log2(e)/sqrt(H) * q_h . B_K^T, for the attention kernel.
//   absorb_query     qt from a caller-supplied q (fused_decode_step's input).
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

// ----------------------------------------------------------- act quant --
constexpr int kAqThreads = 256;

__global__ void __launch_bounds__(kAqThreads) act_quant_kernel(const float* __restrict__ x, int E,
                                                               int Kp, int rot, int rot_blk,
                                                               float rot_scale,
                                                               int8_t* __restrict__ xq,
                                                               float* __restrict__ sx) {
    extern __shared__ float v[];  // [E]
    __shared__ float wmax[kAqThreads / 32];
    const int m = blockIdx.x;
    griddep_wait();
    griddep_launch_dependents();
    const float* xm = x + static_cast<size_t>(m) * E;
    for (int i = threadIdx.x; i < E; i += kAqThreads) v[i] = xm[i];
    if (rot) {
        // stages len = 1, 2, 4, ... < rot_blk; pair p -> (lo, lo + len)
        for (int len = 1; len < rot_blk; len <<= 1) {
            __syncthreads();
            for (int p = threadIdx.x; p < E / 2; p += kAqThreads) {
                const int lo = (p / len) * (2 * len) + (p % len);
                const float a = v[lo], b = v[lo + len];
                v[lo] = __fadd_rn(a, b);
                v[lo + len] = __fsub_rn(a, b);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < E; i += kAqThreads) v[i] = __fmul_rn(v[i], rot_scale);
    }
    __syncthreads();
    float m_abs = 0.f;
    for (int i = threadIdx.x; i < E; i += kAqThreads) m_abs = fmaxf(m_abs, fabsf(v[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m_abs = fmaxf(m_abs, __shfl_xor_sync(0xffffffffu, m_abs, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m_abs;
    __syncthreads();
    m_abs = 0.f;
#pragma unroll
    for (int w = 0; w < kAqThreads / 32; ++w) m_abs = fmaxf(m_abs, wmax[w]);
    const float s = (m_abs == 0.f) ? 1.f : __fdiv_rn(m_abs, 127.f);
    int8_t* q = xq + static_cast<size_t>(m) * Kp;
    for (int i = threadIdx.x; i < Kp; i += kAqThreads) {
        float r = 0.f;
        if (i < E) r = fminf(fmaxf(roundf(__fdiv_rn(v[i], s)), -127.f), 127.f);
        q[i] = static_cast<int8_t>(r);
    }
    if (threadIdx.x == 0) sx[m] = s;
}

// Fast variant (E % 512 == 0): thread t owns elements [16t, 16t + 16).  The
// FWHT stages with len < 16 run in registers, len 16..256 through warp
// shuffles (partner lane t ^ len/16), longer ones through shared memory; every
// butterfly is the same fp32 (a + b, a - b) as the oracle's
// (orc_fwht_f32), so the rotated token -- and everything after it -- is
// bit-identical to the one-pass kernel above.
__global__ void __launch_bounds__(512) act_quant_fast_kernel(const float* __restrict__ x, int E, int Kp, int rot,
                                                             int rot_blk, float rot_scale, int8_t* __restrict__ xq,
                                                             float* __restrict__ sx) {
    extern __shared__ float sv[];  // [E] for the cross-warp stages
    __shared__ float wmax[16];
    const int m = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nw = blockDim.x >> 5;
    griddep_wait();
    griddep_launch_dependents();
    const float4* xm = reinterpret_cast<const float4*>(x + static_cast<size_t>(m) * E) + 4 * t;
    float v[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float4 q = __ldg(xm + i);
        v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
    if (rot) {
#pragma unroll
        for (int len = 1; len < 16; len <<= 1) {
            if (len >= rot_blk) break;
#pragma unroll
            for (int i = 0; i < 16; i += 2 * len)
#pragma unroll
                for (int j = i; j < i + len; ++j) {
                    const float a = v[j], b = v[j + len];
                    v[j] = __fadd_rn(a, b);
                    v[j + len] = __fsub_rn(a, b);
                }
        }
        for (int len = 16; len < rot_blk && len < 512; len <<= 1) {
            const int mk = len >> 4;  // partner thread t ^ mk holds elements +- len
            const bool upper = (t & mk) != 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float o = __shfl_xor_sync(0xffffffffu, v[j], mk);
                v[j] = upper ? __fsub_rn(o, v[j]) : __fadd_rn(v[j], o);
            }
        }
        if (rot_blk > 512) {
#pragma unroll
            for (int j = 0; j < 16; ++j) sv[16 * t + j] = v[j];
            for (int len = 512; len < rot_blk; len <<= 1) {
                __syncthreads();
                for (int p = t; p < E / 2; p += blockDim.x) {
                    const int lo = ((p & ~(len - 1)) << 1) | (p & (len - 1));
                    const float a = sv[lo], b = sv[lo + len];
                    sv[lo] = __fadd_rn(a, b);
                    sv[lo + len] = __fsub_rn(a, b);
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = sv[16 * t + j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], rot_scale);
    }
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) mx = fmaxf(mx, fabsf(v[j]));
    mx = warp_max(mx);
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    mx = 0.f;
    for (int w = 0; w < nw; ++w) mx = fmaxf(mx, wmax[w]);
    const float s = (mx == 0.f) ? 1.f : __fdiv_rn(mx, 127.f);
    uint32_t packed[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t w = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float r = fminf(fmaxf(roundf(__fdiv_rn(v[4 * i + k], s)), -127.f), 127.f);
            w |= (static_cast<uint32_t>(static_cast<int32_t>(r)) & 0xffu) << (8 * k);
        }
        packed[i] = w;
    }
    int8_t* q = xq + static_cast<size_t>(m) * Kp;
    *reinterpret_cast<uint4*>(q + 16 * t) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    for (int i = E + t; i < Kp; i += blockDim.x) q[i] = 0;
    if (t == 0) sx[m] = s;
}

// ------------------------------------------------------ factor access --
WSVD_DEV float bload(const void* b, int bdtype, size_t idx) {
    if (bdtype == F32) return reinterpret_cast<const float*>(b)[idx];
    if (bdtype == BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(b)[idx]);
    return static_cast<float>(reinterpret_cast<const int8_t*>(b)[idx]);
}

// qt[i] = scale * sum_j q[j] * B_K[h][i][j]   (one warp per i)
WSVD_DEV void absorb(const float* q_s, int R, int H, const void* bk, const float* bk_scale,
                     int bdtype, int h, float scale, float* qt_out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const size_t base = static_cast<size_t>(h) * R * H;
    for (int i = warp; i < R; i += nw) {
        float acc = 0.f;
#pragma unroll 4
        for (int j = lane; j < H; j += 32) {
            float b = bload(bk, bdtype, base + static_cast<size_t>(i) * H + j);
            if (bdtype == I8) b *= bk_scale[h * H + j];
            acc = fmaf(q_s[j], b, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) qt_out[i] = acc * scale;
    }
}

// ----------------------------------------------------- append epilogue --
constexpr int kEpThreads = 128;

__global__ void __launch_bounds__(kEpThreads) append_epilogue_kernel(const AppendArgs a) {
    extern __shared__ float sm[];
    float* c = sm;                 // [3][R] latents q, k, v
    float* qh = sm + 3 * a.R;      // [H]
    float* mqs = qh + a.H;         // [R][R] this head's M_QK (layer-step mode)
    const int h = blockIdx.x, m = blockIdx.y;
    const int b = m % a.B, tpos = m / a.B;  // rows are token-major: m = tpos * B + b
    const int R = a.R, H = a.H;
    const bool fold = a.q_out == nullptr && a.qt != nullptr;
    if (fold) {
        // M_QK is a layer constant: staged before the grid-dependency wait, so
        // its loads overlap the predecessor instead of following the split sums
        const float4* src = reinterpret_cast<const float4*>(a.mqk + static_cast<size_t>(h) * R * R);
        for (int i = threadIdx.x; i < R * R / 4; i += kEpThreads) reinterpret_cast<float4*>(mqs)[i] = __ldg(src + i);
    }
    griddep_wait();
    griddep_launch_dependents();
    const int pos = *a.d_len + tpos;

    // ---- latents: fixed-order sum of the K-split partials (+ dequant)
    const int nrow0 = h * 3 * R;
    for (int i = threadIdx.x; i < 3 * R; i += kEpThreads) {
        const size_t o = static_cast<size_t>(m) * a.Nrows + nrow0 + i;
        const size_t stride = static_cast<size_t>(a.M) * a.Nrows;
        float val;
        if (a.wdtype == I8 || a.wdtype == I4) {
            int acc = 0;
            const int* P = reinterpret_cast<const int*>(a.P);
#pragma unroll 8
            for (int s = 0; s < a.splits; ++s) acc += __ldcg(P + s * stride + o);
            val = __fmul_rn(__fmul_rn(static_cast<float>(acc), a.sx[m]), a.a_scale[nrow0 + i]);
        } else {
            // fixed split order: deterministic
            float acc = 0.f;
            const float* P = reinterpret_cast<const float*>(a.P);
#pragma unroll 8
            for (int s = 0; s < a.splits; ++s) acc += __ldcg(P + s * stride + o);
            val = acc;
        }
        c[i] = val;
    }
    __syncthreads();

    // ---- cache append: row [C_K | C_V] at position pos
    const size_t bh = static_cast<size_t>(b) * a.nh + h;
    // rows live inside the (sequence, head) region with the 16-byte XOR swizzle
    uint8_t* region = a.cache + bh * a.cap * a.row_bytes;
    const uint32_t row0 = static_cast<uint32_t>(pos) * a.row_bytes;
    if (a.cdtype == I8) {
        // per (token, head, role) scale: f16(max|c| / 127), 1 when it is 0
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp < 2) {
            const float* src = c + (1 + warp) * R;
            float mx = 0.f;
            for (int i = lane; i < R; i += 32) mx = fmaxf(mx, fabsf(src[i]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            __half hs = __float2half_rn(__fdiv_rn(mx, 127.f));
            float s = __half2float(hs);
            if (s == 0.f) {
                hs = __float2half_rn(1.f);
                s = 1.f;
            }
            // four values per lane and one 32-bit store (R % 4 == 0; the 16-byte
            // swizzle keeps 4-byte groups contiguous): no byte-store tail
            for (int i = 4 * lane; i < R; i += 128) {
                uint32_t w = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int8_t q = static_cast<int8_t>(fminf(fmaxf(roundf(__fdiv_rn(src[i + e], s)), -127.f), 127.f));
                    w |= static_cast<uint32_t>(static_cast<uint8_t>(q)) << (8 * e);
                }
                *reinterpret_cast<uint32_t*>(region + cache_swz(row0 + warp * R + i)) = w;
            }
            if (lane == 0) reinterpret_cast<__half*>(a.cscale + bh * a.cap + pos)[warp] = hs;
        }
    } else if (a.cdtype == BF16) {
        for (int i = 2 * threadIdx.x; i < 2 * R; i += 2 * kEpThreads)  // two values per 32-bit store
            *reinterpret_cast<uint32_t*>(region + cache_swz(row0 + 2 * i)) = pack_bf16x2(c[R + i], c[R + i + 1]);
    } else {
        for (int i = threadIdx.x; i < 2 * R; i += kEpThreads)
            *reinterpret_cast<float*>(region + cache_swz(row0 + 4 * i)) = c[R + i];
    }

    // ---- query
    if (a.q_out != nullptr) {
        // reference API: q_h = c_Q . B_Q (decode.cpp:140) is returned; then the
        // absorbed key side qt = scale * q_h . B_K^T
        const size_t bq0 = static_cast<size_t>(h) * R * H;
        for (int j = threadIdx.x; j < H; j += kEpThreads) {
            float acc = 0.f;
#pragma unroll 16
            for (int i = 0; i < R; ++i) acc = fmaf(c[i], bload(a.bq, a.bdtype, bq0 + static_cast<size_t>(i) * H + j), acc);
            if (a.bdtype == I8) acc *= a.bq_scale[h * H + j];
            qh[j] = acc;
            a.q_out[(static_cast<size_t>(m) * a.nh + h) * H + j] = acc;
        }
        __syncthreads();
        if (a.qt) absorb(qh, R, H, a.bk, a.bk_scale, a.bdtype, h, a.qt_scale,
                         a.qt + (static_cast<size_t>(m) * a.nh + h) * R);
    } else if (a.qt != nullptr) {
        // layer step: q_h is never materialised; qt = c_Q . M_QK with
        // M_QK = scale * B_Q . B_K^T (R x R, folded on the host in fp64)
        for (int i = threadIdx.x; i < R; i += kEpThreads) {
            float acc = 0.f;
#pragma unroll 16
            for (int j = 0; j < R; ++j) acc = fmaf(c[j], mqs[j * R + i], acc);
            a.qt[(static_cast<size_t>(m) * a.nh + h) * R + i] = acc;
        }
    }

    // ---- commit: the last CTA advances the length by T
    if (!a.commit) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int total = gridDim.x * gridDim.y;
        if (atomicAdd(a.done, 1) == total - 1) {
            *a.d_len += a.T;
            *a.done = 0;
            __threadfence();
        }
    }
}

// rows [n][row_bytes] (logical order) -> cache row `pos` of regions 0..n-1
__global__ void push_rows_kernel(const uint8_t* __restrict__ rows, int n, uint8_t* cache, int cap,
                                 int row_bytes, int pos) {
    const int units = row_bytes / 16;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * units) return;
    const int r = i / units, u = i - r * units;
    uint8_t* region = cache + static_cast<size_t>(r) * cap * row_bytes;
    const uint32_t off = static_cast<uint32_t>(pos) * row_bytes + u * 16;
    *reinterpret_cast<uint4*>(region + cache_swz(off)) =
        *reinterpret_cast<const uint4*>(rows + static_cast<size_t>(r) * row_bytes + u * 16);
}

__global__ void __launch_bounds__(kEpThreads) absorb_query_kernel(const float* __restrict__ q, int nh,
                                                                  int R, int H, const void* bk,
                                                                  const float* bk_scale, int bdtype,
                                                                  float scale, float* qt) {
    extern __shared__ float qs[];
    const int h = blockIdx.x, b = blockIdx.y;
    griddep_wait();
    griddep_launch_dependents();
    const size_t o = (static_cast<size_t>(b) * nh + h);
    for (int j = threadIdx.x; j < H; j += kEpThreads) qs[j] = q[o * H + j];
    __syncthreads();
    absorb(qs, R, H, bk, bk_scale, bdtype, h, scale, qt + o * R);
}

// Synthetic latent rows for benchmarks (no prompt to prefill through the
// projection): row t of region r gets N(0, scale^2)-distributed values from a
// counter-based hash (Box-Muller), written in the cache format and swizzle.
WSVD_DEV uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void fill_synthetic_kernel(uint8_t* cache, __half2* cscale, int regions, int cap, int length, int R,
                                      int cdtype, int row_bytes, uint32_t seed, float scale) {
    const size_t n = static_cast<size_t>(regions) * length;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int reg = static_cast<int>(i / length), t = static_cast<int>(i - static_cast<size_t>(reg) * length);
        uint8_t* region = cache + static_cast<size_t>(reg) * cap * row_bytes;
        const uint32_t row0 = static_cast<uint32_t>(t) * row_bytes;
        const uint32_t base = mix32(seed ^ mix32(static_cast<uint32_t>(i) * 0x9e3779b9u));
        float v[128];
        for (int e = 0; e < 2 * R; e += 2) {
            const uint32_t h1 = mix32(base + 2u * e + 1u), h2 = mix32(base + 2u * e + 2u);
            const float u1 = (static_cast<float>(h1 >> 8) + 0.5f) * (1.0f / 16777216.0f);
            const float u2 = static_cast<float>(h2 >> 8) * (1.0f / 16777216.0f);
            const float rad = sqrtf(-2.f * logf(u1)) * scale;
            float sn, cs;
            sincospif(2.f * u2, &sn, &cs);
            v[e] = rad * cs;
            v[e + 1] = rad * sn;
        }
        if (cdtype == BF16) {
            for (int e = 0; e < 2 * R; ++e)
                *reinterpret_cast<__nv_bfloat16*>(region + cache_swz(row0 + 2 * e)) = __float2bfloat16_rn(v[e]);
        } else if (cdtype == F32) {
            for (int e = 0; e < 2 * R; ++e) *reinterpret_cast<float*>(region + cache_swz(row0 + 4 * e)) = v[e];
        } else {
            for (int half = 0; half < 2; ++half) {
                float mx = 0.f;
                for (int e = 0; e < R; ++e) mx = fmaxf(mx, fabsf(v[half * R + e]));
                __half hs = __float2half_rn(__fdiv_rn(mx, 127.f));
                float sc = __half2float(hs);
                if (sc == 0.f) {
                    hs = __float2half_rn(1.f);
                    sc = 1.f;
                }
                for (int e = 0; e < R; ++e)
                    reinterpret_cast<int8_t*>(region)[cache_swz(row0 + half * R + e)] =
                        static_cast<int8_t>(fminf(fmaxf(roundf(__fdiv_rn(v[half * R + e], sc)), -127.f), 127.f));
                reinterpret_cast<__half*>(cscale + static_cast<size_t>(reg) * cap + t)[half] = hs;
            }
        }
    }
}

}  // namespace

cudaError_t launch_fill_synthetic(uint8_t* cache, __half2* cscale, int regions, int cap, int length, int R,
                                  int cdtype, int row_bytes, uint32_t seed, float scale, cudaStream_t s) {
    if (2 * R > 128) return cudaErrorInvalidValue;
    fill_synthetic_kernel<<<1184, 256, 0, s>>>(cache, cscale, regions, cap, length, R, cdtype, row_bytes, seed, scale);
    return cudaGetLastError();
}

cudaError_t launch_act_quant(const float* x, int M, int E, int Kp, int rot, int rot_blk,
                             float rot_scale, int8_t* xq, float* sx, cudaStream_t s) {
    static const bool slow = std::getenv("WSVD_ACT_QUANT_SLOW") != nullptr;  // A/B and parity switch
    if (!slow && E % 512 == 0 && E / 16 <= 512 && (Kp % 16) == 0) {
        const int smem = (rot && rot_blk > 512) ? E * 4 : 0;
        static int attr = 0;
        if (smem > attr) {
            cudaError_t e = cudaFuncSetAttribute(act_quant_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            attr = smem;
        }
        return launch_pdl(act_quant_fast_kernel, dim3(M), dim3(E / 16), smem, s, x, E, Kp, rot, rot_blk, rot_scale,
                          xq, sx);
    }
    const int smem = E * 4;
    static int attr_smem = 0;
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(act_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    return launch_pdl(act_quant_kernel, dim3(M), dim3(kAqThreads), smem, s, x, E, Kp, rot, rot_blk, rot_scale,
                      xq, sx);
}

cudaError_t launch_append_epilogue(const AppendArgs& a, cudaStream_t s) {
    const bool fold = a.q_out == nullptr && a.qt != nullptr;
    const int smem = (3 * a.R + a.H + (fold ? a.R * a.R : 0)) * 4;  // R*R*4 <= 64 KB for R <= 128
    static int attr_smem = 0;
    if (smem > 48 * 1024 && smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(append_epilogue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    return launch_pdl(append_epilogue_kernel, dim3(a.nh, a.M), dim3(kEpThreads), smem, s, a);
}

cudaError_t launch_push_rows(const uint8_t* rows, int n, uint8_t* cache, int cap, int row_bytes,
                             int pos, cudaStream_t s) {
    const int total = n * (row_bytes / 16);
    push_rows_kernel<<<(total + 255) / 256, 256, 0, s>>>(rows, n, cache, cap, row_bytes, pos);
    return cudaGetLastError();
}

cudaError_t launch_absorb_query(const float* q, int B, int nh, int R, int H, const void* bk,
                                const float* bk_scale, int bdtype, float qt_scale, float* qt,
                                cudaStream_t s) {
    return launch_pdl(absorb_query_kernel, dim3(nh, B), dim3(kEpThreads), H * 4, s, q, nh, R, H, bk, bk_scale,
                      bdtype, qt_scale, qt);
}

}  // namespace wsvd_k
