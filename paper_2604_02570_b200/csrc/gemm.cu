// gemm.cu -- skinny (few-token) GEMMs of the decode step.
//
//   latent projection  C[m][n] = x_m . A_all[:, n]   (append_token's vec_mat
//                      calls x.A_K, x.A_V, x.A_Q, decode.cpp:137-139, for every
//                      head at once: N = n_heads * 3 * R columns)
//   O-projection       y[m][e] = heads_row_m . W_o[:, e]   (pipeline.cpp:329)
//
// Weights are stored K-major (one contiguous row of E values per output
// column) so a warp streams 16 weight rows with fully used 32-byte sectors.
// The MMA's M side is the weight rows and its N side the tokens ("swap AB"),
// so a decode batch of 16 tokens exactly fills two m16n8 tiles.  The k order
// inside each 32/64/128-wide block is permuted identically for the weight
// (A) and token (B) fragments, which lets every lane load its fragment with
// one 16-byte load per row; a contraction does not care about k order.
// Partial sums of each K split go to P[split][m][n]; the consumer sums the
// splits in a fixed order, so results are run-to-run deterministic.  Integer
// modes accumulate in int32 and are bit-exact.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kGemmThreads = 128;  // 4 warps x 16 weight rows
constexpr int kRowsPerCta = 64;

template <int WT>
struct GT;
template <>
struct GT<BF16> {
    static constexpr int KB = 32;      // k per block (two k16 MMA steps)
    static constexpr int XB = 2;       // bytes per X element in smem
    static constexpr int XPAD = 64;    // row pad: stride == 64 mod 128 -> conflict-free
    static constexpr int U = 8;        // blocks in flight per lane
};
template <>
struct GT<I8> {
    static constexpr int KB = 64;
    static constexpr int XB = 1;
    static constexpr int XPAD = 64;
    static constexpr int U = 8;
};
template <>
struct GT<I4> {
    static constexpr int KB = 128;
    static constexpr int XB = 1;
    static constexpr int XPAD = 16;    // 32-byte X reads per lane
    static constexpr int U = 4;
};

template <int WT>
WSVD_DEV int x_stride(int KS) {
    return KS * GT<WT>::XB + GT<WT>::XPAD;
}

// Stage X[:, k0:k0+KS] into shared memory (bf16 or int8), zero-padded to Mp rows.
template <int WT>
WSVD_DEV void stage_x(const GemmArgs& a, uint8_t* xs, int k0, int Mp) {
    const int stride = x_stride<WT>(a.KS);
    if (WT == BF16) {
        const float* X = reinterpret_cast<const float*>(a.X);
        const int per_row = a.KS / 8;  // 8 elements per thread-item
        for (int i = threadIdx.x; i < Mp * per_row; i += kGemmThreads) {
            const int m = i / per_row, kk = (i - m * per_row) * 8;
            const int k = k0 + kk;
            uint4 o = make_uint4(0, 0, 0, 0);
            if (m < a.M) {
                const float* src = X + static_cast<size_t>(m) * a.ldx + k;
                float v[8];
                if (k + 8 <= a.K && (a.ldx % 4) == 0) {
                    const float4 p0 = *reinterpret_cast<const float4*>(src);
                    const float4 p1 = *reinterpret_cast<const float4*>(src + 4);
                    v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
                    v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = (k + j < a.K) ? src[j] : 0.f;
                }
                o.x = pack_bf16x2(v[0], v[1]); o.y = pack_bf16x2(v[2], v[3]);
                o.z = pack_bf16x2(v[4], v[5]); o.w = pack_bf16x2(v[6], v[7]);
            }
            *reinterpret_cast<uint4*>(xs + m * stride + kk * 2) = o;
        }
    } else {
        const int8_t* X = reinterpret_cast<const int8_t*>(a.X);
        const int per_row = a.KS / 16;
        for (int i = threadIdx.x; i < Mp * per_row; i += kGemmThreads) {
            const int m = i / per_row, kk = (i - m * per_row) * 16;
            uint4 o = make_uint4(0, 0, 0, 0);
            if (m < a.M) o = *reinterpret_cast<const uint4*>(X + static_cast<size_t>(m) * a.Kp + k0 + kk);
            *reinterpret_cast<uint4*>(xs + m * stride + kk) = o;
        }
    }
}

template <int WT>
WSVD_DEV int w_row_bytes(int KS) {
    return WT == I4 ? KS / 2 : KS * (WT == BF16 ? 2 : 1);
}
// smem pitch of a staged weight row: == 64 (mod 128) so the 8 lanes of a
// shared-memory phase (2 rows x 4 x 16 B) hit distinct banks
template <int WT>
WSVD_DEV int w_stride(int KS) {
    const int b = w_row_bytes<WT>(KS);
    return b + ((64 - (b & 127)) & 127);
}

// One CTA: 64 weight rows x one K split.  Thread 0 streams the 64 rows of
// the split into shared memory with TMA bulk copies (one per row, completion
// on one mbarrier) while all threads convert/stage the token slice; then
// 4 warps run the MMAs out of shared memory.
template <int WT, int MT>
__global__ void __launch_bounds__(kGemmThreads) skinny_mma_kernel(const GemmArgs a) {
    using G = GT<WT>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int split = blockIdx.y;
    const int k0 = split * a.KS;
    const int Mp = MT * 16;
    const int wrb = w_row_bytes<WT>(a.KS);
    const int wst = w_stride<WT>(a.KS);
    uint8_t* ws = smem;                                     // [64][wst]
    uint8_t* xs = smem + kRowsPerCta * wst;                 // [Mp][xstride]
    uint64_t* bar = reinterpret_cast<uint64_t*>(xs + Mp * x_stride<WT>(a.KS));
    const int nc0 = blockIdx.x * kRowsPerCta;
    const int nrows = min(kRowsPerCta, a.N - nc0);

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const size_t full_row = static_cast<size_t>(WT == I4 ? a.Kp / 2 : a.Kp * (WT == BF16 ? 2 : 1));
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.W) + static_cast<size_t>(nc0) * full_row +
                             static_cast<size_t>(WT == I4 ? k0 / 2 : k0 * (WT == BF16 ? 2 : 1));
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nrows * wrb));
        for (int r = 0; r < nrows; ++r) tma_bulk_g2s(ws + r * wst, src + r * full_row, wrb, bar);
    }
    stage_x<WT>(a, xs, k0, Mp);
    __syncthreads();
    mbar_wait(bar, 0);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    if (warp * 16 >= nrows) return;
    const int stride = x_stride<WT>(a.KS);
    const uint32_t wa_lo = smem_u32(ws) + static_cast<uint32_t>((warp * 16 + g) * wst + t * 16);
    const uint32_t wa_hi = wa_lo + static_cast<uint32_t>(8 * wst);
    const uint32_t xbase = smem_u32(xs) + static_cast<uint32_t>(g * stride) +
                           static_cast<uint32_t>(WT == I4 ? t * 32 : t * 16);
    constexpr int KBB = (WT == I4) ? G::KB / 2 : G::KB * (WT == BF16 ? 2 : 1);  // weight bytes per block

    float facc[MT][2][4];
    int iacc[MT][2][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                facc[mt][hh][i] = 0.f;
                iacc[mt][hh][i] = 0;
            }

    const int nblk = a.KS / G::KB;
#pragma unroll 2
    for (int b = 0; b < nblk; ++b) {
        const uint4 wl = lds128(wa_lo + b * KBB);
        const uint4 wh = lds128(wa_hi + b * KBB);
        const uint32_t xk = static_cast<uint32_t>(b * G::KB * G::XB);
        uint32_t la[8], ha[8];
        if (WT == I4) {
            unpack_s4x8(wl.x, la[0], la[1]); unpack_s4x8(wl.y, la[2], la[3]);
            unpack_s4x8(wl.z, la[4], la[5]); unpack_s4x8(wl.w, la[6], la[7]);
            unpack_s4x8(wh.x, ha[0], ha[1]); unpack_s4x8(wh.y, ha[2], ha[3]);
            unpack_s4x8(wh.z, ha[4], ha[5]); unpack_s4x8(wh.w, ha[6], ha[7]);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const uint32_t xa = xbase + static_cast<uint32_t>((mt * 16 + hh * 8) * stride) + xk;
                if (WT == BF16) {
                    const uint4 xv = lds128(xa);
                    mma_bf16_16816(facc[mt][hh], wl.x, wh.x, wl.y, wh.y, xv.x, xv.y);
                    mma_bf16_16816(facc[mt][hh], wl.z, wh.z, wl.w, wh.w, xv.z, xv.w);
                } else if (WT == I8) {
                    const uint4 xv = lds128(xa);
                    mma_s8_16832(iacc[mt][hh], wl.x, wh.x, wl.y, wh.y, xv.x, xv.y);
                    mma_s8_16832(iacc[mt][hh], wl.z, wh.z, wl.w, wh.w, xv.z, xv.w);
                } else {
                    const uint4 x0 = lds128(xa), x1 = lds128(xa + 16);
                    mma_s8_16832(iacc[mt][hh], la[0], ha[0], la[1], ha[1], x0.x, x0.y);
                    mma_s8_16832(iacc[mt][hh], la[2], ha[2], la[3], ha[3], x0.z, x0.w);
                    mma_s8_16832(iacc[mt][hh], la[4], ha[4], la[5], ha[5], x1.x, x1.y);
                    mma_s8_16832(iacc[mt][hh], la[6], ha[6], la[7], ha[7], x1.z, x1.w);
                }
            }
        }
    }

    // D fragment: (row g | g+8, token 2t | 2t+1) of each m16n8 tile
    const int n0 = nc0 + warp * 16;
    const size_t pbase = static_cast<size_t>(split) * a.M * a.N;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int n = n0 + g + ((i & 2) ? 8 : 0);
                const int m = mt * 16 + hh * 8 + 2 * t + (i & 1);
                if (n < a.N && m < a.M) {
                    const size_t o = pbase + static_cast<size_t>(m) * a.N + n;
                    if (WT == BF16) reinterpret_cast<float*>(a.P)[o] = facc[mt][hh][i];
                    else reinterpret_cast<int*>(a.P)[o] = iacc[mt][hh][i];
                }
            }
}

// fp32 weights (config 1): CUDA-core GEMV, one warp per weight row at a time.
constexpr int kF32Rows = 32;
__global__ void __launch_bounds__(kGemmThreads) skinny_f32_kernel(const GemmArgs a) {
    extern __shared__ __align__(16) float xsf[];
    const int split = blockIdx.y;
    const int k0 = split * a.KS;
    const float* X = reinterpret_cast<const float*>(a.X);
    for (int i = threadIdx.x; i < a.M * a.KS; i += kGemmThreads) {
        const int m = i / a.KS, kk = i - m * a.KS;
        const int k = k0 + kk;
        xsf[i] = (k < a.K) ? X[static_cast<size_t>(m) * a.ldx + k] : 0.f;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* W = reinterpret_cast<const float*>(a.W);
    for (int r = warp; r < kF32Rows; r += 4) {
        const int n = blockIdx.x * kF32Rows + r;
        if (n >= a.N) break;
        const float* wrow = W + static_cast<size_t>(n) * a.Kp + k0;
        for (int m0 = 0; m0 < a.M; m0 += 8) {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int k = lane * 4; k < a.KS; k += 128) {
                const float4 w = *reinterpret_cast<const float4*>(wrow + k);
#pragma unroll
                for (int mm = 0; mm < 8; ++mm) {
                    if (m0 + mm < a.M) {
                        const float4 x = *reinterpret_cast<const float4*>(xsf + (m0 + mm) * a.KS + k);
                        acc[mm] = fmaf(w.x, x.x, acc[mm]);
                        acc[mm] = fmaf(w.y, x.y, acc[mm]);
                        acc[mm] = fmaf(w.z, x.z, acc[mm]);
                        acc[mm] = fmaf(w.w, x.w, acc[mm]);
                    }
                }
            }
#pragma unroll
            for (int mm = 0; mm < 8; ++mm) {
                const float s = warp_sum(acc[mm]);
                if (lane == 0 && m0 + mm < a.M)
                    reinterpret_cast<float*>(a.P)[(static_cast<size_t>(split) * a.M + m0 + mm) * a.N + n] = s;
            }
        }
    }
}

template <int WT, int MT>
cudaError_t launch_mma(const GemmArgs& a, cudaStream_t s) {
    const int smem = gemm_smem_bytes(WT, a.M, a.KS);
    auto k = skinny_mma_kernel<WT, MT>;
    static int attr_smem = 0;
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    dim3 grid((a.N + kRowsPerCta - 1) / kRowsPerCta, a.Kp / a.KS);
    k<<<grid, kGemmThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int WT>
cudaError_t launch_wt(const GemmArgs& a, cudaStream_t s) {
    const int mt = (a.M + 15) / 16;
    switch (mt) {
        case 1: return launch_mma<WT, 1>(a, s);
        case 2: return launch_mma<WT, 2>(a, s);
        case 3: case 4: return launch_mma<WT, 4>(a, s);
        case 5: case 6: case 7: case 8: return launch_mma<WT, 8>(a, s);
    }
    return cudaErrorInvalidValue;  // M > 128: caller tiles over M
}

__global__ void reduce_partials_kernel(const float* __restrict__ P, int splits, int MN,
                                       float* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= MN) return;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += P[static_cast<size_t>(k) * MN + i];
    y[i] = s;
}

int w_stride_h(int b) { return b + ((64 - (b & 127)) & 127); }

}  // namespace

int gemm_smem_bytes(int wdtype, int M, int KS) {
    // rows staged = the kernel's MT bucket (1, 2, 4 or 8 tiles of 16)
    const int mt = (M + 15) / 16;
    const int Mp = 16 * (mt <= 2 ? mt : (mt <= 4 ? 4 : 8));
    switch (wdtype) {
        case BF16: return kRowsPerCta * w_stride_h(KS * 2) + Mp * (KS * 2 + GT<BF16>::XPAD) + 16;
        case I8: return kRowsPerCta * w_stride_h(KS) + Mp * (KS + GT<I8>::XPAD) + 16;
        case I4: return kRowsPerCta * w_stride_h(KS / 2) + Mp * (KS + GT<I4>::XPAD) + 16;
        case F32: return M * KS * 4;
    }
    return 0;
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s) {
    switch (a.wdtype) {
        case BF16: return launch_wt<BF16>(a, s);
        case I8: return launch_wt<I8>(a, s);
        case I4: return launch_wt<I4>(a, s);
        case F32: {
            const int smem = gemm_smem_bytes(F32, a.M, a.KS);
            static int attr_smem = 0;
            if (smem > attr_smem) {
                cudaError_t e = cudaFuncSetAttribute(skinny_f32_kernel,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
                attr_smem = smem;
            }
            dim3 grid((a.N + kF32Rows - 1) / kF32Rows, a.Kp / a.KS);
            skinny_f32_kernel<<<grid, kGemmThreads, smem, s>>>(a);
            return cudaGetLastError();
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_partials(const float* P, int splits, int M, int N, float* y,
                                   cudaStream_t s) {
    const int MN = M * N;
    reduce_partials_kernel<<<(MN + 255) / 256, 256, 0, s>>>(P, splits, MN, y);
    return cudaGetLastError();
}

}  // namespace wsvd_k
