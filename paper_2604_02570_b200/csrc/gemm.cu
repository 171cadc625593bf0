// gemm.cu -- skinny (few-token) GEMMs of the decode step.
//
//   latent projection  C[m][n] = x_m . A_all[:, n]   (append_token's vec_mat
//                      calls x.A_K, x.A_V, x.A_Q, decode.cpp:137-139, for every
//                      head at once: N = n_heads * 3 * R columns)
//   O-projection       y[m][e] = vlat_m . W'_o[:, e], W'_o = B_V . W_o
//                      (pipeline.cpp:323-329 with the V up-projection folded in)
//
// Weight layout in HBM ("W-tiles"): every (16-row tile, K split) work item is
// one contiguous block [16 rows][KS] -- rows are output columns, K-major --
// with the 16-byte units of odd rows XOR-ed by 4 so that the MMA fragment
// loads are bank-conflict free.  One TMA bulk copy moves one work item.
//
// The MMA's M side is the weight rows and its N side the tokens ("swap AB"),
// so a decode batch of 16 tokens exactly fills two m16n8 tiles.  The k order
// inside each 32/64/128-wide block is permuted identically for the weight
// (A) and token (B) fragments, which lets every lane load its fragment with
// one 16-byte load per row; a contraction does not care about k order.
// Partial sums of each K split go to P[split][m][n]; consumers sum the
// splits in a fixed order, so results are run-to-run deterministic.  Integer
// modes accumulate in int32 and are bit-exact.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {


template <int WT>
struct GT;
template <>
struct GT<BF16> {
    static constexpr int KB = 32;      // k per block (two k16 MMA steps)
    static constexpr int XB = 2;       // bytes per X element in smem
    static constexpr int XPAD = 64;    // row pad: stride == 64 mod 128 -> conflict-free
};
template <>
struct GT<I8> {
    static constexpr int KB = 64;
    static constexpr int XB = 1;
    static constexpr int XPAD = 64;
};
template <>
struct GT<I4> {
    static constexpr int KB = 128;
    static constexpr int XB = 1;
    static constexpr int XPAD = 16;    // 32-byte X reads per lane
};

template <int WT>
__host__ __device__ __forceinline__ int x_stride(int KS) {
    return KS * GT<WT>::XB + GT<WT>::XPAD;
}

// Stage X[:, k0:k0+KS] into shared memory (bf16 or int8), zero-padded to Mp
// rows.  Loads are issued in batches of 8 per thread before any is consumed,
// so staging costs one memory latency per batch rather than one per item.
// With a.xsplit (bf16 mode, O-projection input): rows [0, Mp/2) hold
// hi = bf16(x) of token rows 0.., rows [Mp/2, Mp) lo = bf16(x - hi) of the
// same tokens; the epilogue adds the two products (~16 mantissa bits of the
// fp32 activation reach the tensor cores).
WSVD_DEV uint32_t pack_lo_bf16x2(float a, float b) {
    const float ha = __bfloat162float(__float2bfloat16_rn(a));
    const float hb = __bfloat162float(__float2bfloat16_rn(b));
    return pack_bf16x2(a - ha, b - hb);
}

template <int WT, int kXThreads>
WSVD_DEV void stage_x(const GemmArgs& a, uint8_t* xs, int k0, int Mp) {
    if (threadIdx.x >= kXThreads) return;  // the first kXThreads threads stage the slice
    const int stride = x_stride<WT>(a.KS);
    constexpr int BATCH = 8;
    if (WT == BF16) {
        const float* X = reinterpret_cast<const float*>(a.X);
        const int per_row = a.KS / 8;  // 8 elements per thread-item
        const int n = Mp * per_row;
        const bool vec = (a.ldx % 4) == 0;
        for (int i0 = threadIdx.x; i0 < n; i0 += kXThreads * BATCH) {
            float4 p[BATCH][2];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int i = i0 + u * kXThreads;
                const int m = i / per_row, kk = (i - m * per_row) * 8;
                const int k = k0 + kk;
                const int ms = (a.xsplit && m >= Mp / 2) ? m - Mp / 2 : m;  // source token row
                p[u][0] = p[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < n && ms < a.M && (!a.xsplit || ms < Mp / 2)) {
                    const float* src = X + static_cast<size_t>(ms) * a.ldx + k;
                    if (k + 8 <= a.K && vec) {
                        p[u][0] = __ldg(reinterpret_cast<const float4*>(src));
                        p[u][1] = __ldg(reinterpret_cast<const float4*>(src + 4));
                    } else {
                        float v[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] = (k + j < a.K) ? src[j] : 0.f;
                        p[u][0] = make_float4(v[0], v[1], v[2], v[3]);
                        p[u][1] = make_float4(v[4], v[5], v[6], v[7]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int i = i0 + u * kXThreads;
                if (i >= n) break;
                const int m = i / per_row, kk = (i - m * per_row) * 8;
                uint4 o;
                if (a.xsplit && m >= Mp / 2) {
                    o.x = pack_lo_bf16x2(p[u][0].x, p[u][0].y); o.y = pack_lo_bf16x2(p[u][0].z, p[u][0].w);
                    o.z = pack_lo_bf16x2(p[u][1].x, p[u][1].y); o.w = pack_lo_bf16x2(p[u][1].z, p[u][1].w);
                } else {
                    o.x = pack_bf16x2(p[u][0].x, p[u][0].y); o.y = pack_bf16x2(p[u][0].z, p[u][0].w);
                    o.z = pack_bf16x2(p[u][1].x, p[u][1].y); o.w = pack_bf16x2(p[u][1].z, p[u][1].w);
                }
                *reinterpret_cast<uint4*>(xs + m * stride + kk * 2) = o;
            }
        }
    } else {
        const int8_t* X = reinterpret_cast<const int8_t*>(a.X);
        const int per_row = a.KS / 16;
        const int n = Mp * per_row;
        for (int i0 = threadIdx.x; i0 < n; i0 += kXThreads * BATCH) {
            uint4 o[BATCH];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int i = i0 + u * kXThreads;
                const int m = i / per_row, kk = (i - m * per_row) * 16;
                o[u] = make_uint4(0, 0, 0, 0);
                if (i < n && m < a.M)
                    o[u] = __ldg(reinterpret_cast<const uint4*>(X + static_cast<size_t>(m) * a.Kp + k0 + kk));
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int i = i0 + u * kXThreads;
                if (i >= n) break;
                const int m = i / per_row, kk = (i - m * per_row) * 16;
                *reinterpret_cast<uint4*>(xs + m * stride + kk) = o[u];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent streaming GEMM.  CTAs are assigned split-aligned: CTA c works on
// K split c % splits and a contiguous run of 16-row tiles, so it stages one
// token slice.  A producer warp streams each work item (one W-tile block) into
// a ring of shared-memory slots with one TMA bulk copy per item (completion on
// the slot's mbarrier); consumer warp w takes items w, w+4, ... and runs the
// MMAs straight from the slot.  One CTA per SM, deep bytes-in-flight, no wave
// quantisation.
// consumer warps: 4, or 8 for 64 token rows (MMA issue then dominates an item).
// Consumer warp w takes items w, w + C, ... of one ring, so the ring needs at
// least C slots: a slot's previous fill must be complete before its next
// waiter arrives (parity waits cannot tell phase u from u - 2).  MT = 8 keeps
// 4 consumers (its 128-row token slice leaves room for 5 slots).
template <int MT>
struct StreamWarps {
    static constexpr int C = MT == 4 ? 8 : 4;
    static constexpr int THREADS = 32 * (C + 1);
};

template <int WT, int MT>
struct StreamCfg {
    static constexpr int MTV = MT;
    static constexpr int XROWS = MT * 16;
    __host__ __device__ static int ksb(int KS) { return WT == I4 ? KS / 2 : KS * (WT == BF16 ? 2 : 1); }
    __host__ __device__ static int item_bytes(int KS) { return 16 * ksb(KS); }
    __host__ __device__ static int xbytes(int KS) { return XROWS * x_stride<WT>(KS); }
    __host__ __device__ static int stages(int KS) {
        const int budget = 222 * 1024 - xbytes(KS) - 256;
        int s = budget / item_bytes(KS);
        return s > 8 ? 8 : s;
    }
    __host__ __device__ static int smem(int KS) { return stages(KS) * item_bytes(KS) + xbytes(KS) + 256; }
};

template <int WT, int MT>
__global__ void __launch_bounds__(StreamWarps<MT>::THREADS, 1) skinny_stream_kernel(const GemmArgs a) {
    constexpr int kStreamConsumers = StreamWarps<MT>::C;
    using G = GT<WT>;
    using S = StreamCfg<WT, MT>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int KS = a.KS;
    const int nst = S::stages(KS);
    const int ksb = S::ksb(KS), xst = x_stride<WT>(KS);
    const int ibytes = S::item_bytes(KS);
    uint8_t* ring = smem;
    uint8_t* xbuf = smem + nst * ibytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + S::xbytes(KS));
    uint64_t* empty = full + 8;

    const int splits = a.Kp / KS;
    const int cps = gridDim.x / splits;  // CTAs per split
    const int s = blockIdx.x % splits, j = blockIdx.x / splits;
    // the layer step's length commit, before any early exit (CTA 0 may own no
    // tile when N/16 < the grid); after the predecessor, which read the length
    if (a.commit_len && blockIdx.x == 0 && threadIdx.x == 0) {
        griddep_wait();
        atomicAdd(a.commit_len, 1);
    }
    if (j >= cps) return;
    const int tiles = (a.N + 15) / 16;
    const int lo = static_cast<int>(static_cast<long>(j) * tiles / cps);
    const int hi = static_cast<int>(static_cast<long>(j + 1) * tiles / cps);
    if (lo >= hi) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kStreamConsumers) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            const uint8_t* W = reinterpret_cast<const uint8_t*>(a.W);
            for (int tile = lo; tile < hi; ++tile) {
                const int k = tile - lo, slot = k % nst;
                const uint32_t ph = static_cast<uint32_t>(k / nst) & 1u;
                mbar_wait(&empty[slot], ph ^ 1u);
                mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(ibytes));
                tma_bulk_g2s(ring + slot * ibytes, W + (static_cast<size_t>(tile) * splits + s) * ibytes, ibytes,
                             &full[slot]);
            }
        }
        return;
    }

    // ------------------------------------------------ consumers
    // the weight stream above needs nothing from the previous kernel; the
    // token slice, the partial outputs and the length commit do
    griddep_wait();
    griddep_launch_dependents();
    stage_x<WT, 32 * kStreamConsumers>(a, xbuf, s * KS, S::XROWS);  // every consumer thread stages
    named_bar_sync(1, 32 * kStreamConsumers);

    const int g = lane >> 2, t = lane & 3;
    const uint32_t swz = static_cast<uint32_t>((g & 1) << 2);  // unit ^= 4 on odd rows
    const uint32_t xbase = smem_u32(xbuf) + static_cast<uint32_t>(g * xst) +
                           static_cast<uint32_t>(WT == I4 ? t * 32 : t * 16);
    const int nblk = KS / G::KB;
    for (int tile = lo + warp; tile < hi; tile += kStreamConsumers) {
        const int k = tile - lo, slot = k % nst;
        const uint32_t ph = static_cast<uint32_t>(k / nst) & 1u;
        mbar_wait(&full[slot], ph);
        const uint32_t rb = smem_u32(ring + slot * ibytes);
        const uint32_t row_lo = rb + static_cast<uint32_t>(g * ksb);
        const uint32_t row_hi = row_lo + static_cast<uint32_t>(8 * ksb);
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
#pragma unroll 2
        for (int b = 0; b < nblk; ++b) {
            // this lane's 16-byte unit of block b: logical unit 4b + t
            const uint32_t uoff = ((static_cast<uint32_t>(4 * b + t)) ^ swz) * 16;
            const uint4 wl = lds128(row_lo + uoff);
            const uint4 wh = lds128(row_hi + uoff);
            const uint32_t xk = static_cast<uint32_t>(b * G::KB * G::XB);
            uint32_t la[8], ha[8];
            if (WT == I4) {
                unpack_s4x8(wl.x, la[0], la[1]); unpack_s4x8(wl.y, la[2], la[3]);
                unpack_s4x8(wl.z, la[4], la[5]); unpack_s4x8(wl.w, la[6], la[7]);
                unpack_s4x8(wh.x, ha[0], ha[1]); unpack_s4x8(wh.y, ha[2], ha[3]);
                unpack_s4x8(wh.z, ha[4], ha[5]); unpack_s4x8(wh.w, ha[6], ha[7]);
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t xa = xbase + static_cast<uint32_t>((mt * 16 + hh * 8) * xst) + xk;
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        // D fragment: (row g | g+8, token 2t | 2t+1) of each m16n8 tile
        const size_t pbase = static_cast<size_t>(s) * a.M * a.N;
        if (WT == BF16 && MT % 2 == 0 && a.xsplit) {
            // token tile mt holds hi, mt + MT/2 lo of the same tokens
#pragma unroll
            for (int mt = 0; mt < MT / 2; ++mt)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int n = tile * 16 + g + ((i & 2) ? 8 : 0);
                        const int m = mt * 16 + hh * 8 + 2 * t + (i & 1);
                        if (n < a.N && m < a.M)
                            reinterpret_cast<float*>(a.P)[pbase + static_cast<size_t>(m) * a.N + n] =
                                facc[mt][hh][i] + facc[mt + MT / 2][hh][i];
                    }
            continue;
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int n = tile * 16 + g + ((i & 2) ? 8 : 0);
                    const int m = mt * 16 + hh * 8 + 2 * t + (i & 1);
                    if (n < a.N && m < a.M) {
                        const size_t o = pbase + static_cast<size_t>(m) * a.N + n;
                        if (WT == BF16) reinterpret_cast<float*>(a.P)[o] = facc[mt][hh][i];
                        else reinterpret_cast<int*>(a.P)[o] = iacc[mt][hh][i];
                    }
                }
    }
}

// fp32 weights (config 1): CUDA-core GEMV over the plain [N][Kp] layout, one
// warp per weight row at a time.
constexpr int kF32Rows = 32;
constexpr int kF32Threads = 128;
__global__ void __launch_bounds__(kF32Threads) skinny_f32_kernel(const GemmArgs a) {
    extern __shared__ __align__(16) float xsf[];
    const int split = blockIdx.y;
    griddep_wait();
    griddep_launch_dependents();
    if (a.commit_len && blockIdx.x == 0 && split == 0 && threadIdx.x == 0) atomicAdd(a.commit_len, 1);
    const int k0 = split * a.KS;
    const float* X = reinterpret_cast<const float*>(a.X);
    for (int i = threadIdx.x; i < a.M * a.KS; i += kF32Threads) {
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
                const float sum = warp_sum(acc[mm]);
                if (lane == 0 && m0 + mm < a.M)
                    reinterpret_cast<float*>(a.P)[(static_cast<size_t>(split) * a.M + m0 + mm) * a.N + n] = sum;
            }
        }
    }
}

// fp32 decode GEMV (M <= kF32RowsM token rows).  Work items are (row, K split)
// pieces of U*128 floats -- U float4 per lane, one coalesced 512-byte warp
// load each -- dealt round-robin to the warps of a persistent grid, so every
// SM streams the same number of bytes; each warp double-buffers its items in
// registers (the next item is in flight while the current one is consumed,
// the first before the grid-dependency wait: weights do not depend on the
// previous kernel).  x sits in shared memory, staged once per CTA.  Partials
// go to P[split][M][N] like the other projection kernels.
constexpr int kF32RowsM = 4;
constexpr int kF32RowsThreads = 256;
template <int M, int U>
__global__ void __launch_bounds__(kF32RowsThreads, 2) skinny_f32_rows_kernel(const GemmArgs a) {
    extern __shared__ __align__(16) float xsf[];
    const int lane = threadIdx.x & 31;
    const float* W = reinterpret_cast<const float*>(a.W);
    const int splits = a.Kp / (U * 128);
    const int items = a.N * splits;
    const int nwarps = gridDim.x * (kF32RowsThreads / 32);
    const int gw = blockIdx.x * (kF32RowsThreads / 32) + (threadIdx.x >> 5);
    float4 w[U], wn[U];
    auto load = [&](int t, float4* dst) {
        const int n = t / splits, sp = t - n * splits;
        const float4* src = reinterpret_cast<const float4*>(W + static_cast<size_t>(n) * a.Kp + sp * U * 128) + lane;
#pragma unroll
        for (int u = 0; u < U; ++u) dst[u] = t < items ? __ldcs(src + u * 32) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    load(gw, w);
    griddep_wait();
    griddep_launch_dependents();
    if (a.commit_len && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.commit_len, 1);
    const float* X = reinterpret_cast<const float*>(a.X);
    if ((a.K & 3) == 0 && (a.ldx & 3) == 0) {
        const int kv = a.Kp >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < M * kv; i += kF32RowsThreads) {
            const int m = i / kv, k = (i - m * kv) * 4;
            reinterpret_cast<float4*>(xsf)[i] = k < a.K ? *reinterpret_cast<const float4*>(X + static_cast<size_t>(m) * a.ldx + k)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
        for (int i = threadIdx.x; i < M * a.Kp; i += kF32RowsThreads) {
            const int m = i / a.Kp, k = i - m * a.Kp;
            xsf[i] = (k < a.K) ? X[static_cast<size_t>(m) * a.ldx + k] : 0.f;
        }
    }
    __syncthreads();
    for (int t = gw; t < items; t += nwarps) {
        load(t + nwarps, wn);
        const int n = t / splits, sp = t - n * splits;
        float acc[M];
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = sp * U * 32 + u * 32 + lane;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const float4 x = reinterpret_cast<const float4*>(xsf + m * a.Kp)[v];
                acc[m] = fmaf(w[u].x, x.x, acc[m]);
                acc[m] = fmaf(w[u].y, x.y, acc[m]);
                acc[m] = fmaf(w[u].z, x.z, acc[m]);
                acc[m] = fmaf(w[u].w, x.w, acc[m]);
            }
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const float sum = warp_sum(acc[m]);
            if (lane == 0) reinterpret_cast<float*>(a.P)[(static_cast<size_t>(sp) * a.M + m) * a.N + n] = sum;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) w[u] = wn[u];
    }
}

// fp32 decode GEMV over a TMA ring (M <= 4 token rows, Kp <= 4096): one CTA
// per SM streams a contiguous run of whole weight rows (Kp * 4 bytes each)
// through 8 stages -- 128 KB in flight per SM, where the register double
// buffer above holds ~32 KB -- and warp w owns stage w (rows i = w mod 8, so
// every fill of a stage is consumed by one warp, in order).  The first stages
// go out before the grid-dependency wait.  One K split: P[0][M][N].
constexpr int kGvW = 8;  // consumer warps = stages
template <int M>
__global__ void __launch_bounds__(32 * (kGvW + 1), 1) gemv_f32_tma_kernel(const GemmArgs a) {
    extern __shared__ __align__(128) uint8_t gsm[];
    const int rb = a.Kp * 4;
    float* xs = reinterpret_cast<float*>(gsm + kGvW * rb);  // [M][Kp]
    uint64_t* full = reinterpret_cast<uint64_t*>(xs + M * a.Kp);
    uint64_t* empty = full + kGvW;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n0 = static_cast<int>(static_cast<long>(blockIdx.x) * a.N / gridDim.x);
    const int n1 = static_cast<int>(static_cast<long>(blockIdx.x + 1) * a.N / gridDim.x);
    const float* W = reinterpret_cast<const float*>(a.W);
    if (tid == 0) {
        for (int i = 0; i < kGvW; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int pre = min(kGvW, n1 - n0);
    if (warp == kGvW && lane == 0)
        for (int i = 0; i < pre; ++i) {
            mbar_arrive_expect_tx(&full[i], rb);
            tma_bulk_g2s(gsm + i * rb, W + static_cast<size_t>(n0 + i) * a.Kp, rb, &full[i]);
        }
    griddep_wait();
    griddep_launch_dependents();
    if (a.commit_len && blockIdx.x == 0 && tid == 0) atomicAdd(a.commit_len, 1);
    if (warp == kGvW) {
        if (lane == 0)
            for (int i = pre; i < n1 - n0; ++i) {
                const int st = i % kGvW;
                mbar_wait(&empty[st], ((i / kGvW) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[st], rb);
                tma_bulk_g2s(gsm + st * rb, W + static_cast<size_t>(n0 + i) * a.Kp, rb, &full[st]);
            }
        return;
    }
    const float* X = reinterpret_cast<const float*>(a.X);
    for (int i = tid; i < M * a.Kp; i += 32 * kGvW) {
        const int m = i / a.Kp, k = i - m * a.Kp;
        xs[i] = k < a.K ? X[static_cast<size_t>(m) * a.ldx + k] : 0.f;
    }
    named_bar_sync(1, 32 * kGvW);
    const int kv = a.Kp / 128;  // float4 per lane per row
    for (int i = warp; i < n1 - n0; i += kGvW) {
        const int st = i % kGvW;
        mbar_wait(&full[st], (i / kGvW) & 1u);
        const float4* wr = reinterpret_cast<const float4*>(gsm + st * rb) + lane;
        float acc[M];
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = 0.f;
#pragma unroll 4
        for (int v = 0; v < kv; ++v) {
            const float4 w = wr[v * 32];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const float4 x = reinterpret_cast<const float4*>(xs + m * a.Kp)[v * 32 + lane];
                acc[m] = fmaf(w.x, x.x, acc[m]);
                acc[m] = fmaf(w.y, x.y, acc[m]);
                acc[m] = fmaf(w.z, x.z, acc[m]);
                acc[m] = fmaf(w.w, x.w, acc[m]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const float sum = warp_sum(acc[m]);
            if (lane == 0) reinterpret_cast<float*>(a.P)[static_cast<size_t>(m) * a.N + n0 + i] = sum;
        }
    }
}

template <int M>
cudaError_t launch_gemv_f32_tma(const GemmArgs& a, cudaStream_t s) {
    const int smem = kGvW * a.Kp * 4 + M * a.Kp * 4 + 2 * kGvW * 8;
    auto k = gemv_f32_tma_kernel<M>;
    static int attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    return launch_pdl(k, dim3(std::min(a.grid, a.N)), dim3(32 * (kGvW + 1)), smem, s, a);
}

template <int M, int U>
cudaError_t launch_f32_rows_u(const GemmArgs& a, cudaStream_t s) {
    const int smem = M * a.Kp * 4;
    auto k = skinny_f32_rows_kernel<M, U>;
    static int attr_smem = 0;
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    const int wpc = kF32RowsThreads / 32;
    static int per_sm = 0;  // resident CTAs per SM (registers / shared memory), at most 4
    if (per_sm == 0) {
        int nb = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kF32RowsThreads, smem) != cudaSuccess) nb = 1;
        per_sm = std::max(1, std::min(4, nb));
    }
    const int items = a.N * (a.Kp / (U * 128));
    const int grid = std::max(1, std::min((items + wpc - 1) / wpc, a.grid * per_sm));
    return launch_pdl(k, dim3(grid), dim3(kF32RowsThreads), smem, s, a);
}

template <int M>
cudaError_t launch_f32_rows(const GemmArgs& a, cudaStream_t s) {
    switch (a.KS / 128) {
        case 2: return launch_f32_rows_u<M, 2>(a, s);
        case 4: return launch_f32_rows_u<M, 4>(a, s);
        default: return launch_f32_rows_u<M, 8>(a, s);
    }
}

template <int WT, int MT>
cudaError_t launch_stream(const GemmArgs& a, cudaStream_t s) {
    using S = StreamCfg<WT, MT>;
    if (S::stages(a.KS) < StreamWarps<MT>::C) return cudaErrorInvalidConfiguration;  // see StreamWarps
    const int smem = S::smem(a.KS);
    auto k = skinny_stream_kernel<WT, MT>;
    static int attr_smem = 0;
    if (smem > attr_smem) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem = smem;
    }
    const int splits = a.Kp / a.KS;
    const int grid = splits <= a.grid ? (a.grid / splits) * splits : splits;
    return launch_pdl(k, dim3(grid), dim3(StreamWarps<MT>::THREADS), smem, s, a);
}

template <int WT>
cudaError_t launch_wt(const GemmArgs& a, cudaStream_t s) {
    if (a.xsplit) {  // hi and lo token tiles: twice the token rows (M <= 64)
        if (WT != BF16) return cudaErrorInvalidValue;
        switch ((a.M + 15) / 16) {
            case 1: return launch_stream<WT, 2>(a, s);
            case 2: return launch_stream<WT, 4>(a, s);
            case 3: case 4: return launch_stream<WT, 8>(a, s);
        }
        return cudaErrorInvalidValue;
    }
    switch ((a.M + 15) / 16) {
        case 1: return launch_stream<WT, 1>(a, s);
        case 2: return launch_stream<WT, 2>(a, s);
        case 3: case 4: return launch_stream<WT, 4>(a, s);
        case 5: case 6: case 7: case 8: return launch_stream<WT, 8>(a, s);
    }
    return cudaErrorInvalidValue;  // M > 128: the caller tiles over M
}

__global__ void reduce_partials_kernel(const float* __restrict__ P, int splits, int MN,
                                       void* __restrict__ y, int act, int y_bf16) {
    griddep_wait();
    griddep_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= MN) return;
    float sum = 0.f;
#pragma unroll 8
    for (int k = 0; k < splits; ++k) sum += __ldcg(P + static_cast<size_t>(k) * MN + i);
    const float v = act == 1 ? tanhf(sum) : sum;  // act 1: the toy FFN's tanh (pipeline.cpp:331-333)
    if (y_bf16) static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(v);
    else static_cast<float*>(y)[i] = v;
}

}  // namespace

bool f32_tma_path(int M, int Kp, int KS) { return M >= 1 && M <= kF32RowsM && KS == Kp && Kp % 128 == 0 && Kp <= 4096; }

bool f32_rows_path(int M, int Kp, int KS) {
    return M <= kF32RowsM && (KS == 256 || KS == 512 || KS == 1024) && Kp % KS == 0 && M * Kp * 4 <= 200 * 1024;
}

bool gemm_fits(int wdtype, int M, int KS) {
    const int mt = (M + 15) / 16;
    auto st = [&](auto cfg) { return decltype(cfg)::stages(KS) >= StreamWarps<decltype(cfg)::MTV>::C; };
    switch (wdtype) {
        case BF16: return mt <= 1 ? st(StreamCfg<BF16, 1>{}) : mt <= 2 ? st(StreamCfg<BF16, 2>{}) : mt <= 4 ? st(StreamCfg<BF16, 4>{}) : st(StreamCfg<BF16, 8>{});
        case I8: return mt <= 1 ? st(StreamCfg<I8, 1>{}) : mt <= 2 ? st(StreamCfg<I8, 2>{}) : mt <= 4 ? st(StreamCfg<I8, 4>{}) : st(StreamCfg<I8, 8>{});
        case I4: return mt <= 1 ? st(StreamCfg<I4, 1>{}) : mt <= 2 ? st(StreamCfg<I4, 2>{}) : mt <= 4 ? st(StreamCfg<I4, 4>{}) : st(StreamCfg<I4, 8>{});
        case F32: return M * KS * 4 <= 200 * 1024;
    }
    return false;
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s) {
    switch (a.wdtype) {
        case BF16: return launch_wt<BF16>(a, s);
        case I8: return launch_wt<I8>(a, s);
        case I4: return launch_wt<I4>(a, s);
        case F32: {
            static const bool no_tma = std::getenv("WSVD_F32_ROWS") != nullptr;  // A/B switch: register GEMV
            if (!no_tma && f32_tma_path(a.M, a.Kp, a.KS)) {
                switch (a.M) {
                    case 1: return launch_gemv_f32_tma<1>(a, s);
                    case 2: return launch_gemv_f32_tma<2>(a, s);
                    case 3: return launch_gemv_f32_tma<3>(a, s);
                    default: return launch_gemv_f32_tma<4>(a, s);
                }
            }
            if (f32_rows_path(a.M, a.Kp, a.KS)) {
                switch (a.M) {
                    case 1: return launch_f32_rows<1>(a, s);
                    case 2: return launch_f32_rows<2>(a, s);
                    case 3: return launch_f32_rows<3>(a, s);
                    default: return launch_f32_rows<4>(a, s);
                }
            }
            const int smem = a.M * a.KS * 4;
            static int attr_smem = 0;
            if (smem > attr_smem) {
                cudaError_t e = cudaFuncSetAttribute(skinny_f32_kernel,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
                attr_smem = smem;
            }
            dim3 grid((a.N + kF32Rows - 1) / kF32Rows, a.Kp / a.KS);
            return launch_pdl(skinny_f32_kernel, grid, dim3(kF32Threads), smem, s, a);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_partials(const float* P, int splits, int M, int N, void* y,
                                   cudaStream_t s, int act, int y_bf16) {
    const int MN = M * N;
    return launch_pdl(reduce_partials_kernel, dim3((MN + 255) / 256), dim3(256), 0, s, P, splits, MN, y, act, y_bf16);
}

}  // namespace wsvd_k
