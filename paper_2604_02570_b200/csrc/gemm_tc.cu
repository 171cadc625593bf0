// gemm_tc.cu -- dense GEMM on the 5th-generation tensor cores for the token
// GEMMs that are real contractions (the decode stack's feed-forward at 128
// sequences, pipeline.cpp:330-334):  D[M][N] = X[M][K] . W[N][K]^T with M <= 128
// token rows, bf16 operands, fp32 accumulation in TMEM.
//
// One CTA per (N tile of 64 columns, K split): warp 0 streams 64-wide K chunks
// of X and W with TMA (2-D tensor maps, 128-byte swizzle) through an 8-stage
// ring -- W stored K-chunk-major so each box is one contiguous block, its
// first stages issued before the grid-dependency wait; the CTAs of a cluster
// (up to 4 consecutive N tiles of one K split) each load a quarter of every X
// chunk and multicast it to all of them.  One elected thread of warp 1 issues
// tcgen05.mma (M = 128, N = 64, K = 16 per instruction, four per chunk) into a
// 64-column TMEM accumulator and frees each stage in every CTA of the cluster
// with a multicast tcgen05.commit; the four warps then read the accumulator
// back with tcgen05.ld (thread r <-> row r) and apply the epilogue: tanh +
// bf16 (the FFN's hidden activations) or fp32 (final / split partials).
// Measured variants (tools/ffn_timing.py): 256-column tiles with more K
// splits, and an in-kernel last-arriver split sum, were both slower.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kBM = 128;              // token rows per tile (TMEM lanes)
constexpr int kBN = 64;               // output columns per CTA (TMEM accumulator columns)
constexpr int kBK = 64;               // K per chunk: one 128-byte swizzle atom of bf16
constexpr int kStages = 8;
constexpr int kMaxCl = 4;             // CTAs per cluster (consecutive N tiles): X chunks are multicast
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kBBytes = kBN * kBK * 2;  // 8 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kSmem = kStages * kStageBytes + 1024 + 256;  // + 1 KB alignment slack + barriers + flags

// Shared-memory matrix descriptor (sm_100), K-major operand in the 128-byte
// swizzle: rows of 128 B, 8-row groups 1024 B apart (SBO); LBO unused.
WSVD_DEV uint64_t sw128_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(16u >> 4) << 16;
    d |= static_cast<uint64_t>(1024u >> 4) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;  // SWIZZLE_128B
    return d;
}
// kind::f16 instruction descriptor: D fp32, A / B bf16, both K-major, M = 128, N = kBN
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

// X rows [32 r, 32 r + 32) of a chunk into the same offset of every CTA of the cluster
WSVD_DEV void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
WSVD_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
WSVD_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(128, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap xmap,
                                                         const __grid_constant__ CUtensorMap wmap,
                                                         const __grid_constant__ TcGemmArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntile = blockIdx.x % a.ntiles, split = blockIdx.x / a.ntiles;
    const int n0 = ntile * kBN;
    const int kchunks = a.K / kBK;
    const int c0 = static_cast<int>(static_cast<long>(split) * kchunks / a.splits);
    const int c1 = static_cast<int>(static_cast<long>(split + 1) * kchunks / a.splits);
    const uint32_t crank = a.cl > 1 ? cluster_rank() : 0u;
    const int kCl = a.cl;
    const uint16_t cmask = static_cast<uint16_t>((1u << kCl) - 1u);
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kCl);  // a stage is free once every CTA's MMAs have read it
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kBN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (kCl > 1) cluster_sync_all();  // every CTA's barriers exist before any multicast lands
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    // the weights never depend on the predecessor: the first stages' W loads go
    // out before it has drained (programmatic dependent launch), X after
    const int pre = min(kStages, c1 - c0);
    if (warp == 0 && lane == 0)
        for (int i = 0; i < pre; ++i) {
            mbar_arrive_expect_tx(&full[i], kStageBytes);  // X from the kCl CTAs' multicasts + own W
            tma_load_2d(smem + i * kStageBytes + kABytes, &wmap, 0, (c0 + i) * a.N + n0, &full[i]);
        }
    griddep_wait();
    griddep_launch_dependents();

    if (warp == 0 && lane == 0) {
        for (int c = c0; c < c1; ++c) {
            const int i = c - c0, s = i % kStages;
            uint8_t* st = smem + s * kStageBytes;
            if (i >= pre) {
                mbar_wait(&empty[s], ((i / kStages) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full[s], kStageBytes);
                tma_load_2d(st + kABytes, &wmap, 0, c * a.N + n0, &full[s]);  // W chunk-major: one contiguous box
            }
            if (kCl > 1)
                tma_load_2d_mc(st + crank * (kABytes / kCl), &xmap, c * kBK, static_cast<int>(crank) * (kBM / kCl),
                               &full[s], cmask);
            else
                tma_load_2d(st, &xmap, c * kBK, 0, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        for (int c = c0; c < c1; ++c) {
            const int i = c - c0, s = i % kStages;
            mbar_wait(&full[s], (i / kStages) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t abase = smem_u32(smem + s * kStageBytes), bbase = abase + kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
                const uint64_t ad = sw128_desc(abase + k * 32), bd = sw128_desc(bbase + k * 32);
                const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
            }
            // the stage's X rows were written into every CTA: free it in all of them
            if (kCl > 1)
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                        smem_u32(&empty[s])),
                    "h"(cmask)
                    : "memory");
            else
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&empty[s]))
                             : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(done))
                     : "memory");
    }
    __syncwarp();
    // ---- epilogue: thread r holds token row r's kBN accumulator columns
    mbar_wait(done, 0u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    auto tmem_group = [&](int g, float (&v)[16]) {
        uint32_t r[16];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(g * 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    };
    auto finish = [&](int g, float (&v)[16]) {  // act + store of the complete sums
        if (row >= a.M) return;
        const int col = n0 + g * 16;
        if (a.act == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = tanhf(v[j]);  // the toy FFN's activation (pipeline.cpp:331-333)
        }
        if (a.out_bf16) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.out) + static_cast<size_t>(row) * a.ldo + col);
            dst[0] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                                pack_bf16x2(v[6], v[7]));
            dst[1] = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]), pack_bf16x2(v[12], v[13]),
                                pack_bf16x2(v[14], v[15]));
        } else {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.out) + static_cast<size_t>(row) * a.ldo + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    };
    if (a.splits == 1) {
#pragma unroll 1
        for (int g = 0; g < kBN / 16; ++g) {
            float v[16];
            tmem_group(g, v);
            finish(g, v);
        }
    } else {
        // K splits: fp32 partial tiles [split][M][ldo]; the caller sums them
        // (launch_reduce_partials, fixed split order)
#pragma unroll 1
        for (int g = 0; g < kBN / 16; ++g) {
            float v[16];
            tmem_group(g, v);
            if (row >= a.M) continue;
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.out) +
                                                    (static_cast<size_t>(split) * (a.ldm ? a.ldm : a.M) + row) * a.ldo +
                                                    n0 + g * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (kCl > 1) cluster_sync_all();  // no CTA leaves while a peer may still arrive on its barriers
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kBN));
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, size_t n4) {
    griddep_wait();
    griddep_launch_dependents();
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    reinterpret_cast<uint2*>(y)[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
}

// one 16-byte unit (8 bf16 of row n, K offset k0) per thread
__global__ void wtiles_to_chunks_kernel(const uint8_t* __restrict__ wt, int N, int Kp, int ks, uint8_t* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // unit index, n-major
    const int upr = Kp / 8;
    if (i >= static_cast<size_t>(N) * upr) return;
    const int n = static_cast<int>(i / upr), k0 = static_cast<int>(i % upr) * 8;
    const int tile = n / 16, rr = n % 16, sp = k0 / ks, u = (k0 % ks) / 8, splits = Kp / ks;
    const size_t src = ((static_cast<size_t>(tile) * splits + sp) * 16 + rr) * ks * 2 + static_cast<size_t>(u ^ ((rr & 1) << 2)) * 16;
    const size_t dst = ((static_cast<size_t>(k0 / 64) * N + n) * 64 + (k0 % 64)) * 2;
    *reinterpret_cast<uint4*>(out + dst) = *reinterpret_cast<const uint4*>(wt + src);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

// bf16 [rows][K] row-major, box kBK x box_rows, 128-byte swizzle, out-of-range rows zero-filled.
// A K-chunk-major matrix [K/64][N][64] is the row-major view [(K/64)*N][64] (K = 64).
bool make_map(CUtensorMap* m, const void* base, int rows, int K, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_gemm_supported(int M, int N, int K) { return M >= 1 && M <= kBM && N % kBN == 0 && K % kBK == 0 && K > 0; }

cudaError_t launch_tc_gemm(const TcGemmArgs& a, cudaStream_t s) {
    if (!tc_gemm_supported(a.M, a.N, a.K) || a.splits < 1 || (a.splits > 1 && (a.act || a.out_bf16)))
        return cudaErrorInvalidValue;
    CUtensorMap xm, wm;
    TcGemmArgs b = a;
    b.ntiles = a.N / kBN;
    b.cl = b.ntiles % 4 == 0 ? 4 : (b.ntiles % 2 == 0 ? 2 : 1);  // clusters never straddle K splits
    if (b.cl > kMaxCl) b.cl = kMaxCl;
    if (!make_map(&xm, a.X, a.M, a.K, kBM / b.cl) || !make_map(&wm, a.W, (a.K / kBK) * a.N, kBK, kBN))
        return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_pdl_cluster(gemm_tc_kernel, dim3(b.ntiles * a.splits), dim3(128), kSmem, s, b.cl, xm, wm, b);
}

cudaError_t launch_wtiles_to_chunks(const void* wt, int N, int Kp, int ks, void* out, cudaStream_t s) {
    if (N % 16 || Kp % 64 || Kp % ks || ks % 8) return cudaErrorInvalidValue;
    const size_t units = static_cast<size_t>(N) * (Kp / 8);
    wtiles_to_chunks_kernel<<<static_cast<unsigned>((units + 255) / 256), 256, 0, s>>>(
        static_cast<const uint8_t*>(wt), N, Kp, ks, static_cast<uint8_t*>(out));
    return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* x, void* y, size_t n, cudaStream_t s) {
    if (n % 4) return cudaErrorInvalidValue;
    const size_t n4 = n / 4;
    return launch_pdl(f32_to_bf16_kernel, dim3(static_cast<unsigned>((n4 + 255) / 256)), dim3(256), 0, s, x,
                      static_cast<__nv_bfloat16*>(y), n4);
}

}  // namespace wsvd_k
