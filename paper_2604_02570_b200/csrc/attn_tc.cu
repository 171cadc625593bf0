// attn_tc.cu -- fused decode attention with EXPLICIT per-head key
// reconstruction on the 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// This is the reference's own algorithm (src/decode.cpp:182-196): every key
// is rebuilt from its latent row, key_j = C_K[j] . B_K (decode.cpp:188), the
// score is q . key_j / sqrt(H), the online softmax accumulates P.C_V in
// latent-V space (decode.cpp:192), and B_V is applied once per head by the
// split-KV combine (decode.cpp:198-203).  The reconstruction is a dense
// contraction of L*r*H MACs per (sequence, head) -- 8.6 GMAC per step at the
// bench workload -- so it runs as tcgen05.mma:
//
//   D[tok][d] (TMEM, fp32) = C_K tile [128 tok x 32] (smem, bf16, the cache
//                            rows exactly as TMA brought them: K-major,
//                            128-byte swizzle)
//                          . B_K^T tile [128 d x 32] (smem, bf16, K-major
//                            core matrices, one TMA per unit)
//
// M = 128 tokens, N = 128 = H, K = 16 per instruction, two instructions per
// 128-token tile, two tiles per 256-token stage, two TMEM buffers of 256
// columns (all 512 columns of the SM).  Warp roles (persistent CTA per SM):
//   warp 8  producer: TMA of the cache stages, and per unit the B_K^T tile and
//           the query row;
//   warp 9  MMA issuer: one elected thread issues tcgen05.mma, commits to the
//           TMEM-full and stage-empty mbarriers; owns the TMEM allocation;
//   warps 0-7 consumers: each thread owns one token of the stage (TMEM lane):
//           tcgen05.ld of its reconstructed key (128 fp32 columns, 16 at a
//           time), dot with q (scaled into the log2 domain), per-thread online
//           softmax, latent-V accumulate from the shared-memory row; per unit a
//           warp merge (transpose-reduce) publishes one partial per warp for
//           the combine kernel of attn.cu.
// Results equal the absorbed-query kernel (attn.cu) up to fp32 reassociation.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int R = 32;                // latent rank (128-byte bf16 cache rows)
constexpr int H = 128;               // head dim (MMA N)
constexpr int kST = 256;             // tokens per stage
constexpr int kNW = 8;               // consumer warps (two warpgroups)
constexpr int kThr = 32 * kNW + 64;  // + producer + MMA warp
constexpr int ROWB = 4 * R;          // bf16 [C_K | C_V]
constexpr int PART = 2 * R;
constexpr int STAGE = kST * ROWB;    // 32 KB
constexpr int NS = 5;                // stage ring depth
constexpr int BT = H * R * 2;        // B_K^T tile bytes (8 KB)
constexpr int QB = H * 4;            // query row bytes
constexpr int UNIT = BT + QB;        // per-unit operand area
constexpr int RING_OFF = 0;
constexpr int UNIT_OFF = NS * STAGE;
constexpr int BAR_OFF = UNIT_OFF + 2 * UNIT;
constexpr int SMEM = BAR_OFF + 256 + 1024;  // + slack to align the base to 1 KB (SW128 atoms)
constexpr uint32_t kTmemCols = 512;  // two buffers x (2 tiles x 128 columns)

static_assert(SMEM <= 227 * 1024, "shared memory budget");

WSVD_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// --------------------------------------------------------- tcgen05 helpers
// Shared-memory matrix descriptor (sm_100): start >> 4 in [0,14), LBO >> 4 in
// [16,30), SBO >> 4 in [32,46), version 1 in [46,48), layout in [61,64).
WSVD_DEV uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(layout & 7u) << 61;
    return d;
}
constexpr uint32_t kLayoutNone = 0, kLayoutSw128 = 2;

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, M = 128, N = 128.
constexpr uint32_t kIdesc = (1u << 4)              // D format F32
                          | (1u << 7)              // A format BF16
                          | (1u << 10)             // B format BF16
                          | (static_cast<uint32_t>(H >> 3) << 17)
                          | (static_cast<uint32_t>(128 >> 4) << 24);

WSVD_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

WSVD_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

WSVD_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
WSVD_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 lanes x 16 consecutive fp32 columns, no wait (pair with tmem_wait)
WSVD_DEV void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
WSVD_DEV void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 16 consecutive fp32 columns: thread i gets lane (taddr.lane + i)
WSVD_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// packed fp32x2 FMA (FFMA2, sm_100): d.{x,y} = a.{x,y} * b.{x,y} + d.{x,y}
WSVD_DEV void ffma2(float2& d, float ax, float ay, float bx, float by) {
    uint64_t dd, aa, bb;
    asm("mov.b64 %0, {%1, %2};" : "=l"(dd) : "f"(d.x), "f"(d.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(ax), "f"(ay));
    asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(bx), "f"(by));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dd));
}

struct TUnit {
    int bh, chunk, t0, ntok;
};

WSVD_DEV void tc_chunking(const AttnArgs& a, int len, int& nch, int& chunk) {
    if (a.chunk > 0) {
        chunk = a.chunk;
    } else {
        const int n = max(1, min(a.max_chunks, (len + 31) / 32));
        chunk = (((len + n - 1) / n) + 31) & ~31;
    }
    nch = (len + chunk - 1) / chunk;
}

WSVD_DEV TUnit tc_unit(int u, int nch, int chunk, int len) {
    TUnit g;
    g.bh = u / nch;
    g.chunk = u - g.bh * nch;
    g.t0 = g.chunk * chunk;
    g.ntok = min(chunk, len - g.t0);
    return g;
}

__global__ void __launch_bounds__(kThr, 1) decode_attn_tc_kernel(const AttnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // the 128-byte swizzle of the MMA operand is a function of the absolute
    // shared address: stages must start on 1 KB boundaries
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem + RING_OFF;
    uint8_t* uarea = smem + UNIT_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;    // [2] TMEM buffer holds a stage's keys
    uint64_t* tempty = tfull + 2;    // [2] consumers drained the buffer
    uint64_t* ufull = tempty + 2;    // [2] unit operands (B_K^T tile, q) landed
    uint64_t* uempty = ufull + 2;    // [2] unit operands no longer needed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uempty + 2);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t cap = static_cast<size_t>(a.cap);

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1 + kNW);  // the MMA commit + every consumer warp
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kNW);
            mbar_init(&ufull[i], 1);
            mbar_init(&uempty[i], 1 + kNW);
        }
        fence_mbar_init();
    }
    if (warp == kNW + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    griddep_wait();
    griddep_launch_dependents();
    const int len = *a.d_len + a.len_add;
    int nch = 0, chunk = 0;
    if (len > 0) tc_chunking(a, len, nch, chunk);
    const int n_units = len > 0 ? a.B * a.nh * nch : 0;

    if (warp == kNW) {
        // ================================================================ producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int slot = 0, j = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
                const TUnit g = tc_unit(u, nch, chunk, len);
                const int ub = j & 1;
                mbar_wait(&uempty[ub], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&ufull[ub], UNIT);
                const int h = g.bh % a.nh;
                tma_bulk_g2s(uarea + ub * UNIT, a.bkt + static_cast<size_t>(h) * BT, BT, &ufull[ub]);
                tma_bulk_g2s(uarea + ub * UNIT + BT, a.q + static_cast<size_t>(g.bh) * H, QB, &ufull[ub]);
                const uint8_t* src = a.cache + (static_cast<size_t>(g.bh) * cap + g.t0) * ROWB;
                for (int s = 0; s * kST < g.ntok; ++s) {
                    const int rows = min(kST, g.ntok - s * kST);
                    const uint32_t rbytes = static_cast<uint32_t>(min(STAGE, ((rows * ROWB + 1023) / 1024) * 1024));
                    mbar_wait(&empty[slot], phase ^ 1u);
                    mbar_arrive_expect_tx(&full[slot], rbytes);
                    tma_bulk_g2s_stream(ring + slot * STAGE, src + static_cast<size_t>(s) * STAGE, rbytes, &full[slot], pol);
                    if (++slot == NS) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == kNW + 1) {
        // ============================================================== MMA issuer
        if (lane == 0) {
            int slot = 0, j = 0, tb = 0;
            uint32_t phase = 0, tph = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
                const TUnit g = tc_unit(u, nch, chunk, len);
                const int ub = j & 1;
                mbar_wait(&ufull[ub], static_cast<uint32_t>(j >> 1) & 1u);
                tc_fence_after();
                const uint32_t bbase = smem_u32(uarea + ub * UNIT);
                for (int s = 0; s * kST < g.ntok; ++s) {
                    const int rows = min(kST, g.ntok - s * kST);
                    mbar_wait(&full[slot], phase);
                    mbar_wait(&tempty[tb], tph ^ 1u);
                    tc_fence_after();
                    const uint32_t abase = smem_u32(ring + slot * STAGE);
                    for (int tile = 0; tile < 2 && tile * 128 < rows; ++tile) {
                        const uint32_t d = tmem + static_cast<uint32_t>(tb * 256 + tile * 128);
#pragma unroll
                        for (int k = 0; k < R / 16; ++k) {
                            // A: 128 token rows of 128 B (SW128, 8-row groups 1024 B apart),
                            //    k-th 32-byte slice of C_K;  B: core matrices of B_K^T,
                            //    K-adjacent 128 B apart, 8-row groups R/8*128 B apart
                            const uint64_t ad = smem_desc(abase + tile * 128 * ROWB + k * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(bbase + k * 2 * 128, 128, (R / 8) * 128, kLayoutNone);
                            mma_bf16(d, ad, bd, k > 0 ? 1u : 0u);
                        }
                    }
                    mma_commit(&tfull[tb]);    // keys of this stage are in TMEM buffer tb
                    mma_commit(&empty[slot]);  // the MMAs no longer read the stage
                    if (++slot == NS) {
                        slot = 0;
                        phase ^= 1u;
                    }
                    if (++tb == 2) {
                        tb = 0;
                        tph ^= 1u;
                    }
                }
                mma_commit(&uempty[ub]);  // B_K^T tile no longer read
            }
        }
        __syncwarp();
    } else {
        // ============================================================ consumers
        const int wg = warp >> 2, wq = warp & 3;  // tile of the stage, TMEM lane quarter
        const float qscale = 1.4426950408889634f * rsqrtf(static_cast<float>(H));
        int slot = 0, j = 0, tb = 0;
        uint32_t phase = 0, tph = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
            const TUnit g = tc_unit(u, nch, chunk, len);
            const int ub = j & 1;
            mbar_wait(&ufull[ub], static_cast<uint32_t>(j >> 1) & 1u);
            const float* qs = reinterpret_cast<const float*>(uarea + ub * UNIT + BT);
            float m = -INFINITY, l = 0.f, acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0.f;
            for (int s = 0; s * kST < g.ntok; ++s) {
                const int rows = min(kST, g.ntok - s * kST);
                const int tok = wg * 128 + wq * 32 + lane;  // this thread's token of the stage
                mbar_wait(&tfull[tb], tph);
                tc_fence_after();
                float sc = 0.f;
                if (wg * 128 < rows) {
                    const uint32_t taddr = tmem + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(tb * 256 + wg * 128);
                    // the 128-term dot as packed fp32x2 FMAs: half the instructions
                    // and two independent chains
                    float2 s2 = make_float2(0.f, 0.f);
                    // two 16-column loads in flight per wait (the TMEM load latency,
                    // not the math, bounds this loop)
#pragma unroll
                    for (int c = 0; c < H / 32; ++c) {
                        uint32_t ka[16], kb[16];
                        tmem_ld16_nowait(taddr + c * 32, ka);
                        tmem_ld16_nowait(taddr + c * 32 + 16, kb);
                        tmem_wait();
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 q4 = *reinterpret_cast<const float4*>(qs + c * 32 + i);
                            ffma2(s2, __uint_as_float(ka[i]), __uint_as_float(ka[i + 1]), q4.x, q4.y);
                            ffma2(s2, __uint_as_float(ka[i + 2]), __uint_as_float(ka[i + 3]), q4.z, q4.w);
                        }
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 q4 = *reinterpret_cast<const float4*>(qs + c * 32 + 16 + i);
                            ffma2(s2, __uint_as_float(kb[i]), __uint_as_float(kb[i + 1]), q4.x, q4.y);
                            ffma2(s2, __uint_as_float(kb[i + 2]), __uint_as_float(kb[i + 3]), q4.z, q4.w);
                        }
                    }
                    sc = s2.x + s2.y;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[tb]);
                if (++tb == 2) {
                    tb = 0;
                    tph ^= 1u;
                }
                mbar_wait(&full[slot], phase);  // (already complete: the MMA consumed it)
                if (tok < rows) {
                    sc *= qscale;
                    if (sc > m) {
                        const float f = ex2(m - sc);
                        l *= f;
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] *= f;
                        m = sc;
                    }
                    const float p = ex2(sc - m);
                    l += p;
                    const uint32_t vrow = smem_u32(ring + slot * STAGE) ;
#pragma unroll
                    for (int c = 0; c < PART / 16; ++c) {
                        const uint4 v = lds128(vrow + cache_swz(static_cast<uint32_t>(tok * ROWB + PART + c * 16)));
                        const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float2 a2 = make_float2(acc[c * 8 + 2 * k], acc[c * 8 + 2 * k + 1]);
                            ffma2(a2, p, p, bf16lo(vw[k]), bf16hi(vw[k]));
                            acc[c * 8 + 2 * k] = a2.x;
                            acc[c * 8 + 2 * k + 1] = a2.y;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == NS) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&uempty[ub]);  // q no longer read
            // ---- warp merge: common max, then a transpose-reduce of acc[R]
            const float M = warp_max(m);
            const float f = (m == -INFINITY) ? 0.f : ex2(m - M);
            const float L = warp_sum(l * f);
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] *= f;
#pragma unroll
            for (int off = 16, n = R; off >= 1; off >>= 1, n >>= 1) {
                const bool up = (lane & off) != 0;
#pragma unroll
                for (int i = 0; i < n / 2; ++i) {
                    const float send = up ? acc[i] : acc[i + n / 2];
                    const float keep = up ? acc[i + n / 2] : acc[i];
                    acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * 16 + warp) * (R + 2);
            wsp[lane] = acc[0];  // lane r holds sum_tokens p . C_V[:, r]
            if (lane == 0) {
                wsp[R] = M;
                wsp[R + 1] = L;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kNW + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

}  // namespace

bool attn_tc_supported(int cdtype, int R_, int H_, int bdtype) {
    return cdtype == BF16 && R_ == R && H_ == H && bdtype == BF16;
}

int attn_tc_btile_bytes() { return BT; }

// B_K^T of one head as the MMA's B operand: element (d, r) at
// (d/8)*(R/8)*128 + (r/8)*128 + (d%8)*16 + (r%8)*2  (K-major core matrices)
size_t attn_tc_btile_offset(int d, int r) {
    return static_cast<size_t>(d / 8) * (R / 8) * 128 + static_cast<size_t>(r / 8) * 128 + (d % 8) * 16 + (r % 8) * 2;
}

cudaError_t launch_decode_attn_tc(const AttnArgs& a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_pdl(decode_attn_tc_kernel, dim3(a.grid), dim3(kThr), SMEM, s, a);
}

}  // namespace wsvd_k
