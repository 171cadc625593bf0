// step2.cu -- the layer chain as ONE persistent kernel whose batch runs as two
// groups half a layer apart (bf16 weights and cache, rank 32, 2 <= B <= 16).
//
// Every layer of pipe::decode_factored's loop (pipeline.cpp:318-336; body
// :320-329) is append_token (decode.cpp:127-153) -> fused_decode_step
// (decode.cpp:155-206) -> heads_row . W_o.  In the one-group kernel (step.cu)
// a layer is: projection P1 -> grid barrier -> attention (HBM-bound, ~36 us
// at the headline shape) -> merges -> grid barrier -> O-projection P3 -> grid
// barrier -> next layer; the latency-bound phases (~20 us a layer) leave HBM
// idle.
//
// Here the sequences split into two groups (rows [0, B0) and [B0, B)).  The
// eight consumer warps and the cache producer stream the groups' attention in
// strict alternation -- group 0 layer l, group 1 layer l, group 0 layer l + 1,
// ... -- through one ring, so every SM streams continuously at full width.
// Everything else a group does (projection P1, the query preparation, the
// merges, the folded O-projection P3, the grid barriers) runs on the group's
// own helper warp, while the consumers stream the OTHER group's half of the
// cache: a group's tail and its next layer's front hide under the other
// group's attention.  The helpers stage their token slices with TMA and run
// the projection tiles on the tensor cores themselves (mma.sync, one warp).
// Each group's arithmetic keeps the one-group kernel's fixed orders (K splits,
// warp states, range-ordered merges, exact two-addend red.add onto zeros), so
// results are run-to-run deterministic.
//
// Warps: 0-7 consumers, 8 the weight producer, 9 the cache producer, 10 / 11
// the groups' helpers.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kNW = 8;                 // consumer warps
constexpr int kWP = kNW;               // the weight producer warp
constexpr int kCP = kNW + 1;           // the cache producer warp
constexpr int kH0 = kNW + 2;           // group g's helper: warp kH0 + g
constexpr int kThr = 32 * (kNW + 4);   // 384 threads
constexpr int kST = 256;               // tokens per attention stage
constexpr int kNB = 4;                 // attention stages
constexpr int kKS = 512;               // K per weight work item
constexpr int kItem = 16 * kKS * 2;    // one weight work item: 16 rows x 512 bf16 = 16 KB
constexpr int kNA = 3;                 // weight ring slots
constexpr int kXS = kKS * 2;           // bytes per bf16 X row of P3 (16-byte units XOR 4 on odd rows)
constexpr int kXF = kKS * 4 + 16;      // bytes per fp32 token row of P1 (padded: conflict-free fragments)
constexpr int kTok = 8;                // token rows per group
constexpr int kMaxU = 4;               // (sequence, head) segments per CTA and group (host-checked)
constexpr int kMaxSplits = 16;         // projection K splits (host-checked)
constexpr int kWS = 36;                // floats per segment state in ws
constexpr int kMaxG = 160;             // CTAs (the range tables)
constexpr int kCut = 32;               // range boundaries fall on multiples of 32 rows
constexpr int kTr = 32;                // trace words per CTA

template <int R>
struct PC {
    static constexpr int ROWB = 4 * R;  // bf16 [C_K | C_V]
    static constexpr int PART = 2 * R;
    static constexpr int STAGE = kST * ROWB;
    static constexpr int RING = kNB * STAGE;
    static constexpr int XST = kTok * kXF;       // staging: P1 fp32 token rows / P3 bf16 X rows
    static constexpr int XB2 = 2 * kTok * kXS;   // P3 X slice: hi rows, then lo rows
    static constexpr int RED = kMaxU * (R * 4 + kNW * (R + 2) * 4 + 4 * R) + (R + 4) * 4;
    static constexpr int PARTB = 4 * 16 * kTok * 4;  // P3 partial tiles [<=4][16][kTok] fp32
    static constexpr int TAB = (kMaxG + 1) * 8 + kMaxU * 32 + 16;  // range table + segments + (pos, nseg)
    // per group: staging | merge area | two range tables (layer parity)
    static constexpr int G_X = 0;
    static constexpr int G_RED = XST;
    static constexpr int G_TAB = G_RED + RED;
    static constexpr int GB = ((G_TAB + 2 * TAB + 1023) / 1024) * 1024;
    static constexpr int B_OFF = kNA * kItem;
    static constexpr int G_OFF = B_OFF + RING;
    static constexpr int MISC = G_OFF + 2 * GB;  // lengths at launch [32], counters
    static constexpr int BAR_OFF = MISC + kStepMaxLayers * 4 + 32;
    static constexpr int SMEM = BAR_OFF + 512;
    static_assert(PARTB <= RED, "P3 partials live in the merge area");
    static_assert(XB2 <= XST, "P3 X slices live in the staging area");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

WSVD_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
WSVD_DEV void split_bf16(float x, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
    hi = *reinterpret_cast<const uint16_t*>(&h);
    lo = *reinterpret_cast<const uint16_t*>(&l);
}
WSVD_DEV uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// phase marks of group a.trace_group at layer a.trace_layer (l, g in scope)
#define PIPE_MARK(k)                                                                                 \
    do {                                                                                             \
        if (a.trace && l == a.trace_layer && g == a.trace_group && lane == 0)                        \
            a.trace[cta * kTr + (k)] = gtimer();                                                     \
    } while (0)

WSVD_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
WSVD_DEV void red_release(unsigned* p) { asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory"); }
WSVD_DEV unsigned atom_add_acq_rel(unsigned* p) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}
WSVD_DEV void wait_count(const unsigned* p, unsigned target) {
    while (static_cast<int>(ld_acquire(p) - target) < 0) {
    }
}
WSVD_DEV void mbar_arrive_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

// Debug build (-DWSVD_PIPE_DEBUG): every wait is bounded -- a thread stuck for
// 2 s records (cta, thread, tag, parity) into mapped host memory, and after
// 4 s the kernel traps, so a protocol error reports where it hangs.
#ifdef WSVD_PIPE_DEBUG
__device__ int* g_pipe_dbg = nullptr;
WSVD_DEV void pipe_stuck(int tag, uint32_t par, uint64_t t0, bool& noted) {
    const uint64_t dt = gtimer() - t0;
    if (!noted && dt > 2000000000ull && g_pipe_dbg) {
        noted = true;
        const int k = atomicAdd(g_pipe_dbg, 1);
        if (k < 1000) {
            g_pipe_dbg[1 + 4 * k] = blockIdx.x;
            g_pipe_dbg[2 + 4 * k] = threadIdx.x;
            g_pipe_dbg[3 + 4 * k] = tag;
            g_pipe_dbg[4 + 4 * k] = static_cast<int>(par);
        }
        __threadfence_system();
    }
    if (dt > 4000000000ull) asm volatile("trap;");
}
WSVD_DEV void pwait(uint64_t* bar, uint32_t par, int tag) {
    const uint64_t t0 = gtimer();
    bool noted = false;
    for (uint32_t n = 0;; ++n) {
        if (mbar_test(bar, par)) return;
        if ((n & 1023u) == 1023u) pipe_stuck(tag, par, t0, noted);
    }
}
WSVD_DEV void gwait(const unsigned* p, unsigned target, int tag) {
    const uint64_t t0 = gtimer();
    bool noted = false;
    for (uint32_t n = 0;; ++n) {
        if (static_cast<int>(ld_acquire(p) - target) >= 0) return;
        if ((n & 1023u) == 1023u) pipe_stuck(tag, target, t0, noted);
    }
}
#else
WSVD_DEV void pwait(uint64_t* bar, uint32_t par, int) { mbar_wait(bar, par); }
WSVD_DEV void gwait(const unsigned* p, unsigned target, int) { wait_count(p, target); }
#endif

// grid-wide barrier among group g's helper warps (one per CTA)
WSVD_DEV void group_sync(int g, unsigned* bar, unsigned target) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        red_release(bar);
        gwait(bar, target, 100 + g);
    }
    __syncwarp();
}

WSVD_DEV long long cut_row(int c, int G, long long T, int pos) {
    if (c >= G) return T;
    if (pos == 0) return 0;
    const long long f = (static_cast<long long>(c) * T) / G;
    const long long bh = f / pos, t = f - bh * pos;
    return bh * pos + (t & ~static_cast<long long>(kCut - 1));
}
struct SegInfo {
    int bh, t0, t1, owners, c0, c1, pad0, pad1;  // bh: group-relative region
};
WSVD_DEV int seg_count(const long long* cut, int c, int G, int pos, int nbh) {
    if (pos == 0) return c < nbh ? (nbh - 1 - c) / G + 1 : 0;
    const long long lo = cut[c], hi = cut[c + 1];
    if (lo >= hi) return 0;
    return static_cast<int>((hi - 1) / pos - lo / pos + 1);
}
WSVD_DEV void seg_at(const long long* cut, int c, int G, int pos, int j, int& bh, int& t0, int& t1) {
    if (pos == 0) {
        bh = c + j * G;
        t0 = t1 = 0;
        return;
    }
    const long long lo = cut[c], hi = cut[c + 1];
    bh = static_cast<int>(lo / pos + j);
    const long long rs = static_cast<long long>(bh) * pos;
    t0 = static_cast<int>(lo > rs ? lo - rs : 0);
    t1 = static_cast<int>(hi < rs + pos ? hi - rs : pos);
}
WSVD_DEV void seg_owners(const long long* cut, int G, int pos, int bh, int& c0, int& c1) {
    if (pos == 0) {
        c0 = bh % G;
        c1 = c0 + 1;
        return;
    }
    const long long r0 = static_cast<long long>(bh) * pos, r1 = r0 + pos;
    int lo = 0, hi = G;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cut[mid] <= r0) lo = mid;
        else hi = mid;
    }
    c0 = lo;
    int c = lo;
    while (c < G && cut[c] < r1) ++c;
    c1 = c;
}
WSVD_DEV uint32_t xrow_off(int m, int u) { return static_cast<uint32_t>(m * kXS + ((u ^ ((m & 1) << 2)) * 16)); }


// one weight item (16 W-rows x kKS) against 8 fp32 token rows (P1): the bf16
// B fragments are packed from the fp32 rows on the fly
WSVD_DEV void item_mma_xf(uint32_t slot_addr, uint32_t xs_addr, int lane, float (&facc)[4]) {
    const int g = lane >> 2, t = lane & 3;
    const uint32_t swz = static_cast<uint32_t>((g & 1) << 2);
    const uint32_t row_lo = slot_addr + static_cast<uint32_t>(g * kKS * 2);
    const uint32_t row_hi = row_lo + static_cast<uint32_t>(8 * kKS * 2);
    const uint32_t xrow = xs_addr + static_cast<uint32_t>(g * kXF + t * 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) facc[i] = 0.f;
#pragma unroll 4
    for (int b = 0; b < kKS / 32; ++b) {
        const uint32_t uoff = ((static_cast<uint32_t>(4 * b + t)) ^ swz) * 16;
        const uint4 wl = lds128(row_lo + uoff);
        const uint4 wh = lds128(row_hi + uoff);
        const uint4 f0 = lds128(xrow + b * 128), f1 = lds128(xrow + b * 128 + 16);  // k = 32b + 8t .. + 7
        mma_bf16_16816(facc, wl.x, wh.x, wl.y, wh.y,
                       pack_bf16x2(__uint_as_float(f0.x), __uint_as_float(f0.y)),
                       pack_bf16x2(__uint_as_float(f0.z), __uint_as_float(f0.w)));
        mma_bf16_16816(facc, wl.z, wh.z, wl.w, wh.w,
                       pack_bf16x2(__uint_as_float(f1.x), __uint_as_float(f1.y)),
                       pack_bf16x2(__uint_as_float(f1.z), __uint_as_float(f1.w)));
    }
}

// one weight item against the 16 bf16 X rows of P3 (8 hi, 8 lo):
// facc[hh][i] = (row g | g+8, token 2t | 2t+1 of half hh)
WSVD_DEV void item_mma_x2(uint32_t slot_addr, uint32_t xs_addr, int lane, float (&facc)[2][4]) {
    const int g = lane >> 2, t = lane & 3;
    const uint32_t swz = static_cast<uint32_t>((g & 1) << 2);
    const uint32_t row_lo = slot_addr + static_cast<uint32_t>(g * kKS * 2);
    const uint32_t row_hi = row_lo + static_cast<uint32_t>(8 * kKS * 2);
    const uint32_t xbase = xs_addr + static_cast<uint32_t>(g * kXS);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int i = 0; i < 4; ++i) facc[hh][i] = 0.f;
#pragma unroll 4
    for (int b = 0; b < kKS / 32; ++b) {
        const uint32_t uoff = ((static_cast<uint32_t>(4 * b + t)) ^ swz) * 16;
        const uint4 wl = lds128(row_lo + uoff);
        const uint4 wh = lds128(row_hi + uoff);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const uint4 xv = lds128(xbase + static_cast<uint32_t>(hh * 8 * kXS) + uoff);
            mma_bf16_16816(facc[hh], wl.x, wh.x, wl.y, wh.y, xv.x, xv.y);
            mma_bf16_16816(facc[hh], wl.z, wh.z, wl.w, wh.w, xv.z, xv.w);
        }
    }
}

// Weight-ring order (one producer thread; the two helpers find their items by
// it): P1_0(0) P1_1(0) P3_0(0), then per layer l >= 1: P1_0(l) P3_1(l-1)
// P1_1(l) P3_0(l), and last P3_1(n-1) -- the order the groups reach them.
WSVD_DEV unsigned wbase(int kind, int g, int l, int n, int np1, int np3) {
    unsigned off = 0;
    auto blk = [&](int k2, int g2, int l2) -> bool {
        if (k2 == kind && g2 == g && l2 == l) return true;
        off += static_cast<unsigned>(k2 == 0 ? np1 : np3);
        return false;
    };
    if (blk(0, 0, 0) || blk(0, 1, 0) || blk(1, 0, 0)) return off;
    for (int li = 1; li < n; ++li)
        if (blk(0, 0, li) || blk(1, 1, li - 1) || blk(0, 1, li) || blk(1, 0, li)) return off;
    blk(1, 1, n - 1);
    return off;
}

WSVD_DEV void spin_ge(const volatile int* p, int v) {
    while (*p < v) {
    }
    __threadfence_block();
}

template <int R>
__global__ void __launch_bounds__(kThr, 1) chain_pipe_kernel(const __grid_constant__ PipeArgs a) {
    static_assert(R == 32, "rank 32: one latent dim per lane");
    using C = PC<R>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nL = a.nlayers;
    int l = 0, g = -1;  // (trace marks)

    uint8_t* ringA = smem;
    uint8_t* ringB = smem + C::B_OFF;
    auto gbase = [&](int gg) { return smem + C::G_OFF + gg * C::GB; };
    auto tab = [&](int gg, int li) { return gbase(gg) + C::G_TAB + (li & 1) * C::TAB; };
    int* posl = reinterpret_cast<int*>(smem + C::MISC);
    volatile int* cnt = reinterpret_cast<volatile int*>(posl + kStepMaxLayers);
    volatile int* bcnt = cnt;        // [2] weight-ring blocks each helper has consumed
    volatile int* tbuilt = cnt + 2;  // [2] range tables each helper has built
    int* tread = const_cast<int*>(cnt + 4);  // [2] (layer, group) table readings finished (8 consumer warps + producer)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + kNA;
    uint64_t* fullB = emptyA + kNA;
    uint64_t* emptyB = fullB + kNB;
    constexpr int NGB = 2 * kMaxU + 2;  // per group: uready[kMaxU] sfull[kMaxU] pbar xbar
    static_assert((2 * kNA + 2 * kNB + 2 * NGB) * 8 <= 512, "mbarriers overflow their region");
    auto uready = [&](int gg) { return fullB + 2 * kNB + gg * NGB; };
    auto sfull = [&](int gg) { return uready(gg) + kMaxU; };
    auto pbar = [&](int gg) { return uready(gg) + 2 * kMaxU; };
    auto xbar = [&](int gg) { return uready(gg) + 2 * kMaxU + 1; };

    if (a.trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[cta * kTr + 10] = smid;
    }
    // ---- projection geometry (shared by the groups and the layers)
    const int splits = a.Kp / kKS;
    const int cps = G / splits;
    const int ps = cta % splits, pj = cta / splits;
    const int ptiles = a.Nrows / 16;
    const int plo = pj < cps ? static_cast<int>(static_cast<long>(pj) * ptiles / cps) : 0;
    const int phi = pj < cps ? static_cast<int>(static_cast<long>(pj + 1) * ptiles / cps) : 0;
    const int np1 = phi - plo;
    const int osplits = a.oKp / kKS;
    // ---- O-projection items (tile, K split) of this CTA (device y): two K
    // splits -- CTA c takes split c % 2 of a run of tiles, the two partial sums
    // meet in y through fp32 red.add onto zeros (exactly two addends: order
    // independent); one K split -- whole tiles, plain stores
    const bool ysplit = osplits == 2;
    int t3lo, nt3, t3step, p3s0, p3ns;
    if (ysplit) {
        const int cps3 = G / 2, pj3 = cta / 2;
        t3lo = pj3 < cps3 ? static_cast<int>(static_cast<long>(pj3) * a.otiles / cps3) : 0;
        nt3 = pj3 < cps3 ? static_cast<int>(static_cast<long>(pj3 + 1) * a.otiles / cps3) - t3lo : 0;
        t3step = 1;
        p3s0 = cta % 2;
        p3ns = 1;
    } else {
        t3lo = cta;
        nt3 = cta < a.otiles ? (a.otiles - 1 - cta) / G + 1 : 0;
        t3step = G;
        p3s0 = 0;
        p3ns = osplits;
    }
    const int np3 = nt3 * p3ns;  // <= 4 (host-checked)
    const int b0g[2] = {0, a.B - a.B / 2};
    const int Bg[2] = {a.B - a.B / 2, a.B / 2};
    const size_t pstride = static_cast<size_t>(kTok) * a.Nrows;

    if (warp == 0) {
        if (lane < 8) cnt[lane] = 0;
        if (lane < kNA) {
            mbar_init(&fullA[lane], 1);
            mbar_init(&emptyA[lane], 1);
        }
        if (lane < kNB) {
            mbar_init(&fullB[lane], 1);
            mbar_init(&emptyB[lane], kNW);
        }
        for (int gg = 0; gg < 2; ++gg) {
            if (lane < kMaxU) {
                mbar_init(&uready(gg)[lane], 1);
                mbar_init(&sfull(gg)[lane], kNW);
            }
            if (lane == 0) {
                mbar_init(pbar(gg), 1);
                mbar_init(xbar(gg), 1);
            }
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (a.cluster > 1) cluster_sync_all();

    auto wsrc = [&](int kind, int li, int i) -> const uint8_t* {
        const StepLayer& Ly = a.layer[li];
        if (kind == 0) return Ly.A + (static_cast<size_t>(plo + i) * splits + ps) * kItem;
        return Ly.Wo + (static_cast<size_t>(t3lo + (i / p3ns) * t3step) * osplits + p3s0 + i % p3ns) * kItem;
    };
    // the weights are constant across steps: the first ring fill goes out
    // before the predecessor has drained (programmatic dependent launch)
    if (warp == kWP && lane == 0)
        for (int i = 0; i < kNA && i < np1; ++i) {
            mbar_arrive_expect_tx(&fullA[i], kItem);
            tma_bulk_g2s(ringA + i * kItem, wsrc(0, 0, i), kItem, &fullA[i]);
        }
    griddep_wait();
    griddep_launch_dependents();
    if (warp == kH0) {
        for (int li = lane; li < nL; li += 32) posl[li] = *static_cast<volatile const int*>(a.layer[li].d_len);
        __syncwarp();
    }
    __syncthreads();  // posl is complete
    const bool rev = (cta & 1) != 0;

    // ================================================================ producers
    if (warp == kWP) {
        if (lane == 0) {
            unsigned ia = 0;  // items issued
            auto block = [&](int kind, int li) {
                const int n = kind == 0 ? np1 : np3;
                for (int i = 0; i < n; ++i, ++ia) {
                    if (kind == 0 && li == 0 && ia < static_cast<unsigned>(kNA) && static_cast<int>(ia) == i)
                        continue;  // issued before the grid-dependency wait
                    const int slot = static_cast<int>(ia % kNA);
                    pwait(&emptyA[slot], ((ia / kNA) & 1u) ^ 1u, 1);
                    mbar_arrive_expect_tx(&fullA[slot], kItem);
                    tma_bulk_g2s(ringA + slot * kItem, wsrc(kind, li, i), kItem, &fullA[slot]);
                }
            };
            block(0, 0);  // group 0's P1 of layer 0
            block(0, 0);  // group 1's (the same items)
            block(1, 0);
            for (int li = 1; li < nL; ++li) {
                block(0, li);
                block(1, li - 1);
                block(0, li);
                block(1, li);
            }
            block(1, nL - 1);
        }
        return;
    }
    if (warp == kCP) {
        if (lane == 0) {
            // the groups' attention streams in strict alternation through one ring
            const uint64_t pol = policy_evict_first();
            unsigned fill = 0;  // stage fills so far: slot fill % kNB, phase (fill / kNB) & 1
            for (int li = 0; li < nL; ++li) {
                const StepLayer& Ly = a.layer[li];
                const size_t cap = static_cast<size_t>(Ly.cap);
                for (int gg = 0; gg < 2; ++gg) {
                    spin_ge(&tbuilt[gg], li + 1);
                    uint8_t* tb = tab(gg, li);
                    const long long* cut = reinterpret_cast<const long long*>(tb);
                    const SegInfo* sinf = reinterpret_cast<const SegInfo*>(cut + kMaxG + 1);
                    const int nseg = reinterpret_cast<const int*>(sinf + kMaxU)[1];
                    for (int p = 0; p < nseg; ++p) {
                        const SegInfo& sg = sinf[rev ? nseg - 1 - p : p];
                        const size_t region = static_cast<size_t>(b0g[gg]) * a.nh + sg.bh;
                        for (int t = sg.t0; t < sg.t1; t += kST) {
                            const int rows = min(kST, sg.t1 - t);
                            // the launch's first fill of each slot is a whole stage: stale
                            // shared memory never meets the tensor cores (rows past the
                            // end are finite cache rows, read times p = 0)
                            const uint32_t rbytes = fill < static_cast<unsigned>(kNB)
                                                        ? static_cast<uint32_t>(C::STAGE)
                                                        : static_cast<uint32_t>(min(C::STAGE, ((rows * C::ROWB + 1023) / 1024) * 1024));
                            const int slot = static_cast<int>(fill % kNB);
                            pwait(&emptyB[slot], ((fill / kNB) & 1u) ^ 1u, 4);
                            mbar_arrive_expect_tx(&fullB[slot], rbytes);
                            const uint8_t* src = Ly.cache + (region * cap + t) * C::ROWB;
                            tma_bulk_g2s_stream(ringB + slot * C::STAGE, src, rbytes, &fullB[slot], pol);
                            ++fill;
                        }
                    }
                    atomicAdd(&tread[gg], 1);
                }
            }
        }
        return;
    }

    const int g8 = lane >> 2, t4 = lane & 3;
    if (warp < kNW) {
        // ===================================================== consumer warps
        // every stage of both groups, in ring order
        unsigned fill = 0;
        constexpr int KR = R / 16;
        for (l = 0; l < nL; ++l) {
            const uint32_t lp = static_cast<uint32_t>(l) & 1u;
            for (int gg = 0; gg < 2; ++gg) {
                g = gg;
                spin_ge(&tbuilt[gg], l + 1);
                uint8_t* tb = tab(gg, l);
                const long long* cut = reinterpret_cast<const long long*>(tb);
                const SegInfo* sinf = reinterpret_cast<const SegInfo*>(cut + kMaxG + 1);
                const int nseg = reinterpret_cast<const int*>(sinf + kMaxU)[1];
                uint8_t* gb = gbase(gg);
                const float* qts = reinterpret_cast<const float*>(gb + C::G_RED);
                float* wst = reinterpret_cast<float*>(gb + C::G_RED) + kMaxU * R;
                for (int p = 0; p < nseg; ++p) {
                    const int j = rev ? nseg - 1 - p : p;
                    const SegInfo& s = sinf[j];
                    const int ntok = s.t1 - s.t0;
                    const int ns = (ntok + kST - 1) / kST;
                    pwait(&uready(gg)[j], lp, 8);
                    if (p == 0) PIPE_MARK(13);
                    uint32_t qf[KR][2];
#pragma unroll
                    for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int k0 = kk * 16 + 2 * t4 + 8 * jj;
                            uint32_t h0, l0, h1, l1;
                            split_bf16(qts[j * R + k0], h0, l0);
                            split_bf16(qts[j * R + k0 + 1], h1, l1);
                            qf[kk][jj] = (g8 == 0) ? (h0 | (h1 << 16)) : (g8 == 1 ? (l0 | (l1 << 16)) : 0u);
                        }
                    float m_w = -INFINITY, lsm = 0.f;
                    float acc[KR][4];
#pragma unroll
                    for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[kk][i] = 0.f;
                    for (int st = 0; st < ns; ++st, ++fill) {
                        const int slot = static_cast<int>(fill % kNB);
                        pwait(&fullB[slot], (fill / kNB) & 1u, 9);
                        const uint32_t sbase = smem_u32(ringB + slot * C::STAGE);
                        const int rows = min(kST, ntok - st * kST);
                        if (warp * 32 < rows) {
                            float sc[2][2];
#pragma unroll
                            for (int grp = 0; grp < 2; ++grp) {
                                const int tb0 = warp * 32 + grp * 16;
                                float d[4] = {0.f, 0.f, 0.f, 0.f};
                                const int ltok = tb0 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
                                for (int kk = 0; kk < KR; ++kk) {
                                    uint32_t a0, a1, a2, a3;
                                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2 + (lane >> 4)) * 16);
                                    ldsm_x4(sbase + cache_swz(off), a0, a1, a2, a3);
                                    mma_bf16_16816(d, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
                                }
                                sc[grp][0] = (t4 == 0 && tb0 + g8 < rows) ? d[0] + d[1] : -INFINITY;
                                sc[grp][1] = (t4 == 0 && tb0 + g8 + 8 < rows) ? d[2] + d[3] : -INFINITY;
                            }
                            const float wm = warp_max(fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1])));
                            if (wm > m_w) {
                                const float f = ex2(m_w - wm);
                                lsm *= f;
#pragma unroll
                                for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                                    for (int i = 0; i < 4; ++i) acc[kk][i] *= f;
                                m_w = wm;
                            }
#pragma unroll
                            for (int grp = 0; grp < 2; ++grp) {
                                const int tb0 = warp * 32 + grp * 16;
                                const float p0 = (sc[grp][0] == -INFINITY) ? 0.f : ex2(sc[grp][0] - m_w);
                                const float p1 = (sc[grp][1] == -INFINITY) ? 0.f : ex2(sc[grp][1] - m_w);
                                lsm += p0 + p1;
                                uint32_t h0, l0, h1, l1;
                                split_bf16(p0, h0, l0);
                                split_bf16(p1, h1, l1);
                                const uint32_t hi2 = h0 | (h1 << 16), lo2 = l0 | (l1 << 16);
                                const int s0 = 8 * t4, s1 = 8 * t4 + 4;
                                const uint32_t xh = __shfl_sync(0xffffffffu, hi2, s0), yh = __shfl_sync(0xffffffffu, hi2, s1);
                                const uint32_t xl = __shfl_sync(0xffffffffu, lo2, s0), yl = __shfl_sync(0xffffffffu, lo2, s1);
                                const uint32_t xx = (g8 == 0) ? xh : xl, yy = (g8 == 0) ? yh : yl;
                                const uint32_t b0 = (g8 < 2) ? __byte_perm(xx, yy, 0x5410) : 0u;
                                const uint32_t b1 = (g8 < 2) ? __byte_perm(xx, yy, 0x7632) : 0u;
                                const int stok = tb0 + (lane & 7) + ((lane >> 4) & 1) * 8;
#pragma unroll
                                for (int mm = 0; mm < KR; ++mm) {
                                    uint32_t a0, a1, a2, a3;
                                    const uint32_t off = static_cast<uint32_t>(stok * C::ROWB + C::PART + (mm * 2 + ((lane >> 3) & 1)) * 16);
                                    ldsm_x4_trans(sbase + cache_swz(off), a0, a1, a2, a3);
                                    mma_bf16_16816(acc[mm], a0, a1, a2, a3, b0, b1);
                                }
                            }
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&emptyB[slot]);
                    }
                    float* wr = wst + (j * kNW + warp) * (R + 2);
                    const float lsum = warp_sum(lsm);
                    if (t4 == 0) {
#pragma unroll
                        for (int mm = 0; mm < KR; ++mm) {
                            wr[mm * 16 + g8] = acc[mm][0] + acc[mm][1];
                            wr[mm * 16 + g8 + 8] = acc[mm][2] + acc[mm][3];
                        }
                    }
                    if (lane == 0) {
                        wr[R] = m_w;
                        wr[R + 1] = lsum;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sfull(gg)[j]);
                }
                if (nseg > 0) PIPE_MARK(5);
                __syncwarp();
                if (lane == 0) atomicAdd(&tread[gg], 1);
            }
        }
        return;
    }

    // ================================================== helper warp of group g
    g = warp - kH0;
    uint8_t* gb = gbase(g);
    uint8_t* xst = gb + C::G_X;
    float* qts = reinterpret_cast<float*>(gb + C::G_RED);  // [kMaxU][R]
    float* wst = qts + kMaxU * R;                           // [kMaxU][kNW][R+2]
    __nv_bfloat16* nrow = reinterpret_cast<__nv_bfloat16*>(wst + kMaxU * kNW * (R + 2));  // [kMaxU][2R]
    float* pst = reinterpret_cast<float*>(nrow + kMaxU * 2 * R);  // [R+2] the pair partner's state
    float* part = reinterpret_cast<float*>(gb + C::G_RED);        // P3 partials (merge area: free during P3)
    const int nbh = Bg[g] * a.nh;   // this group's (sequence, head) regions
    const int rb0 = b0g[g] * a.nh;  // its first region
    unsigned gen = *a.bgen[g];      // this group's barrier generations so far
    unsigned pcnt = 0, xcnt = 0;
    float* Pg = a.P[g];
    // Ring-A gate.  The helpers consume the shared weight ring in the block
    // order of wbase; a helper may wait on an item's fill parity only once the
    // slot's previous fill has landed, else the parity of an older phase
    // satisfies the wait.  Its own blocks run in sequence; across the helpers,
    // a block waits until the other has consumed the block that precedes it:
    // P1_1(0) after P1_0(0); P3_0(l) after P1_1(l); P3_1(l) after P1_0(l + 1),
    // the last one after P3_0(n - 1).  bcnt[g]: group g's consumed blocks
    // (P1_g(l) is its block 2l, P3_g(l) block 2l + 1).
    auto gate = [&](int kind, int li) {
        int need = 0;
        if (kind == 0) need = (g == 1 && li == 0) ? 1 : 0;
        else if (g == 0) need = 2 * li + 1;
        else need = li + 1 < nL ? 2 * li + 3 : 2 * nL;
        if (need > 0) spin_ge(&bcnt[1 - g], need);
    };
    auto block_done = [&]() {
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            bcnt[g] = bcnt[g] + 1;
        }
    };
    auto build_table = [&](int li) {
        // table li goes to buffer li & 1: wait until table li - 2's readers are done
        if (li >= 2) spin_ge(&tread[g], (kNW + 1) * (li - 1));
        uint8_t* tb = tab(g, li);
        long long* cut = reinterpret_cast<long long*>(tb);
        SegInfo* sinf = reinterpret_cast<SegInfo*>(cut + kMaxG + 1);
        int* meta = reinterpret_cast<int*>(sinf + kMaxU);
        const int pos = posl[li];
        const long long T = static_cast<long long>(nbh) * pos;
        for (int c = lane; c <= G; c += 32) cut[c] = cut_row(c, G, T, pos);
        __syncwarp();
        const int nseg = seg_count(cut, cta, G, pos, nbh);
        if (lane < nseg) {
            SegInfo& si = sinf[lane];
            seg_at(cut, cta, G, pos, lane, si.bh, si.t0, si.t1);
            seg_owners(cut, G, pos, si.bh, si.c0, si.c1);
            int owners = 0;
            for (int c = si.c0; c < si.c1; ++c) owners += (cut[c] < cut[c + 1] || pos == 0) ? 1 : 0;
            si.owners = owners;
        }
        if (lane == 0) {
            meta[0] = pos;
            meta[1] = nseg;
            if (a.trace && li == a.trace_layer && g == a.trace_group) a.trace[cta * kTr + 11] = static_cast<uint64_t>(nseg);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            tbuilt[g] = li + 1;
        }
    };
    build_table(0);
    PIPE_MARK(0);

    for (l = 0; l < nL; ++l) {
        const StepLayer& Ly = a.layer[l];
        const uint32_t lp = static_cast<uint32_t>(l) & 1u;
        uint8_t* tb = tab(g, l);
        const long long* cut = reinterpret_cast<const long long*>(tb);
        const SegInfo* sinf = reinterpret_cast<const SegInfo*>(cut + kMaxG + 1);
        const int pos = reinterpret_cast<const int*>(sinf + kMaxU)[0];
        const int nseg = reinterpret_cast<const int*>(sinf + kMaxU)[1];
        auto seg_of = [&](int p) { return rev ? nseg - 1 - p : p; };
        const size_t cap = static_cast<size_t>(Ly.cap);
        if (l > 0) PIPE_MARK(0);
        PIPE_MARK(1);
        // ---- P1: the group's token rows of this CTA's K split (TMA, fp32),
        // its projection items from the weight ring, partials to L2
        if (np1 > 0) {
            const float* xsrc = l == 0 ? a.x : a.layer[l - 1].y;
            if (lane == 0) {
                // the rows were written by other CTAs' generic stores (ordered by
                // the barrier): order them before this thread's async-proxy reads
                asm volatile("fence.proxy.async.global;" ::: "memory");
                mbar_arrive_expect_tx(xbar(g), static_cast<uint32_t>(Bg[g] * kKS * 4));
                for (int m = 0; m < Bg[g]; ++m)
                    tma_bulk_g2s(xst + m * kXF, xsrc + static_cast<size_t>(b0g[g] + m) * a.E + ps * kKS, kKS * 4, xbar(g));
            }
            pwait(xbar(g), xcnt & 1u, 11);
            ++xcnt;
        }
        gate(0, l);
        {
            const unsigned base = wbase(0, g, l, nL, np1, np3);
            float* P = Pg + static_cast<size_t>(ps) * pstride;
            for (int k = 0; k < np1; ++k) {
                const unsigned ia = base + static_cast<unsigned>(k);
                const int slot = static_cast<int>(ia % kNA);
                pwait(&fullA[slot], (ia / kNA) & 1u, 5);
                float facc[4];
                item_mma_xf(smem_u32(ringA + slot * kItem), smem_u32(xst), lane, facc);
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyA[slot]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int n = (plo + k) * 16 + g8 + ((i & 2) ? 8 : 0);
                    const int m = 2 * t4 + (i & 1);
                    if (m < Bg[g]) P[static_cast<size_t>(m) * a.Nrows + n] = facc[i];
                }
            }
        }
        block_done();
        // the first segment's M_QK column does not depend on the projection
        float mq0[R];
        if (nseg > 0) {
            const int h0 = sinf[seg_of(0)].bh % a.nh;
            const float* mq = Ly.mqk + static_cast<size_t>(h0) * R * R + lane;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) mq0[jj] = __ldg(mq + jj * R);
        }
        PIPE_MARK(2);
        group_sync(g, a.bar[g], (++gen) * static_cast<unsigned>(G));  // G1: the group's partials are written
        PIPE_MARK(3);
        if (ysplit) {
            // the group's y rows collect two partial sums: zero this CTA's share
            const size_t ny = static_cast<size_t>(Bg[g]) * a.e_out, yb = static_cast<size_t>(b0g[g]) * a.e_out;
            const size_t y0 = ny * cta / G, y1 = ny * (cta + 1) / G;
            for (size_t i = y0 + lane; i < y1; i += 32) Ly.y[yb + i] = 0.f;
        }
        // segment slots this layer does not use complete their phases anyway
        if (lane == 0)
            for (int j = nseg; j < kMaxU; ++j) {
                mbar_arrive(&uready(g)[j]);
                mbar_arrive_n(&sfull(g)[j], kNW);
            }
        // (a) qt = (sum_split c_Q) . M_QK per segment, ahead of the consumers;
        //     a region's last segment also gets the step's own K / V latents,
        //     rounded to the cache's bf16 and written to row pos (decode.cpp:143-149)
        auto prep = [&](int p, const float (&mqv)[R]) {
            const int j = seg_of(p);
            const SegInfo& s = sinf[j];
            const int bl = s.bh / a.nh, h = s.bh - bl * a.nh;
            const bool own = s.t1 == pos;
            const float* pb = Pg + static_cast<size_t>(bl) * a.Nrows + static_cast<size_t>(h) * 3 * R + lane;
            float pv[3][kMaxSplits];
#pragma unroll
            for (int sp = 0; sp < kMaxSplits; ++sp) {
                pv[0][sp] = sp < splits ? __ldcg(pb + sp * pstride) : 0.f;
                pv[1][sp] = (own && sp < splits) ? __ldcg(pb + sp * pstride + R) : 0.f;
                pv[2][sp] = (own && sp < splits) ? __ldcg(pb + sp * pstride + 2 * R) : 0.f;
            }
            float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int sp = 0; sp < kMaxSplits; ++sp)
#pragma unroll
                for (int r = 0; r < 3; ++r) v[r] += pv[r][sp];
            float qt = 0.f;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) qt = fmaf(__shfl_sync(0xffffffffu, v[0], jj), mqv[jj], qt);
            qts[j * R + lane] = qt;
            if (own) {
                uint8_t* region = Ly.cache + (static_cast<size_t>(rb0) + s.bh) * cap * C::ROWB;
                const uint32_t grow = static_cast<uint32_t>(pos) * C::ROWB;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const __nv_bfloat16 bv = __float2bfloat16_rn(v[1 + half]);
                    nrow[j * 2 * R + half * R + lane] = bv;
                    *reinterpret_cast<__nv_bfloat16*>(region + cache_swz(grow + half * C::PART + 2 * lane)) = bv;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&uready(g)[j]);
        };
        if (nseg > 0) prep(0, mq0);
        for (int p = 1; p < nseg; ++p) {
            const int h = sinf[seg_of(p)].bh % a.nh;
            float mqv[R];
            const float* mq = Ly.mqk + static_cast<size_t>(h) * R * R + lane;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) mqv[jj] = __ldg(mq + jj * R);
            prep(p, mqv);
        }
        PIPE_MARK(4);
        // (b) per segment as the consumers finish it: merge the warp states
        //     (+ the own token); pair regions meet through DSMEM, other shared
        //     regions through L2 (the last part to arrive merges, in range
        //     order: SoftmaxState::merge, decode.cpp:59-75)
        for (int p = 0; p < nseg; ++p) {
            const int j = seg_of(p);
            pwait(&sfull(g)[j], lp, 7);
            const SegInfo& s = sinf[j];
            const float* rbs = wst + j * kNW * (R + 2);
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kNW; ++w) M = fmaxf(M, rbs[w * (R + 2) + R]);
            float Ls = 0.f, av = 0.f;
#pragma unroll
            for (int w = 0; w < kNW; ++w) {
                const float mw = rbs[w * (R + 2) + R];
                if (mw == -INFINITY) continue;
                const float f = ex2(mw - M);
                Ls = fmaf(rbs[w * (R + 2) + R + 1], f, Ls);
                av = fmaf(rbs[w * (R + 2) + lane], f, av);
            }
            if (s.t1 == pos) {
                const float kf = __bfloat162float(nrow[j * 2 * R + lane]);
                const float vf = __bfloat162float(nrow[j * 2 * R + R + lane]);
                const float sn = warp_sum(qts[j * R + lane] * kf);
                const float Mn = fmaxf(M, sn);
                const float fo = ex2(M - Mn), fn = ex2(sn - Mn);
                Ls = fmaf(Ls, fo, fn);
                av = fmaf(av, fo, vf * fn);
                M = Mn;
            }
            const int c0 = s.c0, c1 = s.c1, owners = s.owners;
            const bool pair = a.cluster == 2 && owners == 2 && c1 - c0 == 2 && (c0 & 1) == 0;
            float L2 = Ls, a2 = av;
            if (pair && cta == c0 + 1) {
                const uint32_t dst = cluster_map(smem_u32(pst), 0u);
                st_cluster_f32(dst + 4u * lane, av);
                if (lane == 0) {
                    st_cluster_f32(dst + 4u * R, M);
                    st_cluster_f32(dst + 4u * (R + 1), Ls);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(cluster_map(smem_u32(pbar(g)), 0u));
                continue;
            }
            if (pair) {
                mbar_wait_cluster(pbar(g), pcnt & 1u);
                ++pcnt;
                const float mc = pst[R], lc = pst[R + 1], ac = pst[lane];
                if (mc != -INFINITY) {
                    const float Mn = fmaxf(M, mc);
                    const float fo = ex2(M - Mn), fc = ex2(mc - Mn);
                    L2 = fmaf(lc, fc, Ls * fo);
                    a2 = fmaf(ac, fc, av * fo);
                }
            } else if (owners > 1) {
                float* wsp = a.ws[g] + (static_cast<size_t>(cta) * kMaxU + j) * kWS;
                wsp[lane] = av;
                if (lane == 0) {
                    wsp[R] = M;
                    wsp[R + 1] = Ls;
                }
                __syncwarp();
                unsigned old = 0;
                if (lane == 0) old = atom_add_acq_rel(reinterpret_cast<unsigned*>(Ly.counters) + rb0 + s.bh);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old != static_cast<unsigned>(owners - 1)) continue;
                float M2 = -INFINITY;
                L2 = 0.f;
                a2 = 0.f;
                for (int c = c0; c < c1; ++c) {
                    if (!(cut[c] < cut[c + 1])) continue;
                    const int jc = static_cast<int>(static_cast<long long>(s.bh) - cut[c] / pos);
                    const float* wb = a.ws[g] + (static_cast<size_t>(c) * kMaxU + jc) * kWS;
                    const float mc = __ldcg(wb + R), lc = __ldcg(wb + R + 1), ac = __ldcg(wb + lane);
                    if (mc == -INFINITY) continue;
                    const float Mn = fmaxf(M2, mc);
                    const float fo = ex2(M2 - Mn), fc = ex2(mc - Mn);
                    L2 = fmaf(lc, fc, L2 * fo);
                    a2 = fmaf(ac, fc, a2 * fo);
                    M2 = Mn;
                }
                if (lane == 0) Ly.counters[rb0 + s.bh] = 0;
            }
            // v~ -> the group's O-projection X rows: hi in row bl, lo in row 8 + bl
            const int bl = s.bh / a.nh, h = s.bh - bl * a.nh;
            const int k = h * R + lane, sx = k / kKS, kk = k - sx * kKS;
            const float vo = a2 / L2;
            const __nv_bfloat16 vh = __float2bfloat16_rn(vo);
            const __nv_bfloat16 vl = __float2bfloat16_rn(vo - __bfloat162float(vh));
            uint8_t* xs = a.xo[g] + static_cast<size_t>(sx) * C::XB2;
            const uint32_t eb = static_cast<uint32_t>((kk & 7) * 2);
            *reinterpret_cast<__nv_bfloat16*>(xs + xrow_off(bl, kk >> 3) + eb) = vh;
            *reinterpret_cast<__nv_bfloat16*>(xs + xrow_off(kTok + bl, kk >> 3) + eb) = vl;
        }
        PIPE_MARK(6);
        group_sync(g, a.bar[g], (++gen) * static_cast<unsigned>(G));  // G2: the group's rows are merged
        PIPE_MARK(7);
        if (g == 0 && cta == 0 && lane == 0) *Ly.d_len = posl[l] + 1;  // nobody re-reads it this launch
        if (l + 1 < nL) build_table(l + 1);
        // ---- P3: the group's folded O-projection over its X slices (TMA)
        if (np3 > 0) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                mbar_arrive_expect_tx(xbar(g), static_cast<uint32_t>(p3ns * C::XB2));
                for (int s = 0; s < p3ns; ++s)
                    tma_bulk_g2s(xst + s * C::XB2, a.xo[g] + static_cast<size_t>(p3s0 + s) * C::XB2, C::XB2, xbar(g));
            }
            pwait(xbar(g), xcnt & 1u, 12);
            ++xcnt;
            PIPE_MARK(8);
        }
        gate(1, l);
        {
            const unsigned a3 = wbase(1, g, l, nL, np1, np3);
            for (int j = 0; j < np3; ++j) {
                const unsigned ia = a3 + static_cast<unsigned>(j);
                const int slot = static_cast<int>(ia % kNA), s = j % p3ns;
                pwait(&fullA[slot], (ia / kNA) & 1u, 10);
                float facc[2][4];  // hi rows, lo rows
                item_mma_x2(smem_u32(ringA + slot * kItem), smem_u32(xst + s * C::XB2), lane, facc);
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyA[slot]);
                float* pj3 = part + j * 16 * kTok;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int n = g8 + ((i & 2) ? 8 : 0);
                    const int m = 2 * t4 + (i & 1);
                    pj3[n * kTok + m] = facc[0][i] + facc[1][i];
                }
            }
        }
        block_done();
        PIPE_MARK(12);
        for (int i = lane; i < nt3 * 16 * Bg[g]; i += 32) {
            const int ti = i / (16 * Bg[g]), r = i - ti * 16 * Bg[g];
            const int m = r / 16, n = r - m * 16;
            const int col = (t3lo + ti * t3step) * 16 + n;
            if (col >= a.e_out) continue;
            float v = 0.f;
            for (int s = 0; s < p3ns; ++s) v += part[((ti * p3ns + s) * 16 + n) * kTok + m];
            float* yp = Ly.y + static_cast<size_t>(b0g[g] + m) * a.e_out + col;
            if (ysplit) atomicAdd(yp, v);  // one of exactly two addends onto 0
            else *yp = v;
        }
        PIPE_MARK(9);
        if (l + 1 < nL) group_sync(g, a.bar[g], (++gen) * static_cast<unsigned>(G));  // G3: y rows are the next token
    }
    if (cta == 0 && lane == 0) *a.bgen[g] = gen;
}

}  // namespace

int pipe_set_debug(int* mapped) {
#ifdef WSVD_PIPE_DEBUG
    return cudaMemcpyToSymbol(g_pipe_dbg, &mapped, sizeof(mapped)) == cudaSuccess ? 1 : 0;
#else
    (void)mapped;
    return 0;
#endif
}

bool pipe_supported(int R, int B, int nh, int Kp, int oKp, int otiles, int grid) {
    if (R != 32 || B < 2 || B > 2 * kTok || nh < 1) return false;
    if (grid > kMaxG || grid < 2) return false;
    if (Kp % kKS != 0 || oKp % kKS != 0) return false;
    const int splits = Kp / kKS, osplits = oKp / kKS;
    if (osplits > 2 || splits > grid || splits > kMaxSplits) return false;
    const int bg = B - B / 2;
    if ((bg * nh + grid - 1) / grid + 1 > kMaxU) return false;
    if (osplits == 2 && (otiles + grid / 2 - 1) / (grid / 2) > 4) return false;
    if (osplits == 1 && (otiles + grid - 1) / grid > 4) return false;
    return true;
}
size_t pipe_xo_bytes(int oKp) { return static_cast<size_t>(oKp / kKS) * PC<32>::XB2; }
size_t pipe_ws_bytes(int grid) { return static_cast<size_t>(grid) * kMaxU * kWS * 4; }
size_t pipe_p_bytes(int Kp, int Nrows) { return static_cast<size_t>(Kp / kKS) * kTok * Nrows * 4; }

static bool pipe_attr() {
    static int ok = -1;
    if (ok < 0) {
        ok = cudaFuncSetAttribute(chain_pipe_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, PC<32>::SMEM) ==
                     cudaSuccess
                 ? 1
                 : 0;
        if (!ok) cudaGetLastError();
    }
    return ok == 1;
}

int pipe_resident_ctas_per_sm() {
    if (!pipe_attr()) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, chain_pipe_kernel<32>, kThr, PC<32>::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int pipe_pair_clusters_ok(int grid) {
    if (grid % 2 != 0 || !pipe_attr()) return 0;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = PC<32>::SMEM;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, chain_pipe_kernel<32>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return 2 * n >= grid ? 1 : 0;
}

cudaError_t launch_chain_pipe(const PipeArgs& a, cudaStream_t s) {
    if (!pipe_attr()) return cudaErrorInvalidValue;
    return launch_pdl_cluster(chain_pipe_kernel<32>, dim3(a.grid), dim3(kThr), PC<32>::SMEM, s, a.cluster, a);
}

}  // namespace wsvd_k
