// step.cu -- the decode-layer step as ONE persistent kernel (bf16 weights,
// bf16 latent cache, rank 32), for one layer or a chain of layers.
//
// pipe::decode_factored's per-layer body (reference src/pipeline.cpp:320-329)
// is append_token (decode.cpp:127-153) -> fused_decode_step (decode.cpp:155-206)
// -> heads_row . W_o.  The multi-kernel path (capi.cu layer_step_impl) runs it
// as projection GEMM -> append epilogue -> attention -> combine -> O-projection.
// This kernel runs the same arithmetic with one CTA per SM.  Per layer:
//
//   P1   latent projection P[split][b][n] = x_b . A[:, n] over one K split
//        (swap-AB mma.sync over W-tiles streamed by TMA, as gemm.cu); every
//        partial is stored with its layer step's tag in one 64-bit word, and
//        the helper that prepares a head's query re-reads any word whose tag
//        is stale -- no grid barrier, release or flag between the projection
//        and the attention (WSVD_STEP_G1=1 restores a grid barrier for A/B:
//        ~2 us per layer slower, profiles/r02_step_ab.txt);
//   P2   attention over the cached rows 0 .. pos-1: the B*nh*pos rows of all
//        (sequence, head) regions are cut into G equal contiguous ranges (at
//        32-row boundaries), one per CTA, so every SM streams the same bytes.
//        A range covers a few (sequence, head) segments.  The helper warp
//        derives each segment's absorbed query qt = (sum_split c_Q) . M_QK;
//        the consumer warps run the tensor-core scores K_tile . [qt_hi | qt_lo]
//        and acc += V_tile^T . [p_hi | p_lo] with a warp-uniform running max
//        (SoftmaxState::observe, decode.cpp:35-57, in the log2 domain);
//   merge  per segment, the helper merges the 8 warp states (fixed order);
//        the segment that ends a region also observes the step's own token
//        (its K/V latents from the projection partials, rounded to the
//        cache's bf16 and written to row pos: the reference appends before
//        attending, decode.cpp:143-149).  A region shared by the two CTAs of a
//        cluster pair meets through distributed shared memory; any other
//        shared region publishes its parts and the LAST to arrive merges them
//        in range order (SoftmaxState::merge, decode.cpp:59-75), writing
//        v~ = acc / denom as hi + lo bf16 rows of the O-projection input;
//   G2   grid barrier: every row is merged; the cache length is committed;
//   P3   folded O-projection y = v~ . (B_V . W_o) over W-tiles prefetched into
//        shared memory during P2 (run-to-run deterministic: fixed-order sums,
//        or exactly two red.add addends onto zeros);
//   flag (chains) per CTA: its share of y is written (a release count).  y is
//        the next layer's token (pipeline.cpp:318-336, attention blocks
//        chained): each CTA's next projection waits for exactly the CTAs whose
//        O-projection tiles cover its K split -- no grid barrier between the
//        layers (WSVD_STEP_G3=1 restores it for A/B).
//
// The producer warps drive two rings: warp 8 the weight ring (P1 items, then
// the O-projection items, continuing across layers), warp 9 the cache stream.
// Projection items beyond the 4-slot weight ring are parked in the attention
// ring's stages.  In a chain, the next layer's parked items are loaded while
// this layer finishes: into the stages the O-projection does not use as soon
// as this CTA's attention has consumed them, into the rest once P3 is done --
// so the next layer's projection finds its weights in shared memory when its
// token (this layer's y) is complete.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kNW = 8;               // consumer warps
constexpr int kThr = 32 * kNW + 96;  // + two producer warps (weight ring, cache ring) + one helper warp
constexpr int kHelp = kNW + 2;       // the helper warp
constexpr int kSync = 32 * kNW + 32; // threads in the grid barrier (consumers + helper)
constexpr int kST = 256;             // tokens per attention stage
constexpr int kKS = 512;             // K per weight work item
constexpr int kItem = 16 * kKS * 2;  // one weight work item: 16 rows x 512 bf16 = 16 KB
constexpr int kNA = 4;               // weight ring slots
constexpr int kXS = kKS * 2;         // bytes per staged token row (16-byte units XOR 4 on odd rows)
constexpr int kMaxU = 10;            // (sequence, head) segments per CTA (host-checked)
constexpr int kMaxSplits = 16;       // projection K splits (host-checked)
constexpr int kWS = 36;              // floats per segment state in ws: acc[32], m, l, pad (16 B rows)
constexpr int kMaxG = 160;           // CTAs (the range table)
constexpr int kCut = 32;             // range boundaries fall on multiples of 32 rows (one warp's share)
constexpr int kTr = 32;              // trace words per CTA (WSVD_STEP_TRACE): marks 0-9, smid, segments, marks 12-31

template <int R, int MT>
struct SC {
    static constexpr int ROWB = 4 * R;  // bf16 [C_K | C_V]
    static constexpr int PART = 2 * R;
    static constexpr int STAGE = kST * ROWB;
    static constexpr int XB = MT * 16 * kXS;  // one staged X slice
    static constexpr int XB2 = 2 * XB;        // an O-projection X slice: hi rows, then lo rows
    // per segment: absorbed query, the 8 warp states, the own token's K|V row
    static constexpr int RED = kMaxU * (R * 4 + kNW * (R + 2) * 4 + 4 * R) + (R + 4) * 4;  // + the partner's state
    static constexpr int PARTB = 2 * kNA * 16 * MT * 16 * 4;  // P3 partial tiles [2][kNA][16][MT*16] fp32
    static constexpr bool PART_IN_RED = PARTB <= RED;          // the merge area is free during P3
    static constexpr int CUTB = (kMaxG + 1) * 8 + kMaxU * 32 + 16;  // + the segment table + (pos, nseg)
    // two range tables (layer parity: the next layer's is built during this layer's attention)
    static constexpr int FIXED = kNA * kItem + XB + RED + 2 * CUTB + 768;
    static constexpr int NB_RAW = (227 * 1024 - FIXED) / STAGE;
    static constexpr int NB = NB_RAW > 6 ? 6 : NB_RAW;
    static constexpr int RING = NB * STAGE;
    static constexpr int B_OFF = kNA * kItem;
    static constexpr int X_OFF = B_OFF + NB * STAGE;
    static constexpr int RED_OFF = X_OFF + XB;
    static constexpr int CUT_OFF = RED_OFF + RED;
    static constexpr int BAR_OFF = CUT_OFF + 2 * CUTB;
    static constexpr int SMEM = BAR_OFF + 512;
    static constexpr bool OK = NB_RAW >= 2 && XB2 + (PART_IN_RED ? 0 : PARTB) <= NB * STAGE;
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
// phase marks of layer a.trace_layer (variable l in scope)
#define STEP_MARK(k) \
    do { if (trc && l == a.trace_layer && (tid & 31) == 0) trc[cta * kTr + (k)] = gtimer(); } while (0)

WSVD_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// a projection partial and the layer step that wrote it, as one 64-bit word:
// single-copy atomic, so a reader that sees the step's tag sees its value
// (no release / flag round trips between the projection and its readers)
WSVD_DEV void st_tagged(unsigned long long* p, float v, unsigned tag) {
    const unsigned long long w = (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
WSVD_DEV unsigned long long ld_tagged(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
WSVD_DEV void red_release(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
WSVD_DEV unsigned atom_add_acq_rel(unsigned* p) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}
// wait until the monotone count reaches target (modulo 2^32: the counts wrap
// after ~10^7 steps; the signed difference stays meaningful)
WSVD_DEV void wait_count(const unsigned* p, unsigned target) {
    while (static_cast<int>(ld_acquire(p) - target) < 0) {
    }
}
WSVD_DEV void mbar_arrive_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
// generic-proxy shared-memory writes before async-proxy (TMA) writes to the same bytes
WSVD_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Grid-wide barrier among the consumer and helper warps of every CTA (all
// CTAs are resident: one per SM).  bar is a monotone arrival count; arrival is
// a fire-and-forget release reduction and everyone polls with acquire loads
// (1.2 us on B200 against 2.0 for a count-and-release barrier,
// tools/micro_barrier.cu).
WSVD_DEV void grid_sync(unsigned* bar, unsigned target, uint64_t* tr = nullptr) {
    named_bar_sync(1, kSync);
    if (threadIdx.x == 0) {
        if (tr) tr[25] = gtimer();
        red_release(bar);
        wait_count(bar, target);
        if (tr) tr[7] = gtimer();
    }
    named_bar_sync(1, kSync);
}

// Range table: CTA c attends over the flattened rows [cut[c], cut[c+1]) of the
// (sequence, head)-major row space, T = B*nh*pos rows (the cached rows 0 ..
// pos-1 of every region), cut at multiples of kCut rows inside a region.
WSVD_DEV long long cut_row(int c, int G, long long T, int pos) {
    if (c >= G) return T;
    if (pos == 0) return 0;
    const long long f = (static_cast<long long>(c) * T) / G;
    const long long bh = f / pos, t = f - bh * pos;
    return bh * pos + (t & ~static_cast<long long>(kCut - 1));
}

// Segment j of CTA c: (sequence, head) region bh and its rows [t0, t1).
// pos == 0 (the first token of every sequence): no cached rows; CTA c owns the
// regions bh = c + j*G as empty segments.
struct Seg {
    int bh, t0, t1;
};
// processing order p -> segment (range order): odd CTAs walk their range
// backwards (rev); swap01 exchanges the first two
WSVD_DEV int seg_index(int p, int nseg, bool rev, int swap01) {
    const int q = (swap01 && p < 2) ? 1 - p : p;
    return rev ? nseg - 1 - q : q;
}
// this CTA's segments, resolved once per layer: region, rows, and the CTAs
// [c0, c1) whose ranges reach into the region (owners of them hold a part)
struct SegInfo {
    int bh, t0, t1, owners, c0, c1, pad0, pad1;
};
WSVD_DEV int seg_count(const long long* cut, int c, int G, int pos, int nbh) {
    if (pos == 0) return c < nbh ? (nbh - 1 - c) / G + 1 : 0;
    const long long lo = cut[c], hi = cut[c + 1];
    if (lo >= hi) return 0;
    return static_cast<int>((hi - 1) / pos - lo / pos + 1);
}
WSVD_DEV Seg seg_at(const long long* cut, int c, int G, int pos, int j) {
    Seg s;
    if (pos == 0) {
        s.bh = c + j * G;
        s.t0 = s.t1 = 0;
        return s;
    }
    const long long lo = cut[c], hi = cut[c + 1];
    const long long bh0 = lo / pos;
    s.bh = static_cast<int>(bh0 + j);
    const long long rs = static_cast<long long>(s.bh) * pos;
    s.t0 = static_cast<int>(lo > rs ? lo - rs : 0);
    s.t1 = static_cast<int>(hi < rs + pos ? hi - rs : pos);
    return s;
}
// CTAs whose ranges reach into region bh: [c0, c1) -- those with empty ranges
// among them hold no segment; c0 is the range containing row bh*pos
WSVD_DEV void seg_owners(const long long* cut, int G, int pos, int bh, int& c0, int& c1) {
    if (pos == 0) {
        c0 = bh % G;
        c1 = c0 + 1;
        return;
    }
    const long long r0 = static_cast<long long>(bh) * pos, r1 = r0 + pos;
    int lo = 0, hi = G;  // largest c with cut[c] <= r0
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

// byte offset of 16-byte unit u of staged token row m (odd rows XOR 4: the
// fragment loads of rows g and g + 1 hit disjoint bank quads)
WSVD_DEV uint32_t xrow_off(int m, int u) { return static_cast<uint32_t>(m * kXS + ((u ^ ((m & 1) << 2)) * 16)); }

// fp32 X[rows][ldx] columns [k0, k0 + kKS) -> bf16 smem [MT*16][kXS], zero
// padded.  Every load of the thread is issued before the first is consumed:
// the slice costs one memory latency, not one per item.
template <int MT>
WSVD_DEV void stage_rows(const float* X, int rows, int ldx, int kvalid, int k0, uint8_t* xs, int ctid,
                         uint64_t* issued = nullptr) {
    constexpr int PER = kKS / 8;                       // 8-element items per row
    constexpr int NIT = MT * 16 * PER / (32 * kNW);    // items per thread
    static_assert(MT * 16 * PER % (32 * kNW) == 0, "staging items must divide evenly");
    float4 v[NIT][2];
    const bool vec = (ldx % 4) == 0;
#pragma unroll
    for (int u = 0; u < NIT; ++u) {
        const int i = ctid + u * 32 * kNW;
        const int m = i / PER, kk = (i - m * PER) * 8;
        const int k = k0 + kk;
        v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < rows) {
            const float* src = X + static_cast<size_t>(m) * ldx + k;
            if (k + 8 <= kvalid && vec) {
                v[u][0] = __ldcg(reinterpret_cast<const float4*>(src));
                v[u][1] = __ldcg(reinterpret_cast<const float4*>(src + 4));
            } else {
                float t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) t[j] = (k + j < kvalid) ? __ldcg(src + j) : 0.f;
                v[u][0] = make_float4(t[0], t[1], t[2], t[3]);
                v[u][1] = make_float4(t[4], t[5], t[6], t[7]);
            }
        }
    }
    if (issued) {  // every load of this warp is out
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(issued);
    }
#pragma unroll
    for (int u = 0; u < NIT; ++u) {
        const int i = ctid + u * 32 * kNW;
        const int m = i / PER, kk = (i - m * PER) * 8;
        uint4 o;
        o.x = pack_bf16x2(v[u][0].x, v[u][0].y); o.y = pack_bf16x2(v[u][0].z, v[u][0].w);
        o.z = pack_bf16x2(v[u][1].x, v[u][1].y); o.w = pack_bf16x2(v[u][1].z, v[u][1].w);
        *reinterpret_cast<uint4*>(xs + xrow_off(m, kk / 8)) = o;
    }
}

// One weight work item (16 W-rows x kKS, W-tile layout of gemm.cu) against the
// staged tokens: D fragments facc[mt][hh][i] = (row g | g+8, token 2t | 2t+1).
template <int MT>
WSVD_DEV void item_mma(uint32_t slot_addr, uint32_t xs_addr, int lane, float (&facc)[MT][2][4],
                       int blo = 0, int bhi = kKS / 32) {
    const int g = lane >> 2, t = lane & 3;
    const uint32_t swz = static_cast<uint32_t>((g & 1) << 2);
    const uint32_t row_lo = slot_addr + static_cast<uint32_t>(g * kKS * 2);
    const uint32_t row_hi = row_lo + static_cast<uint32_t>(8 * kKS * 2);
    const uint32_t xbase = xs_addr + static_cast<uint32_t>(g * kXS);  // token rows g (+ 8, 16, ...): same swizzle
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int i = 0; i < 4; ++i) facc[mt][hh][i] = 0.f;
#pragma unroll 4
    for (int b = blo; b < bhi; ++b) {
        const uint32_t uoff = ((static_cast<uint32_t>(4 * b + t)) ^ swz) * 16;
        const uint4 wl = lds128(row_lo + uoff);
        const uint4 wh = lds128(row_hi + uoff);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const uint4 xv = lds128(xbase + static_cast<uint32_t>((mt * 16 + hh * 8) * kXS) + uoff);
                mma_bf16_16816(facc[mt][hh], wl.x, wh.x, wl.y, wh.y, xv.x, xv.y);
                mma_bf16_16816(facc[mt][hh], wl.z, wh.z, wl.w, wh.w, xv.z, xv.w);
            }
    }
}

template <int R, int MT, bool GEN>
__global__ void __launch_bounds__(kThr, 1) layer_step_kernel(const __grid_constant__ StepArgs a) {
    // The production instantiation (GEN = false) has no phase marks and the
    // A/B switches at their defaults (capi.cu); GEN = true reads them (and the
    // WSVD_STEP_TRACE marks) from the arguments.
    uint64_t* const trc = GEN ? a.trace : nullptr;
    const int ab_p3_tma = GEN ? a.p3_tma : 0;
    const int ab_g3 = GEN ? a.g3 : 0;
    const int ab_x_first = GEN ? a.x_first : 1;
    const int ab_l2_next = GEN ? a.l2_next : 1;
    const int ab_chain_pre = GEN ? a.chain_pre : 4;
    const int ab_pre_stages = GEN ? a.pre_stages : 0;
    const int ab_short_seg = GEN ? a.short_seg : 2048;
    // production geometry: CTA pairs and two O-projection K splits (the host
    // launches the generic instantiation otherwise)
    const int kcl = GEN ? a.cluster : 2;
    const int ab_g1 = GEN ? a.g1 : 0;
    static_assert(R == 32, "the fused step is specialised for rank 32 (one latent dim per lane)");
    using C = SC<R, MT>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ringA = smem;
    uint8_t* ringB = smem + C::B_OFF;
    uint8_t* xbuf = smem + C::X_OFF;
    float* qts = reinterpret_cast<float*>(smem + C::RED_OFF);  // [kMaxU][R]
    float* wst = qts + kMaxU * R;                              // [kMaxU][kNW][R+2]
    __nv_bfloat16* nrow = reinterpret_cast<__nv_bfloat16*>(wst + kMaxU * kNW * (R + 2));  // [kMaxU][2R]
    float* pst = reinterpret_cast<float*>(nrow + kMaxU * 2 * R);  // [R+2] the pair partner's state (DSMEM)
    // range table of layer li (buffer li & 1): cut [G+1], segments [kMaxU], meta [0] pos [1] nseg
    auto cut_of = [&](int li) { return reinterpret_cast<long long*>(smem + C::CUT_OFF + (li & 1) * C::CUTB); };
    auto sinf_of = [&](int li) { return reinterpret_cast<SegInfo*>(cut_of(li) + kMaxG + 1); };
    auto meta_of = [&](int li) { return reinterpret_cast<volatile int*>(sinf_of(li) + kMaxU); };
    // tables built so far (helper; readers spin on it -- a count never aliases
    // the way an mbarrier parity can when the builder runs a layer ahead)
    volatile int* tbuilt = reinterpret_cast<volatile int*>(smem + C::BAR_OFF + 504);
    uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* emptyA = fullA + kNA;
    uint64_t* fullB = emptyA + kNA;
    uint64_t* emptyB = fullB + C::NB;
    uint64_t* uready = emptyB + C::NB;  // [kMaxU] segment j's query prepared (helper)
    uint64_t* sfull = uready + kMaxU;   // [kMaxU] segment j's warp states written (consumers)
    uint64_t* p3bar = sfull + kMaxU;    // P3: X slices landed
    uint64_t* wfull = p3bar + 1;        // [2*NB] projection items parked in the attention ring
    uint64_t* wdone = wfull + 2 * C::NB;  // [NB] those items consumed: the stage is free
    uint64_t* b1bar = wdone + C::NB;      // the first segment's producers are seen (gates the parked stages' refill)
    uint64_t* pbar = b1bar + 1;           // the pair partner's state landed (DSMEM)
    uint64_t* xin = pbar + 1;             // every consumer warp has requested its token-slice loads
    uint64_t* p3done = xin + 1;           // the layer's O-projection no longer uses the attention ring
    uint64_t* ybar = p3done + 1;          // pair P3: the odd CTA's split-1 sums landed (DSMEM st.async bytes)
    static_assert((2 * kNA + 2 * C::NB + 2 * kMaxU + 1 + 2 * C::NB + C::NB + 6) * 8 <= 504,
                  "mbarriers overflow their shared-memory region");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int nL = a.nlayers;
    int l = 0;  // the layer (trace marks)

    STEP_MARK(0);
    if (trc && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trc[cta * kTr + 10] = smid;
    }
    // ---- projection geometry (the same for every layer): K split ps, a
    // contiguous run [plo, phi) of the split's 16-row W-tiles (rows n =
    // (head*3 + role)*R + i, capi.cu packing)
    const int splits = a.Kp / kKS;
    const int cps = G / splits;  // CTAs per projection split
    const int ps = cta % splits, pj = cta / splits;
    const int ptiles = a.Nrows / 16;
    const int plo = pj < cps ? static_cast<int>(static_cast<long>(pj) * ptiles / cps) : 0;
    const int phi = pj < cps ? static_cast<int>(static_cast<long>(pj + 1) * ptiles / cps) : 0;
    const int np1 = phi - plo;
    const int osplits = GEN ? a.oKp / kKS : 2;
    // P3 items (tile, K split) of layer l.  Device y with two K splits: CTA c
    // takes split c % 2 of a run of tiles, so it stages only that split's X
    // rows; the two partial sums meet in y through fp32 red.add onto zeros --
    // with exactly two addends the result does not depend on their order
    // (0 + a + b == 0 + b + a), so y stays run-to-run deterministic.
    // Otherwise (host y -- mapped pinned memory, no atomics over the bus -- or
    // one K split) the CTA owns whole tiles with all their splits and sums them
    // itself; host y is a contiguous run of tiles, written as 16-byte stores
    // over 64-128-byte row segments (bus writes drain faster).  The X slices
    // sit at the end of the attention ring, the partial tiles in the merge area.
    struct P3G {
        int t3lo, nt3, t3step, p3s0, p3ns, np3, per, xoff, p3lo;
        bool ycontig, ysplit, pairy;
    };
    auto p3geom_of = [&](int li, int cta) {
        P3G g;
        g.ycontig = a.y_host != 0 && li == nL - 1;
        g.ysplit = !g.ycontig && osplits == 2;
        // CTA pairs: the odd CTA's split-1 sums cross into the even CTA through
        // distributed shared memory, which writes y = split 0 + split 1 with
        // plain stores (no zeroing pass, no atomics; the same fixed order)
        g.pairy = g.ysplit && kcl == 2;
        const int cps3 = G / 2;
        if (g.ysplit) {
            const int pj3 = cta / 2;
            g.t3lo = pj3 < cps3 ? static_cast<int>(static_cast<long>(pj3) * a.otiles / cps3) : 0;
            g.nt3 = pj3 < cps3 ? static_cast<int>(static_cast<long>(pj3 + 1) * a.otiles / cps3) - g.t3lo : 0;
            g.t3step = 1;
            g.p3s0 = cta % 2;
            g.p3ns = 1;
        } else {
            g.t3lo = g.ycontig ? static_cast<int>(static_cast<long>(cta) * a.otiles / G) : cta;
            g.nt3 = g.ycontig ? static_cast<int>(static_cast<long>(cta + 1) * a.otiles / G) - g.t3lo
                              : (cta < a.otiles ? (a.otiles - 1 - cta) / G + 1 : 0);
            g.t3step = g.ycontig ? 1 : G;  // tile i of this CTA: t3lo + i * t3step
            g.p3s0 = 0;
            g.p3ns = osplits;
        }
        g.np3 = g.nt3 * g.p3ns;  // <= kNA (host-checked)
        const int pb = C::PART_IN_RED ? 0 : C::PARTB;
        g.per = (g.p3ns * C::XB2 + pb <= C::RING) ? g.p3ns : 1;  // K splits staged together
        g.xoff = C::RING - g.per * C::XB2;
        g.p3lo = g.xoff - pb;  // first attention-ring byte P3 uses
        return g;
    };
    auto p3geom = [&](int li) { return p3geom_of(li, cta); };
    // Projection items beyond the 4-slot weight ring are parked in the
    // attention ring (2 per stage, in consumption order): the attention cannot
    // start before grid barrier 1 anyway, and with every item in flight at
    // once the projection costs one memory round trip instead of one per ring
    // turn.  Ring-A sequence of a layer: P1 items k < 4 or k >= 4 + nBH, then
    // its P3 items; the sequence continues across the layers of a chain.
    const int nBH = min(max(np1 - kNA, 0), 2 * C::NB);
    const int nA1 = np1 - nBH;
    const int nWS = (nBH + 1) / 2;  // attention stages holding parked items (the first nWS)
    auto parked = [&](int b) -> uint8_t* { return ringB + (b / 2) * C::STAGE + (b & 1) * kItem; };
    if (warp == 0) {
        // the barrier inits spread over warp 0's lanes
        if (lane < kNA) {
            mbar_init(&fullA[lane], 1);
            mbar_init(&emptyA[lane], 1);
        }
        if (lane < C::NB) {
            mbar_init(&fullB[lane], 1);
            mbar_init(&emptyB[lane], kNW);
            mbar_init(&wdone[lane], lane < nWS ? min(2, nBH - 2 * lane) : 1);
        }
        if (lane < kMaxU) {
            mbar_init(&uready[lane], 1);
            mbar_init(&sfull[lane], kNW);
        }
        if (lane < nBH) mbar_init(&wfull[lane], 1);
        if (lane == 0) {
            mbar_init(p3bar, 1);
            mbar_init(b1bar, 1);
            mbar_init(pbar, 1);
            mbar_init(xin, kNW);
            *tbuilt = 0;
            mbar_init(p3done, 1);
            mbar_init(ybar, 1);
        }
        fence_mbar_init();  // every lane: the fence covers the executing thread's inits
    }
    __syncthreads();
    if (kcl > 1) cluster_sync_all();  // the partner's barriers are initialised before any remote arrive
    // ring-A item ia (in-layer sequence) of layer li -> source
    auto a_src = [&](int li, int ia) -> const uint8_t* {
        const StepLayer& Ly = a.layer[li];
        if (ia < nA1) {
            const int k = ia < kNA ? ia : ia + nBH;
            return Ly.A + (static_cast<size_t>(plo + k) * splits + ps) * kItem;
        }
        const P3G g = p3geom(li);
        const int j = ia - nA1;
        return Ly.Wo + (static_cast<size_t>(g.t3lo + (j / g.p3ns) * g.t3step) * osplits + g.p3s0 + j % g.p3ns) * kItem;
    };
    auto parked_src = [&](int li, int b) -> const uint8_t* {
        return a.layer[li].A + (static_cast<size_t>(plo + kNA + b) * splits + ps) * kItem;
    };
    auto issue_parked = [&](int li, int b0, int b1) {
        for (int b = b0; b < b1 && b < nBH; ++b) {
            mbar_arrive_expect_tx(&wfull[b], kItem);
            tma_bulk_g2s(parked(b), parked_src(li, b), kItem, &wfull[b]);
        }
    };
    // The weights are constant across steps: the producer streams layer 0's
    // before the predecessor has drained (programmatic dependent launch); the
    // token, the length and the cache rows wait for it.
    int ia_pre = 0;
    const int na0 = nA1 + p3geom(0).np3;
    if (warp == kNW && lane == 0) {
        for (; ia_pre < kNA && ia_pre < na0; ++ia_pre) {
            mbar_arrive_expect_tx(&fullA[ia_pre], kItem);
            tma_bulk_g2s(ringA + ia_pre * kItem, a_src(0, ia_pre), kItem, &fullA[ia_pre]);
        }
        if (!ab_x_first) issue_parked(0, 0, nBH);
    }
    const int nbh = a.B * a.nh;
    if (warp == kNW + 1 && lane == 0 && a.pos_hint > 0 && ab_pre_stages > 0) {
        // Before the predecessor has drained: request the first stages of this
        // CTA's layer-0 cache range into L2 (a prefetch is only a hint -- L2 is
        // the point of coherence), at the length the host expects
        const long long Th = static_cast<long long>(nbh) * a.pos_hint;
        long long cc[2] = {cut_row(cta, G, Th, a.pos_hint), cut_row(cta + 1, G, Th, a.pos_hint)};
        const long long* ct = cc - cta;  // a two-entry table seen from this CTA
        const int ns = seg_count(ct, cta, G, a.pos_hint, nbh);
        int left = ab_pre_stages;
        for (int p = 0; p < ns && left > 0; ++p) {
            const Seg sg = seg_at(ct, cta, G, a.pos_hint, (cta & 1) ? ns - 1 - p : p);
            for (int t = sg.t0; t < sg.t1 && left > 0; t += kST, --left) {
                const int rows = min(kST, sg.t1 - t);
                prefetch_l2_bulk(a.layer[0].cache + (static_cast<size_t>(sg.bh) * a.layer[0].cap + t) * C::ROWB,
                                 static_cast<uint32_t>(((rows * C::ROWB + 1023) / 1024) * 1024));
            }
        }
    }
    griddep_wait();
    griddep_launch_dependents();
    STEP_MARK(1);

    const unsigned epoch = static_cast<unsigned>(*a.epoch);  // fused launches so far (x-fetch generations)
    const unsigned bgen0 = *a.bgen;                          // grid barriers completed so far
    unsigned gen = bgen0;
    const unsigned p1base = *a.p1gen;                        // layer steps completed so far
    // Odd CTAs walk their segments backwards: the region a pair (2k, 2k+1)
    // shares is then the LAST one both attend (its two parts finish together
    // and meet through distributed shared memory), the region shared with
    // the next pair the FIRST one (its merge through L2 happens early, off
    // the critical path).  Processing order p -> segment (range order) j.
    const bool rev = (cta & 1) != 0;
    const size_t pstride = static_cast<size_t>(a.B) * a.Nrows;

    // ================================================================ producers
    if (warp == kNW || warp == kNW + 1) {
        if (warp == kNW && lane == 0) {
            // the weight ring: every layer's P1 ring items, then its P3 items
            if (ab_x_first && nBH > 0) {
                mbar_wait(xin, 0u);
                issue_parked(0, 0, nBH);
            }
            unsigned ia_g = static_cast<unsigned>(ia_pre);  // items issued this launch
            for (int li = 0; li < nL; ++li) {
                const int na = nA1 + p3geom(li).np3;
                for (int i = (li == 0 ? ia_pre : 0); i < na; ++i) {
                    const int slot = static_cast<int>(ia_g % kNA);
                    mbar_wait(&emptyA[slot], ((ia_g / kNA) & 1u) ^ 1u);
                    if (trc && li == a.trace_layer && i == 0) trc[cta * kTr + 23] = gtimer();
                    mbar_arrive_expect_tx(&fullA[slot], kItem);
                    tma_bulk_g2s(ringA + slot * kItem, a_src(li, i), kItem, &fullA[slot]);
                    ++ia_g;
                }
            }
        } else if (warp == kNW + 1 && lane == 0) {
            // the cache stream, from its own warp: waiting for a ring-A slot
            // never holds it up (divergent lanes of one warp are scheduled as one)
            const uint64_t pol = policy_evict_first();
            uint32_t par = 0;  // per attention-ring slot: parity of its fills so far
            // The first a.chain_pre stages of this CTA's range of layer li into
            // L2, issued once this CTA's previous O-projection is done (every
            // attention stream of that layer has ended -- issued earlier, the
            // prefetch slows the stragglers): HBM is otherwise idle until layer
            // li's attention starts, and those stages then stream from L2
            auto prefetch_cache = [&](int li) {
                if (ab_chain_pre <= 0) return;
                const StepLayer& Ly = a.layer[li];
                const int pos = *static_cast<volatile const int*>(Ly.d_len);
                if (pos <= 0) return;
                const long long T = static_cast<long long>(nbh) * pos;
                long long cc[2] = {cut_row(cta, G, T, pos), cut_row(cta + 1, G, T, pos)};
                const long long* ct = cc - cta;  // a two-entry table seen from this CTA
                const int ns = seg_count(ct, cta, G, pos, nbh);
                int left = ab_chain_pre;
                for (int p = 0; p < ns && left > 0; ++p) {
                    const Seg sg = seg_at(ct, cta, G, pos, rev ? ns - 1 - p : p);
                    for (int t = sg.t0; t < sg.t1 && left > 0; t += kST, --left) {
                        const int rows = min(kST, sg.t1 - t);
                        prefetch_l2_bulk(Ly.cache + (static_cast<size_t>(sg.bh) * Ly.cap + t) * C::ROWB,
                                         static_cast<uint32_t>(((rows * C::ROWB + 1023) / 1024) * 1024));
                    }
                }
            };
            for (int li = 0; li < nL; ++li) {
                const uint32_t lp = static_cast<uint32_t>(li) & 1u;
                if (li > 0) {
                    // this layer's parked projection items: each stage as soon as
                    // the previous layer's attention has consumed it and, where
                    // the previous O-projection stages its rows, once P3 is done
                    const P3G gp = p3geom(li - 1);
                    bool p3w = false;
                    for (int st = 0; st < nWS; ++st) {
                        mbar_wait(&emptyB[st], ((par >> st) & 1u) ^ 1u);
                        if (!p3w && (st + 1) * C::STAGE > gp.p3lo) {
                            mbar_wait(p3done, lp ^ 1u);
                            prefetch_cache(li);  // (HBM is idle: every CTA is past its attention)
                            p3w = true;
                        }
                        issue_parked(li, 2 * st, 2 * st + 2);
                    }
                    // every other stage of the ring may hold P3 data until P3 is done
                    if (!p3w) {
                        mbar_wait(p3done, lp ^ 1u);
                        prefetch_cache(li);
                    }
                }
                while (*tbuilt < li + 1) {
                }
                __threadfence_block();
                const SegInfo* sinf = sinf_of(li);
                const int nseg = meta_of(li)[1];
                const StepLayer& Ly = a.layer[li];
                const size_t cap = static_cast<size_t>(Ly.cap);
                int ib = 0;  // stage fills of this layer: slot ib % NB
                for (int p = 0; p < nseg; ++p) {
                    const SegInfo& sg = sinf[seg_index(p, nseg, rev, meta_of(li)[2])];
                    for (int t = sg.t0; t < sg.t1; t += kST) {
                        const int rows = min(kST, sg.t1 - t);
                        // every slot's first fill of a layer is a whole stage (finite
                        // rows past the end, which the consumers read times p = 0;
                        // the allocation is padded): stale bytes of parked items or
                        // P3 partials never meet the tensor cores
                        const uint32_t rbytes = ib < C::NB ? static_cast<uint32_t>(C::STAGE)
                                                           : static_cast<uint32_t>(min(C::STAGE, ((rows * C::ROWB + 1023) / 1024) * 1024));
                        const int slot = ib % C::NB;
                        if (ib < nWS) {
                            mbar_wait(&wdone[slot], lp);  // its parked projection items are consumed
                            mbar_wait(b1bar, lp);         // and the first segment's producers are seen
                        }
                        mbar_wait(&emptyB[slot], ((par >> slot) & 1u) ^ 1u);
                        par ^= 1u << slot;
                        mbar_arrive_expect_tx(&fullB[slot], rbytes);
                        const uint8_t* src = Ly.cache + (static_cast<size_t>(sg.bh) * cap + t) * C::ROWB;
                        tma_bulk_g2s_stream(ringB + slot * C::STAGE, src, rbytes, &fullB[slot], pol);
                        ++ib;
                    }
                }
                if (ab_l2_next && li + 1 < nL) {
                    // the next layer's items that are loaded last (after this
                    // layer's P3): into L2 now, while this CTA's last stages stream
                    const P3G g = p3geom(li);
                    for (int b = 0; b < nBH; ++b)
                        if ((b / 2 + 1) * C::STAGE > g.p3lo) prefetch_l2_bulk(parked_src(li + 1, b), kItem);
                    for (int i = 0; i < nA1; ++i) prefetch_l2_bulk(a_src(li + 1, i), kItem);
                }
            }
        }
        return;
    }

    // ---- the range / segment table of layer li (helper warp; off the
    // consumers' path: P1 does not need it)
    auto build_table = [&](int li) {
        long long* cut = cut_of(li);
        SegInfo* sinf = sinf_of(li);
        volatile int* meta = meta_of(li);
        const int pos = *static_cast<volatile const int*>(a.layer[li].d_len);
        const long long T = static_cast<long long>(nbh) * pos;
        for (int c = lane; c <= G; c += 32) cut[c] = cut_row(c, G, T, pos);
        __syncwarp();
        const int nseg = seg_count(cut, cta, G, pos, nbh);  // <= kMaxU (host-checked)
        if (lane < nseg) {  // the segment table (64-bit index arithmetic, once)
            const Seg sg = seg_at(cut, cta, G, pos, lane);
            SegInfo& si = sinf[lane];
            si.bh = sg.bh;
            si.t0 = sg.t0;
            si.t1 = sg.t1;
            seg_owners(cut, G, pos, sg.bh, si.c0, si.c1);
            int owners = 0;
            for (int c = si.c0; c < si.c1; ++c) owners += (cut[c] < cut[c + 1] || pos == 0) ? 1 : 0;
            si.owners = owners;
        }
        if (lane == 0) {
            meta[0] = pos;
            meta[1] = nseg;
            // a short first segment would leave the consumers waiting for the
            // second one's query: process the (whole-region) second one first
            const int f = rev ? nseg - 1 : 0;
            meta[2] = (nseg >= 3 && sinf[f].t1 - sinf[f].t0 < ab_short_seg) ? 1 : 0;
            if (trc && li == a.trace_layer) trc[cta * kTr + 11] = static_cast<uint64_t>(nseg);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            *tbuilt = li + 1;
        }
    };
    if (warp == kHelp) build_table(0);

    const int g8 = lane >> 2, t4 = lane & 3;
    uint32_t parc = 0;  // consumers: per attention-ring slot, parity of the fills consumed
    unsigned abase = 0; // ring-A sequence index of the layer's first item
    unsigned pcnt = 0;  // helper: pair-partner states received (pbar phases)
    unsigned p3cnt = 0; // consumers: TMA-staged P3 rounds (p3bar phases)
    unsigned ycnt = 0;  // consumers: pair P3 rounds (ybar phases)
    uint32_t upar = 0;  // consumers: per segment slot, parity of the uready phases consumed
    uint32_t spar = 0;  // helper: per segment slot, parity of the sfull phases consumed
    for (l = 0; l < nL; ++l) {
        const StepLayer& Ly = a.layer[l];
        const uint32_t lp = static_cast<uint32_t>(l) & 1u;
        const P3G g3 = p3geom(l);
        // the O-projection rows, one buffer per layer parity: without a grid
        // barrier between layers, a CTA may merge layer l + 1's rows while
        // another still stages layer l's (it cannot get two layers ahead: G2)
        uint8_t* xo_l = a.xo + static_cast<size_t>(lp) * osplits * C::XB2;
        const bool xt_out = a.xtagged && g3.pairy && l + 1 < nL;  // this layer's y also as tagged bf16 pairs
        if (l > 0) {
            STEP_MARK(0);
            STEP_MARK(1);
        }
        // ---- P1 (consumer warps): latent projection of this CTA's K split
        if (warp < kNW) {
            const float* xsrc = l == 0 ? a.x : a.layer[l - 1].y;
            if (l == 0 && a.x_host && pj < cps) {
                // x lives in mapped (pinned) host memory: the cps CTAs of this K
                // split each fetch 1/cps of its [B][kKS] slice over the bus into
                // the device copy xd and publish a count; all stage from xd once
                // the count is complete (the host bytes cross the bus once)
                const int per = (a.B * kKS / 4 + cps - 1) / cps;  // float4 items per CTA
                for (int i = pj * per + tid; i < min((pj + 1) * per, a.B * kKS / 4); i += 32 * kNW) {
                    const int m = i / (kKS / 4), k4 = i - m * (kKS / 4);
                    const size_t off = static_cast<size_t>(m) * a.E + ps * kKS + 4 * k4;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ps * kKS + 4 * k4 + 4 <= a.E) v = __ldcv(reinterpret_cast<const float4*>(a.x + off));
                    *reinterpret_cast<float4*>(a.xd + off) = v;
                }
                named_bar_sync(2, 32 * kNW);
                if (tid == 0) {
                    red_release(a.xcnt + ps);
                    wait_count(a.xcnt + ps, static_cast<unsigned>(cps) * (epoch + 1u));
                }
                named_bar_sync(2, 32 * kNW);
                xsrc = a.xd;
            } else if (l == 0 && pj < cps && tid == 0) {
                // keep the counters' invariant (cps arrivals per fused launch) in device mode
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.xcnt + ps) : "memory");
            }
            const bool xt_in = l > 0 && a.xtagged && p3geom(l - 1).pairy;
            if (xt_in && np1 > 0) {
                // the token is the previous layer's y as tagged bf16 pairs: every
                // 16-byte unit of the slice from 4 words, each re-read until it
                // carries the previous layer step's tag (no flag round trip)
                const unsigned long long* xs = a.xtag + static_cast<size_t>((l - 1) & 1) * a.B * (a.E / 2);
                const unsigned want = p1base + static_cast<unsigned>(l);
                constexpr int PER = kKS / 8, NIT = MT * 16 * PER / (32 * kNW);
                unsigned long long w[NIT][4];
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int i = tid + u * 32 * kNW, m = i / PER, kk = (i - m * PER) * 8;
                    const unsigned long long* src = xs + static_cast<size_t>(m) * (a.E / 2) + (ps * kKS + kk) / 2;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        w[u][q] = m < a.B ? ld_tagged(src + q) : (static_cast<unsigned long long>(want) << 32);
                }
                for (;;) {
                    bool ok = true;
#pragma unroll
                    for (int u = 0; u < NIT; ++u)
#pragma unroll
                        for (int q = 0; q < 4; ++q) ok = ok && static_cast<unsigned>(w[u][q] >> 32) == want;
                    if (ok) break;
                    __nanosleep(32);
#pragma unroll
                    for (int u = 0; u < NIT; ++u) {
                        const int i = tid + u * 32 * kNW, m = i / PER, kk = (i - m * PER) * 8;
                        const unsigned long long* src = xs + static_cast<size_t>(m) * (a.E / 2) + (ps * kKS + kk) / 2;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (static_cast<unsigned>(w[u][q] >> 32) != want) w[u][q] = ld_tagged(src + q);
                    }
                }
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int i = tid + u * 32 * kNW, m = i / PER, kk = (i - m * PER) * 8;
                    *reinterpret_cast<uint4*>(xbuf + xrow_off(m, kk / 8)) =
                        make_uint4(static_cast<unsigned>(w[u][0]), static_cast<unsigned>(w[u][1]),
                                   static_cast<unsigned>(w[u][2]), static_cast<unsigned>(w[u][3]));
                }
            } else if (l > 0 && !ab_g3 && np1 > 0) {
                // the token is the previous layer's y: wait for the CTAs whose
                // O-projection tiles cover this K split's columns (tile T0 + lane;
                // a tile's producers are its pair's two CTAs, or one CTA)
                if (warp == 0) {
                    const P3G gq = p3geom_of(l - 1, 0);
                    const int t = ps * (kKS / 16) + lane;
                    if (t < a.otiles) {
                        int c0 = t % G, c1 = c0;
                        if (gq.ysplit) {
                            const int cps3 = G / 2, pj3 = ((t + 1) * cps3 - 1) / a.otiles;
                            c0 = 2 * pj3;
                            c1 = 2 * pj3 + 1;
                        }
                        const unsigned yt = p1base + static_cast<unsigned>(l);
                        for (int c = c0; c <= c1; ++c)
                            while (static_cast<int>(ld_acquire(a.yflag + 32 * c) - yt) < 0) __nanosleep(64);
                    }
                    __syncwarp();
                }
                named_bar_sync(2, 32 * kNW);
            }
            if (np1 > 0 && !xt_in) stage_rows<MT>(xsrc, a.B, a.E, a.E, ps * kKS, xbuf, tid, (l == 0) ? xin : nullptr);
            named_bar_sync(2, 32 * kNW);
            STEP_MARK(20);  // the token slice is staged
            // warps 0-3 take the weight-ring items (ring item i on warp i % 4:
            // every fill of a slot is consumed by one warp, in order, so a
            // parity wait never sees an older phase), warps 4-7 the parked ones
            auto emit = [&](int k, const float (&facc)[MT][2][4]) {
                const int tile = plo + k;
                unsigned long long* P = a.Pt + static_cast<size_t>(ps) * pstride;
                const unsigned tag = p1base + static_cast<unsigned>(l) + 1u;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int n = tile * 16 + g8 + ((i & 2) ? 8 : 0);
                            const int m = mt * 16 + hh * 8 + 2 * t4 + (i & 1);
                            if (m < a.B) st_tagged(P + static_cast<size_t>(m) * a.Nrows + n, facc[mt][hh][i], tag);
                        }
            };
            if (warp < kNA) {
                for (int i = warp; i < nA1; i += kNA) {
                    const int k = i < kNA ? i : i + nBH;
                    const unsigned ia = abase + static_cast<unsigned>(i);
                    const int slot = static_cast<int>(ia % kNA);
                    float facc[MT][2][4];
                    mbar_wait(&fullA[slot], (ia / kNA) & 1u);
                    item_mma<MT>(smem_u32(ringA + slot * kItem), smem_u32(xbuf), lane, facc);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&emptyA[slot]);
                    emit(k, facc);
                }
                STEP_MARK(21);  // the weight-ring items are done
            } else {
                for (int b = warp - kNA; b < nBH; b += kNW - kNA) {
                    float facc[MT][2][4];
                    mbar_wait(&wfull[b], lp);
                    item_mma<MT>(smem_u32(parked(b)), smem_u32(xbuf), lane, facc);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wdone[b / 2]);
                    emit(kNA + b, facc);
                }
                STEP_MARK(22);  // the parked items are done
            }
        }
        int nseg = 0, pos = 0;
        long long* cut = cut_of(l);
        const SegInfo* sinf = sinf_of(l);
        named_bar_sync(1, kSync);
        STEP_MARK(2);  // every projection warp of this CTA is done
        // (the projection partials carry their layer step's tag: readers
        // validate each word -- no grid barrier between the projection and
        // the attention)
        if (ab_g1 == 1) grid_sync(a.bar, (++gen) * static_cast<unsigned>(G));  // (A/B: the old grid barrier 1)
        if (tid == 0 && ab_g1 != 0 && nWS > 0) mbar_arrive(b1bar);
        STEP_MARK(3);
        if (warp < kNW || warp == kHelp) {
            while (*tbuilt < l + 1) {  // (built before P1 ended: passes at once)
            }
            __threadfence_block();
            nseg = meta_of(l)[1];
            pos = meta_of(l)[0];
        }
        const int swap01 = meta_of(l)[2];
        auto seg_of = [&](int p) { return seg_index(p, nseg, rev, swap01); };
        const size_t cap = static_cast<size_t>(Ly.cap);

        if (warp == kHelp) {
            // ============================================================ helper warp
            // (a) per segment, in processing order, ahead of the consumers:
            //     qt = (sum_split c_Q) . M_QK (the append epilogue's order: fixed
            //     split order, sequential fma); the segment that ends a region also
            //     gets the step's own K / V latents (summed the same way, rounded to
            //     the cache's bf16 -- the row the reference appends before
            //     attending, decode.cpp:143-149), written to cache row pos
            const unsigned p1t = p1base + static_cast<unsigned>(l) + 1u;  // this layer step's tag
            auto prep = [&](int p) {
                const int j = seg_of(p);
                const SegInfo& s = sinf[j];
                const int b = s.bh / a.nh, h = s.bh - b * a.nh;
                const bool own = s.t1 == pos;
                // M_QK's column (independent of the projection: in flight with the
                // partials' loads)
                float mqv[R];
                const float* mq = Ly.mqk + static_cast<size_t>(h) * R * R + lane;
#pragma unroll
                for (int jj = 0; jj < R; ++jj) mqv[jj] = __ldg(mq + jj * R);
                // every K split's partial of head h's rows, each word validated by
                // its tag (written by this layer step: re-read the stale ones)
                const unsigned long long* pb = a.Pt + static_cast<size_t>(b) * a.Nrows + static_cast<size_t>(h) * 3 * R + lane;
                const unsigned long long fresh = static_cast<unsigned long long>(p1t) << 32;  // a +0.0 of this step
                constexpr int SB = kMaxSplits / 2;  // splits per batch (8: E <= 4096 needs one)
                float v[3] = {0.f, 0.f, 0.f};
                for (int s0 = 0; s0 < splits; s0 += SB) {
                    unsigned long long w[3][SB];
#pragma unroll
                    for (int q = 0; q < SB; ++q)
#pragma unroll
                        for (int r = 0; r < 3; ++r)
                            w[r][q] = (s0 + q < splits && (r == 0 || own)) ? ld_tagged(pb + (s0 + q) * pstride + r * R)
                                                                         : fresh;
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int q = 0; q < SB; ++q)
#pragma unroll
                            for (int r = 0; r < 3; ++r) ok = ok && static_cast<unsigned>(w[r][q] >> 32) == p1t;
                        if (__all_sync(0xffffffffu, ok)) break;
                        __nanosleep(32);
#pragma unroll
                        for (int q = 0; q < SB; ++q)
#pragma unroll
                            for (int r = 0; r < 3; ++r)
                                if (static_cast<unsigned>(w[r][q] >> 32) != p1t) w[r][q] = ld_tagged(pb + (s0 + q) * pstride + r * R);
                    }
#pragma unroll
                    for (int q = 0; q < SB; ++q)
#pragma unroll
                        for (int r = 0; r < 3; ++r)  // +0.0 past `splits` leaves the sum exact
                            v[r] += __uint_as_float(static_cast<unsigned>(w[r][q]));
                }
                if (p == 0) {
                    // the cache stream into the stages that held parked items starts
                    // once the first segment's partials are complete: its burst then
                    // does not queue ahead of the projection loads of CTAs still in P1
                    if (ab_g1 == 0 && nWS > 0 && lane == 0) mbar_arrive(b1bar);  // (waited only with parked stages)
                    if (trc && l == a.trace_layer && lane == 0) trc[cta * kTr + 24] = gtimer();
                }
                float qt = 0.f;
#pragma unroll
                for (int jj = 0; jj < R; ++jj) qt = fmaf(__shfl_sync(0xffffffffu, v[0], jj), mqv[jj], qt);
                qts[j * R + lane] = qt;
                if (own) {
                    uint8_t* region = Ly.cache + static_cast<size_t>(s.bh) * cap * C::ROWB;
                    const uint32_t grow = static_cast<uint32_t>(pos) * C::ROWB;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const __nv_bfloat16 bv = __float2bfloat16_rn(v[1 + half]);
                        nrow[j * 2 * R + half * R + lane] = bv;
                        *reinterpret_cast<__nv_bfloat16*>(region + cache_swz(grow + half * C::PART + 2 * lane)) = bv;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&uready[j]);
            };
            if (nseg > 0) prep(0);
            else if (ab_g1 == 0 && nWS > 0 && lane == 0) mbar_arrive(b1bar);
            if (trc && l == a.trace_layer && lane == 0) trc[cta * kTr + 16] = gtimer();
            for (int p = 1; p < nseg; ++p) prep(p);
            if (nseg > 0) STEP_MARK(4);
            // the next layer's table into the other buffer, while this layer's
            // attention streams (its readers use this layer's buffer)
            if (l + 1 < nL) build_table(l + 1);
            if (l > 0 && !ab_g3 && kcl == 2 && (cta & 1)) {
                // this CTA writes into its even partner's shared memory below
                // (the merge area): the partner is past layer l - 1's O-projection
                // (no grid barrier orders the two; in practice long since)
                if (lane == 0)
                    while (static_cast<int>(ld_acquire(a.yflag + 32 * (cta - 1)) - (p1base + static_cast<unsigned>(l))) < 0)
                        __nanosleep(64);
                __syncwarp();
            }
            // (b) per segment as the consumers finish it: merge the kNW warp states
            //     in warp order (+ the own token for a region's last segment).  A
            //     region held by one CTA is complete.  A region shared by the two
            //     CTAs of a cluster pair: the odd CTA's (later) part crosses into the
            //     even CTA through distributed shared memory and the even CTA
            //     merges.  Any other shared region: every part publishes its state
            //     to L2 and the last to arrive merges them all in range order
            //     (SoftmaxState::merge, decode.cpp:59-75) -- nobody waits.
            for (int p = 0; p < nseg; ++p) {
                const int j = seg_of(p);
                mbar_wait(&sfull[j], (spar >> j) & 1u);
                spar ^= 1u << j;
                if (p == 0) STEP_MARK(15);
                const SegInfo& s = sinf[j];
                const float* rb = wst + j * kNW * (R + 2);
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < kNW; ++w) M = fmaxf(M, rb[w * (R + 2) + R]);
                float Ls = 0.f, av = 0.f;
#pragma unroll
                for (int w = 0; w < kNW; ++w) {
                    const float mw = rb[w * (R + 2) + R];
                    if (mw == -INFINITY) continue;
                    const float f = ex2(mw - M);
                    Ls = fmaf(rb[w * (R + 2) + R + 1], f, Ls);
                    av = fmaf(rb[w * (R + 2) + lane], f, av);
                }
                if (s.t1 == pos) {
                    // SoftmaxState::observe of the own token (decode.cpp:35-57)
                    const float kf = __bfloat162float(nrow[j * 2 * R + lane]);
                    const float vf = __bfloat162float(nrow[j * 2 * R + R + lane]);
                    const float sn = warp_sum(qts[j * R + lane] * kf);
                    const float Mn = fmaxf(M, sn);
                    const float fo = ex2(M - Mn), fn = ex2(sn - Mn);  // fo = 0 when M = -inf
                    Ls = fmaf(Ls, fo, fn);
                    av = fmaf(av, fo, vf * fn);
                    M = Mn;
                }
                const int c0 = s.c0, c1 = s.c1, owners = s.owners;
                const bool pair = kcl == 2 && owners == 2 && c1 - c0 == 2 && (c0 & 1) == 0;
                float L2 = Ls, a2 = av;
                if (pair && cta == c0 + 1) {
                    // the later part of the pair's shared region -> the even CTA
                    const uint32_t dst = cluster_map(smem_u32(pst), 0u);
                    st_cluster_f32(dst + 4u * lane, av);
                    if (lane == 0) {
                        st_cluster_f32(dst + 4u * R, M);
                        st_cluster_f32(dst + 4u * (R + 1), Ls);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(cluster_map(smem_u32(pbar), 0u));
                    continue;
                }
                if (pair) {
                    // this CTA holds the earlier part: it first, the partner's next
                    mbar_wait_cluster(pbar, pcnt & 1u);
                    ++pcnt;
                    const float mc = pst[R], lc = pst[R + 1], ac = pst[lane];
                    if (mc != -INFINITY) {
                        const float Mn = fmaxf(M, mc);
                        const float fo = ex2(M - Mn), fc = ex2(mc - Mn);
                        L2 = fmaf(lc, fc, Ls * fo);
                        a2 = fmaf(ac, fc, av * fo);
                    }
                } else if (owners > 1) {
                    float* wsp = a.ws + (static_cast<size_t>(cta) * kMaxU + j) * kWS;
                    wsp[lane] = av;
                    if (lane == 0) {
                        wsp[R] = M;
                        wsp[R + 1] = Ls;
                    }
                    __syncwarp();
                    unsigned old = 0;
                    if (lane == 0) old = atom_add_acq_rel(reinterpret_cast<unsigned*>(Ly.counters) + s.bh);
                    old = __shfl_sync(0xffffffffu, old, 0);
                    if (old != static_cast<unsigned>(owners - 1)) continue;  // another part merges
                    // ---- last arriver: every part of region bh in range order
                    float M2 = -INFINITY;
                    L2 = 0.f;
                    a2 = 0.f;
                    for (int c = c0; c < c1; ++c) {
                        if (!(cut[c] < cut[c + 1])) continue;
                        const int jc = static_cast<int>(static_cast<long long>(s.bh) - cut[c] / pos);
                        const float* wb = a.ws + (static_cast<size_t>(c) * kMaxU + jc) * kWS;
                        const float mc = __ldcg(wb + R), lc = __ldcg(wb + R + 1), ac = __ldcg(wb + lane);
                        if (mc == -INFINITY) continue;
                        const float Mn = fmaxf(M2, mc);
                        const float fo = ex2(M2 - Mn), fc = ex2(mc - Mn);  // fo = 0 while M2 = -inf
                        L2 = fmaf(lc, fc, L2 * fo);
                        a2 = fmaf(ac, fc, a2 * fo);
                        M2 = Mn;
                    }
                    if (lane == 0) Ly.counters[s.bh] = 0;  // self-resetting for the next step
                }
                // latent output -> X rows of the O-projection, K index h*R + lane:
                // hi = bf16(v) in row b, lo = bf16(v - hi) in row MT*16 + b (~16
                // mantissa bits of the fp32 latent reach the tensor cores)
                const int b = s.bh / a.nh, h = s.bh - b * a.nh;
                const int k = h * R + lane, sx = k / kKS, kk = k - sx * kKS;
                const float vo = a2 / L2;
                const __nv_bfloat16 vh = __float2bfloat16_rn(vo);
                const __nv_bfloat16 vl = __float2bfloat16_rn(vo - __bfloat162float(vh));
                uint8_t* xs = xo_l + static_cast<size_t>(sx) * C::XB2;
                const uint32_t eb = static_cast<uint32_t>((kk & 7) * 2);
                *reinterpret_cast<__nv_bfloat16*>(xs + xrow_off(b, kk >> 3) + eb) = vh;
                *reinterpret_cast<__nv_bfloat16*>(xs + xrow_off(MT * 16 + b, kk >> 3) + eb) = vl;
            }
            STEP_MARK(6);
        } else {
            // ========================================================= consumer warps
            if (g3.ysplit && !g3.pairy) {
                // y collects the two K splits' partial sums (P3): zero this CTA's
                // share now -- after barrier 1, so a y that aliases x is not
                // touched before x is consumed
                const size_t ny = static_cast<size_t>(a.B) * a.e_out;
                const size_t y0 = ny * cta / G, y1 = ny * (cta + 1) / G;
                for (size_t i = y0 + tid; i < y1; i += 32 * kNW) Ly.y[i] = 0.f;
            }
            // ---- P2: attention over this CTA's segments, in processing order
            int slot = 0;
            constexpr int KR = R / 16;
            for (int p = 0; p < nseg; ++p) {
                const int j = seg_of(p);
                const SegInfo& s = sinf[j];
                const int ntok = s.t1 - s.t0;
                const int ns = (ntok + kST - 1) / kST;
                mbar_wait(&uready[j], (upar >> j) & 1u);
                upar ^= 1u << j;
                if (p == 0) {
                    STEP_MARK(13);
                    if (trc && l == a.trace_layer && lane == 0 && (warp == 0 || warp == kNW - 1))
                        trc[cta * kTr + (warp == 0 ? 17 : 18)] = gtimer();
                }
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

                for (int st = 0; st < ns; ++st) {
                    mbar_wait(&fullB[slot], (parc >> slot) & 1u);
                    parc ^= 1u << slot;
                    if (trc && l == a.trace_layer && p == 0 && st == 0 && warp == 0 && lane == 0)
                        trc[cta * kTr + 19] = gtimer();
                    const uint32_t sbase = smem_u32(ringB + slot * C::STAGE);
                    const int rows = min(kST, ntok - st * kST);
                    if (warp * 32 < rows) {
                        // scores D(16 tok x 8) = K(16 x R) . [qt_hi | qt_lo]: lane (g8, t4 = 0)
                        // holds the hi / lo partials of tokens g8 and g8 + 8
                        float sc[2][2];
#pragma unroll
                        for (int grp = 0; grp < 2; ++grp) {
                            const int tb = warp * 32 + grp * 16;
                            float d[4] = {0.f, 0.f, 0.f, 0.f};
                            const int ltok = tb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
                            for (int kk = 0; kk < KR; ++kk) {
                                uint32_t a0, a1, a2, a3;
                                const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2 + (lane >> 4)) * 16);
                                ldsm_x4(sbase + cache_swz(off), a0, a1, a2, a3);
                                mma_bf16_16816(d, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
                            }
                            sc[grp][0] = (t4 == 0 && tb + g8 < rows) ? d[0] + d[1] : -INFINITY;
                            sc[grp][1] = (t4 == 0 && tb + g8 + 8 < rows) ? d[2] + d[3] : -INFINITY;
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
                            const int tb = warp * 32 + grp * 16;
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
                            const int stok = tb + (lane & 7) + ((lane >> 4) & 1) * 8;
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
                    if (++slot == C::NB) slot = 0;
                }
                // this warp's state of segment j -> the helper
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
                if (lane == 0) mbar_arrive(&sfull[j]);
            }
            STEP_MARK(5);
        }
        // G2: every (sequence, head) row is merged; every CTA has read the length
        // (trace: thread 0's arrival -> mark 25, its exit -> mark 7; a mark
        // taken after the barrier by every warp reads the timer early)
        grid_sync(a.bar, (++gen) * static_cast<unsigned>(G), (trc && l == a.trace_layer) ? trc + cta * kTr : nullptr);
        if (cta == 0 && tid == 0) *Ly.d_len = pos + 1;

        if (warp != kHelp) {
            // ---- P3: folded O-projection over the prefetched W'_o items.  The X
            // slices this CTA's items use (hi / lo bf16 rows built by the mergers)
            // land at the end of the attention ring -- all at once, or one K
            // split at a time when they do not fit together.  Item j = (tile j /
            // p3ns, split p3s0 + j % p3ns) runs on warps slot and slot + 4, one
            // half of its K range each, into part[half][j]; the halves and the
            // splits are summed in a fixed order.
            const P3G& g = g3;
            float* part = C::PART_IN_RED ? reinterpret_cast<float*>(smem + C::RED_OFF)
                                         : reinterpret_cast<float*>(ringB + g.p3lo);  // [2][kNA][16 rows][MT*16 tokens]
            uint8_t* xsl = ringB + g.xoff;
            const int half = warp / kNA, hslot = warp % kNA;
            const unsigned a3 = abase + static_cast<unsigned>(nA1);  // ring-A index of P3 item 0
            if (g.np3 > 0) {
                for (int s0 = 0; s0 < g.p3ns; s0 += g.per) {
                    if (ab_p3_tma) {
                        if (tid == 0) {
                            // xo was written by other CTAs' generic stores (ordered by the
                            // barrier); order them before this thread's async-proxy reads
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            mbar_arrive_expect_tx(p3bar, static_cast<uint32_t>(g.per * C::XB2));
                            for (int s = s0; s < s0 + g.per; ++s)
                                tma_bulk_g2s(xsl + (s - s0) * C::XB2, xo_l + static_cast<size_t>(g.p3s0 + s) * C::XB2,
                                             C::XB2, p3bar);
                        }
                        mbar_wait(p3bar, p3cnt & 1u);
                        ++p3cnt;
                    } else {
                        // plain 16-byte loads by every consumer thread, all in flight at once
                        constexpr int V = C::XB2 / 16;  // uint4 per split
                        constexpr int NV = (V + 32 * kNW - 1) / (32 * kNW);
                        for (int s = s0; s < s0 + g.per; ++s) {
                            const uint4* src = reinterpret_cast<const uint4*>(xo_l + static_cast<size_t>(g.p3s0 + s) * C::XB2);
                            uint4* dst = reinterpret_cast<uint4*>(xsl + (s - s0) * C::XB2);
                            uint4 v[NV];
#pragma unroll
                            for (int u = 0; u < NV; ++u) {
                                const int i = tid + u * 32 * kNW;
                                if (i < V) v[u] = __ldcg(src + i);
                            }
#pragma unroll
                            for (int u = 0; u < NV; ++u) {
                                const int i = tid + u * 32 * kNW;
                                if (i < V) dst[i] = v[u];
                            }
                        }
                        named_bar_sync(2, 32 * kNW);
                    }
                    if (s0 == 0) STEP_MARK(8);
                    for (int j = 0; j < g.np3; ++j) {
                        const unsigned ia = a3 + static_cast<unsigned>(j);
                        const int slot = static_cast<int>(ia % kNA), s = j % g.p3ns;
                        if (slot != hslot || s < s0 || s >= s0 + g.per) continue;
                        mbar_wait(&fullA[slot], (ia / kNA) & 1u);
                        if (trc && l == a.trace_layer && tid == 0 && j == 0) trc[cta * kTr + 12] = gtimer();
                        // token columns 0..MT*16-1 are the hi rows, MT*16.. the lo rows
                        float facc[2 * MT][2][4];
                        item_mma<2 * MT>(smem_u32(ringA + slot * kItem), smem_u32(xsl + (s - s0) * C::XB2), lane, facc,
                                         half * kKS / 64, (half + 1) * kKS / 64);
                        if (trc && l == a.trace_layer && tid == 0 && j == 0) trc[cta * kTr + 14] = gtimer();
                        float* pj3 = part + (half * kNA + j) * 16 * MT * 16;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int n = g8 + ((i & 2) ? 8 : 0);
                                    const int m = mt * 16 + hh * 8 + 2 * t4 + (i & 1);
                                    pj3[n * MT * 16 + m] = facc[mt][hh][i] + facc[mt + MT][hh][i];
                                }
                    }
                    if (trc && l == a.trace_layer && (tid & 31) == 0) trc[cta * kTr + 29 + (warp < 4 ? 0 : 1)] = gtimer();
                    named_bar_sync(2, 32 * kNW);  // the X buffer is free again / every partial is written
                }
                // the weight ring's P3 slots are free (both halves have run)
                if (tid < g.np3) mbar_arrive(&emptyA[(a3 + static_cast<unsigned>(tid)) % kNA]);
                if (trc && l == a.trace_layer && tid == 0) trc[cta * kTr + 31] = gtimer();
                // part[(half * kNA + j)] -> sum over halves, then splits
                auto psum = [&](int ti, int n, int m) {
                    float v = 0.f;
                    for (int s = 0; s < g.p3ns; ++s) {
                        const int j = ti * g.p3ns + s;
                        v += part[(j * 16 + n) * MT * 16 + m] + part[((kNA + j) * 16 + n) * MT * 16 + m];
                    }
                    return v;
                };
                // one K split per CTA (pairs): the same sum, straight-line
                auto psum1 = [&](int ti, int n, int m) {
                    return part[(ti * 16 + n) * MT * 16 + m] + part[((kNA + ti) * 16 + n) * MT * 16 + m];
                };
                if (g.pairy) {
                    // [tile][row m][16 columns] fp32 split-1 sums, in the even CTA's merge area
                    float* recv = reinterpret_cast<float*>(smem + C::RED_OFF + (C::PART_IN_RED ? C::PARTB : 0));
                    const int q4 = g.nt3 * a.B * 4;  // 4-column groups
                    if (cta & 1) {
                        // st.async: every 16 bytes complete transaction bytes on the even
                        // CTA's barrier (which expects q4 * 16) -- no release fence
                        const uint32_t dst = cluster_map(smem_u32(recv), 0u), rbar = cluster_map(smem_u32(ybar), 0u);
                        for (int i = tid; i < q4; i += 32 * kNW) {
                            const int ti = i / (a.B * 4), r = i - ti * a.B * 4;
                            const int m = r >> 2, n0 = (r & 3) * 4;
                            st_async_v4(dst + 4u * static_cast<uint32_t>((ti * a.B + m) * 16 + n0), psum1(ti, n0, m),
                                        psum1(ti, n0 + 1, m), psum1(ti, n0 + 2, m), psum1(ti, n0 + 3, m), rbar);
                        }
                        if (trc && l == a.trace_layer && tid == 0) trc[cta * kTr + 26] = gtimer();
                    } else {
                        // this CTA's split-0 sums: <= 4 groups per thread (B <= 32, nt3 <= 4),
                        // in registers (unrolled: a dynamic index would put them in local memory)
                        float own[4][4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = tid + u * 32 * kNW;
                            if (i >= q4) break;
                            const int ti = i / (a.B * 4), r = i - ti * a.B * 4;
                            const int m = r >> 2, n0 = (r & 3) * 4;
#pragma unroll
                            for (int e = 0; e < 4; ++e) own[u][e] = psum1(ti, n0 + e, m);
                        }
                        if (trc && l == a.trace_layer && tid == 0) trc[cta * kTr + 27] = gtimer();
                        if (tid == 0) mbar_arrive_expect_tx(ybar, static_cast<uint32_t>(q4) * 16u);
                        mbar_wait_cluster(ybar, ycnt & 1u);
                        if (trc && l == a.trace_layer && tid == 0) trc[cta * kTr + 26] = gtimer();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = tid + u * 32 * kNW;
                            if (i >= q4) break;
                            const int ti = i / (a.B * 4), r = i - ti * a.B * 4;
                            const int m = r >> 2, n0 = (r & 3) * 4;
                            const int col = (g.t3lo + ti) * 16 + n0;
                            const float4 o = *reinterpret_cast<const float4*>(recv + (ti * a.B + m) * 16 + n0);
                            float* yr = Ly.y + static_cast<size_t>(m) * a.e_out;
                            const float v0 = own[u][0] + o.x, v1 = own[u][1] + o.y;
                            const float v2 = own[u][2] + o.z, v3 = own[u][3] + o.w;
                            if (xt_out) {  // (e_out == E, a multiple of 512: whole groups)
                                unsigned long long* xd = a.xtag + static_cast<size_t>(l & 1) * a.B * (a.E / 2) +
                                                         static_cast<size_t>(m) * (a.E / 2) + col / 2;
                                const unsigned long long tg = static_cast<unsigned long long>(p1base + static_cast<unsigned>(l) + 1u) << 32;
                                const unsigned long long w0 = tg | pack_bf16x2(v0, v1), w1 = tg | pack_bf16x2(v2, v3);
                                asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(xd), "l"(w0), "l"(w1) : "memory");
                            }
                            if (col + 4 <= a.e_out && (a.e_out & 3) == 0) {
                                *reinterpret_cast<float4*>(yr + col) = make_float4(v0, v1, v2, v3);
                            } else {
                                const float v[4] = {v0, v1, v2, v3};
                                for (int e = 0; e < 4; ++e)
                                    if (col + e < a.e_out) yr[col + e] = v[e];
                            }
                        }
                    }
                    ++ycnt;
                } else if (!g.ycontig) {
                    for (int i = tid; i < g.nt3 * 16 * a.B; i += 32 * kNW) {
                        const int ti = i / (16 * a.B), r = i - ti * 16 * a.B;
                        const int m = r / 16, n = r - m * 16;  // n fastest: 64-byte row segments of y
                        const int col = (g.t3lo + ti * g.t3step) * 16 + n;
                        if (col >= a.e_out) continue;
                        float* yp = Ly.y + static_cast<size_t>(m) * a.e_out + col;
                        if (g.ysplit) atomicAdd(yp, psum(ti, n, m));  // red.add: one of exactly two addends onto 0
                        else *yp = psum(ti, n, m);
                    }
                } else {
                    const int q4 = g.nt3 * 4;  // 4-column groups of this CTA's row segment
                    for (int i = tid; i < a.B * q4; i += 32 * kNW) {
                        const int m = i / q4, q = i - m * q4;
                        const int ti = q >> 2, n0 = (q & 3) * 4;
                        const int col = (g.t3lo + ti) * 16 + n0;
                        float v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[e] = psum(ti, n0 + e, m);
                        float* yr = Ly.y + static_cast<size_t>(m) * a.e_out;
                        if (col + 4 <= a.e_out && (a.e_out & 3) == 0) {
                            *reinterpret_cast<float4*>(yr + col) = make_float4(v[0], v[1], v[2], v[3]);
                        } else {
                            for (int e = 0; e < 4; ++e)
                                if (col + e < a.e_out) yr[col + e] = v[e];
                        }
                    }
                }
            }
            STEP_MARK(9);
            // the attention ring and the merge area are free for the next layer's
            // parked items (their generic writes ordered before those TMA writes)
            fence_proxy_async_smem();
            named_bar_sync(2, 32 * kNW);
            if (tid == 0) {
                mbar_arrive(p3done);
                if (trc && l == a.trace_layer) trc[cta * kTr + 28] = gtimer();
                // this CTA's share of y is written (release; with tagged tokens the
                // helper releases it, off the next projection's path)
                if (!a.xtagged) red_release(a.yflag + 32 * cta);
            }
        } else if (a.xtagged) {
            mbar_wait(p3done, lp);  // (this CTA's O-projection is done)
            if (lane == 0) red_release(a.yflag + 32 * cta);
        }
        abase += static_cast<unsigned>(nA1 + g3.np3);
        if (l + 1 < nL && ab_g3) grid_sync(a.bar, (++gen) * static_cast<unsigned>(G));  // (A/B: the old grid barrier 3)
    }
    if (cta == 0 && tid == 0) {
        *a.epoch += 1;  // fused launches run (the x-fetch generations)
        *a.bgen = gen;  // this launch's barriers are all passed (every CTA read bgen before its first)
        *a.p1gen = p1base + static_cast<unsigned>(nL);  // (every CTA read it before the first G2)
    }
}

template <int MT>
cudaError_t launch_mt(const StepArgs& a, cudaStream_t s) {
    using C = SC<32, MT>;
    if constexpr (!C::OK) {
        return cudaErrorInvalidValue;
    } else {
        // the generic instantiation only for traces and non-default A/B switches
        const bool gen = a.trace || a.p3_tma != 0 || a.g3 != 0 || a.x_first != 1 || a.l2_next != 1 ||
                         a.chain_pre != 4 || a.pre_stages != 0 || a.short_seg != 2048 || a.cluster != 2 ||
                         a.oKp / kKS != 2 || a.g1 != 0;
        auto k = gen ? layer_step_kernel<32, MT, true> : layer_step_kernel<32, MT, false>;
        static bool attr[2] = {false, false};
        if (!attr[gen ? 1 : 0]) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e != cudaSuccess) return e;
            attr[gen ? 1 : 0] = true;
        }
        // the counts and the barrier need every CTA resident: one CTA per SM
        // fits (the host checks occupancy once and serialises fused steps of
        // different streams, capi.cu fused_serialize).  A cooperative launch
        // would guarantee it in hardware but costs ~3.5 us per step on B200
        // (profiles/r02_coop.txt); WSVD_STEP_COOP=1 selects it.
        static const bool coop = std::getenv("WSVD_STEP_COOP") != nullptr;
        if (coop) return launch_coop_cluster(k, dim3(a.grid), dim3(kThr), C::SMEM, s, a.cluster, a);
        return launch_pdl_cluster(k, dim3(a.grid), dim3(kThr), C::SMEM, s, a.cluster, a);
    }
}

}  // namespace

bool step_supported(int R, int B, int nh, int Kp, int oKp, int otiles, int grid) {
    if (R != 32 || B < 1 || B > 32 || nh < 1) return false;
    if (grid > kMaxG || grid < 1) return false;
    if (Kp % kKS != 0 || oKp % kKS != 0) return false;
    const int splits = Kp / kKS, osplits = oKp / kKS;
    if (osplits > 2 || splits > grid || splits > kMaxSplits) return false;
    // segments per CTA: at most ceil(B*nh / grid) + 1
    if ((B * nh + grid - 1) / grid + 1 > kMaxU) return false;
    if (((otiles + grid - 1) / grid) * osplits > kNA) return false;       // host y: whole tiles per CTA
    if (osplits == 2 && (otiles + grid / 2 - 1) / (grid / 2) > kNA) return false;  // device y: one split per CTA
    // P3 stages its X slices (at least one K split's hi / lo rows) and the
    // partial tiles in the attention ring
    const int mt = (B + 15) / 16;
    const int ring = (mt == 1 ? SC<32, 1>::NB * SC<32, 1>::STAGE : SC<32, 2>::NB * SC<32, 2>::STAGE);
    return 2 * mt * 16 * kXS + 2 * kNA * 16 * mt * 16 * 4 <= ring;
}

int step_item_k() { return kKS; }

size_t step_xo_bytes(int B, int oKp) { return static_cast<size_t>(oKp / kKS) * 2 * ((B + 15) / 16) * 16 * kXS; }

size_t step_ws_bytes(int grid) { return static_cast<size_t>(grid) * kMaxU * kWS * 4; }

int step_max_units() { return kMaxU; }

int step_ring_stages(int B) { return (B + 15) / 16 == 1 ? SC<32, 1>::NB : SC<32, 2>::NB; }

int step_resident_ctas_per_sm(int B) {
    int n = 0;
    auto probe = [&](auto k, int smem) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kThr, smem) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
    };
    if ((B + 15) / 16 == 1) probe(layer_step_kernel<32, 1, false>, SC<32, 1>::SMEM);
    else probe(layer_step_kernel<32, 2, false>, SC<32, 2>::SMEM);
    return n;
}

template <int MT>
int pair_ok(int grid) {
    using C = SC<32, MT>;
    auto k = layer_step_kernel<32, MT, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return 2 * n >= grid ? 1 : 0;
}

int step_pair_clusters_ok(int B, int grid) {
    if (grid % 2 != 0) return 0;
    return (B + 15) / 16 == 1 ? pair_ok<1>(grid) : pair_ok<2>(grid);
}

cudaError_t launch_layer_step(const StepArgs& a, cudaStream_t s) {
    switch ((a.B + 15) / 16) {
        case 1: return launch_mt<1>(a, s);
        case 2: return launch_mt<2>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace wsvd_k
