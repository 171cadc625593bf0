// step.cu -- the whole decode-layer step as ONE persistent kernel (bf16 weights,
// bf16 latent cache, rank 32).
//
// pipe::decode_factored's per-layer body (reference src/pipeline.cpp:320-329)
// is append_token (decode.cpp:127-153) -> fused_decode_step (decode.cpp:155-206)
// -> heads_row . W_o.  The multi-kernel path (capi.cu layer_step_impl) runs it
// as projection GEMM -> append epilogue -> attention -> combine -> O-projection:
// five launches, each with its own ramp-up and tail, and HBM idle across every
// kernel boundary.  This kernel runs the same arithmetic with one CTA per SM
// and two grid-wide barriers:
//
//   P1  latent projection  P[split][b][n] = x_b . A_all[:, n] over one K split
//       (swap-AB mma.sync over W-tiles streamed by TMA, as gemm.cu), on all
//       eight consumer warps;
//   --  grid barrier 1 (all projection partials written)
//   P2  attention units (sequence, head, chunk) exactly as attn.cu's
//       tensor-core consumer; the helper warp derives each unit's absorbed
//       query from the partials (qt = (sum_split c_Q) . M_QK, the append
//       epilogue's fold), writes the new token's latent row into the cache
//       for the unit holding it (patched into the shared-memory stage), merges
//       each unit's 8 warp states (fixed order) and, for the last chunk of a
//       (sequence, head), merges the chunks in chunk order
//       (SoftmaxState::merge, decode.cpp:59-75) into the bf16 rows of the
//       O-projection input -- through distributed shared memory when the grid
//       runs as 2-CTA clusters (two chunks per pair), else through L2;
//   --  grid barrier 2 (every row complete; the cache length is committed)
//   P3  folded O-projection y = vlat . (B_V . W_o) over W-tiles prefetched
//       into shared memory during P2; each CTA owns whole output tiles and
//       sums their K splits itself -- no atomics, run-to-run deterministic.
//
// One producer warp issues every projection item of the CTA before the
// grid-dependency wait (a 4-slot weight ring plus items parked in the
// attention ring), then the O-projection weights and, once barrier 1 has
// passed, the cache stream.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kNW = 8;               // consumer warps
constexpr int kThr = 32 * kNW + 64;  // + one producer warp + one helper warp
constexpr int kSync = 32 * kNW + 32; // threads in the grid barrier (consumers + helper)
constexpr int kST = 256;             // tokens per attention stage
constexpr int kKS = 512;             // K per weight work item
constexpr int kItem = 16 * kKS * 2;  // one weight work item: 16 rows x 512 bf16 = 16 KB
constexpr int kNA = 4;               // weight ring slots == projection consumer warps
constexpr int kXS = kKS * 2 + 64;    // bytes per staged token row (stride == 64 mod 128)
constexpr int kMaxU = 8;             // attention units per CTA (host-checked)
constexpr int kMaxSplits = 16;       // projection K splits (host-checked)
constexpr int kWS = 36;              // floats per unit state in ws: acc[32], m, l, pad (16 B rows)

template <int R, int MT>
struct SC {
    static constexpr int ROWB = 4 * R;  // bf16 [C_K | C_V]
    static constexpr int PART = 2 * R;
    static constexpr int STAGE = kST * ROWB;
    static constexpr int XB = MT * 16 * kXS;               // one staged X slice
    static constexpr int XB2 = 2 * XB;                     // an O-projection X slice: hi rows, then lo rows
    // per-unit scratch: absorbed queries, the new token's row, the warp states
    // + [kMaxU][R+2] chunk states a cluster peer writes through DSMEM
    static constexpr int RED = kMaxU * (R * 4 + 4 * R + kNW * (R + 2) * 4 + (R + 2) * 4);
    static constexpr int FIXED = kNA * kItem + XB + RED + 768;
    static constexpr int NB_RAW = (225 * 1024 - FIXED) / STAGE;
    static constexpr int NB = NB_RAW > 6 ? 6 : NB_RAW;
    static constexpr int B_OFF = kNA * kItem;
    static constexpr int X_OFF = B_OFF + NB * STAGE;
    static constexpr int RED_OFF = X_OFF + XB;
    static constexpr int BAR_OFF = RED_OFF + RED;
    static constexpr int SMEM = BAR_OFF + 512;
    static constexpr bool OK = NB_RAW >= 2;
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
#define STEP_MARK(k) \
    do { if (a.trace && tid == 0) a.trace[cta * 12 + (k)] = gtimer(); } while (0)

WSVD_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier among the consumer and helper warps of every CTA (all
// CTAs are resident: one per SM).  bar[0] is a monotone arrival count: the
// k-th barrier of the n-th fused step completes when it reaches
// (2n + k) * gridDim.x.  Arrival is a fire-and-forget release reduction and
// everyone polls with acquire loads -- one round trip, 1.2 us on B200
// against 2.0 us for a count-and-release barrier (tools/micro_barrier.cu).
WSVD_DEV void grid_sync(unsigned* bar, unsigned target) {
    named_bar_sync(1, kSync);
    if (threadIdx.x == 0) {
        // release: the CTA's writes (ordered before by bar.sync) become visible
        // to every CTA that acquires the count
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire(bar) < target) {
        }
    }
    named_bar_sync(1, kSync);
}

// split-KV geometry, identical to attn.cu chunking()
WSVD_DEV void step_chunking(const StepArgs& a, int len, int& nch, int& chunk) {
    if (a.chunk > 0) {
        chunk = a.chunk;
    } else {
        const int n = max(1, min(a.max_chunks, (len + 31) / 32));
        chunk = (((len + n - 1) / n) + 31) & ~31;
    }
    nch = (len + chunk - 1) / chunk;
}

// fp32 X[rows][ldx] columns [k0, k0 + kKS) -> bf16 smem [MT*16][kXS], zero padded
template <int MT>
WSVD_DEV void stage_rows(const float* X, int rows, int ldx, int kvalid, int k0, uint8_t* xs, int ctid) {
    constexpr int PER = kKS / 8;  // 8-element items per row
    for (int i = ctid; i < MT * 16 * PER; i += 32 * kNW) {
        const int m = i / PER, kk = (i - m * PER) * 8;
        const int k = k0 + kk;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.f;
        if (m < rows) {
            const float* src = X + static_cast<size_t>(m) * ldx + k;
            if (k + 8 <= kvalid && (ldx % 4) == 0) {
                const float4 p0 = __ldcg(reinterpret_cast<const float4*>(src));
                const float4 p1 = __ldcg(reinterpret_cast<const float4*>(src + 4));
                v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
                v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = (k + j < kvalid) ? __ldcg(src + j) : 0.f;
            }
        }
        uint4 o;
        o.x = pack_bf16x2(v[0], v[1]); o.y = pack_bf16x2(v[2], v[3]);
        o.z = pack_bf16x2(v[4], v[5]); o.w = pack_bf16x2(v[6], v[7]);
        *reinterpret_cast<uint4*>(xs + m * kXS + kk * 2) = o;
    }
}

// One weight work item (16 W-rows x kKS, W-tile layout of gemm.cu) against the
// staged tokens: D fragments facc[mt][hh][i] = (row g | g+8, token 2t | 2t+1).
template <int MT>
WSVD_DEV void item_mma(uint32_t slot_addr, uint32_t xs_addr, int lane, float (&facc)[MT][2][4]) {
    const int g = lane >> 2, t = lane & 3;
    const uint32_t swz = static_cast<uint32_t>((g & 1) << 2);
    const uint32_t row_lo = slot_addr + static_cast<uint32_t>(g * kKS * 2);
    const uint32_t row_hi = row_lo + static_cast<uint32_t>(8 * kKS * 2);
    const uint32_t xbase = xs_addr + static_cast<uint32_t>(g * kXS + t * 16);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int i = 0; i < 4; ++i) facc[mt][hh][i] = 0.f;
#pragma unroll 4
    for (int b = 0; b < kKS / 32; ++b) {
        const uint32_t uoff = ((static_cast<uint32_t>(4 * b + t)) ^ swz) * 16;
        const uint4 wl = lds128(row_lo + uoff);
        const uint4 wh = lds128(row_hi + uoff);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const uint4 xv = lds128(xbase + static_cast<uint32_t>((mt * 16 + hh * 8) * kXS + b * 64));
                mma_bf16_16816(facc[mt][hh], wl.x, wh.x, wl.y, wh.y, xv.x, xv.y);
                mma_bf16_16816(facc[mt][hh], wl.z, wh.z, wl.w, wh.w, xv.z, xv.w);
            }
    }
}

template <int R, int MT>
__global__ void __launch_bounds__(kThr, 1) layer_step_kernel(const StepArgs a) {
    static_assert(R == 32, "the fused step is specialised for rank 32 (one latent dim per lane)");
    using C = SC<R, MT>;
    constexpr int KR = R / 16;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ringA = smem;
    uint8_t* ringB = smem + C::B_OFF;
    uint8_t* xbuf = smem + C::X_OFF;
    float* qts = reinterpret_cast<float*>(smem + C::RED_OFF);                // [kMaxU][R]
    __nv_bfloat16* nrow = reinterpret_cast<__nv_bfloat16*>(qts + kMaxU * R);  // [kMaxU][2R]
    float* wst = qts + 2 * kMaxU * R;                                         // [kMaxU][kNW][R+2]
    float* pst = wst + kMaxU * kNW * (R + 2);                                 // [kMaxU][R+2] peer chunk states
    uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* emptyA = fullA + kNA;
    uint64_t* fullB = emptyA + kNA;
    uint64_t* emptyB = fullB + C::NB;
    uint64_t* uready = emptyB + C::NB;  // [kMaxU] unit j's query / new row prepared (helper)
    uint64_t* sfull = uready + kMaxU;   // [kMaxU] unit j's warp states written (consumers)
    uint64_t* p3bar = sfull + kMaxU;    // P3: chunk states landed (one phase per staged split)
    uint64_t* wfull = p3bar + 1;        // [2*NB] projection items parked in the attention ring
    uint64_t* wdone = wfull + 2 * C::NB;  // [NB] those items consumed: the stage is free
    uint64_t* pbar = wdone + C::NB;       // [kMaxU] unit j's peer chunk state landed (CTA pairs)
    uint64_t* b1bar = pbar + kMaxU;       // grid barrier 1 passed (gates the parked stages' refill)
    static_assert((2 * kNA + 2 * C::NB + 2 * kMaxU + 1 + 2 * C::NB + C::NB + kMaxU + 1) * 8 <= C::SMEM - C::BAR_OFF,
                  "mbarriers overflow their shared-memory region");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;

    STEP_MARK(0);
    if (a.trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[cta * 12 + 10] = smid;
    }
    const int splits = a.Kp / kKS;
    const int cps = G / splits;  // CTAs per projection split
    const int ps = cta % splits, pj = cta / splits;
    const int ptiles = a.Nrows / 16;
    const int plo = pj < cps ? static_cast<int>(static_cast<long>(pj) * ptiles / cps) : 0;
    const int phi = pj < cps ? static_cast<int>(static_cast<long>(pj + 1) * ptiles / cps) : 0;
    const int np1 = phi - plo;
    const int osplits = a.oKp / kKS;
    // P3: this CTA owns output tiles with all their K splits (items (tile,
    // split) in that order), so it sums the splits itself and y is written
    // once with plain stores.  Device y: tiles cta + i*G.  Host y (mapped
    // pinned memory, the host-buffer step): a contiguous run of tiles, written
    // as 16-byte stores over 64-128-byte row segments -- bus writes drain
    // faster (e2e 90.5 -> 88.4 us), device-resident y a little slower.
    const bool ycontig = a.x_host != 0;
    const int t3lo = ycontig ? static_cast<int>(static_cast<long>(cta) * a.otiles / G) : cta;
    const int nt3 = ycontig ? static_cast<int>(static_cast<long>(cta + 1) * a.otiles / G) - t3lo
                            : (cta < a.otiles ? (a.otiles - 1 - cta) / G + 1 : 0);
    const int t3step = ycontig ? 1 : G;  // tile i of this CTA: t3lo + i * t3step
    const int np3 = nt3 * osplits;  // <= kNA (host-checked)
    // Projection items beyond the 4-slot weight ring are parked in the
    // attention ring (2 per stage, in consumption order): the attention cannot
    // start before grid barrier 1 anyway, and with every item in flight at
    // once P1 costs one memory round trip instead of one per ring turn.
    // Ring-A sequence: P1 items k < 4 or k >= 4 + nBH, then the P3 items.
    const int nBH = min(max(np1 - kNA, 0), 2 * C::NB);
    const int nA1 = np1 - nBH;
    const int nWS = (nBH + 1) / 2;  // attention stages holding parked items (the first nWS)
    // Rows past a stage's valid end are read by the MMAs (times p = 0) and must
    // be finite: every slot's first attention stage is copied whole (the cache
    // allocation has a stage of padding), so later partial stages leave finite
    // stale rows -- no zeroing of the ring in the prologue
    if (warp == 0) {
        // the ~50 barrier inits spread over warp 0's lanes (serially they cost
        // ~0.5 us in front of the first weight TMA)
        if (lane < kNA) {
            mbar_init(&fullA[lane], 1);
            mbar_init(&emptyA[lane], 1);
        }
        if (lane < C::NB) {
            mbar_init(&fullB[lane], 1);
            mbar_init(&emptyB[lane], kNW);
            // stage `lane` parks items 4 + 2 lane and 4 + 2 lane + 1
            mbar_init(&wdone[lane], lane < nWS ? min(2, nBH - 2 * lane) : 1);
        }
        if (lane < kMaxU) {
            mbar_init(&uready[lane], 1);
            mbar_init(&sfull[lane], kNW);
            mbar_init(&pbar[lane], 1);
        }
        if (lane < nBH) mbar_init(&wfull[lane], 1);
        if (lane == 0) {
            mbar_init(p3bar, 1);
            mbar_init(b1bar, 1);
        }
        fence_mbar_init();  // every lane: the fence covers the executing thread's inits
    }
    __syncthreads();
    if (a.cluster > 1) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
    // The weights (projection W-tiles, then the folded O-projection) are
    // constant across steps: the producer starts streaming them before the
    // predecessor has drained (programmatic dependent launch), only the token,
    // the length and the cache rows wait for it
    // ring-A item ia -> source (P1 item k(ia), then the P3 items)
    auto a_src = [&](int ia) -> const uint8_t* {
        if (ia < nA1) {
            const int k = ia < kNA ? ia : ia + nBH;
            return a.A + (static_cast<size_t>(plo + k) * splits + ps) * kItem;
        }
        const int j = ia - nA1;
        return a.Wo + (static_cast<size_t>(t3lo + (j / osplits) * t3step) * osplits + j % osplits) * kItem;
    };
    auto parked = [&](int b) -> uint8_t* {  // parked item b (P1 item 4 + b)
        return ringB + (b / 2) * C::STAGE + (b & 1) * kItem;
    };
    int ia_pre = 0;
    if (warp == kNW && lane == 0) {
        for (; ia_pre < kNA && ia_pre < nA1 + np3; ++ia_pre) {
            mbar_arrive_expect_tx(&fullA[ia_pre], kItem);
            tma_bulk_g2s(ringA + ia_pre * kItem, a_src(ia_pre), kItem, &fullA[ia_pre]);
        }
        for (int b = 0; b < nBH; ++b) {
            mbar_arrive_expect_tx(&wfull[b], kItem);
            tma_bulk_g2s(parked(b), a.A + (static_cast<size_t>(plo + kNA + b) * splits + ps) * kItem, kItem,
                         &wfull[b]);
        }
    }
    griddep_wait();
    griddep_launch_dependents();
    STEP_MARK(1);

    const int pos = *a.d_len;  // the new token's row; attention covers pos + 1 rows
    const unsigned epoch = static_cast<unsigned>(*a.epoch);  // fused steps so far (barrier generations)
    const int len = pos + 1;
    int nch, chunk;
    step_chunking(a, len, nch, chunk);
    const int n_units = a.B * a.nh * nch;
    const int nu = cta < n_units ? (n_units - 1 - cta) / G + 1 : 0;  // this CTA's units u = cta + j*G
    if (a.trace && tid == 0) a.trace[cta * 12 + 11] = static_cast<uint64_t>(nu);
    const size_t cap = static_cast<size_t>(a.cap);
    const size_t pstride = static_cast<size_t>(a.B) * a.Nrows;

    // ================================================================ producer
    if (warp == kNW) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int ia = ia_pre;  // the first weight items went out before griddep_wait
            const int na = nA1 + np3;
            auto issue_a = [&]() {
                const int slot = ia % kNA;
                const uint32_t ph = static_cast<uint32_t>(ia / kNA) & 1u;
                mbar_wait(&emptyA[slot], ph ^ 1u);
                mbar_arrive_expect_tx(&fullA[slot], kItem);
                tma_bulk_g2s(ringA + slot * kItem, a_src(ia), kItem, &fullA[slot]);
                ++ia;
            };
            const bool gate_b1 = a.gate_b1 != 0;
            int u = cta, st = 0, ib = 0;
            auto issue_b = [&]() -> bool {
                if (u >= n_units) return false;
                const int bh = u / nch, ck = u - bh * nch;
                const int t0 = ck * chunk, ntok = min(chunk, len - t0);
                const int rows = min(kST, ntok - st * kST);
                const uint32_t rbytes = ib < C::NB ? static_cast<uint32_t>(C::STAGE)
                                                   : static_cast<uint32_t>(min(C::STAGE, ((rows * C::ROWB + 1023) / 1024) * 1024));
                const int slot = ib % C::NB;
                const uint32_t ph = static_cast<uint32_t>(ib / C::NB) & 1u;
                if (ib < nWS) {
                    mbar_wait(&wdone[slot], 0u);  // its parked projection items are consumed
                    if (gate_b1) mbar_wait(b1bar, 0u);
                }
                mbar_wait(&emptyB[slot], ph ^ 1u);
                mbar_arrive_expect_tx(&fullB[slot], rbytes);
                const uint8_t* src = a.cache + (static_cast<size_t>(bh) * cap + t0) * C::ROWB + static_cast<size_t>(st) * C::STAGE;
                tma_bulk_g2s_stream(ringB + slot * C::STAGE, src, rbytes, &fullB[slot], pol);
                ++ib;
                if (++st * kST >= ntok) {
                    st = 0;
                    u += G;
                }
                return true;
            };
            while (ia < na) issue_a();  // projection rest, O-proj weights (as the weight ring frees)
            while (issue_b()) {}        // cache stream; stages with parked items wait for them first
        }
        return;
    }

    const int g8 = lane >> 2, t4 = lane & 3;
    // ---- P1 (consumer warps 0..kNA-1): latent projection of this CTA's K split
    if (warp < kNW) {
        const float* xsrc = a.x;
        if (a.x_host && pj < cps) {
            // x lives in mapped (pinned) host memory: the cps CTAs of this K
            // split (with or without projection tiles) each fetch 1/cps of its
            // [B][kKS] slice over the bus into the device copy xd and publish a
            // count; all stage from xd once the count is complete (the host
            // bytes cross the bus once; the weight stream runs meanwhile)
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
                const unsigned target = static_cast<unsigned>(cps) * (epoch + 1u);
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.xcnt + ps) : "memory");
                while (ld_acquire(a.xcnt + ps) < target) {
                }
            }
            named_bar_sync(2, 32 * kNW);
            xsrc = a.xd;
        } else if (pj < cps && tid == 0) {
            // keep the counters' invariant (cps arrivals per fused step) in device mode
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.xcnt + ps) : "memory");
        }
        if (np1 > 0) stage_rows<MT>(xsrc, a.B, a.E, a.E, ps * kKS, xbuf, tid);
        named_bar_sync(2, 32 * kNW);
        {
            // all kNW consumer warps take items k = warp mod kNW in item order:
            // the weight ring's four (in flight first) and then the parked
            // ones as they land, at most two per warp
            for (int k = warp; k < np1; k += kNW) {
                float facc[MT][2][4];
                if (k >= kNA && k < kNA + nBH) {
                    const int b = k - kNA;
                    mbar_wait(&wfull[b], 0u);
                    item_mma<MT>(smem_u32(parked(b)), smem_u32(xbuf), lane, facc);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&wdone[b / 2]);
                } else {
                    const int ia = k < kNA ? k : k - nBH, slot = ia % kNA;
                    mbar_wait(&fullA[slot], static_cast<uint32_t>(ia / kNA) & 1u);
                    item_mma<MT>(smem_u32(ringA + slot * kItem), smem_u32(xbuf), lane, facc);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&emptyA[slot]);
                }
                const int tile = plo + k;
                float* P = a.P + static_cast<size_t>(ps) * a.B * a.Nrows;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int n = tile * 16 + g8 + ((i & 2) ? 8 : 0);
                            const int m = mt * 16 + hh * 8 + 2 * t4 + (i & 1);
                            if (m < a.B) P[static_cast<size_t>(m) * a.Nrows + n] = facc[mt][hh][i];
                        }
            }
        }
    }
    // helper: the first unit's M_QK column does not depend on the projection;
    // load it while the barrier drains (one L2 round trip off the critical path)
    float mq0[R];
    if (warp == kNW + 1 && nu > 0) {
        const int h0 = ((cta / nch) % a.nh);
        const float* mq = a.mqk + static_cast<size_t>(h0) * R * R + lane;
#pragma unroll
        for (int jj = 0; jj < R; ++jj) mq0[jj] = __ldg(mq + jj * R);
    }
    named_bar_sync(1, kSync);
    STEP_MARK(2);  // every P1 warp of this CTA is done
    grid_sync(a.bar, (2u * epoch + 1u) * G);  // consumers + helper
    if (tid == 0) mbar_arrive(b1bar);
    STEP_MARK(3);

    if (warp == kNW + 1) {
        // ============================================================ helper warp
        // (a) per unit, ahead of the consumers: qt = (sum_split c_Q) . M_QK in
        //     the append epilogue's order (fixed split order, sequential fma);
        //     for the unit holding the new token, its latent row [c_K | c_V] ->
        //     cache and shared memory (the stage is patched by its owner warp)
        auto prep = [&](int j, const float (&mqv)[R]) {
            const int u = cta + j * G;
            const int bh = u / nch, ck = u - bh * nch;
            const int b = bh / a.nh, h = bh - b * a.nh;
            const bool has_new = (ck + 1) * chunk >= len;
            const float* pb = a.P + static_cast<size_t>(b) * a.Nrows + static_cast<size_t>(h) * 3 * R + lane;
            float pv[3][kMaxSplits];
#pragma unroll
            for (int s = 0; s < kMaxSplits; ++s) {
                pv[0][s] = s < splits ? __ldcg(pb + s * pstride) : 0.f;
                pv[1][s] = (has_new && s < splits) ? __ldcg(pb + s * pstride + R) : 0.f;
                pv[2][s] = (has_new && s < splits) ? __ldcg(pb + s * pstride + 2 * R) : 0.f;
            }
            float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int s = 0; s < kMaxSplits; ++s)
#pragma unroll
                for (int r = 0; r < 3; ++r) v[r] += pv[r][s];  // zeros past `splits` leave the sum exact
            float qt = 0.f;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) qt = fmaf(__shfl_sync(0xffffffffu, v[0], jj), mqv[jj], qt);
            qts[j * R + lane] = qt;
            if (has_new) {
                uint8_t* region = a.cache + static_cast<size_t>(bh) * cap * C::ROWB;
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
        if (nu > 0) prep(0, mq0);
        for (int j = 1; j < nu; ++j) {
            const int h = ((cta + j * G) / nch) % a.nh;
            float mqv[R];
            const float* mq = a.mqk + static_cast<size_t>(h) * R * R + lane;
#pragma unroll
            for (int jj = 0; jj < R; ++jj) mqv[jj] = __ldg(mq + jj * R);
            prep(j, mqv);
        }
        // (b) per unit as the consumers finish it: merge the kNW warp states in
        //     warp order.  A unit that is not the last chunk of its (sequence,
        //     head) publishes its state to ws and releases a count; the last
        //     chunk's unit ("home") waits for the others and merges every chunk
        //     in chunk order (SoftmaxState::merge, decode.cpp:59-75) into the
        //     bf16 X rows of the O-projection (xo).  A home unit only waits for
        //     units of an earlier or equal round on lower CTAs, so the waits
        //     cannot form a cycle.
        for (int j = 0; j < nu; ++j) {
            mbar_wait(&sfull[j], 0u);
            const int u = cta + j * G;
            const int bh = u / nch, ck = u - bh * nch;
            const float* rb = wst + j * kNW * (R + 2);
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kNW; ++w) M = fmaxf(M, rb[w * (R + 2) + R]);
            float L = 0.f, av = 0.f;
#pragma unroll
            for (int w = 0; w < kNW; ++w) {
                const float mw = rb[w * (R + 2) + R];
                if (mw == -INFINITY) continue;
                const float f = ex2(mw - M);
                L = fmaf(rb[w * (R + 2) + R + 1], f, L);
                av = fmaf(rb[w * (R + 2) + lane], f, av);
            }
            // CTA pairs (cluster of 2, nch == 2): chunk 0 of a (sequence, head) runs
            // on the even CTA and its home chunk 1 on the odd one in the same round
            // j, so the state crosses through distributed shared memory with one
            // remote mbarrier arrive instead of an L2 publish / poll / load
            const bool pair = a.cluster == 2 && nch == 2;
            if (pair && ck == 0) {
                const uint32_t dst = cluster_map(smem_u32(pst + j * (R + 2)), 1u);
                st_cluster_f32(dst + 4u * lane, av);
                if (lane == 0) {
                    st_cluster_f32(dst + 4u * R, M);
                    st_cluster_f32(dst + 4u * (R + 1), L);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(cluster_map(smem_u32(&pbar[j]), 1u));
                continue;
            }
            if (ck < nch - 1) {
                float* wsp = a.ws + (static_cast<size_t>(bh) * a.max_chunks + ck) * kWS;
                wsp[lane] = av;
                if (lane == 0) {
                    wsp[R] = M;
                    wsp[R + 1] = L;
                }
                __syncwarp();
                if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.counters + bh) : "memory");
                continue;
            }
            if (pair) {
                mbar_wait_cluster(&pbar[j], 0u);
                const float* ps = pst + j * (R + 2);
                const float mc = ps[R], lc = ps[R + 1], ac = ps[lane];
                float M2 = M, L2 = L, a2 = av;
                if (mc != -INFINITY) {  // chunk 0 first, then this chunk (the chunk order of the L2 path)
                    const float Mn = fmaxf(mc, M);
                    const float fc = ex2(mc - Mn), fo = ex2(M - Mn);  // fo = 0 when M = -inf
                    L2 = fmaf(L, fo, lc * fc);
                    a2 = fmaf(av, fo, ac * fc);
                    M2 = Mn;
                }
                av = a2;
                L = L2;
                (void)M2;
            } else if (nch > 1) {
                if (lane == 0)
                    while (ld_acquire(reinterpret_cast<const unsigned*>(a.counters + bh)) < static_cast<unsigned>(nch - 1)) {
                    }
                __syncwarp();
                // one pass over the other chunks in chunk order (online merge):
                // each chunk's (m, l, acc) is one L2 round trip, loaded together
                const float* wb = a.ws + static_cast<size_t>(bh) * a.max_chunks * kWS;
                float M2 = -INFINITY, L2 = 0.f, a2 = 0.f;
                for (int c = 0; c < nch - 1; ++c) {
                    const float mc = __ldcg(wb + c * kWS + R), lc = __ldcg(wb + c * kWS + R + 1);
                    const float ac = __ldcg(wb + c * kWS + lane);
                    if (mc == -INFINITY) continue;
                    const float Mn = fmaxf(M2, mc);
                    const float fo = ex2(M2 - Mn), fc = ex2(mc - Mn);  // fo = 0 while M2 = -inf
                    L2 = fmaf(lc, fc, L2 * fo);
                    a2 = fmaf(ac, fc, a2 * fo);
                    M2 = Mn;
                }
                if (M != -INFINITY) {
                    const float Mn = fmaxf(M2, M);
                    const float fo = ex2(M2 - Mn), fc = ex2(M - Mn);
                    L2 = fmaf(L, fc, L2 * fo);
                    a2 = fmaf(av, fc, a2 * fo);
                }
                av = a2;
                L = L2;
                if (lane == 0) a.counters[bh] = 0;  // self-resetting for the next step
            }
            // latent output -> X rows of the O-projection, K index h*R + lane:
            // hi = bf16(v) in row b, lo = bf16(v - hi) in row MT*16 + b (~16
            // mantissa bits of the fp32 latent reach the tensor cores)
            const int b = bh / a.nh, h = bh - b * a.nh;
            const int k = h * R + lane, s = k / kKS;
            const float vo = av / L;
            const __nv_bfloat16 vh = __float2bfloat16_rn(vo);
            const __nv_bfloat16 vl = __float2bfloat16_rn(vo - __bfloat162float(vh));
            uint8_t* xs = a.xo + static_cast<size_t>(s) * C::XB2;
            reinterpret_cast<__nv_bfloat16*>(xs + static_cast<size_t>(b) * kXS)[k - s * kKS] = vh;
            reinterpret_cast<__nv_bfloat16*>(xs + static_cast<size_t>(MT * 16 + b) * kXS)[k - s * kKS] = vl;
        }
    } else {
        // ========================================================= consumer warps
        // ---- P2: attention units
        int slot = 0;
        uint32_t phase = 0;
        for (int j = 0; j < nu; ++j) {
            const int u = cta + j * G;
            const int bh = u / nch, ck = u - bh * nch;
            const int t0 = ck * chunk, ntok = min(chunk, len - t0);
            const int ns = (ntok + kST - 1) / kST;
            const bool has_new = (t0 + ntok == len);
            mbar_wait(&uready[j], 0u);
            if (j == 0) STEP_MARK(4);
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
            float m_w = -INFINITY, l = 0.f;
            float acc[KR][4];
#pragma unroll
            for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[kk][i] = 0.f;

            for (int s = 0; s < ns; ++s) {
                mbar_wait(&fullB[slot], phase);
                uint8_t* sp = ringB + slot * C::STAGE;
                const uint32_t sbase = smem_u32(sp);
                const int rows = min(kST, ntok - s * kST);
                const bool patch = has_new && s == ns - 1 && (rows - 1) / 32 == warp;
                if (patch) {
                    // the stage was copied before the step's own row existed
                    const uint32_t srow = static_cast<uint32_t>(rows - 1) * C::ROWB;
#pragma unroll
                    for (int half = 0; half < 2; ++half)
                        *reinterpret_cast<__nv_bfloat16*>(sp + cache_swz(srow + half * C::PART + 2 * lane)) =
                            nrow[j * 2 * R + half * R + lane];
                    __syncwarp();
                }
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
                    l *= f;
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
                    l += p0 + p1;
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
                if (patch)  // generic-proxy writes precede the slot's next TMA
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyB[slot]);
                if (++slot == C::NB) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
            // this warp's state of unit j -> the helper
            float* wr = wst + (j * kNW + warp) * (R + 2);
            const float lsum = warp_sum(l);
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
    STEP_MARK(6);
    grid_sync(a.bar, (2u * epoch + 2u) * G);  // every unit state is written; every CTA has read the length
    STEP_MARK(7);
    if (cta == 0 && tid == 0) {
        *a.d_len = len;
        *a.epoch += 1;  // fused steps run (the x-fetch counters' generation)
    }

    // ---- P3: folded O-projection over the prefetched W'_o items
    if (np3 == 0 || warp >= kNW) {
        STEP_MARK(8);
        STEP_MARK(9);
        return;
    }
    // The X slices this CTA's items use (bf16 rows built by the home units)
    // arrive with one TMA bulk copy each
    if (tid == 0) {
        // xo was written by other CTAs' generic stores (ordered by barrier 2);
        // order them before this thread's async-proxy reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_arrive_expect_tx(p3bar, static_cast<uint32_t>(osplits * C::XB2));
        for (int s = 0; s < osplits; ++s)
            tma_bulk_g2s(ringB + s * C::XB2, a.xo + static_cast<size_t>(s) * C::XB2, C::XB2, p3bar);
    }
    mbar_wait(p3bar, 0u);
    named_bar_sync(2, 32 * kNW);
    STEP_MARK(8);
    // item j = (tile i = j / osplits, split s = j % osplits) -> partial tile in
    // shared memory, then the splits are summed in split order
    float* part = reinterpret_cast<float*>(ringB + osplits * C::XB2);  // [np3][16 rows][MT*16 tokens]
    for (int j = 0; j < np3; ++j) {
        const int k = nA1 + j, slot = k % kNA;
        if (slot != warp) continue;
        mbar_wait(&fullA[slot], static_cast<uint32_t>(k / kNA) & 1u);
        const int s = j % osplits;
        // token columns 0..MT*16-1 are the hi rows, MT*16.. the lo rows
        float facc[2 * MT][2][4];
        item_mma<2 * MT>(smem_u32(ringA + slot * kItem), smem_u32(ringB + s * C::XB2), lane, facc);
        float* pj = part + j * 16 * MT * 16;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int n = g8 + ((i & 2) ? 8 : 0);
                    const int m = mt * 16 + hh * 8 + 2 * t4 + (i & 1);
                    pj[n * MT * 16 + m] = facc[mt][hh][i] + facc[mt + MT][hh][i];
                }
    }
    named_bar_sync(2, 32 * kNW);
    if (!ycontig) {
        for (int i = tid; i < nt3 * 16 * a.B; i += 32 * kNW) {
            const int ti = i / (16 * a.B), r = i - ti * 16 * a.B;
            const int m = r / 16, n = r - m * 16;  // n fastest: 64-byte row segments of y
            const int col = (t3lo + ti * G) * 16 + n;
            if (col >= a.e_out) continue;
            float v = 0.f;
            for (int s = 0; s < osplits; ++s) v += part[((ti * osplits + s) * 16 + n) * MT * 16 + m];
            a.y[static_cast<size_t>(m) * a.e_out + col] = v;
        }
        STEP_MARK(9);
        return;
    }
    const int q4 = nt3 * 4;  // 4-column groups of this CTA's row segment
    for (int i = tid; i < a.B * q4; i += 32 * kNW) {
        const int m = i / q4, q = i - m * q4;
        const int ti = q >> 2, n0 = (q & 3) * 4;
        const int col = (t3lo + ti) * 16 + n0;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            v[e] = 0.f;
            for (int s = 0; s < osplits; ++s) v[e] += part[((ti * osplits + s) * 16 + n0 + e) * MT * 16 + m];
        }
        float* yr = a.y + static_cast<size_t>(m) * a.e_out;
        if (col + 4 <= a.e_out && (a.e_out & 3) == 0) {
            *reinterpret_cast<float4*>(yr + col) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
            for (int e = 0; e < 4; ++e)
                if (col + e < a.e_out) yr[col + e] = v[e];
        }
    }
    STEP_MARK(9);
}

template <int MT>
cudaError_t launch_mt(const StepArgs& a, cudaStream_t s) {
    using C = SC<32, MT>;
    if constexpr (!C::OK) {
        return cudaErrorInvalidValue;
    } else {
        auto k = layer_step_kernel<32, MT>;
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e != cudaSuccess) return e;
            attr = true;
        }
        // grid barriers need every CTA resident: one CTA per SM fits (the host
        // checks occupancy once and serialises fused steps of different
        // streams, capi.cu fused_serialize).  A cooperative launch would
        // guarantee it in hardware but costs ~3.5 us per step on B200
        // (59.0 vs 55.5 us, r02_coop.txt); WSVD_STEP_COOP=1 selects it.
        static const bool coop = std::getenv("WSVD_STEP_COOP") != nullptr;
        if (coop) return launch_coop_cluster(k, dim3(a.grid), dim3(kThr), C::SMEM, s, a.cluster, a);
        return launch_pdl_cluster(k, dim3(a.grid), dim3(kThr), C::SMEM, s, a.cluster, a);
    }
}

template <int MT>
int pair_ok(int grid) {
    using C = SC<32, MT>;
    if constexpr (!C::OK) {
        return 0;
    } else {
        auto k = layer_step_kernel<32, MT>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess) return 0;
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
}

}  // namespace

bool step_supported(int R, int B, int nh, int max_units, int max_chunks, int Kp, int oKp, int otiles, int grid) {
    if (R != 32 || B < 1 || B > 32) return false;
    if (Kp % kKS != 0 || oKp % kKS != 0) return false;
    const int splits = Kp / kKS, osplits = oKp / kKS;
    if (osplits > 2 || splits > grid || splits > kMaxSplits) return false;
    if ((max_units + grid - 1) / grid > kMaxU) return false;
    (void)nh;
    if (((otiles + grid - 1) / grid) * osplits > kNA) return false;
    // P3 stages its X slices in the attention ring
    const int mt = (B + 15) / 16;
    const int ring = (mt == 1 ? SC<32, 1>::NB * SC<32, 1>::STAGE : SC<32, 2>::NB * SC<32, 2>::STAGE);
    (void)max_chunks;
    return osplits * 2 * mt * 16 * kXS + kNA * 16 * mt * 16 * 4 <= ring;
}

int step_item_k() { return kKS; }

int step_pair_clusters_ok(int B, int grid) {
    if (grid % 2 != 0) return 0;
    return (B + 15) / 16 == 1 ? pair_ok<1>(grid) : pair_ok<2>(grid);
}

size_t step_xo_bytes(int B, int oKp) { return static_cast<size_t>(oKp / kKS) * 2 * ((B + 15) / 16) * 16 * kXS; }

int step_max_units() { return kMaxU; }

int step_resident_ctas_per_sm(int B) {
    int n = 0;
    auto probe = [&](auto k, int smem) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kThr, smem) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
    };
    if ((B + 15) / 16 == 1) probe(layer_step_kernel<32, 1>, SC<32, 1>::SMEM);
    else probe(layer_step_kernel<32, 2>, SC<32, 2>::SMEM);
    return n;
}

cudaError_t launch_layer_step(const StepArgs& a, cudaStream_t s) {
    switch ((a.B + 15) / 16) {
        case 1: return launch_mt<1>(a, s);
        case 2: return launch_mt<2>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace wsvd_k
