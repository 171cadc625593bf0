// attn.cu -- fused per-head low-rank decode attention for sm_100a.
//
// Replaces wsvd::decode::fused_decode_step (reference src/decode.cpp:155-206).
// The reference rebuilds every key, key_j = C_K[j] . B_K (decode.cpp:188),
// at L*r*H MACs per head.  Scores only need q . key_j, so this kernel uses
// the algebraically identical absorbed query qt = q . B_K^T (r values,
// computed once per (sequence, head) by the append epilogue or
// launch_absorb_query) and streams every latent row exactly once:
//
//   s_j   = qt . C_K[j]                      (log2 domain, 1/sqrt(H) folded in)
//   state = online softmax over s_j with the accumulator in latent-V space
//           (decode.cpp:35-57, 192: acc += p_j * C_V[j])
//   out   = (acc / denom) . B_V              (decode.cpp:198-203, once per head)
//
// Results equal the reference up to floating-point reassociation.
//
// HBM layout: cache[b][h][t][ C_K(R) | C_V(R) ] (one row per token, R = padded
// rank), XOR-swizzled in 16-byte units (cache_swz, common.cuh); int8 rows carry
// a half2 (s_K, s_V) per token in a parallel array.  Work units are
// (sequence, head, chunk of `chunk` tokens); a persistent grid of one CTA per
// SM walks them round-robin.  Warp specialisation: one producer warp keeps a
// ring of TMA bulk copies (cp.async.bulk, completion via mbarrier complete_tx)
// of 256-token stages in flight across unit boundaries -- including the
// unit's absorbed query row -- while 8 consumer warps drain them and hand
// slots back through `empty` mbarriers; no CTA-wide barrier sits in the
// streaming loop.
//
// bf16 caches (the production format) run both contractions of a 16-token
// group on the tensor cores with mma.sync m16n8k16: scores = K_tile . [qt_hi |
// qt_lo] and acc += V_tile^T . [p_hi | p_lo], where x_hi = bf16(x) and
// x_lo = bf16(x - x_hi) keep ~16 significant bits of the fp32 query and
// probabilities (the cache operand is exact bf16, products and sums are fp32).
// fp32 and int8 caches use a CUDA-core path (one token per thread).
//
// At a unit's end every consumer warp publishes its own partial state
// (m, l, acc[R]) -- no CTA-wide or grid-wide synchronisation anywhere in the
// streaming kernel.  A small combine kernel then merges each (sequence, head)'s
// partials in a fixed order (SoftmaxState::merge, decode.cpp:59-75) and
// applies B_V once; results are run-to-run deterministic.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kStageTok = 256;   // tokens per pipeline stage
constexpr int kMaxWarps = 16;    // most consumer warps of any variant (partials per chunk)
constexpr int kDefaultVariant = 0;

// V (tensor-core variants, bf16 cache): bit 0 = transposed score tile,
// bit 1 = 16 consumer warps (else 8)
template <int CD, int R, int V = 0>
struct Cfg {
    static constexpr int EB = (CD == F32) ? 4 : (CD == BF16 ? 2 : 1);
    static constexpr int EPC = 16 / EB;        // elements per 16-byte chunk
    static constexpr int PART = R * EB;        // bytes of the K (and V) half
    static constexpr int NC = PART / 16;       // chunks per half
    static constexpr int ROWB = 2 * PART;
    static constexpr bool MMA = (CD == BF16);
    // int8 cache on the tensor cores (consume_mma_i8): V bit 3 selects the
    // CUDA-core consumer instead (A/B)
    static constexpr bool IMMA = (CD == I8) && !(V & 8) && (R % 16 == 0);
    // tensor-core consumers: 16 warps x one 16-token group per stage (latency
    // hiding: 4 warps per SM sub-partition); CUDA-core consumers: one token per thread
    static constexpr int NW = ((MMA || IMMA) && (V & 2)) ? 16 : 8;
    static constexpr int THREADS = 32 * NW + 64;  // + one producer warp + one merge (helper) warp
    static constexpr int QTB = 512;               // the unit's absorbed query (R <= 128 floats)
    static constexpr int RSTRIDE = R + 4;         // floats per lane row of the reduction scratch
    static constexpr int RED = (MMA || IMMA) ? 0 : NW * 32 * RSTRIDE * 4;
    static constexpr int BUDGET = 222 * 1024;
    // Tokens per stage.  The tensor-core consumers want >= 3 stages in flight,
    // the CUDA-core one >= 2.  int8 tensor-core consumers take 1024-token
    // stages (64 KB at r = 32: fewer per-stage reductions and conversions per
    // token) when three fit, else 512 (the same 32 KB per stage as bf16), else
    // 256 (large ranks); V bit 5 rules out 1024.  bf16 and the CUDA-core
    // consumer take 256-token stages, 128 for large ranks (rows up to 512 B).
    static constexpr int stage_bytes(int st) { return st * ROWB + ((CD == I8) ? 4 * st : 0) + QTB; }
    static constexpr int NEED = (MMA || IMMA) ? 3 : 2;
    static constexpr bool fits(int st) { return NEED * stage_bytes(st) + RED + 4096 <= BUDGET; }
    static constexpr bool BIG = IMMA && !(V & 32) && fits(4 * kStageTok);
    static constexpr int ST = IMMA ? (BIG ? 4 * kStageTok : (fits(2 * kStageTok) ? 2 * kStageTok : kStageTok))
                                   : (fits(kStageTok) ? kStageTok : kStageTok / 2);
    static constexpr int GPW = ST / (16 * NW);  // 16-token groups per warp per stage
    static constexpr int ROWS = ST * ROWB;
    static constexpr int SC = (CD == I8) ? 4 * ST : 0;
    static constexpr int QT_OFF = ROWS + SC;   // absorbed query of the unit (first stage)
    static constexpr int STAGE = QT_OFF + QTB;
    static constexpr int ST_RAW = (BUDGET - RED - 4096) / STAGE;
    static constexpr int STAGES = ST_RAW > 8 ? 8 : ST_RAW;
    static constexpr int BAR_OFF = STAGES * STAGE;
    static constexpr int RED_OFF = BAR_OFF + 256;
    static constexpr int MISC_OFF = RED_OFF + RED;
    // >= 2 stages; every tensor-core warp owns whole 16-token groups (pairs for
    // the int8 P.V k-steps)
    static constexpr bool OK = ST_RAW >= 2 && (!(MMA || IMMA) || (GPW >= 1 && (!IMMA || GPW % 2 == 0)));
    static constexpr int SMEM = OK ? MISC_OFF : 0;
    static_assert(PART % 16 == 0, "latent half must be a multiple of 16 bytes");
    static_assert(R * 4 <= QTB, "query row must fit the stage's query area");
};

WSVD_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16 bytes of cache -> EPC floats
template <int CD>
WSVD_DEV void chunk_to_f32(const uint4& v, float* f);
template <>
WSVD_DEV void chunk_to_f32<F32>(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
template <>
WSVD_DEV void chunk_to_f32<BF16>(const uint4& v, float* f) {
    f[0] = bf16lo(v.x); f[1] = bf16hi(v.x); f[2] = bf16lo(v.y); f[3] = bf16hi(v.y);
    f[4] = bf16lo(v.z); f[5] = bf16hi(v.z); f[6] = bf16lo(v.w); f[7] = bf16hi(v.w);
}
// signed bytes -> float through the 2^23 magic: float(0x4B0000uu) - (2^23 + 128)
// Exact int <-> float conversions for |v| < 2^22 on the full-rate FP32 / INT
// pipes (I2F / F2I issue at a quarter rate and were hot in the int8 consumers:
// profiles/r01_i8_full_summary.json).  The int8 MMA sums stay below 2^22
// (128 * 127 * 127 for the scores at r <= 128, 32 * 127 * 127 for P.V) and the
// quantised probabilities below 128; f2i_rn_small rounds to nearest even like
// __float2int_rn.  Results are bit-identical to the conversion instructions.
WSVD_DEV float i2f_small(int v) { return __int_as_float(v + 0x4B400000) - 12582912.0f; }
WSVD_DEV int f2i_rn_small(float x) { return __float_as_int(x + 12582912.0f) - 0x4B400000; }

WSVD_DEV void s8x4_to_f32(uint32_t w, float* f) {
    const uint32_t u = w ^ 0x80808080u;
    f[0] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7650)) - 8388736.0f;
    f[1] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7651)) - 8388736.0f;
    f[2] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7652)) - 8388736.0f;
    f[3] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7653)) - 8388736.0f;
}
template <>
WSVD_DEV void chunk_to_f32<I8>(const uint4& v, float* f) {
    s8x4_to_f32(v.x, f); s8x4_to_f32(v.y, f + 4); s8x4_to_f32(v.z, f + 8); s8x4_to_f32(v.w, f + 12);
}

WSVD_DEV float load_b(const void* b, int bdtype, size_t idx) {
    if (bdtype == F32) return reinterpret_cast<const float*>(b)[idx];
    if (bdtype == BF16)
        return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(b)[idx]);
    return static_cast<float>(reinterpret_cast<const int8_t*>(b)[idx]);
}

// x -> (bf16(x), bf16(x - bf16(x))) as raw 16-bit patterns
WSVD_DEV void split_bf16(float x, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
    hi = *reinterpret_cast<const uint16_t*>(&h);
    lo = *reinterpret_cast<const uint16_t*>(&l);
}

struct Unit {
    int bh, chunk, t0, ntok;
};

// Split of one (sequence, head) into chunks for this launch.  a.chunk > 0
// fixes the chunk length (tests); otherwise up to a.max_chunks chunks of equal
// length (a multiple of 32 tokens), so every unit carries real work.
WSVD_DEV void chunking(const AttnArgs& a, int len, int& nch, int& chunk) {
    if (a.cluster > 1) {  // exactly one chunk per cluster CTA (trailing ones may be empty)
        nch = a.cluster;
        chunk = (((len + nch - 1) / nch) + 31) & ~31;
        return;
    }
    if (a.chunk > 0) {
        chunk = a.chunk;
    } else {
        const int n = max(1, min(a.max_chunks, (len + 31) / 32));
        chunk = (((len + n - 1) / n) + 31) & ~31;
    }
    nch = (len + chunk - 1) / chunk;
}

WSVD_DEV Unit unit_geom(int u, int nch, int chunk, int len) {
    Unit g;
    g.bh = u / nch;
    g.chunk = u - g.bh * nch;
    g.t0 = g.chunk * chunk;
    g.ntok = min(chunk, len - g.t0);
    return g;
}

// ----------------------------------------------------------------------------
// Tensor-core consumer (bf16 cache) of one warp over one unit.  The warp owns
// GPW 16-token groups of every 256-token stage.
//
// TS = 0: scores D(16 tok x 8) = K(16 tok x R) . [qt_hi | qt_lo](R x 8): the
//   lane (g8, t4 = 0) holds the hi / lo partial scores of tokens g8, g8 + 8;
//   four shuffles per group build the P fragment of the P.V MMA.
// TS = 1: transposed tile S(16 x 8 tok) = Q(16 x R) . K^T with Q rows 0 and 1
//   both the query (hi part in one MMA, lo part in a second accumulating one):
//   lanes g8 in {0,1} hold the full scores of exactly the token pair their P
//   fragment needs -- no shuffles, 4x the score MMAs.
// Both: P.V as acc(R x 8) += V^T(R x 16 tok) . [p_hi | p_lo](16 tok x 8), the
// x_hi = bf16(x), x_lo = bf16(x - x_hi) split keeping ~16 bits of the fp32
// query and probabilities; the running max is a warp-uniform reference moved
// lazily (only when a score exceeds it by 2^8, decided by one vote), so no
// per-stage shuffle reduction sits on the critical path.
template <class C, int R, int TS>
WSVD_DEV void consume_mma(const AttnArgs& a, const Unit& g, uint8_t* smem, uint64_t* full, uint64_t* empty,
                          int& slot, uint32_t& phase, int warp, int lane) {
    constexpr int KR = R / 16;
    constexpr int GPW = C::GPW;
    const int g8 = lane >> 2, t4 = lane & 3;
    const bool qlane = g8 < 2;
    float m_w = -INFINITY, l = 0.f;
    const int ns = (g.ntok + C::ST - 1) / C::ST;
    uint32_t qa[KR][2][2];  // TS=0: B fragments [kk][b0/b1][unused]; TS=1: A frags [kk][hi/lo][a0/a2]
    float acc[KR][4];
#pragma unroll
    for (int kk = 0; kk < KR; ++kk)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[kk][i] = 0.f;
    for (int s = 0; s < ns; ++s) {
        mbar_wait(&full[slot], phase);
        const uint8_t* sp = smem + slot * C::STAGE;
        const uint32_t sbase = smem_u32(sp);
        if (s == 0) {
            const float* q = reinterpret_cast<const float*>(sp + C::QT_OFF);
#pragma unroll
            for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k0 = kk * 16 + 2 * t4 + 8 * j;
                    uint32_t h0, l0, h1, l1;
                    split_bf16(q[k0], h0, l0);
                    split_bf16(q[k0 + 1], h1, l1);
                    if (TS == 0) {
                        qa[kk][j][0] = (g8 == 0) ? (h0 | (h1 << 16)) : (g8 == 1 ? (l0 | (l1 << 16)) : 0u);
                    } else {
                        qa[kk][0][j] = qlane ? (h0 | (h1 << 16)) : 0u;
                        qa[kk][1][j] = qlane ? (l0 | (l1 << 16)) : 0u;
                    }
                }
        }
        const int rows = min(C::ST, g.ntok - s * C::ST);
        // ---- scores: sc[grp][i], i = the lane's 4 token slots of the group
        float sc[GPW][4];
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            if (TS == 0) {
                float d[4] = {0.f, 0.f, 0.f, 0.f};
                const int ltok = tb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
                for (int kk = 0; kk < KR; ++kk) {
                    uint32_t a0, a1, a2, a3;
                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2 + (lane >> 4)) * 16);
                    ldsm_x4(sbase + cache_swz(off), a0, a1, a2, a3);
                    mma_bf16_16816(d, a0, a1, a2, a3, qa[kk][0][0], qa[kk][1][0]);
                }
                // slots 0/1: tokens g8, g8 + 8 (valid on t4 == 0)
                sc[grp][0] = (t4 == 0 && tb + g8 < rows) ? d[0] + d[1] : -INFINITY;
                sc[grp][1] = (t4 == 0 && tb + g8 + 8 < rows) ? d[2] + d[3] : -INFINITY;
                sc[grp][2] = sc[grp][3] = -INFINITY;
            } else {
#pragma unroll
                for (int tile = 0; tile < 2; ++tile) {
                    float d[4] = {0.f, 0.f, 0.f, 0.f};
                    const uint32_t rowoff = static_cast<uint32_t>((tb + tile * 8 + (lane & 7)) * C::ROWB);
#pragma unroll
                    for (int kk = 0; kk + 1 < KR; kk += 2) {
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(sbase + cache_swz(rowoff + (kk * 2 + (lane >> 3)) * 16), b0, b1, b2, b3);
                        mma_bf16_16816(d, qa[kk][0][0], 0u, qa[kk][0][1], 0u, b0, b1);
                        mma_bf16_16816(d, qa[kk][1][0], 0u, qa[kk][1][1], 0u, b0, b1);
                        mma_bf16_16816(d, qa[kk + 1][0][0], 0u, qa[kk + 1][0][1], 0u, b2, b3);
                        mma_bf16_16816(d, qa[kk + 1][1][0], 0u, qa[kk + 1][1][1], 0u, b2, b3);
                    }
                    if constexpr (KR & 1) {
                        constexpr int kk = KR - 1;
                        uint32_t b0, b1;
                        ldsm_x2(sbase + cache_swz(rowoff + (kk * 2 + ((lane >> 3) & 1)) * 16), b0, b1);
                        mma_bf16_16816(d, qa[kk][0][0], 0u, qa[kk][0][1], 0u, b0, b1);
                        mma_bf16_16816(d, qa[kk][1][0], 0u, qa[kk][1][1], 0u, b0, b1);
                    }
                    const int tok = tb + tile * 8 + 2 * t4;
                    sc[grp][2 * tile] = (qlane && tok < rows) ? d[0] : -INFINITY;
                    sc[grp][2 * tile + 1] = (qlane && tok + 1 < rows) ? d[1] : -INFINITY;
                }
            }
        }
        // ---- lazily moved reference max
        float lm = -INFINITY;
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp)
#pragma unroll
            for (int i = 0; i < 4; ++i) lm = fmaxf(lm, sc[grp][i]);
        if (__any_sync(0xffffffffu, lm > m_w + 8.f)) {
            const float wm = warp_max(lm);
            const float f = ex2(m_w - wm);
            l *= f;
#pragma unroll
            for (int kk = 0; kk < KR; ++kk)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[kk][i] *= f;
            m_w = wm;
        }
        // ---- probabilities and P.V
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            float p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = (sc[grp][i] == -INFINITY) ? 0.f : ex2(sc[grp][i] - m_w);
            uint32_t b[2];
            if (TS == 0) {
                l += p[0] + p[1];
                uint32_t h0, l0, h1, l1;
                split_bf16(p[0], h0, l0);
                split_bf16(p[1], h1, l1);
                const uint32_t hi2 = h0 | (h1 << 16), lo2 = l0 | (l1 << 16);
                // lane (g8 in {0,1}, t4) needs p of tokens 2t4, 2t4+1 (+8): held by
                // lanes 4*(2t4) and 4*(2t4+1) as (token, token + 8) pairs
                const int s0 = 8 * t4, s1 = 8 * t4 + 4;
                const uint32_t xh = __shfl_sync(0xffffffffu, hi2, s0), yh = __shfl_sync(0xffffffffu, hi2, s1);
                const uint32_t xl = __shfl_sync(0xffffffffu, lo2, s0), yl = __shfl_sync(0xffffffffu, lo2, s1);
                const uint32_t x = (g8 == 0) ? xh : xl, y = (g8 == 0) ? yh : yl;
                b[0] = (g8 < 2) ? __byte_perm(x, y, 0x5410) : 0u;
                b[1] = (g8 < 2) ? __byte_perm(x, y, 0x7632) : 0u;
            } else {
                if (g8 == 0) l += (p[0] + p[1]) + (p[2] + p[3]);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    uint32_t h0, l0, h1, l1;
                    split_bf16(p[2 * j], h0, l0);
                    split_bf16(p[2 * j + 1], h1, l1);
                    b[j] = (g8 == 0) ? (h0 | (h1 << 16)) : (g8 == 1 ? (l0 | (l1 << 16)) : 0u);
                }
            }
            const int stok = tb + (lane & 7) + ((lane >> 4) & 1) * 8;
#pragma unroll
            for (int mm = 0; mm < KR; ++mm) {
                uint32_t a0, a1, a2, a3;
                const uint32_t off = static_cast<uint32_t>(stok * C::ROWB + C::PART + (mm * 2 + ((lane >> 3) & 1)) * 16);
                ldsm_x4_trans(sbase + cache_swz(off), a0, a1, a2, a3);
                mma_bf16_16816(acc[mm], a0, a1, a2, a3, b[0], b[1]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == C::STAGES) {
            slot = 0;
            phase ^= 1u;
        }
    }
    const float lsum = warp_sum(l);
    float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * kMaxWarps + warp) * (R + 2);
    if (t4 == 0) {
#pragma unroll
        for (int mm = 0; mm < KR; ++mm) {
            wsp[mm * 16 + g8] = acc[mm][0] + acc[mm][1];      // r = mm*16 + g8
            wsp[mm * 16 + g8 + 8] = acc[mm][2] + acc[mm][3];  // r = mm*16 + g8 + 8
        }
    }
    if (lane == 0) {
        wsp[R] = m_w;
        wsp[R + 1] = lsum;
    }
}

// ----------------------------------------------------------------------------
// Tensor-core consumer for INT8 caches (per-token scales s_K, s_V).
// Scores on the integer tensor cores: the absorbed query is split into two
// int8 rows, qt ~ s1.q1 + s2.q2 (s1 = max|qt|/127, s2 = s1/254, ~15 bits), and
// D(16 tok x 8) = K_int8(16 x 32) . [q1 | q2](32 x 8) (mma.m16n8k32.s8, exact
// int32), score = (d1.s1 + d2.s2).s_K.  P.V on the f16 tensor cores:
// acc(16 x 8 r) += [p'_hi ; p'_lo](16 x 16 tok) . V(16 tok x 8 r) with
// p' = p.s_V split into f16 hi / lo (~22 bits) and V converted exactly from
// int8 (ldmatrix.trans pairs of bytes -> f16x2: r = 2n and 2n+1 of each
// 16-byte unit feed two MMAs).  Results equal the CUDA-core consumer up to fp32
// reassociation and the ~1e-5 relative query split.
template <class C, int R>
WSVD_DEV void consume_mma_i8(const AttnArgs& a, const Unit& g, uint8_t* smem, uint64_t* full, uint64_t* empty,
                             int& slot, uint32_t& phase, int warp, int lane) {
    constexpr int K32 = (R + 31) / 32;  // s8 MMA k-steps for the scores (the last may be half: R % 32 == 16)
    constexpr int UV = R / 16;      // 16-byte units of the V half
    const int g8 = lane >> 2, t4 = lane & 3;
    float m_w = -INFINITY, l = 0.f;
    const int ns = (g.ntok + C::ST - 1) / C::ST;
    uint32_t qf[K32][2];            // B fragments (int8 x4): b0 / b1 of each k-step
    float s1 = 1.f, s2 = 1.f;
    float acc[UV][2][4];            // [unit][even|odd r][D fragment]
#pragma unroll
    for (int u = 0; u < UV; ++u)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[u][e][i] = 0.f;
    for (int s = 0; s < ns; ++s) {
        mbar_wait(&full[slot], phase);
        const uint8_t* sp = smem + slot * C::STAGE;
        const uint32_t sbase = smem_u32(sp);
        if (s == 0) {
            const float* q = reinterpret_cast<const float*>(sp + C::QT_OFF);
            float mx = 0.f;
#pragma unroll
            for (int k = 0; k < R; ++k) mx = fmaxf(mx, fabsf(q[k]));
            s1 = (mx == 0.f) ? 1.f : mx / 127.f;
            s2 = s1 / 254.f;
#pragma unroll
            for (int kk = 0; kk < K32; ++kk)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    uint32_t w1 = 0, w2 = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (kk * 32 + 16 * j >= R) break;  // the padded half of a last k-step
                        const float v = q[kk * 32 + 16 * j + 4 * t4 + e];
                        const float h = rintf(v / s1);
                        const float lo = rintf(fmaf(-h, s1, v) / s2);  // oracle: orc_i8_query_split
                        w1 |= (static_cast<uint32_t>(static_cast<int32_t>(h)) & 0xffu) << (8 * e);
                        w2 |= (static_cast<uint32_t>(static_cast<int32_t>(fminf(fmaxf(lo, -127.f), 127.f))) & 0xffu) << (8 * e);
                    }
                    qf[kk][j] = (g8 == 0) ? w1 : (g8 == 1 ? w2 : 0u);
                }
        }
        const int rows = min(C::ST, g.ntok - s * C::ST);
        const __half2* sc2 = reinterpret_cast<const __half2*>(sp + C::ROWS);
        constexpr int GPW = C::GPW;
        float sc[GPW][2];
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            int d[4] = {0, 0, 0, 0};
            const int ltok = tb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
            for (int kk = 0; kk < K32; ++kk) {
                uint32_t a0, a1, a2 = 0u, a3 = 0u;
                if (kk * 32 + 16 < R) {
                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2 + (lane >> 4)) * 16);
                    ldsm_x4(sbase + cache_swz(off), a0, a1, a2, a3);
                } else {  // r in [32kk, 32kk + 16): the upper half of the k-step is zero
                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2) * 16);
                    ldsm_x2(sbase + cache_swz(off), a0, a1);
                }
                mma_s8_16832(d, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
            }
            const int t0 = tb + g8, t1 = tb + g8 + 8;
            if (a.dbg_scores && t4 == 0) {  // test hook: the int32 score accumulators (hi, lo query parts)
                int* dbg = a.dbg_scores + (static_cast<size_t>(g.bh) * a.cap + g.t0 + s * C::ST) * 2;
                if (t0 < rows) { dbg[2 * t0] = d[0]; dbg[2 * t0 + 1] = d[1]; }
                if (t1 < rows) { dbg[2 * t1] = d[2]; dbg[2 * t1 + 1] = d[3]; }
            }
            const float k0 = __low2float(sc2[t0]), k1 = __low2float(sc2[t1]);
            sc[grp][0] = (t4 == 0 && t0 < rows)
                ? fmaf(i2f_small(d[0]), s1, i2f_small(d[1]) * s2) * k0 : -INFINITY;
            sc[grp][1] = (t4 == 0 && t1 < rows)
                ? fmaf(i2f_small(d[2]), s1, i2f_small(d[3]) * s2) * k1 : -INFINITY;
        }
        float lm = -INFINITY;
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) lm = fmaxf(lm, fmaxf(sc[grp][0], sc[grp][1]));
        // lazily moved reference max: rescale only when a score exceeds it by
        // more than 2^8 (p <= 256 in between), one vote instead of a reduction
        if (__any_sync(0xffffffffu, lm > m_w + 8.f)) {
            const float wm = warp_max(lm);
            const float f = ex2(m_w - wm);
            l *= f;
#pragma unroll
            for (int u = 0; u < UV; ++u)
#pragma unroll
                for (int e = 0; e < 2; ++e)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[u][e][i] *= f;
            m_w = wm;
        }
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            const int t0 = tb + g8, t1 = tb + g8 + 8;
            const float p0 = (sc[grp][0] == -INFINITY) ? 0.f : ex2(sc[grp][0] - m_w);
            const float p1 = (sc[grp][1] == -INFINITY) ? 0.f : ex2(sc[grp][1] - m_w);
            l += p0 + p1;
            // p' = p . s_V, split into f16 hi / lo
            const float q0 = p0 * __high2float(sc2[t0]), q1 = p1 * __high2float(sc2[t1]);
            const __half h0 = __float2half_rn(q0), h1 = __float2half_rn(q1);
            const __half e0 = __float2half_rn(q0 - __half2float(h0)), e1 = __float2half_rn(q1 - __half2float(h1));
            const uint32_t hi2 = static_cast<uint32_t>(__half_as_ushort(h0)) | (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
            const uint32_t lo2 = static_cast<uint32_t>(__half_as_ushort(e0)) | (static_cast<uint32_t>(__half_as_ushort(e1)) << 16);
            // A fragment of P (rows 0 = hi, 1 = lo; k = tokens): lane (g8 in {0,1}, t4)
            // needs tokens 2t4, 2t4+1 (a0) and 2t4+8, 2t4+9 (a2), held by lanes
            // 4*(2t4), 4*(2t4+1) as (token, token + 8) pairs
            const int s0 = 8 * t4, s1l = 8 * t4 + 4;
            const uint32_t xh = __shfl_sync(0xffffffffu, hi2, s0), yh = __shfl_sync(0xffffffffu, hi2, s1l);
            const uint32_t xl = __shfl_sync(0xffffffffu, lo2, s0), yl = __shfl_sync(0xffffffffu, lo2, s1l);
            const uint32_t xx = (g8 == 0) ? xh : xl, yy = (g8 == 0) ? yh : yl;
            const uint32_t pa0 = (g8 < 2) ? __byte_perm(xx, yy, 0x5410) : 0u;  // tokens 2t4, 2t4+1
            const uint32_t pa2 = (g8 < 2) ? __byte_perm(xx, yy, 0x7632) : 0u;  // tokens 2t4+8, 2t4+9
            // V: for each 16-byte unit, matrices (tokens 0-7) and (tokens 8-15)
            const int vtok = tb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
            for (int u = 0; u < UV; ++u) {
                uint32_t v0, v1;
                const uint32_t off = static_cast<uint32_t>(vtok * C::ROWB + C::PART + u * 16);
                ldsm_x2_trans(sbase + cache_swz(off), v0, v1);
                // v0 = (tok 2t4: r 2g8, 2g8+1 | tok 2t4+1: r 2g8, 2g8+1) of this unit; v1 = +8 tokens
                const uint32_t x0 = v0 ^ 0x80808080u, x1 = v1 ^ 0x80808080u;
                const uint32_t be0 = s8pair_to_f16x2(x0, 0x4240), bo0 = s8pair_to_f16x2(x0, 0x4341);
                const uint32_t be1 = s8pair_to_f16x2(x1, 0x4240), bo1 = s8pair_to_f16x2(x1, 0x4341);
                mma_f16_16816(acc[u][0], pa0, 0u, pa2, 0u, be0, be1);
                mma_f16_16816(acc[u][1], pa0, 0u, pa2, 0u, bo0, bo1);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == C::STAGES) {
            slot = 0;
            phase ^= 1u;
        }
    }
    // D fragment: lane (g8 in {0,1} = hi / lo row, t4) holds columns 2t4, 2t4+1 of
    // each MMA; column c of the even (odd) MMA of unit u is r = 16u + 2c (+1)
    const float lsum = warp_sum(l);
    float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * kMaxWarps + warp) * (R + 2);
#pragma unroll
    for (int u = 0; u < UV; ++u)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float v = acc[u][e][i] + __shfl_xor_sync(0xffffffffu, acc[u][e][i], 4);  // hi + lo rows
                if (g8 == 0) wsp[16 * u + 2 * (2 * t4 + i) + e] = v;
            }
    if (lane == 0) {
        wsp[R] = m_w;
        wsp[R + 1] = lsum;
    }
}

// ----------------------------------------------------------------------------
// INT8 cache, both contractions on the integer tensor cores (the default at
// r <= 32, where 1024-token stages fit; variant bit 4 swaps it with consume_mma_i8).
// Scores as consume_mma_i8.  P.V: per stage, p' = p.s_V is split against the
// warp's stage maximum b into two int8 columns, p' ~ s1.h + s2.l (s1 = b/127,
// s2 = s1/254, ~15 bits of b), and the transposed product D(16 r x 8) =
// V^T_int8(16 r x 32 tok) . [h | l](32 tok x 8) runs on mma.m16n8k32.s8 with
// exact int32 sums -- one MMA per 16 latent columns per 32 tokens, a quarter
// of the f16 P.V's, and no int8 -> f16 conversion of V.  The stage's sums are
// scaled into fp32 accumulators once.  V^T fragments are byte gathers of
// ldmatrix.trans pairs: k = 4 t4 + i of a 16-token half is token (2t4, 2t4+1,
// 2t4+8, 2t4+9)[i], row g8 is r = 2 g8 and row g8 + 8 is r = 2 g8 + 1; the P
// fragment uses the same token order.
template <class C, int R>
WSVD_DEV void consume_imma_i8(const AttnArgs& a, const Unit& g, uint8_t* smem, uint64_t* full, uint64_t* empty,
                              int& slot, uint32_t& phase, int warp, int lane) {
    constexpr int K32 = (R + 31) / 32;
    constexpr int UV = R / 16;
    constexpr int GPW = C::GPW;
    static_assert(GPW % 2 == 0, "32-token P.V k-steps pair the warp's 16-token groups");
    const int g8 = lane >> 2, t4 = lane & 3;
    float m_w = -INFINITY, l = 0.f;
    const int ns = (g.ntok + C::ST - 1) / C::ST;
    uint32_t qf[K32][2];
    float s1 = 1.f, s2 = 1.f;
    float acc[UV][2];               // [unit][r = 16u + 2 g8 | 16u + 2 g8 + 1] (lanes t4 = 0)
#pragma unroll
    for (int u = 0; u < UV; ++u) acc[u][0] = acc[u][1] = 0.f;
    // P fragment byte gather: x = word of lane 8 t4 (tokens 2t4, 2t4+8), y = lane
    // 8 t4 + 4 (2t4+1, 2t4+9); words are [h(t0), h(t1), l(t0), l(t1)]
    const uint32_t asel = (g8 == 0) ? 0x5140u : 0x7362u;
    const int src_x = 8 * t4, src_y = 8 * t4 + 4;
    // scores of stage sl (tokens of this warp) -> sc; -INF past the unit's end
    auto scores = [&](int s, int sl, float (&sc)[GPW][2]) {
        const uint8_t* sp = smem + sl * C::STAGE;
        const uint32_t sbase = smem_u32(sp);
        const int rows = min(C::ST, g.ntok - s * C::ST);
        const __half2* sc2 = reinterpret_cast<const __half2*>(sp + C::ROWS);
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            int d[4] = {0, 0, 0, 0};
            const int ltok = tb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
            for (int kk = 0; kk < K32; ++kk) {
                uint32_t a0, a1, a2 = 0u, a3 = 0u;
                if (kk * 32 + 16 < R) {
                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2 + (lane >> 4)) * 16);
                    ldsm_x4(sbase + cache_swz(off), a0, a1, a2, a3);
                } else {
                    const uint32_t off = static_cast<uint32_t>(ltok * C::ROWB + (kk * 2) * 16);
                    ldsm_x2(sbase + cache_swz(off), a0, a1);
                }
                mma_s8_16832(d, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
            }
            const int t0 = tb + g8, t1 = tb + g8 + 8;
            if (a.dbg_scores && t4 == 0) {  // test hook: the int32 score accumulators (hi, lo query parts)
                int* dbg = a.dbg_scores + (static_cast<size_t>(g.bh) * a.cap + g.t0 + s * C::ST) * 2;
                if (t0 < rows) { dbg[2 * t0] = d[0]; dbg[2 * t0 + 1] = d[1]; }
                if (t1 < rows) { dbg[2 * t1] = d[2]; dbg[2 * t1 + 1] = d[3]; }
            }
            const float k0 = __low2float(sc2[t0]), k1 = __low2float(sc2[t1]);
            sc[grp][0] = (t4 == 0 && t0 < rows)
                ? fmaf(i2f_small(d[0]), s1, i2f_small(d[1]) * s2) * k0 : -INFINITY;
            sc[grp][1] = (t4 == 0 && t1 < rows)
                ? fmaf(i2f_small(d[2]), s1, i2f_small(d[3]) * s2) * k1 : -INFINITY;
        }
    };
    mbar_wait(&full[slot], phase);
    {
        const float* q = reinterpret_cast<const float*>(smem + slot * C::STAGE + C::QT_OFF);
        float mx = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) mx = fmaxf(mx, fabsf(q[k]));
        s1 = (mx == 0.f) ? 1.f : mx / 127.f;
        s2 = s1 / 254.f;
#pragma unroll
        for (int kk = 0; kk < K32; ++kk)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                uint32_t w1 = 0, w2 = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (kk * 32 + 16 * j >= R) break;
                    const float v = q[kk * 32 + 16 * j + 4 * t4 + e];
                    const float h = rintf(v / s1);
                    const float lo = rintf(fmaf(-h, s1, v) / s2);  // oracle: orc_i8_query_split
                    w1 |= (static_cast<uint32_t>(static_cast<int32_t>(h)) & 0xffu) << (8 * e);
                    w2 |= (static_cast<uint32_t>(static_cast<int32_t>(fminf(fmaxf(lo, -127.f), 127.f))) & 0xffu) << (8 * e);
                }
                qf[kk][j] = (g8 == 0) ? w1 : (g8 == 1 ? w2 : 0u);
            }
    }
    float sc[GPW][2];
    scores(0, slot, sc);
    for (int s = 0; s < ns; ++s) {
        // software pipeline: the next stage's score MMAs are issued before this
        // stage's softmax and P.V, so their latencies overlap
        const int cur = slot;
        if (++slot == C::STAGES) {
            slot = 0;
            phase ^= 1u;
        }
        float scn[GPW][2];
        if (s + 1 < ns) {
            mbar_wait(&full[slot], phase);
            scores(s + 1, slot, scn);
        }
        const uint8_t* sp = smem + cur * C::STAGE;
        const uint32_t sbase = smem_u32(sp);
        const __half2* sc2 = reinterpret_cast<const __half2*>(sp + C::ROWS);
        float lm = -INFINITY;
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) lm = fmaxf(lm, fmaxf(sc[grp][0], sc[grp][1]));
        if (__any_sync(0xffffffffu, lm > m_w + 8.f)) {
            const float wm = warp_max(lm);
            const float f = ex2(m_w - wm);
            l *= f;
#pragma unroll
            for (int u = 0; u < UV; ++u) {
                acc[u][0] *= f;
                acc[u][1] *= f;
            }
            m_w = wm;
        }
        // p' = p . s_V and the warp's stage maximum
        float pp[GPW][2];
        float bm = 0.f;
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int tb = (warp * GPW + grp) * 16;
            const float p0 = (sc[grp][0] == -INFINITY) ? 0.f : ex2(sc[grp][0] - m_w);
            const float p1 = (sc[grp][1] == -INFINITY) ? 0.f : ex2(sc[grp][1] - m_w);
            l += p0 + p1;
            pp[grp][0] = p0 * __high2float(sc2[tb + g8]);
            pp[grp][1] = p1 * __high2float(sc2[tb + g8 + 8]);
            bm = fmaxf(bm, fmaxf(pp[grp][0], pp[grp][1]));
        }
        bm = warp_max(bm);
        const float ps1 = bm * (1.f / 127.f), ps2 = ps1 * (1.f / 254.f);
        const float pi1 = bm > 0.f ? __fdividef(127.f, bm) : 0.f, pi2 = pi1 * 254.f;
        uint32_t pa[GPW];
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            const int h0 = f2i_rn_small(pp[grp][0] * pi1), h1 = f2i_rn_small(pp[grp][1] * pi1);
            const int l0 = max(-127, min(127, f2i_rn_small(fmaf(i2f_small(-h0), ps1, pp[grp][0]) * pi2)));
            const int l1 = max(-127, min(127, f2i_rn_small(fmaf(i2f_small(-h1), ps1, pp[grp][1]) * pi2)));
            const uint32_t w = (static_cast<uint32_t>(h0) & 0xffu) | ((static_cast<uint32_t>(h1) & 0xffu) << 8) |
                               ((static_cast<uint32_t>(l0) & 0xffu) << 16) | (static_cast<uint32_t>(l1) << 24);
            const uint32_t x = __shfl_sync(0xffffffffu, w, src_x), y = __shfl_sync(0xffffffffu, w, src_y);
            pa[grp] = (g8 < 2) ? __byte_perm(x, y, asel) : 0u;
        }
        // P.V transposed: D(16 r x 8) = V^T(16 r x 32 tok) . [h | l](32 tok x 8),
        // one MMA per 16-byte unit per 32 tokens; row g8 of the unit is r = 2 g8,
        // row g8 + 8 is r = 2 g8 + 1; lane (g8, t4 = 0) gets (h, l) sums of both
        int dI[UV][4];
#pragma unroll
        for (int u = 0; u < UV; ++u) dI[u][0] = dI[u][1] = dI[u][2] = dI[u][3] = 0;
#pragma unroll
        for (int j = 0; j < GPW / 2; ++j) {
            const int tb = (warp * GPW + 2 * j) * 16;
            const int vtok = tb + (lane & 7) + (lane >> 3) * 8;  // matrices: tokens 0-7, 8-15, 16-23, 24-31
#pragma unroll
            for (int u = 0; u < UV; ++u) {
                uint32_t m0, m1, m2, m3;
                const uint32_t off = static_cast<uint32_t>(vtok * C::ROWB + C::PART + u * 16);
                ldsm_x4_trans(sbase + cache_swz(off), m0, m1, m2, m3);
                mma_s8_16832(dI[u], __byte_perm(m0, m1, 0x6420), __byte_perm(m0, m1, 0x7531),
                             __byte_perm(m2, m3, 0x6420), __byte_perm(m2, m3, 0x7531), pa[2 * j], pa[2 * j + 1]);
            }
        }
#pragma unroll
        for (int u = 0; u < UV; ++u) {
            acc[u][0] = fmaf(i2f_small(dI[u][0]), ps1, fmaf(i2f_small(dI[u][1]), ps2, acc[u][0]));
            acc[u][1] = fmaf(i2f_small(dI[u][2]), ps1, fmaf(i2f_small(dI[u][3]), ps2, acc[u][1]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur]);
#pragma unroll
        for (int grp = 0; grp < GPW; ++grp) {
            sc[grp][0] = scn[grp][0];
            sc[grp][1] = scn[grp][1];
        }
    }
    const float lsum = warp_sum(l);
    float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * kMaxWarps + warp) * (R + 2);
    if (t4 == 0) {
#pragma unroll
        for (int u = 0; u < UV; ++u) {
            wsp[16 * u + 2 * g8] = acc[u][0];
            wsp[16 * u + 2 * g8 + 1] = acc[u][1];
        }
    }
    if (lane == 0) {
        wsp[R] = m_w;
        wsp[R + 1] = lsum;
    }
}

// One chunk per (sequence, head) -- max_chunks == 1, no fixed chunk length --
// means one CTA holds every partial of a unit, so the attention kernel merges
// them itself and the combine launch is skipped.  Latent outputs only (the
// layer step): the operator API's B_V up-projection stays in the combine
// kernel, whose 128 threads per head do it in parallel (one warp inside the
// attention kernel measured 4x slower for the whole launch).
__host__ __device__ inline bool attn_finalizes(const AttnArgs& a) {
    return a.chunk == 0 && (a.max_chunks == 1 || a.cluster > 1) && a.out == nullptr && !a.no_finalize;
}

// Merge of one unit's nw warp partials (fixed warp order, SoftmaxState::merge,
// decode.cpp:59-75) by one warp into the latent output -- the combine kernel's
// work for a single chunk.  The partials were written by this CTA's warps
// before a CTA barrier.
// Merged (m, l, acc) of one unit's nw warp partials, fixed warp order.
template <int R>
WSVD_DEV void unit_state(const AttnArgs& a, int bh, int ck, int nw, int lane, float& M, float& L,
                         float (&acc)[(R + 31) / 32]) {
    constexpr int RI = (R + 31) / 32;
    const float* wsb = a.ws + (static_cast<size_t>(bh) * a.max_chunks + ck) * kMaxWarps * (R + 2);
    M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, wsb[w * (R + 2) + R]);
    L = 0.f;
#pragma unroll
    for (int i = 0; i < RI; ++i) acc[i] = 0.f;
    for (int w = 0; w < nw; ++w) {
        const float m = wsb[w * (R + 2) + R];
        if (m == -INFINITY) continue;
        const float f = ex2(m - M);
        L = fmaf(wsb[w * (R + 2) + R + 1], f, L);
#pragma unroll
        for (int i = 0; i < RI; ++i)
            if (lane + 32 * i < R) acc[i] = fmaf(wsb[w * (R + 2) + lane + 32 * i], f, acc[i]);
    }
}

// Cluster merge (a.cluster = C CTAs = the C chunks of one (sequence, head),
// one unit per CTA): chunk ck < C-1 writes its merged state into the last
// CTA's shared memory (DSMEM) and arrives on its barrier; the last CTA merges
// the chunks in chunk order and writes the latent output -- no combine launch.
template <int R>
WSVD_DEV void cluster_merge_unit(const AttnArgs& a, int bh, int ck, int nw, int lane, float* cst, uint64_t* cbar) {
    constexpr int RI = (R + 31) / 32;
    const int C = a.cluster;
    float M, L, acc[RI];
    unit_state<R>(a, bh, ck, nw, lane, M, L, acc);
    if (ck < C - 1) {
        const uint32_t dst = cluster_map(smem_u32(cst + ck * (R + 2)), static_cast<uint32_t>(C - 1));
#pragma unroll
        for (int i = 0; i < RI; ++i)
            if (lane + 32 * i < R) st_cluster_f32(dst + 4u * (lane + 32 * i), acc[i]);
        if (lane == 0) {
            st_cluster_f32(dst + 4u * R, M);
            st_cluster_f32(dst + 4u * (R + 1), L);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(cluster_map(smem_u32(cbar), static_cast<uint32_t>(C - 1)));
        return;
    }
    mbar_wait_cluster(cbar, 0u);
    float M2 = -INFINITY, L2 = 0.f, a2[RI];
#pragma unroll
    for (int i = 0; i < RI; ++i) a2[i] = 0.f;
    for (int c = 0; c < C; ++c) {  // chunk order; the last chunk is this CTA's own state
        const float mc = c < C - 1 ? cst[c * (R + 2) + R] : M;
        const float lc = c < C - 1 ? cst[c * (R + 2) + R + 1] : L;
        if (mc == -INFINITY) continue;
        const float Mn = fmaxf(M2, mc);
        const float fo = ex2(M2 - Mn), fc = ex2(mc - Mn);
        L2 = fmaf(lc, fc, L2 * fo);
#pragma unroll
        for (int i = 0; i < RI; ++i) {
            const float ac = c < C - 1 ? (lane + 32 * i < R ? cst[c * (R + 2) + lane + 32 * i] : 0.f) : acc[i];
            a2[i] = fmaf(ac, fc, a2[i] * fo);
        }
        M2 = Mn;
    }
#pragma unroll
    for (int i = 0; i < RI; ++i)
        if (a.vlat && lane + 32 * i < R) a.vlat[static_cast<size_t>(bh) * R + lane + 32 * i] = a2[i] / L2;
}

template <int R>
WSVD_DEV void finalize_unit(const AttnArgs& a, int bh, int nw, int lane) {
    constexpr int RI = (R + 31) / 32;  // latent columns per lane
    const float* wsb = a.ws + static_cast<size_t>(bh) * a.max_chunks * kMaxWarps * (R + 2);
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, wsb[w * (R + 2) + R]);
    float L = 0.f, acc[RI];
#pragma unroll
    for (int i = 0; i < RI; ++i) acc[i] = 0.f;
    for (int w = 0; w < nw; ++w) {
        const float m = wsb[w * (R + 2) + R];
        if (m == -INFINITY) continue;  // a warp that saw no token
        const float f = ex2(m - M);
        L = fmaf(wsb[w * (R + 2) + R + 1], f, L);
#pragma unroll
        for (int i = 0; i < RI; ++i)
            if (lane + 32 * i < R) acc[i] = fmaf(wsb[w * (R + 2) + lane + 32 * i], f, acc[i]);
    }
    float vt[RI];
#pragma unroll
    for (int i = 0; i < RI; ++i) {
        vt[i] = acc[i] / L;
        if (a.vlat && lane + 32 * i < R) a.vlat[static_cast<size_t>(bh) * R + lane + 32 * i] = vt[i];
    }
}

template <int CD, int R, int V>
__global__ void __launch_bounds__(Cfg<CD, R, V>::THREADS, 1) decode_attn_kernel(const AttnArgs a) {
    using C = Cfg<CD, R, V>;
    constexpr int NC = C::NC, EPC = C::EPC;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* empty = full + C::STAGES;
    float* red = reinterpret_cast<float*>(smem + C::RED_OFF);
    // in-kernel merge (attn_finalizes): unit slots between the consumers and
    // the helper warp, 16 units deep
    __shared__ uint64_t ufull[16], uempty[16];
    __shared__ uint64_t cbar;                  // cluster merge: the other chunks' states landed
    __shared__ float cst[8 * (R + 2)];         // cluster merge: chunk states written by the peers

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t cap = static_cast<size_t>(a.cap);

    // Rows (and int8 scales) past a stage's valid end are read by the MMAs
    // (times p = 0) and must be finite: each slot's first stage is copied
    // whole (the cache and scale allocations carry a stage of padding), so
    // later partial stages leave finite stale rows -- no ring zeroing.
    if (tid == 0) {
        for (int i = 0; i < C::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], C::NW);
        }
        for (int i = 0; i < 16; ++i) {
            mbar_init(&ufull[i], C::NW);
            mbar_init(&uempty[i], 1);
        }
        mbar_init(&cbar, a.cluster > 1 ? a.cluster - 1 : 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (a.cluster > 1) cluster_sync_all();  // every CTA's cbar is initialised before a remote arrive
    griddep_wait();  // the appended row, qt and the length come from the predecessor
    griddep_launch_dependents();
    const int len = *a.d_len + a.len_add;
    if (len <= 0) return;
    int nch, chunk;
    chunking(a, len, nch, chunk);
    const int n_units = a.B * a.nh * nch;

    // ======================================================== producer warp
    if (warp == C::NW) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int slot = 0, issued = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const Unit g = unit_geom(u, nch, chunk, len);
                const uint8_t* src = a.cache + (static_cast<size_t>(g.bh) * cap + g.t0) * C::ROWB;
                const __half2* ssrc = a.cscale + static_cast<size_t>(g.bh) * cap + g.t0;
                for (int s = 0; s * C::ST < g.ntok; ++s) {
                    const int rows = min(C::ST, g.ntok - s * C::ST);
                    // whole 16-byte units; the swizzle only permutes within 1 KB blocks,
                    // so copy the covering blocks (rows past the end are masked)
                    const bool first = issued++ < C::STAGES;  // the slot's first use: copy it whole
                    const uint32_t rbytes = first ? static_cast<uint32_t>(C::ST * C::ROWB)
                        : static_cast<uint32_t>(min(C::ST * C::ROWB, ((rows * C::ROWB + 1023) / 1024) * 1024));
                    const uint32_t sbytes = (CD == I8) ? (first ? static_cast<uint32_t>(C::ST * 4)
                                                                : static_cast<uint32_t>((rows * 4 + 15) & ~15))
                                                       : 0u;
                    const uint32_t qbytes = (s == 0) ? static_cast<uint32_t>(R * 4) : 0u;
                    mbar_wait(&empty[slot], phase ^ 1u);
                    uint8_t* dst = smem + slot * C::STAGE;
                    mbar_arrive_expect_tx(&full[slot], rbytes + sbytes + qbytes);
                    tma_bulk_g2s_stream(dst, src + static_cast<size_t>(s) * C::ST * C::ROWB, rbytes,
                                        &full[slot], pol);
                    if (CD == I8)
                        tma_bulk_g2s_stream(dst + C::ROWS, ssrc + s * C::ST, sbytes, &full[slot], pol);
                    if (s == 0)
                        tma_bulk_g2s(dst + C::QT_OFF, a.qt + static_cast<size_t>(g.bh) * R, qbytes, &full[slot]);
                    if (++slot == C::STAGES) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ========================================================= helper warp
    // merges each unit's warp partials as the consumers publish them (off the
    // consumers' path: a merge costs ~2 L2 round trips)
    if (warp == C::NW + 1) {
        if constexpr (!(V & 4)) {
            if (attn_finalizes(a)) {
                int jl = 0;
                for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++jl) {
                    const int us = jl & 15;
                    mbar_wait(&ufull[us], static_cast<uint32_t>(jl >> 4) & 1u);
                    const Unit ug = unit_geom(u, nch, chunk, len);
                    if (a.cluster > 1)
                        cluster_merge_unit<R>(a, ug.bh, ug.chunk, C::NW, lane, cst, &cbar);
                    else
                        finalize_unit<R>(a, ug.bh, C::NW, lane);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&uempty[us]);
                }
            }
        }
        return;
    }

    // ====================================================== consumer warps
    const int g8 = lane >> 2, t4 = lane & 3;
    int slot = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit g = unit_geom(u, nch, chunk, len);
        float m_w = -INFINITY, l = 0.f;
        const int ns = (g.ntok + C::ST - 1) / C::ST;

        if (g.ntok <= 0) {
            // an empty trailing chunk (cluster mode at short lengths): no stage
            // was issued for it; publish an empty state
            float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * kMaxWarps + warp) * (R + 2);
            for (int j = lane; j < R; j += 32) wsp[j] = 0.f;
            if (lane == 0) {
                wsp[R] = -INFINITY;
                wsp[R + 1] = 0.f;
            }
        } else if constexpr ((C::MMA || C::IMMA) && (V & 4)) {
            // pipeline probe (WSVD_ATTN_VARIANT bit 2): drain the stages without
            // computing -- the streaming ceiling of this producer structure
            const int ns = (g.ntok + C::ST - 1) / C::ST;
            for (int s = 0; s < ns; ++s) {
                mbar_wait(&full[slot], phase);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == C::STAGES) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        } else if constexpr (C::MMA) {
            consume_mma<C, R, (V & 1)>(a, g, smem, full, empty, slot, phase, warp, lane);
        } else if constexpr (C::IMMA && (C::BIG != static_cast<bool>(V & 16))) {
            // int8 P.V on the int8 tensor cores where 1024-token stages fit (r <= 32),
            // else (measured faster at r = 48) the f16 P.V; bit 4 swaps them
            consume_imma_i8<C, R>(a, g, smem, full, empty, slot, phase, warp, lane);
        } else if constexpr (C::IMMA) {
            consume_mma_i8<C, R>(a, g, smem, full, empty, slot, phase, warp, lane);
        } else {
            // ------------------------------------------ CUDA-core path (f32, int8)
            float qr[NC][EPC];
            float acc[NC][EPC];
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int e = 0; e < EPC; ++e) acc[c][e] = 0.f;
            for (int s = 0; s < ns; ++s) {
                mbar_wait(&full[slot], phase);
                const uint8_t* sp = smem + slot * C::STAGE;
                if (s == 0) {
                    const float* q = reinterpret_cast<const float*>(sp + C::QT_OFF);
#pragma unroll
                    for (int c = 0; c < NC; ++c)
#pragma unroll
                        for (int e = 0; e < EPC; ++e) qr[c][e] = q[c * EPC + e];
                }
                const int rows = min(C::ST, g.ntok - s * C::ST);
                const bool valid = tid < rows;
                const uint32_t sbase = smem_u32(sp);
                const uint32_t rlog = static_cast<uint32_t>(tid * C::ROWB);
                float sk = 1.f, sv = 1.f;
                if (CD == I8) {
                    const __half2 scv = reinterpret_cast<const __half2*>(sp + C::ROWS)[tid];
                    sk = __low2float(scv);
                    sv = __high2float(scv);
                }
                float sacc[2] = {0.f, 0.f};
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    float f[EPC];
                    chunk_to_f32<CD>(lds128(sbase + cache_swz(rlog + c * 16)), f);
#pragma unroll
                    for (int e = 0; e < EPC; ++e) sacc[e & 1] = fmaf(qr[c][e], f[e], sacc[e & 1]);
                }
                const float scv = valid ? (sacc[0] + sacc[1]) * sk : -INFINITY;
                const float wm = warp_max(scv);
                if (wm > m_w) {
                    const float f = ex2(m_w - wm);
                    l *= f;
#pragma unroll
                    for (int c = 0; c < NC; ++c)
#pragma unroll
                        for (int e = 0; e < EPC; ++e) acc[c][e] *= f;
                    m_w = wm;
                }
                if (valid) {
                    const float p = ex2(scv - m_w);
                    l += p;
                    const float pv = p * sv;
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        float f[EPC];
                        chunk_to_f32<CD>(lds128(sbase + cache_swz(rlog + C::PART + c * 16)), f);
#pragma unroll
                        for (int e = 0; e < EPC; ++e) acc[c][e] = fmaf(pv, f[e], acc[c][e]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == C::STAGES) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
            // reduce 32 lanes through a shared-memory transpose
            float* wr = red + warp * 32 * C::RSTRIDE;
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int e = 0; e < EPC; e += 4)
                    *reinterpret_cast<float4*>(wr + lane * C::RSTRIDE + c * EPC + e) =
                        make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]);
            const float lsum = warp_sum(l);
            float* wsp = a.ws + ((static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * kMaxWarps + warp) * (R + 2);
            for (int j = lane; j < R; j += 32) {
                float sum = 0.f;
#pragma unroll 8
                for (int r = 0; r < 32; ++r) sum += wr[r * C::RSTRIDE + j];
                wsp[j] = sum;
            }
            if (lane == 0) {
                wsp[R] = m_w;
                wsp[R + 1] = lsum;
            }
            __syncwarp();  // scratch reuse by the next unit
        }
        // each warp published its own partial (m, l, acc[R])
        if constexpr (!(V & 4)) {
            if (attn_finalizes(a)) {
                // hand unit g to the helper warp (its slot must be free: the
                // helper has merged the unit 16 before)
                __syncwarp();
                if (lane == 0) {
                    const int jl = (u - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x);
                    mbar_wait(&uempty[jl & 15], (static_cast<uint32_t>(jl >> 4) & 1u) ^ 1u);
                    mbar_arrive(&ufull[jl & 15]);
                }
            }
        }
    }
}

// Split-KV combine (SoftmaxState::merge, decode.cpp:59-75, over the chunk x
// warp partials in a fixed order) and the single B_V up-projection per head
// (decode.cpp:198-203).  One CTA per (sequence, head).
inline int combine_smem(int max_chunks, int ppc, int R) {
    return (max_chunks * ppc * (R + 3) + R + (R > 128 ? R : 128) + 8) * 4;
}

__global__ void __launch_bounds__(128) attn_combine_kernel(const AttnArgs a, int parts_per_chunk) {
    extern __shared__ float sm[];  // parts [np][R+2], then vt [R]
    const int bh = blockIdx.x, tid = threadIdx.x, R = a.R;
    griddep_wait();
    griddep_launch_dependents();
    const int len = *a.d_len + a.len_add;
    if (len <= 0) return;
    int nch, chunk;
    chunking(a, len, nch, chunk);
    const int np = nch * parts_per_chunk;
    float* part = sm;
    float* vt = sm + a.max_chunks * parts_per_chunk * (R + 2);
    // stage every partial of this (sequence, head) with coalesced loads
    // (workspace layout [bh][max_chunks][kMaxWarps][R+2]; this variant used
    // the first parts_per_chunk warp slots of each chunk)
    const int pw = parts_per_chunk * (R + 2);
    const float* wsb = a.ws + static_cast<size_t>(bh) * a.max_chunks * kMaxWarps * (R + 2);
    const int n = np * (R + 2);
    // 8 independent L2 loads in flight per thread (the partials were just
    // written by the attention kernel and sit in L2)
    for (int i0 = tid; i0 < n; i0 += 8 * 128) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * 128;
            const int c = i / pw, r = i - c * pw;
            v[u] = i < n ? __ldcg(wsb + static_cast<size_t>(c) * kMaxWarps * (R + 2) + r) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * 128 < n) part[i0 + u * 128] = v[u];
    }
    __syncthreads();
    // parallel merge: block max of the partial maxima, per-partial factors,
    // then G = 128 / R thread groups each sum a fixed residue class of the
    // partials for every latent column (fixed order: deterministic)
    float* fac = vt + R;             // [np]
    float* red = fac + a.max_chunks * parts_per_chunk;  // [max(128, R)] + [4] + [4]
    const int warp = tid >> 5, lane = tid & 31;
    float M = -INFINITY;
    for (int p = tid; p < np; p += 128) M = fmaxf(M, part[p * (R + 2) + R]);
    M = warp_max(M);
    float* wred = red + (R > 128 ? R : 128);
    if (lane == 0) wred[warp] = M;
    __syncthreads();
    M = fmaxf(fmaxf(wred[0], wred[1]), fmaxf(wred[2], wred[3]));
    float Lp = 0.f;
    for (int p = tid; p < np; p += 128) {
        const float m = part[p * (R + 2) + R];
        const float f = m == -INFINITY ? 0.f : ex2(m - M);  // a warp that saw no token of its chunk
        fac[p] = f;
        Lp = fmaf(part[p * (R + 2) + R + 1], f, Lp);
    }
    Lp = warp_sum(Lp);
    if (lane == 0) wred[4 + warp] = Lp;
    __syncthreads();
    const float L = (wred[4] + wred[5]) + (wred[6] + wred[7]);
    const int G = R >= 128 ? 1 : 128 / R;
    for (int i = tid; i < G * R; i += 128) {
        const int g = i / R, r = i - g * R;
        float s = 0.f;
        for (int p = g; p < np; p += G) s = fmaf(part[p * (R + 2) + r], fac[p], s);
        red[i] = s;
    }
    __syncthreads();
    for (int r = tid; r < R; r += 128) {
        float acc = 0.f;
        for (int g = 0; g < G; ++g) acc += red[g * R + r];
        vt[r] = acc / L;
        if (a.vlat) a.vlat[static_cast<size_t>(bh) * R + r] = acc / L;
    }
    if (a.out == nullptr) return;  // the layer step folds B_V into W_o
    __syncthreads();
    const int h = bh % a.nh;
    const size_t bvo = static_cast<size_t>(h) * R * a.H;
    for (int col = tid; col < a.H; col += blockDim.x) {
        float o = 0.f;
#pragma unroll 8
        for (int j = 0; j < R; ++j) o = fmaf(vt[j], load_b(a.bv, a.bdtype, bvo + j * a.H + col), o);
        if (a.bdtype == I8) o *= a.bv_scale[h * a.H + col];
        a.out[static_cast<size_t>(bh) * a.H + col] = o;
    }
}

int g_combine_smem_attr = 0;

template <int CD, int R, int V>
cudaError_t launch_v(const AttnArgs& a, cudaStream_t s) {
    using C = Cfg<CD, R, V>;
    if constexpr (!C::OK) {
        return cudaErrorInvalidValue;
    } else {
        auto k = decode_attn_kernel<CD, R, V>;
        static bool attr_set = false;
        if (!attr_set) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e != cudaSuccess) return e;
            attr_set = true;
        }
        cudaError_t e = launch_pdl_cluster(k, dim3(a.grid), dim3(C::THREADS), C::SMEM, s, a.cluster, a);
        if (e != cudaSuccess) return e;
        if (attn_finalizes(a) && !(V & 4)) return cudaSuccess;  // merged in the kernel
        const int csmem = combine_smem(a.max_chunks, C::NW, R);
        if (csmem > g_combine_smem_attr) {  // one (non-template) kernel: track its attribute globally
            e = cudaFuncSetAttribute(attn_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
            if (e != cudaSuccess) return e;
            g_combine_smem_attr = csmem;
        }
        return launch_pdl(attn_combine_kernel, dim3(a.B * a.nh), dim3(128), csmem, s, a,
                          static_cast<int>(C::NW));
    }
}

// tensor-core variant (bf16 cache); WSVD_ATTN_VARIANT overrides it for A/B runs
int attn_variant() {
    static const int v = [] {
        const char* e = std::getenv("WSVD_ATTN_VARIANT");
        return e ? (std::atoi(e) & 63) : kDefaultVariant;
    }();
    return v;
}

template <int CD, int R>
cudaError_t launch_t(const AttnArgs& a, cudaStream_t s) {
    if constexpr (R > 64) {
        return launch_v<CD, R, 0>(a, s);  // large ranks: the default consumers only
    } else if constexpr (CD == I8) {
        // WSVD_ATTN_VARIANT bit 3: the CUDA-core int8 consumer; bit 1: 16 consumer warps (A/B)
        if (attn_variant() & 8) return launch_v<CD, R, 8>(a, s);
        if (attn_variant() & 4) return launch_v<CD, R, 4>(a, s);  // streaming probe (no compute)
        // bit 4: the f16 P.V consumer (consume_mma_i8); bit 5: 512-token stages
        switch (attn_variant() & 50) {
            case 0: return launch_v<CD, R, 0>(a, s);
            case 2: return launch_v<CD, R, 2>(a, s);
            case 16: return launch_v<CD, R, 16>(a, s);
            case 32: return launch_v<CD, R, 32>(a, s);
            default: return launch_v<CD, R, 18>(a, s);
        }
    } else if constexpr (CD != BF16) {
        return launch_v<CD, R, 0>(a, s);
    } else {
        if constexpr (R != 32) {
            return launch_v<CD, R, kDefaultVariant>(a, s);
        } else {
            switch (attn_variant() & 7) {
                case 0: return launch_v<CD, R, 0>(a, s);
                case 1: return launch_v<CD, R, 1>(a, s);
                case 2: return launch_v<CD, R, 2>(a, s);
                case 3: return launch_v<CD, R, 3>(a, s);
                case 4: return launch_v<CD, R, 4>(a, s);
                default: return launch_v<CD, R, 6>(a, s);
            }
        }
    }
}

template <int CD>
int smem_for(int R) {
    switch (R) {
        case 16: return Cfg<CD, 16>::SMEM;
        case 32: return Cfg<CD, 32>::SMEM;
        case 48: return Cfg<CD, 48>::SMEM;
        case 64: return Cfg<CD, 64>::SMEM;
        case 80: return Cfg<CD, 80>::SMEM;
        case 96: return Cfg<CD, 96>::SMEM;
        case 112: return Cfg<CD, 112>::SMEM;
        case 128: return Cfg<CD, 128>::SMEM;
    }
    return 0;
}

template <int CD>
cudaError_t launch_cd(const AttnArgs& a, cudaStream_t s) {
    switch (a.R) {
        case 16: return launch_t<CD, 16>(a, s);
        case 32: return launch_t<CD, 32>(a, s);
        case 48: return launch_t<CD, 48>(a, s);
        case 64: return launch_t<CD, 64>(a, s);
        case 80: return launch_t<CD, 80>(a, s);
        case 96: return launch_t<CD, 96>(a, s);
        case 112: return launch_t<CD, 112>(a, s);
        case 128: return launch_t<CD, 128>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

int attn_smem_bytes(int cdtype, int R) {
    switch (cdtype) {
        case F32: return smem_for<F32>(R);
        case BF16: return smem_for<BF16>(R);
        case I8: return smem_for<I8>(R);
    }
    return 0;
}

int attn_parts_per_chunk() { return kMaxWarps; }

int attn_occupancy(int cdtype, int R) {
    return attn_smem_bytes(cdtype, R) > 0 ? 1 : 0;  // persistent: one CTA per SM
}

cudaError_t launch_attn_combine(const AttnArgs& a, int parts_per_chunk, cudaStream_t s) {
    const int csmem = combine_smem(a.max_chunks, parts_per_chunk, a.R);
    if (csmem > g_combine_smem_attr) {
        cudaError_t e = cudaFuncSetAttribute(attn_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
        if (e != cudaSuccess) return e;
        g_combine_smem_attr = csmem;
    }
    return launch_pdl(attn_combine_kernel, dim3(a.B * a.nh), dim3(128), csmem, s, a, parts_per_chunk);
}

template <int CD, int R>
bool cluster_ok_t(int Cn) {
    using C = Cfg<CD, R, 0>;
    if constexpr (!C::OK) {
        return false;
    } else {
        auto k = decode_attn_kernel<CD, R, 0>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(Cn);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(Cn);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return n >= 1;
    }
}

template <int CD>
bool cluster_ok_cd(int R, int Cn) {
    switch (R) {
        case 16: return cluster_ok_t<CD, 16>(Cn);
        case 32: return cluster_ok_t<CD, 32>(Cn);
        case 48: return cluster_ok_t<CD, 48>(Cn);
        case 64: return cluster_ok_t<CD, 64>(Cn);
        case 80: return cluster_ok_t<CD, 80>(Cn);
        case 96: return cluster_ok_t<CD, 96>(Cn);
        case 112: return cluster_ok_t<CD, 112>(Cn);
        case 128: return cluster_ok_t<CD, 128>(Cn);
    }
    return false;
}

cudaError_t launch_decode_attn(const AttnArgs& a, cudaStream_t s) {
    switch (a.cdtype) {
        case F32: return launch_cd<F32>(a, s);
        case BF16: return launch_cd<BF16>(a, s);
        case I8: return launch_cd<I8>(a, s);
    }
    return cudaErrorInvalidValue;
}

bool attn_cluster_ok(int cdtype, int R, int Cn) {
    static int memo[3][5][4] = {};  // 0 unknown, 1 yes, 2 no; [dtype][R/16][log2 C - 1]
    const int ri = R / 16, ci = Cn == 2 ? 0 : Cn == 4 ? 1 : Cn == 8 ? 2 : 3;
    if (R % 16 || ri < 1 || ri > 4 || ci > 2 || cdtype < 0 || cdtype > 2) return false;
    int& m = memo[cdtype][ri][ci];
    if (m == 0) {
        bool ok = false;
        switch (cdtype) {
            case F32: ok = cluster_ok_cd<F32>(R, Cn); break;
            case BF16: ok = cluster_ok_cd<BF16>(R, Cn); break;
            case I8: ok = cluster_ok_cd<I8>(R, Cn); break;
        }
        m = ok ? 1 : 2;
    }
    return m == 1;
}

}  // namespace wsvd_k
