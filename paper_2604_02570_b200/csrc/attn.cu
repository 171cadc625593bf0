// attn.cu -- fused per-head low-rank decode attention for sm_100a.
//
// Replaces wsvd::decode::fused_decode_step (reference src/decode.cpp:155-206).
// The reference rebuilds every key, key_j = C_K[j] . B_K (decode.cpp:188),
// at L*r*H MACs per head.  Scores only need q . key_j, so this kernel uses
// the algebraically identical absorbed query qt = q . B_K^T (r values,
// computed once per (sequence, head) by the append epilogue or
// launch_absorb_query) and streams the latent rows once:
//
//   s_j   = qt . C_K[j]                      (log2 domain, 1/sqrt(H) folded in)
//   state = online softmax over s_j with the accumulator in latent-V space
//           (decode.cpp:35-57, 192: acc += p_j * C_V[j])
//   out   = (acc / denom) . B_V              (decode.cpp:198-203, once per head)
//
// Results equal the reference up to floating-point reassociation.
//
// HBM layout: cache[b][h][t][ C_K(R) | C_V(R) ] (one row per token, R = padded
// rank), int8 rows carry a half2 (s_K, s_V) scale per token in a parallel
// array.  Work is split into units (sequence, head, chunk of `chunk` tokens);
// a persistent grid walks the units round-robin.  Per CTA, one thread keeps a
// ring of TMA bulk copies (cp.async.bulk + mbarrier complete_tx) of
// 128-token stages in flight across unit boundaries while 4 warps consume:
// one token per thread per stage, warp-uniform running max, per-lane
// accumulators.  At a unit's end the CTA reduces its 128 partial states and
// either finalises (single chunk) or publishes a partial (m, l, acc[R]); the
// last CTA to finish a (sequence, head) merges the partials in chunk order
// (SoftmaxState::merge, decode.cpp:59-75) and applies B_V -- the split-KV
// combine is fused, deterministic and needs no second launch.
#include "common.cuh"
#include "kernels.h"

using namespace wsvd_dev;

namespace wsvd_k {

namespace {

constexpr int kThreads = 128;
constexpr int kStageTok = 128;

template <int CD, int R>
struct Cfg {
    static constexpr int EB = (CD == F32) ? 4 : (CD == BF16 ? 2 : 1);
    static constexpr int EPC = 16 / EB;        // elements per 16-byte chunk
    static constexpr int PART = R * EB;        // bytes of the K (and V) half
    static constexpr int NC = PART / 16;       // chunks per half
    static constexpr int ROWB = 2 * PART;
    static constexpr bool POW2 = (NC & (NC - 1)) == 0;
    // per-lane rotation of the chunk order keeps ld.shared.v4 at <= 2-way bank
    // conflicts for rows that are multiples of 128 B (or 64 B)
    static constexpr bool ROT = POW2 && NC > 1 && (ROWB % 64 == 0);
    static constexpr int ROT_SHIFT = ROWB >= 128 ? 0 : 1;
    static constexpr int SC = (CD == I8) ? 4 * kStageTok : 0;
    static constexpr int STAGE = kStageTok * ROWB + SC;
    static constexpr int RSTRIDE = R + 4;      // floats per lane row of the reduction scratch
    static constexpr int RED = 4 * 32 * RSTRIDE * 4;
    static constexpr int BUDGET = 110 * 1024;
    static constexpr int ST_RAW = (BUDGET - RED - 2048) / STAGE;
    static constexpr int STAGES = ST_RAW > 8 ? 8 : (ST_RAW < 2 ? 2 : ST_RAW);
    static constexpr int BAR_OFF = STAGES * STAGE;
    static constexpr int RED_OFF = BAR_OFF + 128;
    static constexpr int MISC_OFF = RED_OFF + RED;                  // wpart[4][R+2], vt[R]
    static constexpr int SMEM = MISC_OFF + (4 * (R + 2) + R + 8) * 4;
    static_assert(PART % 16 == 0, "latent half must be a multiple of 16 bytes");
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

struct Unit {
    int bh, chunk, t0, ntok;
};

WSVD_DEV Unit unit_geom(int u, int nch, int chunk, int len) {
    Unit g;
    g.bh = u / nch;
    g.chunk = u - g.bh * nch;
    g.t0 = g.chunk * chunk;
    g.ntok = min(chunk, len - g.t0);
    return g;
}

template <int CD, int R>
__global__ void __launch_bounds__(kThreads, 2) decode_attn_kernel(const AttnArgs a) {
    using C = Cfg<CD, R>;
    constexpr int NC = C::NC, EPC = C::EPC;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    float* red = reinterpret_cast<float*>(smem + C::RED_OFF);
    float* wpart = reinterpret_cast<float*>(smem + C::MISC_OFF);  // [4][R+2]
    float* vt = wpart + 4 * (R + 2);                               // [R]
    int* sflag = reinterpret_cast<int*>(vt + R);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int len = *a.d_len;
    if (len <= 0) return;
    const int nch = (len + a.chunk - 1) / a.chunk;
    const int n_units = a.B * a.nh * nch;
    const size_t cap = static_cast<size_t>(a.cap);

    if (tid == 0) {
        for (int i = 0; i < C::STAGES; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // ---------------- producer cursor (thread 0 only)
    int pu = blockIdx.x, ps = 0, pslot = 0;
    const uint64_t pol = policy_evict_first();
    auto issue_next = [&]() {
        // load the next stage of this CTA's unit sequence into pslot
        if (pu >= n_units) return;
        const Unit g = unit_geom(pu, nch, a.chunk, len);
        const int t = g.t0 + ps * kStageTok;
        const int rows = min(kStageTok, g.ntok - ps * kStageTok);
        uint8_t* dst = smem + pslot * C::STAGE;
        const uint32_t rbytes = static_cast<uint32_t>(rows * C::ROWB);
        uint32_t sbytes = 0;
        if (CD == I8) sbytes = static_cast<uint32_t>((rows * 4 + 15) & ~15);
        mbar_arrive_expect_tx(&bars[pslot], rbytes + sbytes);
        const uint8_t* src = a.cache + (static_cast<size_t>(g.bh) * cap + t) * C::ROWB;
        tma_bulk_g2s_stream(dst, src, rbytes, &bars[pslot], pol);
        if (CD == I8) {
            const __half2* ssrc = a.cscale + static_cast<size_t>(g.bh) * cap + t;
            tma_bulk_g2s_stream(dst + kStageTok * C::ROWB, ssrc, sbytes, &bars[pslot], pol);
        }
        pslot = (pslot + 1 == C::STAGES) ? 0 : pslot + 1;
        if (++ps * kStageTok >= g.ntok) {
            ps = 0;
            pu += gridDim.x;
        }
    };
    if (tid == 0)
        for (int i = 0; i < C::STAGES; ++i) issue_next();

    // ---------------- per-lane chunk rotation
    const int rot = C::ROT ? ((lane >> C::ROT_SHIFT) & (NC - 1)) : 0;
    uint32_t koff[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) koff[c] = static_cast<uint32_t>(((c + rot) % NC) * 16);

    int cslot = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit g = unit_geom(u, nch, a.chunk, len);

        // absorbed query chunks in this lane's rotated order
        float qr[NC][EPC];
        const float* qsrc = a.qt + static_cast<size_t>(g.bh) * R;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const float4* p4 = reinterpret_cast<const float4*>(qsrc + (koff[c] / 16) * EPC);
#pragma unroll
            for (int e = 0; e < EPC / 4; ++e) {
                const float4 v = __ldg(p4 + e);
                qr[c][4 * e] = v.x; qr[c][4 * e + 1] = v.y;
                qr[c][4 * e + 2] = v.z; qr[c][4 * e + 3] = v.w;
            }
        }
        float acc[NC][EPC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < EPC; ++e) acc[c][e] = 0.f;
        float m_w = -INFINITY, l = 0.f;

        const int ns = (g.ntok + kStageTok - 1) / kStageTok;
        for (int s = 0; s < ns; ++s) {
            mbar_wait(&bars[cslot], phase);
            const uint8_t* st = smem + cslot * C::STAGE;
            const int rows = min(kStageTok, g.ntok - s * kStageTok);
            const bool valid = tid < rows;
            const uint32_t row = smem_u32(st) + static_cast<uint32_t>(tid * C::ROWB);

            float sk = 1.f, sv = 1.f;
            if (CD == I8) {
                const __half2 sc = reinterpret_cast<const __half2*>(st + kStageTok * C::ROWB)[tid];
                sk = __low2float(sc);
                sv = __high2float(sc);
            }
            // ---- score: qt . C_K[t]
            float sacc[2] = {0.f, 0.f};
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                float f[EPC];
                chunk_to_f32<CD>(lds128(row + koff[c]), f);
#pragma unroll
                for (int e = 0; e < EPC; ++e) sacc[e & 1] = fmaf(qr[c][e], f[e], sacc[e & 1]);
            }
            const float sc = valid ? (sacc[0] + sacc[1]) * sk : -INFINITY;

            // ---- online softmax, warp-uniform running max (exp2 domain)
            const float wm = warp_max(sc);
            if (wm > m_w) {
                const float f = ex2(m_w - wm);
                l *= f;
#pragma unroll
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int e = 0; e < EPC; ++e) acc[c][e] *= f;
                m_w = wm;
            }
            const float p = valid ? ex2(sc - m_w) : 0.f;
            l += p;
            // ---- latent-V accumulate (rows past the stage end hold stale smem)
            if (valid) {
                const float pv = p * sv;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    float f[EPC];
                    chunk_to_f32<CD>(lds128(row + C::PART + koff[c]), f);
#pragma unroll
                    for (int e = 0; e < EPC; ++e) acc[c][e] = fmaf(pv, f[e], acc[c][e]);
                }
            }

            __syncthreads();  // slot fully consumed
            if (tid == 0) issue_next();
            cslot = (cslot + 1 == C::STAGES) ? 0 : cslot + 1;
            if (cslot == 0) phase ^= 1u;
        }

        // ---- reduce 32 lanes: transpose through shared memory
        float* wr = red + warp * 32 * C::RSTRIDE;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int e = 0; e < EPC; e += 4) {
                float4 v = make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]);
                *reinterpret_cast<float4*>(wr + lane * C::RSTRIDE + (koff[c] / 16) * EPC + e) = v;
            }
        const float lsum = warp_sum(l);
        __syncwarp();
        for (int j = lane; j < R; j += 32) {
            float s = 0.f;
#pragma unroll 8
            for (int r = 0; r < 32; ++r) s += wr[r * C::RSTRIDE + j];
            wpart[warp * (R + 2) + j] = s;
        }
        if (lane == 0) {
            wpart[warp * (R + 2) + R] = m_w;
            wpart[warp * (R + 2) + R + 1] = lsum;
        }
        __syncthreads();

        // ---- merge the 4 warps
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, wpart[w * (R + 2) + R]);
        float fw[4], L = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float mw = wpart[w * (R + 2) + R];
            fw[w] = (mw == -INFINITY) ? 0.f : ex2(mw - M);
            L = fmaf(wpart[w * (R + 2) + R + 1], fw[w], L);
        }
        float accj = 0.f;
        if (tid < R) {
#pragma unroll
            for (int w = 0; w < 4; ++w) accj = fmaf(wpart[w * (R + 2) + tid], fw[w], accj);
        }

        bool finalize = true;
        if (nch > 1) {
            float* wsu = a.ws + (static_cast<size_t>(g.bh) * a.max_chunks + g.chunk) * (R + 2);
            if (tid < R) wsu[tid] = accj;
            if (tid == R) wsu[R] = M;
            if (tid == R + 1) wsu[R + 1] = L;
            __threadfence();
            __syncthreads();
            if (tid == 0) *sflag = (atomicAdd(&a.counters[g.bh], 1) == nch - 1);
            __syncthreads();
            finalize = *sflag != 0;
            if (finalize) {
                __threadfence();
                const float* wsb = a.ws + static_cast<size_t>(g.bh) * a.max_chunks * (R + 2);
                M = -INFINITY;
                for (int c = 0; c < nch; ++c) M = fmaxf(M, __ldcg(wsb + c * (R + 2) + R));
                L = 0.f;
                accj = 0.f;
                for (int c = 0; c < nch; ++c) {
                    const float f = ex2(__ldcg(wsb + c * (R + 2) + R) - M);
                    L = fmaf(__ldcg(wsb + c * (R + 2) + R + 1), f, L);
                    if (tid < R) accj = fmaf(__ldcg(wsb + c * (R + 2) + tid), f, accj);
                }
                if (tid == 0) a.counters[g.bh] = 0;
            }
        }
        if (finalize) {
            // latent output, then one B_V up-projection (decode.cpp:198-203)
            if (tid < R) vt[tid] = accj / L;
            __syncthreads();
            const int h = g.bh % a.nh;
            const size_t bvo = static_cast<size_t>(h) * R * a.H;
            for (int col = tid; col < a.H; col += kThreads) {
                float o = 0.f;
                for (int j = 0; j < R; ++j) o = fmaf(vt[j], load_b(a.bv, a.bdtype, bvo + j * a.H + col), o);
                if (a.bdtype == I8) o *= a.bv_scale[h * a.H + col];
                a.out[static_cast<size_t>(g.bh) * a.H + col] = o;
            }
        }
        __syncthreads();  // scratch reuse by the next unit
    }
}

template <int CD, int R>
cudaError_t launch_t(const AttnArgs& a, cudaStream_t s) {
    using C = Cfg<CD, R>;
    auto k = decode_attn_kernel<CD, R>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    k<<<a.grid, kThreads, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int CD>
int smem_for(int R) {
    switch (R) {
        case 16: return Cfg<CD, 16>::SMEM;
        case 32: return Cfg<CD, 32>::SMEM;
        case 48: return Cfg<CD, 48>::SMEM;
        case 64: return Cfg<CD, 64>::SMEM;
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

int attn_occupancy(int cdtype, int R) {
    const int sm = attn_smem_bytes(cdtype, R);
    if (sm <= 0) return 0;
    int occ = (227 * 1024) / (sm + 1024);
    if (occ > 2) occ = 2;  // __launch_bounds__(128, 2)
    return occ < 1 ? 1 : occ;
}

cudaError_t launch_decode_attn(const AttnArgs& a, cudaStream_t s) {
    switch (a.cdtype) {
        case F32: return launch_cd<F32>(a, s);
        case BF16: return launch_cd<BF16>(a, s);
        case I8: return launch_cd<I8>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace wsvd_k
