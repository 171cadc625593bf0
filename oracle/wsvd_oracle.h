/*
 * wsvd_oracle.h -- CPU oracle for the WSVD per-head low-rank decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * algorithm (/root/reference/proj, C++20, fp64).  It is the checker the parity
 * tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the
 * CUDA path against.  The product (paper_2604_02570_b200/) never links, loads
 * or calls anything in oracle/.
 *
 * Parity pinning: every fp64 routine here is checked against the reference
 * itself (oracle/_ref/libwsvdref.so, compiled from the reference sources by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/
 * (generated from the reference by tests/golden/make_golden.py).
 *
 * Reference citations are path:line into /root/reference/proj.
 */
#ifndef WSVD_ORACLE_H
#define WSVD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- rng ----
 * Restates src/rng.cpp: std::mt19937_64 seeded with splitmix64-hashed
 * (seed, stream) pairs (rng.cpp:19-21), 53-bit uniforms (rng.hpp:24),
 * Box-Muller normals with a cached spare (rng.cpp:23-36), reject-sampled
 * index (rng.cpp:38-44). */
typedef struct {
    uint64_t mt[312];
    int mti;
    int has_spare;
    double spare;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
void orc_rng_stream(orc_rng* r, uint64_t seed, uint64_t stream_id);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
uint64_t orc_rng_index(orc_rng* r, uint64_t n);
/* Rng::normal_matrix (rng.cpp:46-50): row-major fill, stddev * normal(). */
void orc_rng_normal_fill(orc_rng* r, double* out, size_t n, double stddev);

/* ------------------------------------------------------------ counters ---
 * decode::TrafficCounter (decode.hpp:13-49); stream order matches the
 * reference enum: LatentK, LatentV, FullK, FullV, WeightsB, Query, Output. */
enum { ORC_LATENT_K = 0, ORC_LATENT_V, ORC_FULL_K, ORC_FULL_V, ORC_WEIGHTS_B, ORC_QUERY,
       ORC_OUTPUT, ORC_NSTREAMS };
typedef struct {
    uint64_t loads[ORC_NSTREAMS];
    uint64_t stores[ORC_NSTREAMS];
    uint64_t flops[ORC_NSTREAMS];
} orc_counter;

/* --------------------------------------------------------------- layer ---
 * decode::LayerFactors (decode.hpp:71-79) in a padded, ragged-rank-aware
 * layout: A[h][role][E][rmax], B[h][role][rmax][H]; ranks[h][role] is the
 * true rank (role 0=q, 1=k, 2=v).  Only the first rank columns of A / rows
 * of B are ever read, as in the reference. */
typedef struct {
    size_t E, H, nh, rmax;
    const int32_t* ranks; /* [nh][3] */
    const double* A;      /* [nh][3][E][rmax] */
    const double* B;      /* [nh][3][rmax][H] */
} orc_layer;

/* Latent cache of ONE sequence: ck/cv [nh][cap][rmax] (reference keeps a
 * growing Matrix per head, decode.hpp:83-96). */

/* decode::append_token (decode.cpp:127-153) for one token of one sequence:
 * writes ck/cv rows at position pos and q_out[nh][H]. */
int orc_append_token(const orc_layer* f, double* ck, double* cv, size_t cap, size_t pos,
                     const double* x, double* q_out, orc_counter* c);

/* decode::fused_decode_step (decode.cpp:155-206): tiled online softmax with
 * per-row key reconstruction and latent-V accumulation.  Returns 0, or
 * -1 (ShapeError: empty cache) / -2 (ConfigError: tile 0). */
int orc_fused_decode_step(const orc_layer* f, const double* ck, const double* cv, size_t cap,
                          size_t len, const double* q, size_t tile, double* out, orc_counter* c);

/* Test-oracle of tests/test_decode.cpp:68-94 / acceptance_main.cpp:109-135:
 * rebuild dense K,V, full-row softmax. */
void orc_reconstruct_then_attend(const orc_layer* f, const double* ck, const double* cv,
                                 size_t cap, size_t len, const double* q, double* out);

/* SoftmaxState (decode.cpp:35-75), exposed for the merge tests. */
typedef struct {
    double max_score, denom;
    double* acc; /* caller-owned, width w */
    size_t w;
    int empty;
} orc_softmax;
void orc_softmax_observe(orc_softmax* s, double score, const double* value);
void orc_softmax_merge(orc_softmax* s, const orc_softmax* o);

/* traffic_report (decode.cpp:452-487), fused mode only. */
int orc_traffic_match_fused(const orc_counter* c, uint64_t seq_len, uint64_t n_heads,
                            uint64_t head_dim, uint64_t rank_k);

/* Batched driver: the same per-sequence routines over B sequences, split
 * over `threads` pthreads by (sequence, head) -- the CPU baseline "port"
 * arm.  ck/cv [B][nh][cap][rmax], x [B][E], q [B][nh][H], out [B][nh][H]. */
int orc_batched_append(const orc_layer* f, double* ck, double* cv, size_t B, size_t cap,
                       size_t pos, const double* x, double* q_out, int threads);
int orc_batched_decode(const orc_layer* f, const double* ck, const double* cv, size_t B,
                       size_t cap, size_t len, const double* q, size_t tile, double* out,
                       int threads);
/* the same, also returning every (sequence, head)'s latent output
 * v~ = acc / denom (decode.cpp:198, before the B_V up-projection),
 * latent [B][nh][rmax] (zero past the head's V rank) */
int orc_batched_decode_latent(const orc_layer* f, const double* ck, const double* cv, size_t B,
                              size_t cap, size_t len, const double* q, size_t tile, double* out,
                              double* latent, int threads);

/* ------------------------------------------------- storage-format rules ---
 * The device stores factors, tokens and latents in narrower formats; the
 * oracle applies the SAME rounding to its inputs so that both sides compute
 * on identical values.  double -> float is IEEE round-to-nearest-even;
 * float -> bf16 / fp16 are RNE as well (cvt.rn on the device). */
float orc_f32(double v);
double orc_bf16(double v);             /* double -> f32 -> bf16, as a double */
uint16_t orc_bf16_bits(float v);       /* f32 -> bf16 bits (RNE) */
uint16_t orc_f16_bits(float v);        /* f32 -> fp16 bits (RNE, subnormals kept) */
float orc_f16_to_f32(uint16_t h);

/* quant.cpp:34-37 */
int orc_qmax(int bits);
/* quant.cpp:99-119: per-column RTN with clip-grid search (0.50..1.00 step
 * 0.05, first grid point wins ties); fp64, llround (ties away from zero).
 * w [rows][cols] -> q [rows][cols] int8, scales [cols], returns clip. */
double orc_quantize_weight(const double* w, size_t rows, size_t cols, int bits, int8_t* q,
                           double* scales);
/* quant.cpp:131-150: per-row activation quantization (fp64 reference). */
void orc_quantize_activation_f64(const double* x, size_t rows, size_t cols, int bits,
                                 int8_t* q, double* scales);

/* Composed INT path: the device arithmetic, restated
 * with the same fp32 operation sequence. */
/* In-place fp32 FWHT of v[n] (n power of two), stages len = 1,2,4,...;
 * (lo, hi) -> (lo + hi, lo - hi); then times `scale`. */
void orc_fwht_f32(float* v, size_t n, float scale);
/* S1 rotation of one token: block-diagonal H_blk/sqrt(blk), blk = E when E
 * is a power of two, else 128 (E = 5120 = 40 x 128). */
size_t orc_rot_block(size_t E);
void orc_rotate_token_f32(const float* x, float* xr, size_t E);
/* Per-token int8: m = max|v|, s = m / 127 (fp32), s = 1 if m == 0,
 * q = clamp(roundf(v / s), -127, 127).  Returns s. */
float orc_quant_token_f32(const float* v, size_t n, int8_t* q);
/* int32 latent accumulate acc[c] = sum_i xq[i] * wq[c][i] over K-major
 * weights wq [ncols][E]. */
void orc_int_gemv(const int8_t* xq, const int8_t* wq, size_t E, size_t ncols, int32_t* acc);
/* Dequantised latent: ((float)acc * sx) * sw, fp32, no contraction. */
float orc_dequant_latent(int32_t acc, float sx, float sw);
/* Int8 cache row rule (quantize_activation rule per (token, head, role)):
 * s = f16(max|c| / 127); s := 1 when it is 0; q = clamp(roundf(c / s)).
 * Returns the fp16 bits of the scale. */
uint16_t orc_quant_cache_row(const float* c, size_t n, int8_t* q);
/* Sign-extend the nibbles of a packed int4 row (lo nibble = even index). */
void orc_unpack_int4(const uint8_t* packed, size_t n, int8_t* out);

/* INT8-cache attention, the integer score stage of the absorbed form
 * (attn.cu consume_mma_i8 / consume_imma_i8): the fp32
 * absorbed query split into int8 hi / lo parts, and every cached row's int32
 * accumulators against them, acc [L][2] = (hi, lo).  R <= 256. */
void orc_i8_query_split(const float* q, size_t R, int8_t* h, int8_t* l, float* s1, float* s2);
void orc_i8_scores(const float* q, size_t R, const int8_t* rows, size_t L, size_t ld, int32_t* acc);

#ifdef __cplusplus
}
#endif
#endif
