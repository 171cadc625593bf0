/*
 * wsvd_b200.h -- C ABI of the B200-native WSVD decode path.
 *
 * This is the drop-in boundary for the reference's decode operator API
 * (/root/reference/proj/include/wsvd/decode.hpp, namespace wsvd::decode).
 * Everything below is extern "C", takes plain pointers and sizes, and never
 * exposes CUDA or torch types (streams are passed as `void*` holding a
 * cudaStream_t; NULL = the legacy default stream).  The C++ host API
 * (include/wsvd/decode.hpp in this repo) and the Python package are built on
 * these entry points; INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Ownership: the library owns all device memory behind a handle; tensors
 * passed as `const float* x` etc. are DEVICE pointers unless the name ends in
 * `_host`.  Every call returns WSVD_OK or a negative status; the message of
 * the last failure on the calling thread is returned by wsvd_last_error().
 * The status codes mirror the reference exception hierarchy
 * (include/wsvd/errors.hpp:9-31) and its CLI exit codes
 * (tools/wsvd_main.cpp:632-653).
 *
 * There is no CPU fallback: on a machine without an sm_100 device every
 * compute entry point fails with WSVD_ECUDA.
 */
#ifndef WSVD_B200_H
#define WSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WSVD_ABI_VERSION 1

/* status codes (errors.hpp:9-31) */
#define WSVD_OK 0
#define WSVD_ESHAPE (-1)   /* ShapeError: empty cache, head-count / width mismatch */
#define WSVD_ECONFIG (-2)  /* ConfigError: tile 0, unknown dtype, bad option */
#define WSVD_ENUMERIC (-3) /* NumericError: non-finite input, counter mismatch */
#define WSVD_ECUDA (-4)    /* CUDA runtime / launch failure, no device */
#define WSVD_EIO (-5)      /* IoError */
#define WSVD_ENCCL (-6)    /* NCCL unavailable or failed */

/* storage formats */
typedef enum {
    WSVD_F32 = 0,  /* fp32 storage, fp32 math (config 1) */
    WSVD_BF16 = 1, /* bf16 storage, fp32 accumulate (config 2) */
    WSVD_I8 = 2,   /* int8 values + scales, int32-exact accumulate (W8A8, INT8 cache) */
    WSVD_I4 = 3    /* int4 values packed two per byte + scales (W4A8 weights) */
} wsvd_dtype;

/* roles of a factored head (factorize.hpp:15 Role::Q/K/V) */
typedef enum { WSVD_ROLE_Q = 0, WSVD_ROLE_K = 1, WSVD_ROLE_V = 2 } wsvd_role;

/* traffic streams, decode.hpp:16-24 order; counters are [loads(7) | stores(7) | flops(7)] */
typedef enum {
    WSVD_STREAM_LATENT_K = 0,
    WSVD_STREAM_LATENT_V,
    WSVD_STREAM_FULL_K,
    WSVD_STREAM_FULL_V,
    WSVD_STREAM_WEIGHTS_B,
    WSVD_STREAM_QUERY,
    WSVD_STREAM_OUTPUT,
    WSVD_STREAM_COUNT
} wsvd_stream;

typedef struct wsvd_layer_s* wsvd_layer_t; /* device factors of one layer (or head shard) */
typedef struct wsvd_cache_s* wsvd_cache_t; /* device latent cache of `batch` sequences */
typedef struct wsvd_comm_s* wsvd_comm_t;   /* NCCL communicator for the O-proj all-reduce */

/* Geometry of a layer object; replaces decode::LayerFactors' embed_dim /
 * head_dim / heads.size() (decode.hpp:76-79).  A head-sharded rank holds
 * heads [head_offset, head_offset + n_heads) of the full layer. */
typedef struct {
    int32_t embed_dim;    /* E */
    int32_t head_dim;     /* H */
    int32_t n_heads;      /* heads held by this object */
    int32_t head_offset;  /* first global head (0 when unsharded) */
    int32_t weight_dtype; /* wsvd_dtype of A and B factors */
    int32_t act_rotation; /* I8/I4 only: 1 = activations are rotated by S1 = Hadamard
                             (linalg.cpp:219-243; block H_128 when E is not a power of 2)
                             before per-token quantisation (quant.cpp:131-150) */
    int32_t device;       /* CUDA device ordinal */
} wsvd_layer_desc;

const char* wsvd_last_error(void);
int wsvd_abi_version(void);
/* number of visible sm_100 devices (0 on a machine without one) */
int wsvd_device_count(int32_t* n);

/* ---------------------------------------------------------------- layer --
 * ranks: [n_heads][3] true ranks (q, k, v) per head, as in
 * factorize::HeadFactors::rank (factorize.hpp:20-27).  Ranks may differ per
 * head and role; the device zero-pads every head to one common width, which
 * leaves results unchanged (SURVEY.md section 8(b) "Ragged ranks"). */
int wsvd_layer_create(const wsvd_layer_desc* desc, const int32_t* ranks, wsvd_layer_t* out);
int wsvd_layer_destroy(wsvd_layer_t layer);
/* padded latent width used on the device */
int wsvd_layer_rank_pad(wsvd_layer_t layer, int32_t* rpad);

/* Upload one head's factors given in the reference HeadFactors layout:
 * a row-major E x rank, b row-major rank x H, fp64 (factorize.hpp:20-27).
 * F32 / BF16 layers round them (double -> float -> bf16, RNE).  I8 / I4
 * layers quantise them on the host with the reference weight quantiser
 * (quant.cpp:99-119, per-column scales, clip-grid search), after rotating a
 * by S1 when act_rotation is set (insert_rotations, quant.cpp:182-189). */
int wsvd_layer_set_head(wsvd_layer_t layer, int32_t head, int32_t role, const double* a,
                        const double* b);
/* Upload already-quantised factors (quant::QuantizedFactors, quant.hpp:98-107;
 * checkpoint files .q.a.i8 / .q.a.scale.wsvd, checkpoint.cpp:220-244):
 * a_q row-major E x rank int8 (I4: values in [-7, 7]), a_scales[rank];
 * b_q row-major rank x H, b_scales[H].  The factors must already carry the
 * rotations (S1 a S2^T, S2 b). */
int wsvd_layer_set_head_quantized(wsvd_layer_t layer, int32_t head, int32_t role,
                                  const int8_t* a_q, const double* a_scales, const int8_t* b_q,
                                  const double* b_scales);
/* O-projection rows of this shard (pipeline.cpp:329 `heads_row * W_o`):
 * w_o_rows is row-major (n_heads * H) x e_out fp64, the rows of W_o that
 * multiply this shard's heads.  dtype F32 or BF16. */
int wsvd_layer_set_oproj(wsvd_layer_t layer, const double* w_o_rows, int32_t e_out,
                         int32_t dtype);

/* ---------------------------------------------------------------- cache --
 * decode::LatentCache (decode.hpp:83-96) for `batch` sequences that advance
 * together; capacity is the maximum length (preallocated, no regrowth).
 * cache_dtype F32 / BF16 / I8 (I8 rows carry one fp16 scale per
 * (token, head, K|V), the quantize_activation rule). */
int wsvd_cache_create(wsvd_layer_t layer, int32_t batch, int32_t capacity, int32_t cache_dtype,
                      wsvd_cache_t* out);
int wsvd_cache_destroy(wsvd_cache_t cache);
/* Raises the capacity to at least `capacity` rows, keeping the committed rows
 * (reallocates and copies; synchronises the device).  The reference's cache
 * grows row by row (Matrix::append_row); the C++ drop-in grows by doubling. */
int wsvd_cache_grow(wsvd_cache_t cache, int32_t capacity);
int wsvd_cache_capacity(wsvd_cache_t cache, int32_t* capacity);
/* empties the cache (length 0) */
int wsvd_cache_reset(wsvd_cache_t cache);
/* decode with another factor set of identical geometry (the reference passes
 * the LayerFactors to every call, decode.hpp:100-111); WSVD_ESHAPE when the
 * head count, padded rank, E or H differ (decode.cpp:159-162). */
int wsvd_cache_bind_layer(wsvd_cache_t cache, wsvd_layer_t layer);
int wsvd_cache_length(wsvd_cache_t cache, int32_t* len);
/* Re-reads the committed length from the device into the host mirror (after
 * steps replayed inside a caller's CUDA graph, which the host does not see). */
int wsvd_cache_sync_length(wsvd_cache_t cache, int32_t* len);
/* Benchmark utility: rows 0..length-1 of every (sequence, head) become
 * synthetic N(0, scale^2) latents in the cache format (no projection), and the
 * cache length becomes `length` -- the reference's decode-bench prefill of
 * random latents (wsvd_main.cpp:393-396) without the per-token projection. */
int wsvd_cache_fill_synthetic(wsvd_cache_t cache, int32_t length, uint64_t seed, float scale);
/* LatentCache::push + bump_length for every sequence and head at once:
 * ck / cv host fp64 [batch][n_heads][rpad] (entries beyond a head's rank are
 * ignored and stored as 0). */
int wsvd_cache_push_host(wsvd_cache_t cache, const double* ck, const double* cv);
/* latent_k(h) / latent_v(h) of sequence b, dequantised to fp64:
 * ck, cv host [len][rpad]. */
int wsvd_cache_read_host(wsvd_cache_t cache, int32_t b, int32_t head, double* ck, double* cv);
/* raw device rows of sequence b, head h: rows [len][row_bytes] and (I8 only)
 * fp16 scale pairs [len][2]; for bit-exact checks. */
int wsvd_cache_row_bytes(wsvd_cache_t cache, int32_t* row_bytes);
/* Attention algorithm of a cache (both give the reference's results up to fp32
 * reassociation; SURVEY.md 7 "hard parts"):
 *   WSVD_ATTN_ABSORBED     scores against the absorbed query qt = q . B_K^T
 *                          (r MACs per cached token; default, all dtypes);
 *   WSVD_ATTN_EXPLICIT_TC  the reference's explicit key rebuild
 *                          key_j = C_K[j] . B_K (decode.cpp:188) on tcgen05
 *                          tensor cores into TMEM (bf16 cache and factors,
 *                          rank 32, head dim 128; ECONFIG otherwise). */
#define WSVD_ATTN_ABSORBED 0
#define WSVD_ATTN_EXPLICIT_TC 1
int wsvd_cache_set_attention_mode(wsvd_cache_t cache, int32_t mode);
int wsvd_cache_attention_mode(wsvd_cache_t cache, int32_t* mode);

/* ---- checkpoints of the reference (wsvd::ckpt, src/checkpoint.cpp:168-333):
 * manifest.json + WSVDMAT1 fp64 / WSVDI8T1 int8 tensor files.  Host-only
 * readers (no device needed) and a device-layer loader.  IO and format
 * errors return WSVD_EIO (the reference's IoError). */
/* info = {embed_dim, head_dim, n_heads, n_layers, weight_bits, activation_bits,
 *         has_factors, has_quantized} */
int wsvd_ckpt_info(const char* dir, int64_t info[8]);
/* fp64 factors of (layer, head, role): a [E][rank], b [rank][H]; null buffers
 * only return the rank */
int wsvd_ckpt_head(const char* dir, int32_t layer, int32_t head, int32_t role, int32_t* rank, double* a, double* b);
/* quantised factors Q(S1 A S2^T) [E][rank], Q(S2 B) [rank][H] and their
 * per-column scales (quant.cpp:344-358) */
int wsvd_ckpt_head_quantized(const char* dir, int32_t layer, int32_t head, int32_t role, int32_t* rank,
                             int8_t* a_q, double* a_scales, int8_t* b_q, double* b_scales);
/* a dense weight by manifest name (e.g. "layer0.w_o"); *rows x *cols must hold
 * it when out is non-null */
int wsvd_ckpt_weight(const char* dir, const char* name, int64_t* rows, int64_t* cols, double* out);
/* device layer of heads [head_begin, head_end) of `layer`: quantised factors
 * for WSVD_I8 / WSVD_I4 (act_rotation on), fp64 factors otherwise; with
 * oproj_dtype >= 0 also the W_o rows of those heads (wsvd_layer_set_oproj) */
int wsvd_layer_load_checkpoint(const char* dir, int32_t layer, int32_t head_begin, int32_t head_end,
                               int32_t weight_dtype, int32_t oproj_dtype, int32_t device, wsvd_layer_t* out);

/* How wsvd_layer_step(_graph/_host) runs for this cache: *fused = 1 when the
 * whole step is the single persistent kernel of step.cu (bf16, rank 32,
 * batch <= 32), 0 for the multi-kernel path; *launches = kernels per step. */
int wsvd_cache_step_info(wsvd_cache_t cache, int32_t* fused, int32_t* launches);
int wsvd_cache_read_raw(wsvd_cache_t cache, int32_t b, int32_t head, void* rows_host,
                        uint16_t* scales_host);

/* ------------------------------------------------------------ operators --
 * append_token (decode.cpp:127-153), batched over the cache's sequences:
 * x [batch][E] fp32, q_out [batch][n_heads][H] fp32 (may be NULL).  Writes
 * the new latent rows at position length() and increments the length. */
int wsvd_append_token(wsvd_cache_t cache, const float* x, float* q_out, void* stream);
/* Appends T tokens per sequence at once (prefill): x [batch][T][E] fp32. */
int wsvd_prefill(wsvd_cache_t cache, const float* x, int32_t T, void* stream);
/* fused_decode_step (decode.cpp:155-206), batched: q [batch][n_heads][H] fp32,
 * out [batch][n_heads][H] fp32.  tile_len mirrors TileConfig::tile_len
 * (decode.hpp:51-53): 0 is rejected (WSVD_ECONFIG); any other value gives
 * the same result up to reassociation, as in the reference. */
int wsvd_fused_decode_step(wsvd_cache_t cache, const float* q, int32_t tile_len, float* out,
                           void* stream);
/* The attention kernel alone, with the absorbed query of the most recent
 * wsvd_append_token / wsvd_fused_decode_step on this cache (no append):
 * out [batch][n_heads][H].  Used to time the dominant kernel in isolation. */
int wsvd_decode_attention(wsvd_cache_t cache, float* out, void* stream);
/* One attention-layer decode step for every sequence (pipeline.cpp:320-329):
 * append x, attend with that token's own query, O-project this shard's
 * heads.  y [batch][e_out] fp32 = this shard's partial sum (complete when
 * unsharded).  attn_out [batch][n_heads][H] may be NULL. */
int wsvd_layer_step(wsvd_cache_t cache, const float* x, float* attn_out, float* y, void* stream);
/* Same, through host buffers: copies x_host [batch][E] in, y_host
 * [batch][e_out] out (pinned or pageable), synchronising the stream. */
int wsvd_layer_step_host(wsvd_cache_t cache, const float* x_host, float* y_host, void* stream);
/* Capture wsvd_layer_step into a CUDA graph bound to (x, y, stream); later
 * calls with the same arguments replay it (1 launch instead of ~5). */
int wsvd_layer_step_graph(wsvd_cache_t cache, const float* x, float* y, void* stream);

/* ------------------------------------------------------ feed-forward --
 * The reference model's per-layer feed-forward after the O-projection
 * (pipe::decode_factored, pipeline.cpp:330-334): out = tanh(o . ff1) . ff2,
 * ff1 [embed_dim][hidden], ff2 [hidden][embed_dim] (row-major fp32, stored on
 * the device as bf16 W-tiles); two skinny tensor-core GEMMs (the projection
 * kernel), the split sums with the tanh fused.  o, out: [rows][embed_dim]
 * fp32 device buffers (rows <= 128; out may alias o). */
typedef struct wsvd_ffn_s* wsvd_ffn_t;
int wsvd_ffn_create(int32_t embed_dim, int32_t hidden, const float* ff1, const float* ff2, int32_t device,
                    wsvd_ffn_t* out);
int wsvd_ffn_destroy(wsvd_ffn_t ffn);
int wsvd_ffn_forward(wsvd_ffn_t ffn, const float* o, int32_t rows, float* out, void* stream);

/* -------------------------------------------------------------- chains --
 * pipe::decode_factored's layer loop (pipeline.cpp:318-336) over the
 * attention blocks of n layers, one token per sequence: layer 0 takes x,
 * layer l > 0 takes layer l - 1's output ys[l - 1] (the attention blocks of a
 * decode stack chained, no FFN between them), and every layer appends to its
 * own cache.  caches[l]: n distinct caches of one geometry (batch, heads,
 * embed_dim, rank, e_out == embed_dim), each bound to its layer with an
 * O-projection; ys[l]: [batch][E] fp32 device buffers.  When every layer runs
 * the fused step (wsvd_cache_step_info) and n <= 32, the chain is ONE
 * persistent kernel launch -- the next layer's projection weights load while
 * a layer finishes; otherwise it is n wsvd_layer_step calls. */
int wsvd_chain_step(wsvd_cache_t const* caches, int32_t n, const float* x, float* const* ys, void* stream);
/* Same through host buffers, synchronising the stream: x_host [batch][E] in,
 * y_host [batch][E] = the last layer's output out (pinned or pageable); the
 * intermediate outputs stay on the device. */
int wsvd_chain_step_host(wsvd_cache_t const* caches, int32_t n, const float* x_host, float* y_host,
                         void* stream);

/* Copies internal per-step buffers of the last append to the host, for
 * bit-exact parity checks of the integer path: what = 0 quantised tokens
 * int8 [rows][Kp]; 1 token scales fp32 [rows]; 2 projection accumulators
 * summed over K splits, int32 (I8/I4) or fp32, [rows][n_heads*3*rpad];
 * 3 absorbed queries fp32 [batch][n_heads][rpad].  *bytes is in/out. */
int wsvd_cache_debug_copy(wsvd_cache_t cache, int32_t what, void* host, int64_t* bytes);
/* Test hook, INT8 caches: flags bit 0 makes the following attention launches
 * record every cached row's int32 score accumulators -- the rows times the
 * hi and lo int8 parts of the split absorbed query --
 * read back with wsvd_cache_debug_copy(what = 5) as int32
 * [batch][n_heads][capacity][2].  Off by default (no cost). */
int wsvd_cache_set_debug(wsvd_cache_t cache, int32_t flags);

/* ----------------------------------------------------- host utilities ---
 * The reference weight quantiser (quant::quantize_weight, quant.cpp:99-119):
 * per-column symmetric round-to-nearest (ties away from zero), clip ratio
 * searched over 0.50..1.00 (first minimum wins), zero columns get scale 1.
 * w row-major rows x cols fp64 -> q int8 (values in +-(2^(bits-1)-1)),
 * scales[cols], *clip.  Host only; what wsvd_layer_set_head uses for I8/I4. */
int wsvd_quantize_weight(const double* w, int64_t rows, int64_t cols, int32_t bits, int8_t* q,
                         double* scales, double* clip);

/* ----------------------------------------------------- traffic counters --
 * Closed-form TrafficCounter increments (decode.cpp:132-149, 176-203;
 * test_decode.cpp:229-292) for one call on this cache, ADDED to counter21
 * (= [loads(7) | stores(7) | flops(7)] per stream, times batch). */
int wsvd_traffic_append(wsvd_cache_t cache, uint64_t* counter21);
int wsvd_traffic_fused(wsvd_cache_t cache, int32_t tile_len, uint64_t* counter21);

/* ------------------------------------------------------ multi-GPU (NCCL) --
 * Head-sharded layers: each rank holds n_heads/G
 * heads and the matching W_o rows; after wsvd_layer_step the partial y is
 * summed across ranks by one ncclAllReduce.  NCCL is loaded at run time
 * (dlopen libnccl.so.2); WSVD_ENCCL when absent. */
int wsvd_nccl_unique_id(uint8_t id[128]);
int wsvd_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                     wsvd_comm_t* out);
int wsvd_comm_destroy(wsvd_comm_t comm);
int wsvd_allreduce_sum_f32(wsvd_comm_t comm, float* buf, int64_t count, void* stream);

/* ------------------------------------------- comparison baselines (dense.cu) --
 * The reference's uncompressed and shared-latent baselines on the device
 * (decode.hpp:114-170; decode.cpp:208-432), fp32: dense per-head K/V caches
 * (FullKvCache) with the attention of eager_decode_step / flash_decode_step
 * (one softmax over the cached rows; the two schedules differ only in their
 * traffic tallies), and the GEMV / GEMM blocks of append_token_dense,
 * append_token_shared and shared_decode_step(materialize).  Device pointers;
 * row-major matrices. */
typedef struct wsvd_dense_cache_s* wsvd_dense_cache_t;
int wsvd_dense_cache_create(int32_t n_heads, int32_t head_dim, int32_t device, wsvd_dense_cache_t* out);
int wsvd_dense_cache_destroy(wsvd_dense_cache_t cache);
int wsvd_dense_cache_length(wsvd_dense_cache_t cache, int32_t* len);
/* FullKvCache::push of every head + bump_length: k, v [n_heads][head_dim] */
int wsvd_dense_cache_append(wsvd_dense_cache_t cache, const float* k, const float* v, void* stream);
/* keys(head) / values(head) to the host as fp64 [len][head_dim] */
int wsvd_dense_cache_read_host(wsvd_dense_cache_t cache, int32_t head, double* k, double* v);
/* softmax(q . k_j / sqrt(H)) . V per head: q, out [n_heads][head_dim];
 * tile_len as TileConfig (0 -> WSVD_ECONFIG) */
int wsvd_dense_decode_step(wsvd_dense_cache_t cache, const float* q, int32_t tile_len, float* out, void* stream);
/* the same over caller buffers keys / values [n_heads][ld][head_dim] (len rows
 * valid), scores scratch [n_heads][ld] */
int wsvd_dense_attend(const float* keys, const float* values, int32_t n_heads, int32_t len, int32_t ld,
                      int32_t head_dim, const float* q, float* scores, float* out, void* stream);
/* y[n] = sum_k x[k] w[k][n] (vec_mat, decode.cpp:97-110) */
int wsvd_vecmat_f32(const float* x, const float* w, int32_t k, int32_t n, float* y, void* stream);
/* c[m][n] = a[m][k] . b[k][n] (matmul, matrix.cpp) */
int wsvd_matmul_f32(const float* a, const float* b, int32_t m, int32_t k, int32_t n, float* c, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WSVD_B200_H */
