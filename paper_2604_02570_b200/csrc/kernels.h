// kernels.h -- launch interface between the C ABI (capi.cu) and the kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace wsvd_k {

enum DType { F32 = 0, BF16 = 1, I8 = 2, I4 = 3 };

// ---------------------------------------------------------------- GEMM --
// Partial skinny GEMM  P[split][m][n] = sum_{k in split} X[m][k] * W[n][k]
// (W K-major).  bf16: X fp32 -> bf16, fp32 partials.  i8 / i4: X int8,
// int32 partials (exact).  f32: CUDA-core fp32.
// bf16 / i8 / i4 weights are W-tiles: [N/16][Kp/KS][16][KS bytes-of-row],
// 16-byte units of odd rows XOR 4 (see pack in capi.cu); f32 is plain [N][Kp].
struct GemmArgs {
    const void* W;   // W-tiles (bf16 / i8 / i4) or [N][Kp] (f32)
    const void* X;   // fp32 [M][ldx] (f32 / bf16 modes) or int8 [M][Kp]
    void* P;         // [splits][M][N] fp32 or int32
    int M, N, K;     // K: valid columns of X (fp32 modes); Kp: padded K
    int Kp, KS;      // KS: K per split (Kp % KS == 0)
    int ldx;         // row stride of fp32 X (elements)
    int wdtype;      // DType
    int grid;        // SM count: the streaming kernel runs floor(grid/splits)*splits CTAs
    int* commit_len; // non-null: one thread adds 1 to it (the layer step's length commit)
    int xsplit;      // bf16 only: X as hi + lo bf16 token tiles (fp32-grade activations), M <= 64
};
// true when M token rows with split KS fit the streaming kernel's shared memory
bool gemm_fits(int wdtype, int M, int KS);
// fp32 weights, M <= 4 token rows, KS in {256, 512, 1024}: the balanced row-piece GEMV
bool f32_rows_path(int M, int Kp, int KS);
// fp32 weights, M <= 4 token rows, one K split (KS == Kp <= 4096): the TMA-ring GEMV
bool f32_tma_path(int M, int Kp, int KS);
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s);

// Sum split partials into fp32 y [M][N] (fixed split order).
// act 1: tanh of the sum (the toy FFN's hidden activation); y_bf16: y is bf16
cudaError_t launch_reduce_partials(const float* P, int splits, int M, int N, void* y,
                                   cudaStream_t s, int act = 0, int y_bf16 = 0);

// ------------------------------------------- dense GEMM on tcgen05 (gemm_tc.cu) --
// D[M][N] = X[M][K] . W[N][K]^T, bf16 operands: X row-major [M][K], W K-chunk-
// major [K/64][N][64] (each 64-wide K slice of all rows contiguous), fp32
// accumulation in TMEM; M <= 128 token rows, N % 64 == 0 (64-column CTA
// tiles; up to four of a K split share each X chunk by TMA multicast), K % 64 == 0.
// One split: epilogue act 1 = tanh, out bf16 or fp32 [M][ldo]; `splits` > 1:
// fp32 partials [splits][M][ldo] for launch_reduce_partials.
struct TcGemmArgs {
    const void* X;
    const void* W;
    void* out;         // bf16 (out_bf16) or fp32 [M][ldo] after act; fp32 [splits][M][ldo] partials
    int M, N, K, ldo, splits, act, out_bf16;
    int ntiles, cl;    // set by launch_tc_gemm
    int ldm;           // partials: rows between K splits (0: M)
};
bool tc_gemm_supported(int M, int N, int K);
cudaError_t launch_tc_gemm(const TcGemmArgs& a, cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* x, void* y, size_t n, cudaStream_t s);  // n % 4 == 0
// bf16 W-tiles [N/16][Kp/ks][16][ks] (gemm.cu layout) -> K-chunk-major [Kp/64][N][64]
cudaError_t launch_wtiles_to_chunks(const void* wt, int N, int Kp, int ks, void* out, cudaStream_t s);

// ------------------------------------------------------ activation quant --
// Per token: optional S1 rotation (FWHT over blocks of rot_blk, times
// rot_scale), s = max|v|/127, q = clamp(roundf(v/s)); xq [M][Kp] zero-padded.
cudaError_t launch_act_quant(const float* x, int M, int E, int Kp, int rot, int rot_blk,
                             float rot_scale, int8_t* xq, float* sx, cudaStream_t s);

// ------------------------------------------------------ append epilogue --
struct AppendArgs {
    const void* P;        // projection partials [splits][M][Nrows] (fp32 or int32)
    int splits, M, Nrows;
    int wdtype;           // DType of projection (int modes dequantise)
    const float* a_scale; // [Nrows] per-row weight scales (int modes)
    const float* sx;      // [M] per-token activation scales (int modes)
    int T, B;             // tokens per sequence in this call, sequences (row m = t*B + b)
    int nh, R, H;         // local heads, padded rank, head dim
    // cache
    uint8_t* cache;       // [B][nh][cap][row_bytes]
    __half2* cscale;      // [B][nh][cap] (int8 cache)
    int cdtype, cap, row_bytes;
    int* d_len;           // committed length (read at start, += T by the last CTA)
    int* done;            // CTA completion counter (self-resetting)
    // query path (only when T == 1)
    const void* bq;       // B_Q [nh][R][H]
    const void* bk;       // B_K [nh][R][H]
    const float* bq_scale;  // [nh][H] (int modes)
    const float* bk_scale;
    int bdtype;
    float* q_out;         // [M][nh][H] or null
    float* qt;            // [M][nh][R] absorbed query (log2 domain) or null
    float qt_scale;       // log2(e) / sqrt(H)
    const float* mqk;     // [nh][R][R] qt_scale * B_Q . B_K^T (used when q_out is null)
    int commit;           // 1: the last CTA advances *d_len by T
};
cudaError_t launch_append_epilogue(const AppendArgs& a, cudaStream_t s);

// synthetic N(0, scale^2) latent rows 0..length-1 of every region (benchmarks)
cudaError_t launch_fill_synthetic(uint8_t* cache, __half2* cscale, int regions, int cap, int length, int R,
                                  int cdtype, int row_bytes, uint32_t seed, float scale, cudaStream_t s);

// host-provided rows [n][row_bytes] -> row `pos` of cache regions 0..n-1 (swizzled)
cudaError_t launch_push_rows(const uint8_t* rows, int n, uint8_t* cache, int cap, int row_bytes,
                             int pos, cudaStream_t s);

// q [B][nh][H] -> qt [B][nh][R] = qt_scale * q . B_K^T
cudaError_t launch_absorb_query(const float* q, int B, int nh, int R, int H, const void* bk,
                                const float* bk_scale, int bdtype, float qt_scale, float* qt,
                                cudaStream_t s);

// ------------------------------------------------------------ attention --
struct AttnArgs {
    const uint8_t* cache;   // [B][nh][cap][row_bytes]
    const __half2* cscale;  // [B][nh][cap]
    const float* qt;        // [B][nh][R]
    const void* bv;         // B_V [nh][R][H]
    const float* bv_scale;  // [nh][H]
    int bdtype;
    float* out;             // [B][nh][H] (null: latent output only)
    float* vlat;            // [B][nh][R] latent output acc/denom (may be null)
    float* ws;              // [B*nh][max_chunks][warps][R+2]
    int* counters;          // [B*nh], zero between launches (self-resetting)
    const int* d_len;       // committed rows (device); the kernel attends over *d_len + len_add
    int len_add;            // 1 when the step's own row is appended but not yet committed
    int B, nh, H, R, cap, chunk, max_chunks, cdtype, row_bytes;
    int grid;               // persistent CTAs
    int no_finalize;        // A/B switch: always merge in the combine kernel (WSVD_ATTN_COMBINE=1)
    int cluster;            // > 1: clusters of that many CTAs, one unit per CTA and exactly `cluster`
                            // chunks per (sequence, head); the chunks merge through DSMEM
    // explicit key reconstruction (attn_tc.cu): per-head B_K^T tiles and the query
    const uint8_t* bkt;     // [nh][attn_tc_btile_bytes()] bf16, MMA B-operand layout
    const float* q;         // [B][nh][H] query rows
    int* dbg_scores;        // test hook (int8 cache): [B*nh][cap][2] int32 score accumulators, or null
};
int attn_smem_bytes(int cdtype, int R);
int attn_occupancy(int cdtype, int R);  // resident CTAs per SM (0 if unsupported)
int attn_parts_per_chunk();             // warp partials published per unit
cudaError_t launch_decode_attn(const AttnArgs& a, cudaStream_t s);
// clusters of C attention CTAs can be scheduled (the cluster-merge mode)
bool attn_cluster_ok(int cdtype, int R, int C);
// split-KV combine alone (attn.cu): merges parts_per_chunk warp partials per chunk
cudaError_t launch_attn_combine(const AttnArgs& a, int parts_per_chunk, cudaStream_t s);

// tcgen05 explicit-reconstruction attention (attn_tc.cu): bf16 cache, R = 32, H = 128
bool attn_tc_supported(int cdtype, int R, int H, int bdtype);
int attn_tc_btile_bytes();
size_t attn_tc_btile_offset(int d, int r);
cudaError_t launch_decode_attn_tc(const AttnArgs& a, cudaStream_t s);  // + launch_attn_combine(a, 8)

// ------------------------------------------------- fused layer step (step.cu) --
// projection -> append -> attention -> merge -> folded O-projection as one
// persistent kernel (bf16 weights / cache, rank 32, batch <= 32), for one layer
// or for a chain of layers in one launch (layer l + 1's token = layer l's y:
// pipe::decode_factored's layer loop, pipeline.cpp:318-336, attention blocks
// only).
constexpr int kStepMaxLayers = 32;
struct StepLayer {         // one layer of the launch (all share the geometry below)
    const uint8_t* A;      // projection W-tiles (bf16, K split 512)
    const float* mqk;      // [nh][R][R]
    uint8_t* cache;        // [B][nh][cap][4R] bf16, swizzled
    int* counters;         // [B*nh] segments arrived per (sequence, head), self-resetting
    const uint8_t* Wo;     // folded O-projection W-tiles (bf16, K split 512)
    int* d_len;            // committed length (the new row goes to *d_len)
    float* y;              // [B][e_out] fp32 output; the next layer's token
    int cap;
    int pad_;
};
struct StepArgs {
    const float* x;        // [B][E] fp32 tokens of layer 0 (device, or mapped host memory when x_host)
    int x_host;            // x is pinned host memory: fetched once over the bus into xd
    int y_host;            // the last layer's y is mapped host memory (plain stores, whole tiles per CTA)
    float* xd;             // [B][E] device copy of a host x
    unsigned* xcnt;        // [kMaxSplits] per-K-split fetch counters (monotone)
    int* epoch;            // fused launches run so far (x-fetch counter generations)
    unsigned* bgen;        // grid-barrier generations completed so far
    unsigned* bar;         // grid barrier count (monotone, wrap-safe compares)
    unsigned* yflag;       // [grid][32] per CTA: layers whose O-projection outputs (y) it has written
    unsigned long long* xtag;  // [2][B][E/2] chained tokens (layer parity): bf16 pairs | layer-step tag << 32
    int xtagged;           // 1: pair O-projections also write xtag; the next projection stages from it
    unsigned* p1gen;       // layer steps run so far (the flags' base)
    int g3;                // A/B: 1 a grid barrier between chained layers instead of the y flags
    int short_seg;         // rows: a first segment shorter than this is processed second (0: never)
    int g1;                // A/B: 1 a grid barrier after the projection instead of the per-CTA
                           // flags; 2 the cache stream starts at this CTA's projection end
    unsigned long long* Pt;  // [splits][B][Nrows] projection partials, each (layer-step tag << 32 | fp32 bits)
    float* ws;             // [grid][kMaxU][36] segment states (step_ws_bytes)
    uint8_t* xo;           // [osplits][2][MT*16][1024] bf16 hi / lo X rows of the O-projection (swizzled)
    uint64_t* trace;       // [grid][24] %globaltimer at the phase marks of layer trace_layer, or null
    int trace_layer;
    int B, nh, E, Kp, Nrows, e_out, oKp, otiles;
    int grid;
    int cluster;           // 2: CTA pairs (the region a pair shares meets through DSMEM), else 1
    int pos_hint;          // the host's expected length of layer 0 (-1: unknown, e.g. graph replays)
    int pre_stages;        // layer-0 cache stages per CTA prefetched into L2 before the grid-dependency wait
    int p3_tma;            // O-projection input rows staged by TMA (1) or by plain loads (0)
    int x_first;           // parked projection weights go out after the token slice is requested
    int l2_next;           // prefetch the next layer's late weight items into L2 during the tail
    int chain_pre;         // the next layer's first cache stages per CTA prefetched into L2 during the tail
    int nlayers;           // 1 .. kStepMaxLayers
    StepLayer layer[kStepMaxLayers];
};
bool step_supported(int R, int B, int nh, int Kp, int oKp, int otiles, int grid);

// The layer chain with the batch as two groups half a layer apart (step2.cu):
// one group's latency-bound phases run under the other's attention stream.
struct PipeArgs {
    const float* x;        // [B][E] layer-0 tokens (device)
    unsigned* bar[2];      // per group: grid barrier count (monotone, wrap-safe compares)
    unsigned* bgen[2];     // per group: barrier generations completed
    float* P[2];           // per group: [splits][8][Nrows] projection partials
    uint8_t* xo[2];        // per group: [osplits][16][1024] bf16 hi / lo O-projection rows (swizzled)
    float* ws[2];          // per group: [grid][6][36] segment states
    uint64_t* trace;       // [grid][24] phase marks of (trace_group, trace_layer), or null
    int trace_layer, trace_group;
    int B, nh, E, Kp, Nrows, e_out, oKp, otiles;
    int grid, cluster;
    int nlayers;
    StepLayer layer[kStepMaxLayers];
};
bool pipe_supported(int R, int B, int nh, int Kp, int oKp, int otiles, int grid);
size_t pipe_xo_bytes(int oKp);            // per group
size_t pipe_ws_bytes(int grid);           // per group
size_t pipe_p_bytes(int Kp, int Nrows);   // per group
int pipe_resident_ctas_per_sm();
int pipe_pair_clusters_ok(int grid);
cudaError_t launch_chain_pipe(const PipeArgs& a, cudaStream_t s);
int pipe_set_debug(int* mapped);  // debug builds (-DWSVD_PIPE_DEBUG): where stuck waits are recorded
int step_item_k();
size_t step_xo_bytes(int B, int oKp);  // bytes of StepArgs::xo
size_t step_ws_bytes(int grid);        // bytes of StepArgs::ws
int step_max_units();  // (sequence, head) segments one CTA of the fused step can hold
int step_ring_stages(int B);  // attention-ring stages of the fused step
int step_resident_ctas_per_sm(int B);  // occupancy of the fused step kernel (>= 1 to run)
int step_pair_clusters_ok(int B, int grid);  // 1 when the grid can run as resident CTA pairs
cudaError_t launch_layer_step(const StepArgs& a, cudaStream_t s);

}  // namespace wsvd_k
