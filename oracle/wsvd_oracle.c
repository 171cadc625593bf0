/*
 * wsvd_oracle.c -- TEST INFRASTRUCTURE ONLY (see wsvd_oracle.h).
 *
 * Plain-C restatement of the reference decode path, kept in the reference's
 * loop and operation order so that fp64 results agree with the reference
 * objects bit-for-bit (checked in tests/test_oracle.py).  Compiled with
 * -ffp-contract=off so that no multiply-add is fused behind our back.
 */
#include "wsvd_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ================================================================ rng === */

/* std::mt19937_64 (seed sequence: the standard single-seed initialisation). */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->mti = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

static uint64_t splitmix64(uint64_t x) {
    /* rng.cpp:9-14 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void orc_rng_stream(orc_rng* r, uint64_t seed, uint64_t stream_id) {
    /* rng.cpp:19-21 */
    orc_rng_seed(r, splitmix64(splitmix64(seed) ^ splitmix64(stream_id * 0x632be59bd9b4e019ULL + 1)));
}

uint64_t orc_rng_u64(orc_rng* r) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
    if (r->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
        }
        for (; i < 311; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
        }
        uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }

double orc_rng_normal(orc_rng* r) {
    /* rng.cpp:23-36 (Box-Muller with a cached spare) */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 1.0 - orc_rng_uniform(r);
    double u2 = orc_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    double a = 2.0 * 3.141592653589793 * u2; /* std::numbers::pi */
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}

uint64_t orc_rng_index(orc_rng* r, uint64_t n) {
    /* rng.cpp:38-44 */
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v = orc_rng_u64(r);
    while (v >= limit) v = orc_rng_u64(r);
    return v % n;
}

void orc_rng_normal_fill(orc_rng* r, double* out, size_t n, double stddev) {
    for (size_t i = 0; i < n; ++i) out[i] = stddev * orc_rng_normal(r);
}

/* ============================================================ decode === */

/* decode.cpp:97-110 -- row vector (len m) times matrix (m x n, row stride ld);
 * zero entries of x are skipped exactly like the reference. */
static void vec_mat(const double* x, size_t m, const double* mat, size_t ld, size_t n,
                    double* out) {
    for (size_t j = 0; j < n; ++j) out[j] = 0.0;
    for (size_t i = 0; i < m; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        const double* row = mat + i * ld;
        for (size_t j = 0; j < n; ++j) out[j] += xi * row[j];
    }
}

/* matrix.cpp:210-218 */
static double dot(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static const double* fa(const orc_layer* f, size_t h, int role) {
    return f->A + (h * 3 + (size_t)role) * f->E * f->rmax;
}
static const double* fb(const orc_layer* f, size_t h, int role) {
    return f->B + (h * 3 + (size_t)role) * f->rmax * f->H;
}
static size_t rank_of(const orc_layer* f, size_t h, int role) {
    return (size_t)f->ranks[h * 3 + (size_t)role];
}

/* Column-restricted vec_mat over the padded A (E x rmax, first r columns). */
static void vec_mat_cols(const double* x, size_t m, const double* mat, size_t ld, size_t r,
                         double* out) {
    vec_mat(x, m, mat, ld, r, out);
}

void orc_softmax_observe(orc_softmax* s, double score, const double* value) {
    /* decode.cpp:35-57 */
    if (s->empty) {
        s->max_score = score;
        s->denom = 1.0;
        memcpy(s->acc, value, s->w * sizeof(double));
        s->empty = 0;
        return;
    }
    if (score <= s->max_score) {
        const double w = exp(score - s->max_score);
        s->denom += w;
        for (size_t i = 0; i < s->w; ++i) s->acc[i] += w * value[i];
    } else {
        const double c = exp(s->max_score - score);
        s->denom = s->denom * c + 1.0;
        for (size_t i = 0; i < s->w; ++i) s->acc[i] = s->acc[i] * c + value[i];
        s->max_score = score;
    }
}

void orc_softmax_merge(orc_softmax* s, const orc_softmax* o) {
    /* decode.cpp:59-75 */
    if (o->empty) return;
    if (s->empty) {
        s->max_score = o->max_score;
        s->denom = o->denom;
        memcpy(s->acc, o->acc, s->w * sizeof(double));
        s->empty = 0;
        return;
    }
    const double m = s->max_score > o->max_score ? s->max_score : o->max_score;
    const double c1 = exp(s->max_score - m);
    const double c2 = exp(o->max_score - m);
    s->denom = s->denom * c1 + o->denom * c2;
    for (size_t i = 0; i < s->w; ++i) s->acc[i] = s->acc[i] * c1 + o->acc[i] * c2;
    s->max_score = m;
}

static void counter_add(orc_counter* c, int kind, int stream, uint64_t n) {
    if (!c) return;
    if (kind == 0) c->loads[stream] += n;
    else if (kind == 1) c->stores[stream] += n;
    else c->flops[stream] += n;
}

/* One head of append_token (decode.cpp:135-150). */
static void append_head(const orc_layer* f, size_t h, double* ck_h, double* cv_h, size_t pos,
                        const double* x, double* q_h, orc_counter* c, double* scratch) {
    const size_t E = f->E, H = f->H, R = f->rmax;
    const size_t rq = rank_of(f, h, 0), rk = rank_of(f, h, 1), rv = rank_of(f, h, 2);
    double* ck = scratch;
    double* cv = scratch + R;
    double* cq = scratch + 2 * R;
    vec_mat_cols(x, E, fa(f, h, 1), R, rk, ck);
    vec_mat_cols(x, E, fa(f, h, 2), R, rv, cv);
    vec_mat_cols(x, E, fa(f, h, 0), R, rq, cq);
    vec_mat(cq, rq, fb(f, h, 0), H, H, q_h);
    double* krow = ck_h + pos * R;
    double* vrow = cv_h + pos * R;
    for (size_t j = 0; j < R; ++j) {
        krow[j] = j < rk ? ck[j] : 0.0;
        vrow[j] = j < rv ? cv[j] : 0.0;
    }
    counter_add(c, 2, ORC_LATENT_K, E * rk);
    counter_add(c, 1, ORC_LATENT_K, rk);
    counter_add(c, 2, ORC_LATENT_V, E * rv);
    counter_add(c, 1, ORC_LATENT_V, rv);
    counter_add(c, 2, ORC_QUERY, E * rq + rq * H);
}

int orc_append_token(const orc_layer* f, double* ck, double* cv, size_t cap, size_t pos,
                     const double* x, double* q_out, orc_counter* c) {
    if (pos >= cap) return -1;
    double* scratch = (double*)malloc(3 * f->rmax * sizeof(double));
    counter_add(c, 0, ORC_QUERY, f->E); /* decode.cpp:132 */
    for (size_t h = 0; h < f->nh; ++h) {
        append_head(f, h, ck + h * cap * f->rmax, cv + h * cap * f->rmax, pos, x, q_out + h * f->H,
                    c, scratch);
    }
    free(scratch);
    return 0;
}

/* One head of fused_decode_step (decode.cpp:168-204). */
static void decode_head(const orc_layer* f, size_t h, const double* ck_h, const double* cv_h,
                        size_t len, const double* q_h, size_t tile, double* out_h,
                        orc_counter* c, double* scratch, double* latent_h) {
    const size_t H = f->H, R = f->rmax;
    const size_t rk = rank_of(f, h, 1), rv = rank_of(f, h, 2);
    const double* bk = fb(f, h, 1);
    const double* bv = fb(f, h, 2);
    const double inv_sqrt_h = 1.0 / sqrt((double)H);
    double* key = scratch;                     /* H */
    double* acc_state = scratch + H;           /* R */
    double* acc_local = scratch + H + R;       /* R */
    double* latent_out = scratch + H + 2 * R;  /* R */

    counter_add(c, 0, ORC_WEIGHTS_B, rk * H + rv * H);
    counter_add(c, 0, ORC_QUERY, H);
    orc_softmax state = {0.0, 0.0, acc_state, rv, 1};
    for (size_t t0 = 0; t0 < len; t0 += tile) {
        const size_t t1 = t0 + tile < len ? t0 + tile : len;
        counter_add(c, 0, ORC_LATENT_K, (t1 - t0) * rk);
        counter_add(c, 0, ORC_LATENT_V, (t1 - t0) * rv);
        orc_softmax local = {0.0, 0.0, acc_local, rv, 1};
        for (size_t j = t0; j < t1; ++j) {
            vec_mat(ck_h + j * R, rk, bk, H, H, key);
            counter_add(c, 2, ORC_LATENT_K, rk * H);
            const double score = dot(q_h, key, H) * inv_sqrt_h;
            counter_add(c, 2, ORC_QUERY, H);
            orc_softmax_observe(&local, score, cv_h + j * R);
            counter_add(c, 2, ORC_LATENT_V, rv);
        }
        orc_softmax_merge(&state, &local);
    }
    for (size_t i = 0; i < rv; ++i) latent_out[i] = state.acc[i] / state.denom;
    if (latent_h) { /* the latent output v~ = acc / denom (decode.cpp:198), before B_V */
        for (size_t i = 0; i < R; ++i) latent_h[i] = i < rv ? latent_out[i] : 0.0;
    }
    vec_mat(latent_out, rv, bv, H, H, out_h);
    counter_add(c, 2, ORC_OUTPUT, rv * H);
    counter_add(c, 1, ORC_OUTPUT, H);
}

int orc_fused_decode_step(const orc_layer* f, const double* ck, const double* cv, size_t cap,
                          size_t len, const double* q, size_t tile, double* out, orc_counter* c) {
    if (len == 0) return -1; /* decode.cpp:158 ShapeError */
    if (tile == 0) return -2; /* decode.cpp:113 ConfigError */
    if (tile > len) tile = len;
    double* scratch = (double*)malloc((f->H + 3 * f->rmax) * sizeof(double));
    for (size_t h = 0; h < f->nh; ++h) {
        decode_head(f, h, ck + h * cap * f->rmax, cv + h * cap * f->rmax, len, q + h * f->H, tile,
                    out + h * f->H, c, scratch, NULL);
    }
    free(scratch);
    return 0;
}

void orc_reconstruct_then_attend(const orc_layer* f, const double* ck, const double* cv,
                                 size_t cap, size_t len, const double* q, double* out) {
    /* tests/test_decode.cpp:68-94 (matmul ikj order, matrix.cpp:152-168) */
    const size_t H = f->H, R = f->rmax;
    const double inv_sqrt = 1.0 / sqrt((double)H);
    double* keys = (double*)malloc(len * H * sizeof(double));
    double* values = (double*)malloc(len * H * sizeof(double));
    double* scores = (double*)malloc(len * sizeof(double));
    for (size_t h = 0; h < f->nh; ++h) {
        const size_t rk = rank_of(f, h, 1), rv = rank_of(f, h, 2);
        const double* ckh = ck + h * cap * R;
        const double* cvh = cv + h * cap * R;
        for (size_t j = 0; j < len; ++j) {
            vec_mat(ckh + j * R, rk, fb(f, h, 1), H, H, keys + j * H);
            vec_mat(cvh + j * R, rv, fb(f, h, 2), H, H, values + j * H);
        }
        double mx = -INFINITY;
        for (size_t j = 0; j < len; ++j) {
            scores[j] = dot(q + h * H, keys + j * H, H) * inv_sqrt;
            if (j == 0 || scores[j] > mx) mx = scores[j];
        }
        double denom = 0.0;
        for (size_t j = 0; j < len; ++j) {
            scores[j] = exp(scores[j] - mx);
            denom += scores[j];
        }
        for (size_t col = 0; col < H; ++col) {
            double acc = 0.0;
            for (size_t j = 0; j < len; ++j) acc += scores[j] * values[j * H + col];
            out[h * H + col] = acc / denom;
        }
    }
    free(keys);
    free(values);
    free(scores);
}

int orc_traffic_match_fused(const orc_counter* c, uint64_t seq_len, uint64_t n_heads,
                            uint64_t head_dim, uint64_t rank_k) {
    /* decode.cpp:452-487, Mode::Fused */
    if (n_heads == 0) return -1;
    const uint64_t eta = seq_len * rank_k, gamma = seq_len * rank_k * head_dim;
    const uint64_t loads = c->loads[ORC_LATENT_K], flops = c->flops[ORC_LATENT_K];
    if (loads % n_heads || flops % n_heads) return 0;
    return loads / n_heads == eta && flops / n_heads == gamma;
}

/* ------------------------------------------------------ batched drivers */

typedef struct {
    const orc_layer* f;
    double* ck;
    double* cv;
    const double* ckc;
    const double* cvc;
    size_t B, cap, pos, len, tile;
    const double* x;
    const double* q;
    double* qo;
    double* out;
    double* lat; /* decode: [B][nh][rmax] latent outputs, or NULL */
    size_t next;
    pthread_mutex_t mu;
    int mode; /* 0 append, 1 decode */
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    const orc_layer* f = j->f;
    const size_t R = f->rmax, H = f->H;
    double* scratch = (double*)malloc((H + 3 * R + 3 * R) * sizeof(double));
    for (;;) {
        pthread_mutex_lock(&j->mu);
        size_t i = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (i >= j->B * f->nh) break;
        const size_t b = i / f->nh, h = i % f->nh;
        const size_t cache_off = (b * f->nh + h) * j->cap * R;
        if (j->mode == 0) {
            append_head(f, h, j->ck + cache_off, j->cv + cache_off, j->pos, j->x + b * f->E,
                        j->qo + (b * f->nh + h) * H, NULL, scratch);
        } else {
            decode_head(f, h, j->ckc + cache_off, j->cvc + cache_off, j->len,
                        j->q + (b * f->nh + h) * H, j->tile, j->out + (b * f->nh + h) * H, NULL,
                        scratch, j->lat ? j->lat + (b * f->nh + h) * R : NULL);
        }
    }
    free(scratch);
    return NULL;
}

static int run_batch(batch_job* j, int threads) {
    if (threads < 1) threads = 1;
    pthread_mutex_init(&j->mu, NULL);
    j->next = 0;
    pthread_t* tids = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, batch_worker, j);
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids);
    pthread_mutex_destroy(&j->mu);
    return 0;
}

int orc_batched_append(const orc_layer* f, double* ck, double* cv, size_t B, size_t cap,
                       size_t pos, const double* x, double* q_out, int threads) {
    if (pos >= cap) return -1;
    batch_job j;
    memset(&j, 0, sizeof j);
    j.f = f; j.ck = ck; j.cv = cv; j.B = B; j.cap = cap; j.pos = pos; j.x = x; j.qo = q_out;
    j.mode = 0;
    return run_batch(&j, threads);
}

int orc_batched_decode(const orc_layer* f, const double* ck, const double* cv, size_t B,
                       size_t cap, size_t len, const double* q, size_t tile, double* out,
                       int threads) {
    if (len == 0) return -1;
    if (tile == 0) return -2;
    batch_job j;
    memset(&j, 0, sizeof j);
    j.f = f; j.ckc = ck; j.cvc = cv; j.B = B; j.cap = cap; j.len = len; j.q = q; j.out = out;
    j.tile = tile > len ? len : tile;
    j.mode = 1;
    return run_batch(&j, threads);
}

int orc_batched_decode_latent(const orc_layer* f, const double* ck, const double* cv, size_t B,
                              size_t cap, size_t len, const double* q, size_t tile, double* out,
                              double* latent, int threads) {
    if (len == 0) return -1;
    if (tile == 0) return -2;
    batch_job j;
    memset(&j, 0, sizeof j);
    j.f = f; j.ckc = ck; j.cvc = cv; j.B = B; j.cap = cap; j.len = len; j.q = q; j.out = out;
    j.lat = latent;
    j.tile = tile > len ? len : tile;
    j.mode = 1;
    return run_batch(&j, threads);
}

/* ================================================ storage-format rules === */

float orc_f32(double v) { return (float)v; }

static uint32_t f32_bits(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    return u;
}
static float bits_f32(uint32_t u) {
    float v;
    memcpy(&v, &u, 4);
    return v;
}

uint16_t orc_bf16_bits(float v) {
    uint32_t u = f32_bits(v);
    if ((u & 0x7fffffffU) > 0x7f800000U) return (uint16_t)((u >> 16) | 0x40); /* NaN */
    u += 0x7fffU + ((u >> 16) & 1U);
    return (uint16_t)(u >> 16);
}

double orc_bf16(double v) {
    return (double)bits_f32((uint32_t)orc_bf16_bits((float)v) << 16);
}

uint16_t orc_f16_bits(float v) {
    uint32_t u = f32_bits(v);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000U);
    float a = fabsf(v);
    if (a != a) return (uint16_t)(sign | 0x7e00U);
    if (a >= 65520.0f) return (uint16_t)(sign | 0x7c00U);
    if (a < 0x1.0p-14f) {
        /* subnormal: integer multiple of 2^-24, round half to even */
        float m = a * 16777216.0f; /* exact */
        float fl = floorf(m);
        float rem = m - fl;
        uint32_t n = (uint32_t)fl;
        if (rem > 0.5f || (rem == 0.5f && (n & 1U))) ++n;
        return (uint16_t)(sign | n);
    }
    uint32_t ua = f32_bits(a);
    int e = (int)((ua >> 23) & 0xff) - 127 + 15;
    uint32_t mant = ua & 0x7fffffU;
    uint32_t h = ((uint32_t)e << 10) | (mant >> 13);
    uint32_t rem = mant & 0x1fffU;
    if (rem > 0x1000U || (rem == 0x1000U && (h & 1U))) ++h;
    return (uint16_t)(sign | h);
}

float orc_f16_to_f32(uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000U) << 16;
    uint32_t e = ((uint32_t)h >> 10) & 0x1fU;
    uint32_t m = (uint32_t)h & 0x3ffU;
    if (e == 0) {
        float v = (float)m * 0x1.0p-24f;
        return sign ? -v : v;
    }
    if (e == 31) return bits_f32(sign | 0x7f800000U | (m << 13));
    return bits_f32(sign | ((e - 15 + 127) << 23) | (m << 13));
}

int orc_qmax(int bits) { return (bits == 4 || bits == 8) ? (1 << (bits - 1)) - 1 : -1; }

static long long clampll(long long v, long long lim) {
    return v < -lim ? -lim : (v > lim ? lim : v);
}

double orc_quantize_weight(const double* w, size_t rows, size_t cols, int bits, int8_t* q,
                           double* scales) {
    /* quant.cpp:40-119 */
    const long long lim = orc_qmax(bits);
    const double qd = (double)lim;
    double* maxabs = (double*)calloc(cols, sizeof(double));
    double* s = (double*)malloc(cols * sizeof(double));
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) {
            const double a = fabs(w[i * cols + j]);
            if (a > maxabs[j]) maxabs[j] = a;
        }
    double best_clip = 10.0 / 20.0, best_err = -1.0;
    for (int g = 10; g <= 20; ++g) {
        const double clip = (double)g / 20.0;
        for (size_t j = 0; j < cols; ++j) s[j] = maxabs[j] == 0.0 ? 1.0 : clip * maxabs[j] / qd;
        double err = 0.0;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                long long qi = clampll(llround(w[i * cols + j] / s[j]), lim);
                const double d = w[i * cols + j] - (double)qi * s[j];
                err += d * d;
            }
        if (best_err < 0.0 || err < best_err) {
            best_err = err;
            best_clip = clip;
        }
    }
    for (size_t j = 0; j < cols; ++j)
        scales[j] = maxabs[j] == 0.0 ? 1.0 : best_clip * maxabs[j] / qd;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j)
            q[i * cols + j] = (int8_t)clampll(llround(w[i * cols + j] / scales[j]), lim);
    free(maxabs);
    free(s);
    return best_clip;
}

void orc_quantize_activation_f64(const double* x, size_t rows, size_t cols, int bits,
                                 int8_t* q, double* scales) {
    /* quant.cpp:131-150 */
    const long long lim = orc_qmax(bits);
    const double qd = (double)lim;
    for (size_t i = 0; i < rows; ++i) {
        double m = 0.0;
        for (size_t j = 0; j < cols; ++j) {
            const double a = fabs(x[i * cols + j]);
            if (a > m) m = a;
        }
        const double s = m == 0.0 ? 1.0 : m / qd;
        scales[i] = s;
        for (size_t j = 0; j < cols; ++j)
            q[i * cols + j] = (int8_t)clampll(llround(x[i * cols + j] / s), lim);
    }
}

void orc_fwht_f32(float* v, size_t n, float scale) {
    for (size_t len = 1; len < n; len <<= 1)
        for (size_t i = 0; i < n; i += 2 * len)
            for (size_t j = i; j < i + len; ++j) {
                const float a = v[j], b = v[j + len];
                v[j] = a + b;
                v[j + len] = a - b;
            }
    for (size_t i = 0; i < n; ++i) v[i] = v[i] * scale;
}

size_t orc_rot_block(size_t E) {
    if (E && !(E & (E - 1))) return E;
    if (E % 128 == 0) return 128;
    return 0;
}

void orc_rotate_token_f32(const float* x, float* xr, size_t E) {
    const size_t blk = orc_rot_block(E);
    const float scale = (float)(1.0 / sqrt((double)blk));
    memcpy(xr, x, E * sizeof(float));
    for (size_t b0 = 0; b0 < E; b0 += blk) orc_fwht_f32(xr + b0, blk, scale);
}

float orc_quant_token_f32(const float* v, size_t n, int8_t* q) {
    float m = 0.0f;
    for (size_t i = 0; i < n; ++i) m = fmaxf(m, fabsf(v[i]));
    const float s = m == 0.0f ? 1.0f : m / 127.0f;
    for (size_t i = 0; i < n; ++i) {
        float r = roundf(v[i] / s);
        r = r < -127.0f ? -127.0f : (r > 127.0f ? 127.0f : r);
        q[i] = (int8_t)r;
    }
    return s;
}

void orc_int_gemv(const int8_t* xq, const int8_t* wq, size_t E, size_t ncols, int32_t* acc) {
    for (size_t c = 0; c < ncols; ++c) {
        int32_t s = 0;
        const int8_t* row = wq + c * E;
        for (size_t i = 0; i < E; ++i) s += (int32_t)xq[i] * (int32_t)row[i];
        acc[c] = s;
    }
}

float orc_dequant_latent(int32_t acc, float sx, float sw) {
    volatile float t = (float)acc * sx; /* volatile: keep the two roundings */
    return t * sw;
}

uint16_t orc_quant_cache_row(const float* c, size_t n, int8_t* q) {
    float m = 0.0f;
    for (size_t i = 0; i < n; ++i) m = fmaxf(m, fabsf(c[i]));
    uint16_t h = orc_f16_bits(m / 127.0f);
    float s = orc_f16_to_f32(h);
    if (s == 0.0f) {
        h = 0x3c00U;
        s = 1.0f;
    }
    for (size_t i = 0; i < n; ++i) {
        float r = roundf(c[i] / s);
        r = r < -127.0f ? -127.0f : (r > 127.0f ? 127.0f : r);
        q[i] = (int8_t)r;
    }
    return h;
}

void orc_unpack_int4(const uint8_t* packed, size_t n, int8_t* out) {
    for (size_t i = 0; i < n; ++i) {
        const uint8_t b = packed[i >> 1];
        int v = (i & 1) ? (b >> 4) : (b & 0xf);
        out[i] = (int8_t)(v >= 8 ? v - 16 : v);
    }
}

/* ======================= int8-cache attention: the integer score stage === */
/* The absorbed query of an INT8 cache is split into two int8 vectors
 * (paper_2604_02570_b200/csrc/attn.cu consume_mma_i8 / consume_imma_i8; SURVEY
 * Appendix A.5 "if the absorbed form is used for INT8 configs, the oracle must
 * implement the same absorbed form"): s1 = max|q| / 127 (1 when q == 0),
 * s2 = s1 / 254, h = rint(q / s1), l = clamp(rint(fma(-h, s1, q) / s2), +-127)
 * with rint = round half to even, all in fp32.  Each cached int8 row c_j then
 * gives the exact int32 accumulators hi_j = sum_t c_j[t] h[t] and
 * lo_j = sum_t c_j[t] l[t]; the score is (hi_j s1 + lo_j s2) * s_cK[j] in the
 * log2 domain.  rows: L x ld int8 (the first R columns are C_K). */
void orc_i8_query_split(const float* q, size_t R, int8_t* h, int8_t* l, float* s1_out, float* s2_out) {
    float mx = 0.0f;
    for (size_t k = 0; k < R; ++k) mx = fmaxf(mx, fabsf(q[k]));
    const float s1 = (mx == 0.0f) ? 1.0f : mx / 127.0f;
    const float s2 = s1 / 254.0f;
    for (size_t k = 0; k < R; ++k) {
        const float hv = rintf(q[k] / s1);
        float lv = rintf(fmaf(-hv, s1, q[k]) / s2);
        lv = fminf(fmaxf(lv, -127.0f), 127.0f);
        h[k] = (int8_t)hv;
        l[k] = (int8_t)lv;
    }
    *s1_out = s1;
    *s2_out = s2;
}

void orc_i8_scores(const float* q, size_t R, const int8_t* rows, size_t L, size_t ld, int32_t* acc) {
    int8_t h[256], l[256];
    float s1, s2;
    orc_i8_query_split(q, R, h, l, &s1, &s2);
    for (size_t j = 0; j < L; ++j) {
        int32_t a = 0, b = 0;
        for (size_t t = 0; t < R; ++t) {
            a += (int32_t)rows[j * ld + t] * (int32_t)h[t];
            b += (int32_t)rows[j * ld + t] * (int32_t)l[t];
        }
        acc[2 * j] = a;
        acc[2 * j + 1] = b;
    }
}
