/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH (see etap_oracle.h).
 * Plain-C, binary64 restatement of the reference's ETAP decode algorithm and its oracle.
 * Build: oracle/Makefile (gcc -O2, no -ffast-math, no FMA contraction).
 */
#include "etap_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------- generator
 * src/matrix.cpp:23-48 (SplitMix64: next, uniform01, uniform01_open_at_zero, normal) and
 * src/matrix.cpp:153-165 (matrix_from_seed: one draw pair per normal element). */
typedef struct {
    uint64_t state;
} splitmix64;

static uint64_t sm_next(splitmix64* s) {
    s->state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double sm_uniform01(splitmix64* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }

static double sm_uniform01_open0(splitmix64* s) {
    return (double)((sm_next(s) >> 11) + 1) * 0x1.0p-53;
}

static double sm_normal(splitmix64* s) {
    const double two_pi = 6.283185307179586476925286766559;
    const double u1 = sm_uniform01_open0(s);
    const double u2 = sm_uniform01(s);
    return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

void oracle_matrix_from_seed(int64_t rows, int64_t cols, uint64_t seed, int dist, double* out) {
    splitmix64 s = {seed};
    const int64_t n = rows * cols;
    if (dist == 1) {
        for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * sm_uniform01(&s) - 1.0;
    } else {
        for (int64_t i = 0; i < n; ++i) out[i] = sm_normal(&s);
    }
}

/* ------------------------------------------------------------- rounding */
static double round_int_even(double m) { /* src/matrix.cpp:50-57 */
    const double f = floor(m);
    const double frac = m - f;
    if (frac > 0.5) return f + 1.0;
    if (frac < 0.5) return f;
    return fmod(f, 2.0) == 0.0 ? f : f + 1.0;
}

double oracle_round_half(double x) { /* src/matrix.cpp:167-184 */
    if (isnan(x)) return NAN;
    const double ax = fabs(x);
    if (ax >= 65520.0) return copysign(INFINITY, x);
    if (ax == 0.0) return x;
    int e = 0;
    frexp(ax, &e);
    const int exp2 = e - 1;
    const int q = exp2 < -14 ? -24 : exp2 - 10;
    const double scaled = ldexp(ax, -q);
    return copysign(ldexp(round_int_even(scaled), q), x);
}

/* bfloat16: 8 significant bits, exponent range of binary32 (subnormal quantum 2^-133).
 * Same construction as round_half with the bf16 parameters. */
double oracle_bf16_round(double x) {
    if (isnan(x)) return NAN;
    const double ax = fabs(x);
    if (ax == 0.0) return x;
    int e = 0;
    frexp(ax, &e);
    int q = e - 8;
    if (q < -133) q = -133;
    const double r = ldexp(round_int_even(ldexp(ax, -q)), q);
    if (r > 3.3895313892515355e38) return copysign(INFINITY, x);
    return copysign(r, x);
}

void oracle_bf16_round_array(const double* in, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_bf16_round(in[i]);
}

void oracle_bf16_bits(const double* in, uint16_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const float f = (float)oracle_bf16_round(in[i]); /* exact */
        uint32_t u;
        memcpy(&u, &f, 4);
        out[i] = isnan(in[i]) ? (uint16_t)0x7FC0 : (uint16_t)(u >> 16);
    }
}

void oracle_bf16_widen(const uint16_t* in, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t u = (uint32_t)in[i] << 16;
        float f;
        memcpy(&f, &u, 4);
        out[i] = (double)f;
    }
}

/* ------------------------------------------------------------- attention_ref
 * src/attention.cpp:44-77: per query row: s_j = scale * (q . k_j) with the dot summed in
 * column order, m = max_j s_j, p_j = exp(s_j - m), l = sum p_j, o = (sum_j p_j v_j) / l,
 * L = m + log l. */
void oracle_attention_ref(const double* q, int64_t n_q, const double* k, int64_t n_kv,
                          int64_t d_qk, const double* v, int64_t ldv, int64_t d_v, double scale,
                          double* o, double* l) {
    double* s = (double*)malloc(sizeof(double) * (size_t)(n_kv > 0 ? n_kv : 1));
    for (int64_t i = 0; i < n_q; ++i) {
        const double* qi = q + i * d_qk;
        double m = -INFINITY;
        for (int64_t j = 0; j < n_kv; ++j) {
            const double* kj = k + j * d_qk;
            double dot = 0.0;
            for (int64_t c = 0; c < d_qk; ++c) dot += qi[c] * kj[c];
            s[j] = scale * dot;
            if (s[j] > m) m = s[j];
        }
        double sum = 0.0;
        double* oi = o + i * d_v;
        for (int64_t c = 0; c < d_v; ++c) oi[c] = 0.0;
        for (int64_t j = 0; j < n_kv; ++j) {
            const double p = exp(s[j] - m);
            sum += p;
            const double* vj = v + j * ldv;
            for (int64_t c = 0; c < d_v; ++c) oi[c] += p * vj[c];
        }
        for (int64_t c = 0; c < d_v; ++c) oi[c] /= sum;
        l[i] = m + log(sum);
    }
    free(s);
}

/* ------------------------------------------------------------- run_etap (exact64)
 * src/etap.cpp:102-148 with block_update_impl (etap.cpp:15-79). Accumulator O^T is kept as
 * d_v x r (queries as columns), split into halves of ceil(d_v/2) and floor(d_v/2) rows
 * (etap.cpp:83-94); both halves use the same per-column rescale. */
int oracle_run_etap(const double* q, int64_t n_q, const double* k, int64_t n_kv, int64_t d_qk,
                    const double* v, int64_t ldv, int64_t d_v, double scale, int64_t b_r,
                    int64_t b_c, int negate_rescale, double* o, double* l) {
    if (b_r < 1 || b_c < 1) return 1; /* etap.cpp:104-106 */
    const int64_t t_c = (n_kv + b_c - 1) / b_c; /* kv_block_count, tiled_standard.cpp:21-23 */
    const int64_t d_lower = (d_v + 1) / 2;
    const double sign = negate_rescale ? -1.0 : 1.0;
    double* ot = (double*)malloc(sizeof(double) * (size_t)(d_v * b_r)); /* O^T, d_v x r */
    double* st = (double*)malloc(sizeof(double) * (size_t)(b_c * b_r)); /* S^T, b x r */
    double* mm = (double*)malloc(sizeof(double) * (size_t)b_r);
    double* ll = (double*)malloc(sizeof(double) * (size_t)b_r);
    double* resc = (double*)malloc(sizeof(double) * (size_t)b_r);
    double* colsum = (double*)malloc(sizeof(double) * (size_t)b_r);
    for (int64_t i0 = 0; i0 < n_q; i0 += b_r) {
        const int64_t r = (b_r < n_q - i0) ? b_r : n_q - i0;
        const double* qi = q + i0 * d_qk;
        for (int64_t e = 0; e < d_v * r; ++e) ot[e] = 0.0; /* make_etap_accumulator */
        for (int64_t c = 0; c < r; ++c) { mm[c] = -INFINITY; ll[c] = 0.0; }
        for (int64_t j = 0; j < t_c; ++j) {
            const int64_t k0 = j * b_c;
            const int64_t b = (b_c < n_kv - k0) ? b_c : n_kv - k0;
            /* S^T = K_j Q_i^T (gemm F,T: row dot products, matrix.cpp:72-82), then * scale */
            for (int64_t row = 0; row < b; ++row) {
                const double* kr = k + (k0 + row) * d_qk;
                for (int64_t c = 0; c < r; ++c) {
                    const double* qc = qi + c * d_qk;
                    double acc = 0.0;
                    for (int64_t kk = 0; kk < d_qk; ++kk) acc += kr[kk] * qc[kk];
                    st[row * r + c] = scale * acc;
                }
            }
            /* column max, rescale = exp(m_old - m_new) (etap.cpp:40-47) */
            for (int64_t c = 0; c < r; ++c) {
                double mx = mm[c];
                for (int64_t row = 0; row < b; ++row)
                    if (st[row * r + c] > mx) mx = st[row * r + c];
                resc[c] = exp(mm[c] - mx);
                mm[c] = mx;
                colsum[c] = 0.0;
            }
            /* P = exp(S^T - m), column sums (etap.cpp:49-58); P overwrites S^T */
            for (int64_t row = 0; row < b; ++row)
                for (int64_t c = 0; c < r; ++c) {
                    const double e = exp(st[row * r + c] - mm[c]);
                    st[row * r + c] = e;
                    colsum[c] += e;
                }
            for (int64_t c = 0; c < r; ++c) ll[c] = resc[c] * ll[c] + colsum[c]; /* :59-60 */
            /* O^T_half = sign*rescale*O^T_half + V_half^T P (etap.cpp:62-74); gemm T,F is the
             * outer-product order over the KV rows (matrix.cpp:83-92) */
            for (int half = 0; half < 2; ++half) {
                const int64_t c0 = half == 0 ? 0 : d_lower;
                const int64_t nd = half == 0 ? d_lower : d_v - d_lower;
                if (nd <= 0) continue;
                double* vp = (double*)calloc((size_t)(nd * r), sizeof(double));
                for (int64_t row = 0; row < b; ++row) {
                    const double* vr = v + (k0 + row) * ldv + c0;
                    const double* pr = st + row * r;
                    for (int64_t dd = 0; dd < nd; ++dd) {
                        const double a = vr[dd];
                        for (int64_t c = 0; c < r; ++c) vp[dd * r + c] += a * pr[c];
                    }
                }
                for (int64_t dd = 0; dd < nd; ++dd)
                    for (int64_t c = 0; c < r; ++c) {
                        double* acc = ot + (c0 + dd) * r + c;
                        *acc = sign * resc[c] * *acc + vp[dd * r + c];
                    }
                free(vp);
            }
        }
        /* epilogue: normalize, one transpose per query block, L = m + log l (:131-145) */
        for (int64_t c = 0; c < r; ++c) {
            for (int64_t dd = 0; dd < d_v; ++dd) o[(i0 + c) * d_v + dd] = ot[dd * r + c] / ll[c];
            l[i0 + c] = mm[c] + log(ll[c]);
        }
    }
    free(ot); free(st); free(mm); free(ll); free(resc); free(colsum);
    return 0;
}

/* ------------------------------------------------------------- batched paged MLA */
typedef struct {
    const uint16_t* q;
    const uint16_t* kv_pool;
    const int32_t* block_table;
    const int32_t* seqlens;
    int64_t max_pages, heads, n_units, next;
    double scale;
    double* o;
    double* l;
    pthread_mutex_t mu;
} mla_job;

static double widen1(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* one sequence: attention_ref for each of its heads (attention.cpp:44-77 per query row) with
 * K rows gathered through the block table and V = K[:, :512] */
static void mla_one_seq(mla_job* J, int64_t b) {
    const int64_t H = J->heads, D = 576, DV = 512;
    const int64_t n = J->seqlens[b] > 0 ? J->seqlens[b] : 0;
    double* o = J->o + b * H * DV;
    double* l = J->l + b * H;
    if (n == 0) {
        for (int64_t i = 0; i < H * DV; ++i) o[i] = 0.0;
        for (int64_t h = 0; h < H; ++h) l[h] = -INFINITY;
        return;
    }
    double* qd = (double*)malloc(sizeof(double) * (size_t)(H * D));
    for (int64_t i = 0; i < H * D; ++i) qd[i] = widen1(J->q[b * H * D + i]);
    double* s = (double*)malloc(sizeof(double) * (size_t)(n * H));
    double* kr = (double*)malloc(sizeof(double) * (size_t)D);
    double* m = (double*)malloc(sizeof(double) * (size_t)H);
    double* sum = (double*)malloc(sizeof(double) * (size_t)H);
    for (int64_t h = 0; h < H; ++h) { m[h] = -INFINITY; sum[h] = 0.0; }
    const int32_t* bt = J->block_table + b * J->max_pages;
    for (int64_t j = 0; j < n; ++j) {
        const uint16_t* src = J->kv_pool + ((int64_t)bt[j / 64] * 64 + (j % 64)) * D;
        for (int64_t c = 0; c < D; ++c) kr[c] = widen1(src[c]);
        for (int64_t h = 0; h < H; ++h) {
            const double* qh = qd + h * D;
            double dot = 0.0;
            for (int64_t c = 0; c < D; ++c) dot += qh[c] * kr[c];
            const double sv = J->scale * dot;
            s[j * H + h] = sv;
            if (sv > m[h]) m[h] = sv;
        }
    }
    for (int64_t i = 0; i < H * DV; ++i) o[i] = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        const uint16_t* src = J->kv_pool + ((int64_t)bt[j / 64] * 64 + (j % 64)) * D;
        for (int64_t c = 0; c < DV; ++c) kr[c] = widen1(src[c]);
        for (int64_t h = 0; h < H; ++h) {
            const double p = exp(s[j * H + h] - m[h]);
            sum[h] += p;
            double* oh = o + h * DV;
            for (int64_t c = 0; c < DV; ++c) oh[c] += p * kr[c];
        }
    }
    for (int64_t h = 0; h < H; ++h) {
        for (int64_t c = 0; c < DV; ++c) o[h * DV + c] /= sum[h];
        l[h] = m[h] + log(sum[h]);
    }
    free(qd); free(s); free(kr); free(m); free(sum);
}

static void* mla_worker(void* arg) {
    mla_job* J = (mla_job*)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int64_t u = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (u >= J->n_units) break;
        mla_one_seq(J, u);
    }
    return NULL;
}

int oracle_mla_decode_bf16(const uint16_t* q, const uint16_t* kv_pool, int64_t num_pages,
                           const int32_t* block_table, int64_t max_pages,
                           const int32_t* seqlens, int64_t batch, int64_t heads, double scale,
                           int nthreads, double* o, double* l) {
    (void)num_pages;
    mla_job J;
    J.q = q; J.kv_pool = kv_pool; J.block_table = block_table; J.seqlens = seqlens;
    J.max_pages = max_pages; J.heads = heads; J.n_units = batch; J.next = 0;
    J.scale = scale; J.o = o; J.l = l;
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, mla_worker, &J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&J.mu);
    return 0;
}
