/*
 * qvg_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference codec's hot path
 * (/root/reference/pkg/src/qvgcodec, "Q/" below) with every floating-point
 * operation order spelled out, so that it reproduces the reference's
 * numpy/OpenBLAS results bit for bit.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library;
 * the product path (paper_2602_02958_b200) never links or calls it.
 *
 * Third-party arithmetic the reference delegates to (numpy 2.3.5 +
 * scipy-openblas 0.3.30, SkylakeX kernel) and how it is restated here:
 *   - ndarray.sum / np.mean      -> numpy pairwise_sum (8 accumulators,
 *                                   blocks of 128, recursive halving), with
 *                                   the add identity 0.0 as the initial value
 *   - rows @ centroids.T (dgemm) -> one sequential fp64 FMA chain per output,
 *                                   k = 0..d-1, starting from 0.0
 *   - np.cumsum / np.add.at      -> strictly sequential fp64 additions
 *   - np.rint / np.ceil / frexp  -> IEEE round-half-even / ceil / exponent
 * These orders are pinned by tests/golden (fixtures produced by the
 * reference itself, script tests/golden/make_golden.py) and by
 * tests/test_oracle_numerics.py.
 *
 * The k-means++ random draws (numpy Generator(Philox(stage_seed)).random())
 * are data-independent, so callers pass them in pre-drawn (K per stage).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Minimal plane-parallel for-loop over pthreads (planes are independent,
 * SPEC.md:76-77); body(i, ctx) is called for i in [0, n). */
typedef struct { int64_t n; int64_t next; pthread_mutex_t mu; void (*body)(int64_t, void *); void *ctx; } qo_pool;
static void *qo_worker(void *arg)
{
    qo_pool *p = arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->n) return NULL;
        p->body(i, p->ctx);
    }
}
static void qo_parallel_for(int64_t n, int n_threads, void (*body)(int64_t, void *), void *ctx)
{
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    qo_pool p = {n, 0, PTHREAD_MUTEX_INITIALIZER, body, ctx};
    pthread_t th[256];
    for (int t = 1; t < n_threads; t++) pthread_create(&th[t], NULL, qo_worker, &p);
    qo_worker(&p);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
}

#define QO_OK 0
#define QO_ERR_NONFINITE 2
#define QO_ERR_DIM 1
#define QO_ERR_EMPTY 3
#define QO_ERR_CONFIG 5

/* ---------------------------------------------------------------------- */
/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src).     */
/* Used by every ndarray.sum() in Q/clustering.py:38,59,62,70,99,106,143,  */
/* 154 and by np.mean in Q/metrics.py:27 / Q/prq.py:171.                   */
/* ---------------------------------------------------------------------- */
static double pw_strided(const double *a, int64_t n, int64_t stride)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += a[i * stride];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j * stride];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) s += a[i * stride];
        return s;
    }
    int64_t h = n / 2;
    h -= h % 8;
    return pw_strided(a, h, stride) + pw_strided(a + h * stride, n - h, stride);
}

/* reduction result = identity (0.0) + pairwise(all n) */
double qo_pairwise_sum(const double *a, int64_t n) { return 0.0 + pw_strided(a, n, 1); }

/* ---------------------------------------------------------------------- */
/* FP8 E4M3 (Q/lowprec.py:36-92) and bf16 rounding (Q/lowprec.py:112-120) */
/* ---------------------------------------------------------------------- */
double qo_e4m3_decode(uint8_t b)
{
    int e = (b >> 3) & 0xF, m = b & 7;
    double v;
    if (e == 0xF && m == 7) return NAN;
    if (e == 0) v = m * ldexp(1.0, -9);
    else v = (8 + m) * ldexp(1.0, e - 10);
    return (b & 0x80) ? -v : v;
}

/* x finite and >= 0.  round_up != 0 -> ceil on the grid ("up"), else RNE. */
uint8_t qo_e4m3_encode(double x, int round_up)
{
    if (x > 448.0) x = 448.0;
    if (x == 0.0) return 0;
    int e2;
    frexp(x, &e2);            /* x = f * 2^e2, f in [0.5, 1) */
    int e = e2 - 1;
    if (e < -6) e = -6;
    double sc = ldexp(x, -(e - 3)); /* exact: power-of-two scaling */
    double kd = round_up ? ceil(sc) : nearbyint(sc);
    int64_t k = (int64_t)kd;
    if (k == 16) { e += 1; k = 8; }
    if (e >= 8 && k > 14) k = 14;
    if (e > 8) e = 8;
    if (k >= 8) return (uint8_t)(((e + 7) << 3) | (int)(k - 8));
    return (uint8_t)k;
}

float qo_round_bf16(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    memcpy(&f, &u, 4);
    return f;
}

/* ---------------------------------------------------------------------- */
/* Group quantizer + packing: Q/quant.py:40-55 (_group_scales,            */
/* _quantize_groups), :78-100 (pack_payload), :134-148 (quantize_matrix).  */
/* ---------------------------------------------------------------------- */
int qo_quantize_matrix(const double *x, int64_t n, int d, int bits, int gsize,
                       uint8_t *payload, uint8_t *scales)
{
    if (gsize < 1 || d % gsize) return QO_ERR_DIM;
    int64_t cnt = n * (int64_t)d;
    for (int64_t i = 0; i < cnt; i++)
        if (!isfinite(x[i])) return QO_ERR_NONFINITE;
    int qmax = (1 << (bits - 1)) - 1;
    int per = 8 / bits;
    uint8_t mask = (uint8_t)((1 << bits) - 1);
    memset(payload, 0, (size_t)((cnt * bits + 7) / 8));
    int64_t ng = cnt / gsize;
    for (int64_t g = 0; g < ng; g++) {
        const double *v = x + g * gsize;
        double amax = 0.0;
        for (int j = 0; j < gsize; j++) { double a = fabs(v[j]); if (a > amax) amax = a; }
        uint8_t code = 0x38;                       /* zero group -> 1.0 */
        if (amax != 0.0) code = qo_e4m3_encode(amax / (double)qmax, 1);
        scales[g] = code;
        double s = qo_e4m3_decode(code);
        for (int j = 0; j < gsize; j++) {
            double q = nearbyint(v[j] / s);       /* np.rint: half-even */
            if (q > qmax) q = qmax;
            if (q < -qmax) q = -qmax;
            int64_t idx = g * gsize + j;
            uint8_t u = (uint8_t)((int)q) & mask;
            payload[idx / per] |= (uint8_t)(u << ((idx % per) * bits));
        }
    }
    return QO_OK;
}

/* Q/quant.py:103-116 (unpack_payload) + :151-168 (dequantize_plane): f32 q*s */
void qo_dequantize_matrix(const uint8_t *payload, const uint8_t *scales, int64_t n, int d,
                          int bits, int gsize, float *out)
{
    int per = 8 / bits;
    int sign = 1 << (bits - 1);
    int mask = (1 << bits) - 1;
    int64_t cnt = n * (int64_t)d;
    for (int64_t i = 0; i < cnt; i++) {
        int u = (payload[i / per] >> ((i % per) * bits)) & mask;
        int q = (u ^ sign) - sign;
        float s = (float)qo_e4m3_decode(scales[i / gsize]);
        out[i] = (float)q * s;
    }
}

/* ---------------------------------------------------------------------- */
/* k-means (Q/clustering.py)                                              */
/* ---------------------------------------------------------------------- */

/* ((a - b) ** 2).sum() over one row of d, numpy pairwise (no FMA). */
static double row_sqdist(const double *a, const double *b, int d, double *tmp)
{
    for (int k = 0; k < d; k++) { double t = a[k] - b[k]; tmp[k] = t * t; }
    return 0.0 + pw_strided(tmp, d, 1);
}

/* Q/clustering.py:36-44 _pick: total = pairwise(w); cum = sequential cumsum;
 * searchsorted(cum, r*total, side="right").clip(0, n-1). */
static int64_t pick(const double *w, int64_t n, double r)
{
    double total = qo_pairwise_sum(w, n);
    if (total <= 0.0) {
        int64_t i = (int64_t)(r * (double)n);
        return i < n - 1 ? i : n - 1;
    }
    double target = r * total, c = 0.0;
    int64_t i = 0;
    for (; i < n; i++) {
        c += w[i];
        if (c > target) break;
    }
    return i < n - 1 ? i : n - 1;
}

/* Q/clustering.py:47-63 kmeans_pp_init, draws[0..k-1] = successive rng.random() */
int qo_kmeans_pp(const double *rows, int64_t n, int d, int k, const double *draws,
                 double *cent_out, int64_t *chosen_out)
{
    if (n < 1) return QO_ERR_EMPTY;
    double *d2 = malloc(sizeof(double) * n);
    double *tmp = malloc(sizeof(double) * d);
    int64_t c = (int64_t)(draws[0] * (double)n);
    if (c > n - 1) c = n - 1;
    if (chosen_out) chosen_out[0] = c;
    memcpy(cent_out, rows + c * d, sizeof(double) * d);
    for (int64_t i = 0; i < n; i++) d2[i] = row_sqdist(rows + i * d, rows + c * d, d, tmp);
    for (int p = 1; p < k; p++) {
        c = pick(d2, n, draws[p]);
        if (chosen_out) chosen_out[p] = c;
        memcpy(cent_out + (int64_t)p * d, rows + c * d, sizeof(double) * d);
        for (int64_t i = 0; i < n; i++) {
            double v = row_sqdist(rows + i * d, rows + c * d, d, tmp);
            if (v < d2[i]) d2[i] = v;
        }
    }
    free(d2);
    free(tmp);
    return QO_OK;
}

/* Q/clustering.py:66-71 _assign: argmin(c2 - 2*(X C^T)), first minimum. */
void qo_assign(const double *rows, int64_t n, int d, const double *cent, int k, int32_t *assign)
{
    double *c2 = malloc(sizeof(double) * k);
    double *tmp = malloc(sizeof(double) * d);
    for (int j = 0; j < k; j++) {
        for (int t = 0; t < d; t++) tmp[t] = cent[(int64_t)j * d + t] * cent[(int64_t)j * d + t];
        c2[j] = 0.0 + pw_strided(tmp, d, 1);
    }
    for (int64_t i = 0; i < n; i++) {
        const double *x = rows + i * d;
        int best = 0;
        double bv = 0.0;
        for (int j = 0; j < k; j++) {
            const double *c = cent + (int64_t)j * d;
            double acc = 0.0;
            for (int t = 0; t < d; t++) acc = fma(x[t], c[t], acc);
            double v = c2[j] - 2.0 * acc;
            if (j == 0 || v < bv) { bv = v; best = j; }
        }
        assign[i] = best;
    }
    free(c2);
    free(tmp);
}

/* flat ((rows - cent[assign]) ** 2).sum() — pairwise over n*d */
static double objective(const double *rows, int64_t n, int d, const double *cent,
                        const int32_t *assign, double *scratch /* n*d */)
{
    for (int64_t i = 0; i < n; i++) {
        const double *c = cent + (int64_t)assign[i] * d;
        for (int t = 0; t < d; t++) { double v = rows[i * d + t] - c[t]; scratch[i * d + t] = v * v; }
    }
    return qo_pairwise_sum(scratch, n * d);
}

/* Q/clustering.py:74-107 lloyd_step. cent is updated in place; returns objective. */
static double lloyd_step(const double *rows, int64_t n, int d, double *cent, int k,
                         int32_t *assign, double *scratch)
{
    qo_assign(rows, n, d, cent, k, assign);
    int64_t *cnt = calloc(k, sizeof(int64_t));
    double *nc = calloc((size_t)k * d, sizeof(double));
    for (int64_t i = 0; i < n; i++) {               /* np.add.at: row order */
        cnt[assign[i]]++;
        double *dst = nc + (int64_t)assign[i] * d;
        for (int t = 0; t < d; t++) dst[t] += rows[i * d + t];
    }
    int n_empty = 0;
    for (int j = 0; j < k; j++) {
        double *dst = nc + (int64_t)j * d;
        if (cnt[j] > 0) { for (int t = 0; t < d; t++) dst[t] /= (double)cnt[j]; }
        else { memcpy(dst, cent + (int64_t)j * d, sizeof(double) * d); n_empty++; }
    }
    if (n_empty) {                                  /* Q/clustering.py:97-104 */
        double *dist = malloc(sizeof(double) * n);
        double *tmp = malloc(sizeof(double) * d);
        for (int64_t i = 0; i < n; i++)
            dist[i] = row_sqdist(rows + i * d, nc + (int64_t)assign[i] * d, d, tmp);
        for (int j = 0; j < k; j++) {
            if (cnt[j] > 0) continue;
            int64_t r = 0;
            for (int64_t i = 1; i < n; i++) if (dist[i] > dist[r]) r = i;
            memcpy(nc + (int64_t)j * d, rows + r * d, sizeof(double) * d);
            assign[r] = j;
            dist[r] = -1.0;
        }
        free(dist);
        free(tmp);
    }
    memcpy(cent, nc, sizeof(double) * k * d);
    free(nc);
    free(cnt);
    return objective(rows, n, d, cent, assign, scratch);
}

/* Q/clustering.py:74-107 lloyd_step as an entry point: cent [k][d] updated in
   place, assign [n] out, returns the objective against the new centroids. */
double qo_lloyd_step(const double *rows, int64_t n, int d, double *cent, int k, int32_t *assign)
{
    double *scratch = malloc(sizeof(double) * n * d);
    double obj = lloyd_step(rows, n, d, cent, k, assign, scratch);
    free(scratch);
    return obj;
}

/* Q/clustering.py:110-160 kmeans.  init == NULL -> k-means++ with draws. */
int qo_kmeans(const double *rows, int64_t n, int d, int k, int max_iters, double tol,
              const double *draws, const double *init, double *cent, int32_t *assign,
              double *obj_out, int32_t *iters_out)
{
    if (n < 1) return QO_ERR_EMPTY;
    if (k < 1 || k > 256) return QO_ERR_CONFIG;
    if (init) memcpy(cent, init, sizeof(double) * k * d);
    else qo_kmeans_pp(rows, n, d, k, draws, cent, NULL);
    double *scratch = malloc(sizeof(double) * n * d);
    qo_assign(rows, n, d, cent, k, assign);
    double prev = objective(rows, n, d, cent, assign, scratch);
    int it = 0;
    for (int s = 0; s < max_iters; s++) {
        double obj = lloyd_step(rows, n, d, cent, k, assign, scratch);
        it++;
        double den = prev > 2.2250738585072014e-308 ? prev : 2.2250738585072014e-308;
        if ((prev - obj) / den < tol) break;
        prev = obj;
    }
    qo_assign(rows, n, d, cent, k, assign);
    double obj = objective(rows, n, d, cent, assign, scratch);
    if (obj_out) *obj_out = obj;
    if (iters_out) *iters_out = it;
    free(scratch);
    return QO_OK;
}

/* ---------------------------------------------------------------------- */
/* PRQ chain: Q/smoothing.py:23-41 + Q/prq.py:38-80 (prq_compress).       */
/* x: (n,d) f32 plane.  draws: [stages][k].  warm: [stages][k][d] or NULL. */
/* Outputs: payload, scales, cent_bf16 [stages][k][d] (bf16-exact f32),    */
/* assign [stages][n] u8, optional cent_f64 [stages][k][d], iters[stages]. */
/* ---------------------------------------------------------------------- */
int qo_prq_compress(const float *x, int64_t n, int d, int bits, int gsize, int stages, int k,
                    int max_iters, double tol, const double *draws, const double *warm,
                    uint8_t *payload, uint8_t *scales, float *cent_bf16, uint8_t *assign_out,
                    double *cent_f64_out, int32_t *iters_out)
{
    if (n < 1 || d < 1) return QO_ERR_EMPTY;
    if (gsize < 1 || d % gsize) return QO_ERR_DIM;
    for (int64_t i = 0; i < n * d; i++)
        if (!isfinite(x[i])) return QO_ERR_NONFINITE;
    double *res = malloc(sizeof(double) * n * d);
    for (int64_t i = 0; i < n * d; i++) res[i] = (double)x[i];
    double *cent = malloc(sizeof(double) * k * d);
    int32_t *asg = malloc(sizeof(int32_t) * n);
    int rc = QO_OK;
    for (int t = 0; t < stages; t++) {
        int32_t it = 0;
        rc = qo_kmeans(res, n, d, k, max_iters, tol, draws ? draws + (int64_t)t * k : NULL,
                       warm ? warm + (int64_t)t * k * d : NULL, cent, asg, NULL, &it);
        if (rc) break;
        if (iters_out) iters_out[t] = it;
        if (cent_f64_out) memcpy(cent_f64_out + (int64_t)t * k * d, cent, sizeof(double) * k * d);
        float *cb = cent_bf16 + (int64_t)t * k * d;
        for (int64_t j = 0; j < (int64_t)k * d; j++) cb[j] = qo_round_bf16((float)cent[j]);
        for (int64_t i = 0; i < n; i++) {
            assign_out[(int64_t)t * n + i] = (uint8_t)asg[i];
            const float *c = cb + (int64_t)asg[i] * d;
            for (int j = 0; j < d; j++) res[i * d + j] = res[i * d + j] - (double)c[j];
        }
    }
    if (!rc) rc = qo_quantize_matrix(res, n, d, bits, gsize, payload, scales);
    free(res);
    free(cent);
    free(asg);
    return rc;
}

/* Q/prq.py:113-132 prq_decompress_onepass: f64(q*s) + C_S[pi_S] + ... + C_1[pi_1] -> f32 */
void qo_prq_decompress(const uint8_t *payload, const uint8_t *scales, const float *cent_bf16,
                       const uint8_t *assign, int64_t n, int d, int bits, int gsize, int stages,
                       int k, float *out)
{
    qo_dequantize_matrix(payload, scales, n, d, bits, gsize, out);
    for (int64_t i = 0; i < n; i++)
        for (int j = 0; j < d; j++) {
            double acc = (double)out[i * d + j];
            for (int t = stages - 1; t >= 0; t--)
                acc += (double)cent_bf16[((int64_t)t * k + assign[(int64_t)t * n + i]) * d + j];
            out[i * d + j] = (float)acc;
        }
}

/* Batched drivers for the CPU baseline: P independent planes, plane-parallel
 * over n_threads threads (planes are independent).  Layouts
 * are the device layouts of include/qvg.h. */
typedef struct {
    const float *x; int64_t n; int d, bits, gsize, stages, k, max_iters; double tol;
    const double *draws; uint8_t *payload, *scales; float *cent; uint8_t *assign;
    int32_t *iters; float *out; int rc;
} qo_batch;

static void compress_one(int64_t p, void *v)
{
    qo_batch *b = v;
    int64_t n = b->n, d = b->d, pb = (n * d * b->bits + 7) / 8, sb = n * d / b->gsize;
    int64_t sk = (int64_t)b->stages * b->k;
    int rc = qo_prq_compress(b->x + p * n * d, n, b->d, b->bits, b->gsize, b->stages, b->k,
                             b->max_iters, b->tol, b->draws ? b->draws + p * sk : NULL, NULL,
                             b->payload + p * pb, b->scales + p * sb, b->cent + p * sk * d,
                             b->assign + p * b->stages * n, NULL,
                             b->iters ? b->iters + p * b->stages : NULL);
    if (rc) b->rc = rc;
}

int qo_prq_compress_batch(const float *x, int64_t P, int64_t n, int d, int bits, int gsize,
                          int stages, int k, int max_iters, double tol, const double *draws,
                          uint8_t *payload, uint8_t *scales, float *cent_bf16, uint8_t *assign,
                          int32_t *iters, int n_threads)
{
    qo_batch b = {x, n, d, bits, gsize, stages, k, max_iters, tol, draws, payload, scales,
                  cent_bf16, assign, iters, NULL, 0};
    qo_parallel_for(P, n_threads, compress_one, &b);
    return b.rc;
}

static void decompress_one(int64_t p, void *v)
{
    qo_batch *b = v;
    int64_t n = b->n, d = b->d, pb = (n * d * b->bits + 7) / 8, sb = n * d / b->gsize;
    int64_t sk = (int64_t)b->stages * b->k;
    qo_prq_decompress(b->payload + p * pb, b->scales + p * sb, b->cent + p * sk * d,
                      b->assign + p * b->stages * n, n, b->d, b->bits, b->gsize, b->stages, b->k,
                      b->out + p * n * d);
}

void qo_prq_decompress_batch(const uint8_t *payload, const uint8_t *scales, const float *cent_bf16,
                             const uint8_t *assign, int64_t P, int64_t n, int d, int bits,
                             int gsize, int stages, int k, float *out, int n_threads)
{
    qo_batch b = {NULL, n, d, bits, gsize, stages, k, 0, 0.0, NULL, (uint8_t *)payload,
                  (uint8_t *)scales, (float *)cent_bf16, (uint8_t *)assign, NULL, out, 0};
    qo_parallel_for(P, n_threads, decompress_one, &b);
}

/* Given-metas quantize (the K5 contract): residual chain from x and the
 * stored bf16 centroids/assignments (Q/smoothing.py:40 per stage), then
 * quantize_matrix (Q/quant.py:134).  Batched over planes. */
static void quantize_one(int64_t p, void *v)
{
    qo_batch *b = v;
    int64_t n = b->n, d = b->d, pb = (n * d * b->bits + 7) / 8, sb = n * d / b->gsize;
    int64_t S = b->stages, k = b->k;
    double *res = malloc(sizeof(double) * n * d);
    const float *xp = b->x + p * n * d;
    for (int64_t i = 0; i < n; i++)
        for (int64_t j = 0; j < d; j++) {
            double r = (double)xp[i * d + j];
            for (int64_t t = 0; t < S; t++)
                r = r - (double)b->cent[((p * S + t) * k + b->assign[(p * S + t) * n + i]) * d + j];
            res[i * d + j] = r;
        }
    int rc = qo_quantize_matrix(res, n, b->d, b->bits, b->gsize, b->payload + p * pb,
                                b->scales + p * sb);
    if (rc) b->rc = rc;
    free(res);
}

int qo_quantize_given_metas_batch(const float *x, int64_t P, int64_t n, int d, int bits, int gsize,
                                  int stages, int k, const float *cent_bf16, const uint8_t *assign,
                                  uint8_t *payload, uint8_t *scales, int n_threads)
{
    qo_batch b = {x, n, d, bits, gsize, stages, k, 0, 0.0, NULL, payload, scales,
                  (float *)cent_bf16, (uint8_t *)assign, NULL, NULL, 0};
    qo_parallel_for(P, n_threads, quantize_one, &b);
    return b.rc;
}

/* ---------------------------------------------------------------------- */
/* Attention oracle (no reference symbol): per head,        */
/* O = softmax(q K^T * scale) V over [K_cache ; K_cur], all in fp64.       */
/* q: [nq][h][d] f32, kc/vc: [h][nc][d] f32 (dequantized cache),           */
/* kn/vn: [ncur][h][d] f32 (current chunk), out: [nq][h][d] f64.           */
/* ---------------------------------------------------------------------- */
typedef struct {
    const float *q, *kc, *vc, *kn, *vn; int64_t nc, ncur; int h, d; double scale; double *out;
} qo_att;

static void attention_row(int64_t qi, void *v)
{
    qo_att *a = v;
    int64_t i = qi / a->h, nc = a->nc, nkv = a->nc + a->ncur;
    int hh = (int)(qi % a->h), h = a->h, d = a->d;
    double *s = malloc(sizeof(double) * nkv);
    const float *qv = a->q + (i * h + hh) * d;
    double mx = -INFINITY;
    for (int64_t j = 0; j < nkv; j++) {
        const float *kv = j < nc ? a->kc + ((int64_t)hh * nc + j) * d
                                 : a->kn + ((j - nc) * h + hh) * d;
        double acc = 0.0;
        for (int t = 0; t < d; t++) acc += (double)qv[t] * (double)kv[t];
        s[j] = acc * a->scale;
        if (s[j] > mx) mx = s[j];
    }
    double den = 0.0;
    for (int64_t j = 0; j < nkv; j++) { s[j] = exp(s[j] - mx); den += s[j]; }
    double *o = a->out + (i * h + hh) * d;
    for (int t = 0; t < d; t++) o[t] = 0.0;
    for (int64_t j = 0; j < nkv; j++) {
        const float *vv = j < nc ? a->vc + ((int64_t)hh * nc + j) * d
                                 : a->vn + ((j - nc) * h + hh) * d;
        double w = s[j] / den;
        for (int t = 0; t < d; t++) o[t] += w * (double)vv[t];
    }
    free(s);
}

void qo_attention(const float *q, const float *kc, const float *vc, const float *kn,
                  const float *vn, int64_t nq, int64_t nc, int64_t ncur, int h, int d,
                  double scale, double *out, int n_threads)
{
    qo_att a = {q, kc, vc, kn, vn, nc, ncur, h, d, scale, out};
    qo_parallel_for(nq * h, n_threads, attention_row, &a);
}
