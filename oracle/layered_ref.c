/*
 * oracle/layered_ref.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, FP64 restatement of the reference layered belief-propagation
 * decoder (/root/reference/pkg/src/qcldpc/decoder.py).  It is the CPU checker
 * the parity tests compare the CUDA path against, and the CPU arm that
 * bench.py times beside it ("cpu_baseline", kind "port").  Nothing in the
 * product package may link or call it; only tests/, __graft_entry__.smoke()
 * and bench.py's reference/cpu_baseline legs do.
 *
 * Parity is pinned against the reference itself: tests/golden/make_golden.py
 * imports the reference package in the build container and dumps its outputs
 * (per-layer states, sweeps, full decodes); tests/test_oracle.py checks this
 * file against those fixtures.
 *
 * Arithmetic follows the reference operation by operation:
 *   phi(x)        = log1p(2 / expm1(clip(x, eps, clip)))       decoder.py:96-105
 *   q             = clip(L[v] - r_old, +-clip)                 decoder.py:219-220
 *   ph            = phi(|q|)                                    decoder.py:225
 *   total (uniform-degree layer)   left fold over the row      decoder.py:233 (sum(axis=2))
 *   total (ragged layer)           a0 + pairwise(a1..)         decoder.py:240 (np.add.reduceat)
 *   mag           = phi(total - ph)                             decoder.py:235/241
 *   sign          = (q<0) ^ XOR_row(q<0) ^ syndrome             decoder.py:234/242-243
 *   r_new         = clip(sign ? -mag : mag)                     decoder.py:244-245
 *   L[v]          = clip(q + r_new)                             decoder.py:248-250
 *   hard decision = (L < 0)  (-0.0 -> 0)                        decoder.py:264-266
 *   ET bookkeeping: freeze words/iterations at first sweep whose hard
 *   decision satisfies the syndrome                             decoder.py:292-311
 * numpy's pairwise summation (n<8: left fold from 0.0; else 8 accumulators,
 * ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail) is restated in pw_sum.
 * Transcendentals come from libm; numpy's SIMD expm1/log1p differ from libm
 * by 1 ulp on ~2% of inputs, so FP64 posteriors are
 * compared with a ulp-level tolerance, decisions bit-exactly.
 *
 * Layouts are the reference's: posterior (B, n) row-major; edge messages
 * (B, total_edges * z) with slot s, edge j of the slot, offset k at
 * (slot_offsets[s] + j) * z + k (decoder.py:79-83, 216); syndrome (B, m) in
 * ORIGINAL check order row * z + k (decoder.py:168-170).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct {
    int z, n_cols, n_slots, n_layers, n_edges;
    const int32_t *edge_shift, *edge_col, *slot_off, *slot_row, *layer_start;
} orc_code;

static inline double clampd(double x, double lo, double hi) {
    /* np.clip semantics for finite bounds: NaN-free inputs only */
    return x < lo ? lo : (x > hi ? hi : x);
}

double orc_phi(double x, double eps, double clip) {
    x = clampd(x, eps, clip);
    return log1p(2.0 / expm1(x));
}

void orc_phi_array(const double *x, int64_t n, double eps, double clip, double *out) {
    for (int64_t i = 0; i < n; i++) out[i] = orc_phi(x[i], eps, clip);
}

/* numpy pairwise_sum for the contiguous-free reduce loop (n < 128 here). */
static double pw_sum(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r += a[i];
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
}

static int layer_is_uniform(const orc_code *c, int layer) {
    int s0 = c->layer_start[layer], s1 = c->layer_start[layer + 1];
    int d0 = c->slot_off[s0 + 1] - c->slot_off[s0];
    for (int s = s0 + 1; s < s1; s++)
        if (c->slot_off[s + 1] - c->slot_off[s] != d0) return 0;
    return 1;
}

static int max_degree(const orc_code *c) {
    int m = 0;
    for (int s = 0; s < c->n_slots; s++) {
        int d = c->slot_off[s + 1] - c->slot_off[s];
        if (d > m) m = d;
    }
    return m;
}

/* One layer on one frame.  post: n doubles; msg: n_edges*z doubles; syn: m bytes or NULL. */
static void layer_one(const orc_code *c, int layer, double *post, double *msg, const uint8_t *syn,
                      double clip, double eps, double *q, double *ph) {
    const int z = c->z;
    const int uniform = layer_is_uniform(c, layer);
    for (int s = c->layer_start[layer]; s < c->layer_start[layer + 1]; s++) {
        const int e0 = c->slot_off[s], d = c->slot_off[s + 1] - e0;
        const int row = c->slot_row[s];
        for (int k = 0; k < z; k++) {
            int parity = syn ? (syn[(int64_t)row * z + k] != 0) : 0;
            for (int j = 0; j < d; j++) {
                int e = e0 + j;
                int pos = k + c->edge_shift[e];
                if (pos >= z) pos -= z;
                int64_t v = (int64_t)c->edge_col[e] * z + pos;
                double qq = clampd(post[v] - msg[(int64_t)e * z + k], -clip, clip);
                q[j] = qq;
                ph[j] = orc_phi(fabs(qq), eps, clip);
                parity ^= (qq < 0);
            }
            double total;
            if (uniform) {
                total = ph[0];
                for (int j = 1; j < d; j++) total += ph[j];
            } else {
                total = ph[0] + pw_sum(ph + 1, d - 1);
            }
            for (int j = 0; j < d; j++) {
                int e = e0 + j;
                int pos = k + c->edge_shift[e];
                if (pos >= z) pos -= z;
                int64_t v = (int64_t)c->edge_col[e] * z + pos;
                double mag = orc_phi(total - ph[j], eps, clip);
                int neg = (q[j] < 0) ^ parity;
                double r = clampd(neg ? -mag : mag, -clip, clip);
                msg[(int64_t)e * z + k] = r;
                post[v] = clampd(q[j] + r, -clip, clip);
            }
        }
    }
}

static int64_t n_vars(const orc_code *c) { return (int64_t)c->n_cols * c->z; }
static int64_t n_checks(const orc_code *c) { return (int64_t)c->n_slots * c->z; }
static int64_t n_msgs(const orc_code *c) { return (int64_t)c->n_edges * c->z; }

/* Apply `layer` (or every layer in order when layer < 0) to a (B, ...) state. */
void orc_layer_update(const orc_code *c, int layer, double *post, double *msg, const uint8_t *syn,
                      int64_t batch, double clip, double eps) {
    int dmax = max_degree(c);
    double *q = (double *)malloc(sizeof(double) * dmax * 2);
    double *ph = q + dmax;
    for (int64_t b = 0; b < batch; b++) {
        const uint8_t *sb = syn ? syn + b * n_checks(c) : NULL;
        if (layer >= 0) {
            layer_one(c, layer, post + b * n_vars(c), msg + b * n_msgs(c), sb, clip, eps, q, ph);
        } else {
            for (int l = 0; l < c->n_layers; l++)
                layer_one(c, l, post + b * n_vars(c), msg + b * n_msgs(c), sb, clip, eps, q, ph);
        }
    }
    free(q);
}

/* H x == syndrome over GF(2), evaluated from the posterior signs of one frame. */
static int frame_satisfied(const orc_code *c, const double *post, const uint8_t *syn) {
    const int z = c->z;
    for (int s = 0; s < c->n_slots; s++) {
        int row = c->slot_row[s];
        for (int k = 0; k < z; k++) {
            int p = 0;
            for (int e = c->slot_off[s]; e < c->slot_off[s + 1]; e++) {
                int pos = k + c->edge_shift[e];
                if (pos >= z) pos -= z;
                p ^= post[(int64_t)c->edge_col[e] * z + pos] < 0;
            }
            int want = syn ? (syn[(int64_t)row * z + k] != 0) : 0;
            if (p != want) return 0;
        }
    }
    return 1;
}

static void decode_frame(const orc_code *c, const double *llr, const uint8_t *syn, int max_iter,
                         int early_term, double clip, double eps, uint8_t *word, uint8_t *conv,
                         int64_t *iters, double *post_out) {
    const int64_t n = n_vars(c);
    double *post = (double *)malloc(sizeof(double) * n);
    double *msg = (double *)calloc((size_t)n_msgs(c), sizeof(double));
    int dmax = max_degree(c);
    double *q = (double *)malloc(sizeof(double) * dmax * 2);
    for (int64_t v = 0; v < n; v++) post[v] = clampd(llr[v], -clip, clip);
    int done = 0;
    *iters = max_iter;
    *conv = 0;
    for (int t = 1; t <= max_iter && !done; t++) {
        for (int l = 0; l < c->n_layers; l++) layer_one(c, l, post, msg, syn, clip, eps, q, q + dmax);
        if (early_term && frame_satisfied(c, post, syn)) {
            for (int64_t v = 0; v < n; v++) word[v] = post[v] < 0;
            *conv = 1;
            *iters = t;
            done = 1;
        }
    }
    if (!done) {
        for (int64_t v = 0; v < n; v++) word[v] = post[v] < 0;
        *conv = (uint8_t)frame_satisfied(c, post, syn);
    }
    if (post_out) memcpy(post_out, post, sizeof(double) * n);
    free(q);
    free(msg);
    free(post);
}

/* Batch decode; frames are independent (decoder.py:18-21), so host threads
 * split them (the reference splits a batch over a ThreadPoolExecutor,
 * bench.py:139-150).  post_out (B, n) may be NULL; otherwise it receives each
 * frame's posterior after its own last sweep. */
typedef struct {
    const orc_code *c;
    const double *llr;
    const uint8_t *syn;
    int64_t batch;
    int max_iter, early_term;
    double clip, eps;
    uint8_t *words, *converged;
    int64_t *iterations;
    double *post_out;
    int64_t next; /* shared frame counter */
    pthread_mutex_t lock;
} decode_job;

static void *decode_worker(void *arg) {
    decode_job *j = (decode_job *)arg;
    const int64_t n = n_vars(j->c), m = n_checks(j->c);
    for (;;) {
        pthread_mutex_lock(&j->lock);
        int64_t b = j->next++;
        pthread_mutex_unlock(&j->lock);
        if (b >= j->batch) break;
        decode_frame(j->c, j->llr + b * n, j->syn ? j->syn + b * m : NULL, j->max_iter, j->early_term,
                     j->clip, j->eps, j->words + b * n, j->converged + b, j->iterations + b,
                     j->post_out ? j->post_out + b * n : NULL);
    }
    return NULL;
}

int orc_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

void orc_decode(const orc_code *c, const double *llr, const uint8_t *syn, int64_t batch, int max_iter,
                int early_term, double clip, double eps, int threads, uint8_t *words, uint8_t *converged,
                int64_t *iterations, double *post_out) {
    decode_job job = {c, llr, syn, batch, max_iter, early_term, clip, eps, words, converged,
                      iterations, post_out, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = orc_threads();
    if (threads > batch) threads = (int)(batch > 0 ? batch : 1);
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (int t = 1; t < threads; t++) pthread_create(&tid[t], NULL, decode_worker, &job);
    decode_worker(&job);
    for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
    free(tid);
}

/* Syndrome of hard words (B, n) -> (B, m) in original check order. */
void orc_syndrome(const orc_code *c, const uint8_t *words, int64_t batch, uint8_t *out) {
    const int z = c->z;
    const int64_t n = n_vars(c), m = n_checks(c);
    for (int64_t b = 0; b < batch; b++)
        for (int s = 0; s < c->n_slots; s++)
            for (int k = 0; k < z; k++) {
                int p = 0;
                for (int e = c->slot_off[s]; e < c->slot_off[s + 1]; e++) {
                    int pos = k + c->edge_shift[e];
                    if (pos >= z) pos -= z;
                    p ^= words[b * n + (int64_t)c->edge_col[e] * z + pos] & 1;
                }
                out[b * m + (int64_t)c->slot_row[s] * z + k] = (uint8_t)p;
            }
}

