/*
 * ubqp_oracle.c — plain, slow, obviously-correct CPU oracle for the hot path of
 * Lewis, "A Diversified Multi-Start Algorithm for Unconstrained Binary Quadratic
 * Problems Leveraging the GPU" (arXiv 1706.00037).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path
 * (paper_1706_00037_b200/csrc); neither includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * O1..O10 / R1..R18 = SURVEY.md §8(c) definitions and readings (restated in DESIGN.md).
 *
 * Solutions are passed as one byte per variable (x_i in {0,1}), row-major
 * [K][n]; the packed-bit convention of the C-ABI is handled by the tests.
 * All objective arithmetic is exact int64 (R1, R18).  No blocking, fusion or
 * reordering: every function is the textbook loop of its definition.
 *
 * Parity pins: see tests/test_oracle_pins.py (brute force, closed forms,
 * SPEC worked examples, SplitMix64 KAT, Glover's illustration).
 *   O4 (Glover diversification): pinned only by Glover's own x = 0 example and
 *   the definition; the paper prints no vectors ("parity unpinned by the paper").
 *   O8 (round loop) quality vs Tables 1'/2: parity unpinned (no instance files).
 *   O4b (blend) and O11 (path relinking) are readings R11b / R19 of passages that
 *   print no operator; pinned by reductions, invariants, brute force and hand tables.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* O1  f(x) = x^t Q x = sum_i sum_j Q_ij x_i x_j   (eq. (P))     */
/* ------------------------------------------------------------------------- */
static int64_t xQx(int n, const int32_t *Q, const uint8_t *x)
{
    int64_t f = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            f += (int64_t)Q[(int64_t)i * n + j] * (int64_t)x[i] * (int64_t)x[j];
    return f;
}

typedef struct {
    int n;
    const int32_t *Q;
    const uint8_t *X;
    int64_t *f;
    int64_t begin, end;
} eval_job;

static void *eval_worker(void *arg)
{
    eval_job *j = (eval_job *)arg;
    for (int64_t k = j->begin; k < j->end; ++k)
        j->f[k] = xQx(j->n, j->Q, j->X + k * (int64_t)j->n);
    return NULL;
}

/* Evaluate K solutions; threads split the solution list only (the
 * result is independent of the degree of parallelism). */
int oracle_eval_batch(int n, const int32_t *Q, int64_t K, const uint8_t *X,
                      int64_t *f_out, int nthreads)
{
    if (n < 0 || K < 0) return 1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    eval_job jobs[256];
    int64_t per = (K + nthreads - 1) / nthreads;
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].n = n; jobs[t].Q = Q; jobs[t].X = X; jobs[t].f = f_out;
        jobs[t].begin = (int64_t)t * per;
        jobs[t].end = jobs[t].begin + per > K ? K : jobs[t].begin + per;
        if (jobs[t].begin >= jobs[t].end) break;
        if (nthreads == 1) { eval_worker(&jobs[t]); continue; }
        pthread_create(&th[t], NULL, eval_worker, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    return 0;
}

int64_t oracle_eval(int n, const int32_t *Q, const uint8_t *x) { return xQx(n, Q, x); }

/* ------------------------------------------------------------------------- */
/* O2  Delta_i = f(x xor e_i) - f(x) = (1 - 2 x_i)(Q_ii + 2 sum_{j!=i} Q_ij x_j)  */
/*     ("effect ... of flipping one bit")                  */
/* ------------------------------------------------------------------------- */
void oracle_gains(int n, const int32_t *Q, const uint8_t *x, int64_t *Delta)
{
    for (int i = 0; i < n; ++i) {
        int64_t s = 0;
        for (int j = 0; j < n; ++j)
            if (j != i) s += (int64_t)Q[(int64_t)i * n + j] * (int64_t)x[j];
        Delta[i] = (int64_t)(1 - 2 * (int)x[i]) * ((int64_t)Q[(int64_t)i * n + i] + 2 * s);
    }
}

/* ------------------------------------------------------------------------- */
/* O3  random solutions ("randomly generated x"; R12) */
/*     SplitMix64 finaliser; word(g,w) = mix(seed + (g*W64 + w + 1)*golden).   */
/* ------------------------------------------------------------------------- */
uint64_t oracle_splitmix_word(uint64_t seed, int64_t g, int64_t W64, int64_t w)
{
    uint64_t z = seed + ((uint64_t)g * (uint64_t)W64 + (uint64_t)w + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* O10: slot i on rank r of `world` <-> global index g = (r + floor(i/B) world) B + (i mod B):
 * blocks of B consecutive g, dealt round robin (B = 1: g = r + i world).  Every output depends
 * on g only, so results do not depend on (world, B). */
static int64_t global_index(int64_t i, int rank, int world, int block)
{
    return ((int64_t)rank + (i / block) * (int64_t)world) * block + i % block;
}

void oracle_random(int n, uint64_t seed, int64_t k_local, int rank, int world, int block, uint8_t *X)
{
    int64_t W64 = (n + 63) / 64;
    for (int64_t i = 0; i < k_local; ++i) {
        int64_t g = global_index(i, rank, world, block);
        for (int j = 0; j < n; ++j) {
            uint64_t word = oracle_splitmix_word(seed, g, W64, j / 64);
            X[i * n + j] = (uint8_t)((word >> (j % 64)) & 1u);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O4  Glover (1998) diversification generator, enumerated by the loop counter */
/*     ("based on the loop counter"; R11)               */
/*     t -> (h, q, c):  h = floor((1 + isqrt(1 + 4t)) / 2),  r = t - h(h-1),   */
/*     q = floor(r/2) + 1,  c = r mod 2.  t is taken mod n(n+1).               */
/*     x = seed xor M(h,q), M(h,q) = {j = q-1 + k h < n};  complement if c=1.  */
/* ------------------------------------------------------------------------- */
static int64_t isqrt64(int64_t v)
{
    /* plain integer square root by bisection: largest s with s*s <= v */
    int64_t lo = 0, hi = 3037000499LL; /* floor(sqrt(2^63-1)) */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo + 1) / 2;
        if (mid <= v / mid) lo = mid; else hi = mid - 1;
    }
    return lo;
}

void oracle_glover_params(int64_t t, int n, int64_t *h, int64_t *q, int *c)
{
    int64_t period = (int64_t)n * ((int64_t)n + 1);
    t = t % period;
    int64_t hh = (1 + isqrt64(1 + 4 * t)) / 2;
    int64_t r = t - hh * (hh - 1);
    *h = hh;
    *q = r / 2 + 1;
    *c = (int)(r % 2);
}

void oracle_diversify(int n, const uint8_t *seed, int64_t t0, int64_t k_local, int rank,
                      int world, int block, uint8_t *X)
{
    for (int64_t i = 0; i < k_local; ++i) {
        int64_t g = global_index(i, rank, world, block);
        int64_t h, q; int c;
        oracle_glover_params(t0 + g, n, &h, &q, &c);
        uint8_t *x = X + i * n;
        for (int j = 0; j < n; ++j) x[j] = seed[j];
        for (int64_t j = q - 1; j < n; j += h) x[j] = (uint8_t)(1 - x[j]);
        if (c == 1)
            for (int j = 0; j < n; ++j) x[j] = (uint8_t)(1 - x[j]);
    }
}

/* ------------------------------------------------------------------------- */
/* O4b blend ("diversification approaches based on blending (or breeding) two  */
/*     solutions"; reading R11b).  Parent p = parents[g mod P]; */
/*     (h, q, c) from t = t0 + g as in O4; the child takes p's bit on the mask  */
/*     M(h,q) = {q-1, q-1+h, ...} (its complement within n bits when c = 1) and */
/*     the seed's (incumbent's) bit everywhere else.  With p = NOT seed this is */
/*     exactly O4.                                                               */
/* ------------------------------------------------------------------------- */
void oracle_blend(int n, const uint8_t *seed, const uint8_t *parents, int64_t n_parents, int64_t t0,
                  int64_t k_local, int rank, int world, int block, uint8_t *X)
{
    for (int64_t i = 0; i < k_local; ++i) {
        int64_t g = global_index(i, rank, world, block);
        const uint8_t *p = parents + (g % n_parents) * (int64_t)n;
        int64_t h, q; int c;
        oracle_glover_params(t0 + g, n, &h, &q, &c);
        uint8_t *x = X + i * n;
        for (int j = 0; j < n; ++j) {
            int in_m = (j >= q - 1) && ((j - (q - 1)) % h == 0);
            int take_parent = c == 1 ? !in_m : in_m;
            x[j] = take_parent ? p[j] : seed[j];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O5  batch statistics {sum f, count, max_key}  (R14)            */
/*     max_key = ((f + 2^40) << 22) | (2^22 - 1 - g): highest f, then lowest g */
/* ------------------------------------------------------------------------- */
int64_t oracle_max_key(int64_t f, int64_t g)
{
    return (int64_t)(((uint64_t)(f + (1LL << 40)) << 22) | (uint64_t)((1LL << 22) - 1 - g));
}

void oracle_stats(int64_t k_local, const int64_t *f, int rank, int world, int block, int64_t *out4)
{
    int64_t sum = 0, best = -1;
    for (int64_t i = 0; i < k_local; ++i) {
        sum += f[i];
        int64_t key = oracle_max_key(f[i], global_index(i, rank, world, block));
        if (key > best) best = key;
    }
    out4[0] = sum; out4[1] = k_local; out4[2] = best; out4[3] = 0;
}

/* ------------------------------------------------------------------------- */
/* O6  screen: T(lambda) = Mean + lambda (Max - Mean)  (P:49;    */
/*     R8 strict, R16 binary64 without contraction).  survivors ascending.   */
/* ------------------------------------------------------------------------- */
double oracle_threshold(double lambda, int64_t mean_sum, int64_t mean_count, int64_t max_value)
{
    double mean = (double)mean_sum / (double)mean_count;
    double diff = (double)max_value - mean;
    double scaled = lambda * diff;
    return mean + scaled;
}

int64_t oracle_screen(int64_t k_local, const int64_t *f, double T, int32_t *surv)
{
    int64_t m = 0;
    for (int64_t i = 0; i < k_local; ++i)
        if ((double)f[i] > T) surv[m++] = (int32_t)i;   /* f > T, "if xQx > Screening_value" */
    return m;
}

/* ------------------------------------------------------------------------- */
/* O7  steepest ascent on 1-bit flips (R9)   */
/*   loop: k* = argmax_j Delta_j (lowest j on ties); stop if Delta_k* <= 0 or */
/*   flips == max_flips; f += Delta_k*; d = 1 - 2 x_k*; x_k* ^= 1;            */
/*   Delta_l += 2 Q_{l,k*} d (1 - 2 x_l) for l != k*; Delta_k* = -Delta_k*.   */
/* ------------------------------------------------------------------------- */
static int64_t ascend_one(int n, const int32_t *Q, uint8_t *x, int64_t f, int max_flips,
                          int32_t *flips_out, int64_t *Delta)
{
    oracle_gains(n, Q, x, Delta);
    int flips = 0;
    for (;;) {
        int kstar = 0;
        for (int j = 1; j < n; ++j)
            if (Delta[j] > Delta[kstar]) kstar = j;   /* strict: keeps the lowest index */
        if (n == 0 || Delta[kstar] <= 0 || flips == max_flips) break;
        f += Delta[kstar];
        int64_t d = 1 - 2 * (int64_t)x[kstar];
        x[kstar] = (uint8_t)(1 - x[kstar]);
        for (int l = 0; l < n; ++l)
            if (l != kstar)
                Delta[l] += 2 * (int64_t)Q[(int64_t)l * n + kstar] * d * (1 - 2 * (int64_t)x[l]);
        Delta[kstar] = -Delta[kstar];
        ++flips;
    }
    *flips_out = flips;
    return f;
}

typedef struct {
    int n; const int32_t *Q; uint8_t *X; int64_t *f; int32_t *flips; int max_flips;
    int64_t begin, end;
} ascend_job;

static void *ascend_worker(void *arg)
{
    ascend_job *j = (ascend_job *)arg;
    int64_t *Delta = (int64_t *)malloc(sizeof(int64_t) * (size_t)(j->n > 0 ? j->n : 1));
    for (int64_t k = j->begin; k < j->end; ++k)
        j->f[k] = ascend_one(j->n, j->Q, j->X + k * (int64_t)j->n, j->f[k], j->max_flips,
                             &j->flips[k], Delta);
    free(Delta);
    return NULL;
}

/* In place: X[m][n] (start solutions -> local optima), f[m] (start values ->
 * final values; the caller passes f(x) of each start), flips[m] out. */
int oracle_ascend_batch(int n, const int32_t *Q, int64_t m, uint8_t *X, int64_t *f,
                        int32_t *flips, int max_flips, int nthreads)
{
    if (n < 0 || m < 0) return 1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    ascend_job jobs[256];
    int64_t per = (m + nthreads - 1) / nthreads;
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (ascend_job){n, Q, X, f, flips, max_flips, (int64_t)t * per, 0};
        jobs[t].end = jobs[t].begin + per > m ? m : jobs[t].begin + per;
        if (jobs[t].begin >= jobs[t].end) break;
        if (nthreads == 1) { ascend_worker(&jobs[t]); continue; }
        pthread_create(&th[t], NULL, ascend_worker, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O11 path relinking (NEXT-4: Glover's "Scatter Search / Path Relinking      */
/*     Phase"; the paper defers "solution polishing";      */
/*     DESIGN.md reading R19).  From x0 toward the guide y: D = {j: x0_j !=   */
/*     y_j}; |D| forced steps, each flipping the j in D of largest gain       */
/*     Delta_j (lowest j on ties; the move may worsen f), D -= {j}, gains     */
/*     updated as in O7.  Result: the best strictly interior point (1 <= s <  */
/*     |D|; highest f, earliest s on ties); s_best = -1 when |D| < 2.         */
/* ------------------------------------------------------------------------- */
static void relink_one(int n, const int32_t *Q, const uint8_t *x0, const uint8_t *y, int64_t f0,
                       uint8_t *xbest, int64_t *fbest, int32_t *sbest, int32_t *len, int32_t *path,
                       int64_t *Delta, uint8_t *x, uint8_t *D)
{
    int nd = 0;
    for (int j = 0; j < n; ++j) {
        x[j] = x0[j];
        xbest[j] = x0[j];
        D[j] = (uint8_t)(x0[j] != y[j]);
        nd += D[j];
    }
    oracle_gains(n, Q, x, Delta);
    int64_t f = f0;
    *fbest = INT64_MIN;
    *sbest = -1;
    *len = nd;
    for (int s = 1; s <= nd; ++s) {
        int k = -1;
        for (int j = 0; j < n; ++j)
            if (D[j] && (k < 0 || Delta[j] > Delta[k])) k = j;   /* strict: lowest j on ties */
        f += Delta[k];
        int64_t d = 1 - 2 * (int64_t)x[k];
        x[k] = (uint8_t)(1 - x[k]);
        D[k] = 0;
        for (int l = 0; l < n; ++l)
            if (l != k)
                Delta[l] += 2 * (int64_t)Q[(int64_t)l * n + k] * d * (1 - 2 * (int64_t)x[l]);
        Delta[k] = -Delta[k];
        if (path) path[s - 1] = k;
        if (s < nd && f > *fbest) {
            *fbest = f;
            *sbest = s;
            for (int j = 0; j < n; ++j) xbest[j] = x[j];
        }
    }
}

typedef struct {
    int n; const int32_t *Q; const uint8_t *X0; const int64_t *f0; const uint8_t *Y; int64_t n_guides;
    uint8_t *Xb; int64_t *fb; int32_t *sb; int32_t *len; int32_t *path; int64_t begin, end;
} relink_job;

static void *relink_worker(void *arg)
{
    relink_job *j = (relink_job *)arg;
    size_t nn = (size_t)(j->n > 0 ? j->n : 1);
    int64_t *Delta = (int64_t *)malloc(sizeof(int64_t) * nn);
    uint8_t *x = (uint8_t *)malloc(nn), *D = (uint8_t *)malloc(nn);
    for (int64_t i = j->begin; i < j->end; ++i)
        relink_one(j->n, j->Q, j->X0 + i * (int64_t)j->n, j->Y + (i % j->n_guides) * (int64_t)j->n, j->f0[i],
                   j->Xb + i * (int64_t)j->n, &j->fb[i], &j->sb[i], &j->len[i],
                   j->path ? j->path + i * (int64_t)j->n : NULL, Delta, x, D);
    free(Delta); free(x); free(D);
    return NULL;
}

/* X0[m][n] initiating solutions with values f0[m]; guide of i = Y[i mod n_guides];
 * out: Xb[m][n] best interior points, fb[m] (INT64_MIN if none), sb[m] (-1 if none),
 * len[m] = |D|, path[m][n] flip order (optional, may be NULL). */
int oracle_relink_batch(int n, const int32_t *Q, int64_t m, const uint8_t *X0, const int64_t *f0,
                        const uint8_t *Y, int64_t n_guides, uint8_t *Xb, int64_t *fb, int32_t *sb,
                        int32_t *len, int32_t *path, int nthreads)
{
    if (n < 1 || m < 0 || n_guides < 1) return 1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    relink_job jobs[256];
    int64_t per = (m + nthreads - 1) / nthreads;
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (relink_job){n, Q, X0, f0, Y, n_guides, Xb, fb, sb, len, path, (int64_t)t * per, 0};
        jobs[t].end = jobs[t].begin + per > m ? m : jobs[t].begin + per;
        if (jobs[t].begin >= jobs[t].end) break;
        if (nthreads == 1) { relink_worker(&jobs[t]); continue; }
        pthread_create(&th[t], NULL, relink_worker, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* first-derivative start: x_i = 1 iff sum_j Q_ij > 0 */
void oracle_first_derivative_start(int n, const int32_t *Q, uint8_t *x)
{
    for (int i = 0; i < n; ++i) {
        int64_t s = 0;
        for (int j = 0; j < n; ++j) s += Q[(int64_t)i * n + j];
        x[i] = (uint8_t)(s > 0 ? 1 : 0);
    }
}
