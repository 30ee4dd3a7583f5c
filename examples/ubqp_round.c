/* ubqp_round.c — one round of the diversified multi-start (Figure 2) driven from
 * plain C through the C-ABI of include/ubqp.h (no Python, no torch): host arrays in and out.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/ubqp_round.c -Lpaper_1706_00037_b200 -lubqp \
 *       -Wl,-rpath,$PWD/paper_1706_00037_b200 -o ubqp_round && ./ubqp_round [n] [K] [prefix]
 *
 * With a prefix, Q is written to prefix.Q (int32, row-major) and the round's results to
 * prefix.out (statistics, T, then one "slot f flips" line per survivor) -- tests/test_gpu_c_abi.py
 * checks them against the oracle.
 * Q: symmetric, coefficients uniform in [-100, 100] from a small xorshift generator (this
 * example only; the tests and bench use inputs/generate_Q). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "ubqp.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t xorshift(void) {
    rng_state ^= rng_state << 13;
    rng_state ^= rng_state >> 7;
    rng_state ^= rng_state << 17;
    return rng_state;
}

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_) {                                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, ubqp_last_error(h)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 2500;
    const int64_t K = argc > 2 ? atoll(argv[2]) : 65536;
    int32_t *Q = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j) {
            int32_t v = (int32_t)(xorshift() % 201) - 100;
            Q[(size_t)i * n + j] = v;
            Q[(size_t)j * n + i] = v;
        }
    ubqp_t h = NULL;
    if (ubqp_create(0, NULL, &h)) { fprintf(stderr, "ubqp_create failed\n"); return 1; }
    printf("libubqp ABI %d\n", ubqp_version());
    CHECK(ubqp_load_Q(h, n, Q, K));
    const int W64 = (n + 63) / 64;
    uint64_t *seed = (uint64_t *)calloc(W64, sizeof(uint64_t));
    CHECK(ubqp_first_derivative(h, seed));                     /* incumbent */
    CHECK(ubqp_diversify(h, seed, 0, K, 0, 1));                /* Glover diversification */
    ubqp_stats st;
    CHECK(ubqp_eval_batch(h, UBQP_EMIT_GAINS, NULL, &st));     /* f = x^T Q x + gains */
    const int64_t maxv = (st.max_key >> 22) - ((int64_t)1 << 40);
    int32_t *surv = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
    int64_t m = 0;
    double T = 0;
    CHECK(ubqp_screen(h, 0.5, st.sum, st.count, maxv, surv, &m, &T)); /* T(0.5) */
    int64_t *f = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int32_t *flips = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    int64_t best = -1;
    CHECK(ubqp_ascend(h, surv, m, 10 * n, f, flips, NULL, &best)); /* steepest ascent */
    int64_t total = 0;
    for (int64_t i = 0; i < m; ++i) total += flips[i];
    if (argc > 3) {
        char path[4096];
        snprintf(path, sizeof path, "%s.Q", argv[3]);
        FILE *fq = fopen(path, "wb");
        if (!fq || fwrite(Q, sizeof(int32_t), (size_t)n * n, fq) != (size_t)n * n) { fprintf(stderr, "write %s\n", path); return 1; }
        fclose(fq);
        snprintf(path, sizeof path, "%s.out", argv[3]);
        FILE *fo = fopen(path, "w");
        if (!fo) { fprintf(stderr, "write %s\n", path); return 1; }
        fprintf(fo, "%lld %lld %lld %.17g %lld %lld\n", (long long)st.sum, (long long)st.count, (long long)st.max_key, T,
                (long long)m, (long long)best);
        for (int64_t i = 0; i < m; ++i) fprintf(fo, "%d %lld %d\n", surv[i], (long long)f[i], flips[i]);
        fclose(fo);
    }
    printf("n=%d K=%lld mean=%.1f max=%lld T=%.1f survivors=%lld flips=%lld best f=%lld (g=%lld)\n", n,
           (long long)K, (double)st.sum / (double)st.count, (long long)maxv, T, (long long)m, (long long)total,
           best >= 0 ? (long long)((best >> 22) - ((int64_t)1 << 40)) : 0LL,
           best >= 0 ? (long long)(((int64_t)1 << 22) - 1 - (best & (((int64_t)1 << 22) - 1))) : -1LL);
    ubqp_destroy(h);
    free(Q); free(seed); free(surv); free(f); free(flips);
    return 0;
}
