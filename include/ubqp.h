/*
 * ubqp.h — C-ABI of the B200 (sm_100a) hot path of Lewis's GPU diversified
 * multi-start for the Unconstrained Binary Quadratic Problem (arXiv 1706.00037):
 *
 *     (P)  maximise f(x) = x^t Q x,  x in {0,1}^n,  Q symmetric
 *
 * One round of the method (Figure 2) is the call sequence
 *     ubqp_diversify | ubqp_random | ubqp_set_batch   -> a batch of K_r solutions
 *     ubqp_eval_batch                                 -> f = xQx (+ 1-flip gains, stats)
 *     [caller all-reduces the stats across ranks]
 *     ubqp_screen                                     -> survivors of T(lambda)
 *     ubqp_ascend                                     -> 1-flip local optima + best key
 * with, beyond that core: ubqp_blend (blend / breeding diversification),
 * ubqp_relink (path relinking), and the real-valued Q path ubqp_load_Q_real /
 * ubqp_eval_batch_real / ubqp_screen_real / ubqp_ascend_real.
 * Implemented by libubqp.so (paper_1706_00037_b200/csrc).  No torch types, no NCCL.
 * ABI version 2.00 (ubqp_version() == 200): 2.00 widened ubqp_stats_real to int128 sums and
 * maxima of an exact evaluation image and added ubqp_set_option.
 * Citations: P:n = PAPER.md line n (section in brackets), S:n = SPEC.md line n.
 *
 * Conventions (all calls)
 *  - Return value: UBQP_OK or an error code; never throws.  On error the outputs are
 *    unspecified and ubqp_last_error(h) holds a message.  UBQP_E_CUDA is sticky: the
 *    handle must be destroyed.
 *  - Memory: every array argument may be a DEVICE pointer (on the handle's device)
 *    or a HOST pointer (pageable or pinned); the library detects which with
 *    cudaPointerGetAttributes.  Device arrays are read/written in stream order on the
 *    handle's stream and the call returns without synchronising; host arrays are
 *    copied through the stream and the call synchronises before returning.  The
 *    caller owns every buffer it passes; the handle owns Q, the batch and workspace.
 *  - Solutions: bit j of a solution is bit (j & 63) of 64-bit word (j >> 6); a
 *    solution is W64 = ceil(n/64) words, least significant bit first.  Padding bits
 *    (j >= n) are ignored on input and written as 0.
 *  - Sharding (multi-GPU, O10): slot i of a rank's batch is global
 *    solution g = (rank + floor(i/B)*world)*B + (i mod B) -- blocks of B consecutive g dealt
 *    round robin, B = ubqp_set_option(UBQP_OPT_SHARD_BLOCK), default 2 (B = 1: plain cyclic,
 *    g = rank + i*world).  B = 2 keeps each (c = 0, c = 1) complement pair of Glover's generator
 *    on one rank: with plain cyclic sharding and an even world every complemented solution
 *    (almost never a survivor) lands on the odd ranks and the ascent work on the even ones.
 *    Every output depends on g only, so results are identical for any world size and B.
 *    K (global batch) <= 2^22.
 *  - max_key = ((f + 2^40) << 22) | (2^22 - 1 - g): int64, larger = better; MAX over
 *    keys picks the highest f, ties to the lowest g (a valid NCCL int64 MAX operand).
 *    -1 means "no solution".
 */
#ifndef UBQP_H
#define UBQP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ubqp_ctx *ubqp_t;

enum {
    UBQP_OK = 0,
    UBQP_E_INVALID = 1,       /* null/negative/mismatched argument, bad slot, non-finite lambda */
    UBQP_E_NOT_SYMMETRIC = 2, /* Q != Q^t ("square symmetric matrix") */
    UBQP_E_RANGE = 3,         /* a coefficient outside [-127, 127] or an overflow bound fails */
    UBQP_E_STATE = 4,         /* call order: no Q loaded, no batch, mean_count <= 0, ... */
    UBQP_E_NOMEM = 5,         /* device allocation failed */
    UBQP_E_CUDA = 6           /* CUDA error (sticky) */
};

/* ubqp_eval_batch flags */
enum { UBQP_EMIT_GAINS = 1 };

/* batch statistics of ubqp_eval_batch (T(lambda) inputs): sum of f, count,
 * best max_key; reserved = 0.  int64 so the caller can all-reduce SUM/SUM/MAX. */
typedef struct {
    int64_t sum;
    int64_t count;
    int64_t max_key;
    int64_t reserved;
} ubqp_stats;

/* ABI version (major*100 + minor). */
int ubqp_version(void);

/* Create a handle bound to CUDA device `device` and stream `cuda_stream`
 * (a cudaStream_t; NULL = the handle creates and owns a non-blocking stream).
 * Errors: E_INVALID (out == NULL, bad device), E_CUDA. */
int ubqp_create(int device, void *cuda_stream, ubqp_t *out);

/* Destroy a handle and free its device memory (synchronises its stream). */
int ubqp_destroy(ubqp_t h);

/* Message of the last error on h (static string if h == NULL). Never NULL. */
const char *ubqp_last_error(ubqp_t h);

/* ReadQ/MoveQtoGPU (Figure 2; "the transfer of Q occurs only once").
 * Q: n*n int32, row-major, host or device.  Validates symmetry (E_NOT_SYMMETRIC) and
 * |Q_ij| <= 127 (E_RANGE: the evaluation runs on int8 tensor cores, exact),
 * then builds the device copies: Q8 int8 [ceil(n/256)*256][n_pad] (n_pad =
 * ceil(n/128)*128, zero padded) and diag int32.  k_max = workspace capacity in
 * solutions per batch (1 <= k_max <= 2^22).  n >= 1, n <= 16384.  Replaces any earlier
 * Q and batch.  Synchronises. */
int ubqp_load_Q(ubqp_t h, int32_t n, const int32_t *Q, int64_t k_max);

/* Diversify (Figure 2 line "Diversify(x, best_xQx, i, Q_cols)"; Glover 1998
 * diversification generator; "number of variables to be changed ... based on the
 * loop counter").  For slot i, t = t0 + g (g = rank + i*world), taken mod n(n+1):
 *   h = floor((1 + isqrt(1 + 4t))/2), r = t - h(h-1), q = floor(r/2) + 1, c = r mod 2,
 *   x = seed xor {bits q-1, q-1+h, q-1+2h, ... < n}, complemented within n bits if c = 1.
 * seed_bits: W64 words; 0 <= t0 <= 2^62.  Fills the handle's batch with k_local solutions
 * (0 <= k_local <= k_max).  Errors: E_INVALID, E_STATE (no Q). */
int ubqp_diversify(ubqp_t h, const uint64_t *seed_bits, int64_t t0, int64_t k_local,
                   int32_t rank, int32_t world);

/* Blend diversification ("Different diversification approaches based on blending
 * (or breeding) two solutions to generate new ones were implemented"; the operator is not
 * printed -- DESIGN.md reading R11b).  Slot i (global index g, t = t0 + g, (h, q, c)
 * as in ubqp_diversify) takes parent p = parents[g mod n_parents]'s bits on the Glover
 * mask M(h,q) (on its complement within n bits when c = 1) and seed_bits' elsewhere:
 *   x = seed xor (mask_c and (p xor seed)).
 * p = NOT seed reproduces ubqp_diversify exactly; p = seed gives the seed.  Every child
 * lies on a shortest seed-p path (path relinking).  parents: n_parents * W64 words,
 * host or device (host parents are staged in a handle-owned buffer, grown on demand,
 * synchronising the stream when it grows); 1 <= n_parents <= 2^22.  Bits >= n of seed
 * and parents are ignored.  Errors: E_INVALID, E_STATE (no Q), E_NOMEM. */
int ubqp_blend(ubqp_t h, const uint64_t *seed_bits, const uint64_t *parents, int64_t n_parents,
               int64_t t0, int64_t k_local, int32_t rank, int32_t world);

/* EvaluateRandomStarts' random solutions: bit j of slot i is bit
 * (j & 63) of SplitMix64-mix(seed + (g*W64 + (j>>6) + 1) * 0x9E3779B97F4A7C15),
 * g = the global index of slot i (see Sharding).  Fills the batch with k_local solutions. */
int ubqp_random(ubqp_t h, uint64_t seed, int64_t k_local, int32_t rank, int32_t world);

/* Load caller solutions bits[k_local][W64] as the batch (rank/world set their g). */
int ubqp_set_batch(ubqp_t h, const uint64_t *bits, int64_t k_local, int32_t rank,
                   int32_t world);

/* CalculateFirstDerivativeSolution (Figure 2; "simply sum the i^th row of Q
 * ... and if that sum is positive, then set x_i = 1"): bits_out[W64] gets x_i = 1 iff
 * sum_j Q_ij > 0 (for a real-valued Q: the exact row sums of its evaluation image, R22).
 * Requires a loaded Q; does not touch the batch. */
int ubqp_first_derivative(ubqp_t h, uint64_t *bits_out);

/* Copy the current batch out: bits_out[k_local][W64]. */
int ubqp_get_batch(ubqp_t h, uint64_t *bits_out);

/* Evaluate (Figure 2 "xQx <- Evaluate(x)"; "the GPU, which excels at matrix
 * multiplication"): for every slot k of the batch, f_k = x_k^t Q x_k computed as
 * Y = X Q on int8 tensor cores (int32 exact) with the row-dot f_k = sum_j x_kj Y_kj and the
 * statistics fused into the kernel (one launch; device f_out / stats_out are written by it).  flags & UBQP_EMIT_GAINS additionally stores the 1-flip
 * gains Delta_kj = Q_jj + 2(1 - 2 x_kj) Y_kj = f(x xor e_j) - f(x) on the device
 * for ubqp_ascend / ubqp_get_gains.  f_out: int64[k_local] (may be NULL); stats_out:
 * one ubqp_stats (may be NULL) = {sum f, k_local, max_key over the batch, 0}.
 * Errors: E_STATE (no batch). */
int ubqp_eval_batch(ubqp_t h, int flags, int64_t *f_out, ubqp_stats *stats_out);

/* Copy gains of slots [slot0, slot0+count) out as int32 [count][n] (requires the last
 * ubqp_eval_batch to have used UBQP_EMIT_GAINS; else E_STATE). */
int ubqp_get_gains(ubqp_t h, int64_t slot0, int64_t count, int32_t *gains_out);

/* Screen (Figure 2 "if xQx > Screening_value"; T(lambda) = Mean + lambda(Max - Mean),
 * P:49): mean = (double)mean_sum/(double)mean_count; T = mean + lambda*(max_value -
 * mean) in IEEE binary64 without contraction; survivors = {k : f_k > T} = {k : f_k >
 * floor(T)} of the last evaluated batch, in ascending slot order, written to
 * surv_out[0..m) (capacity k_local).  *m_out (host) = m; *T_out (host, may be NULL) = T.
 * Synchronises (m is returned to the host).  Errors: E_INVALID (lambda not finite),
 * E_STATE (mean_count <= 0 or no evaluated batch). */
int ubqp_screen(ubqp_t h, double lambda, int64_t mean_sum, int64_t mean_count,
                int64_t max_value, int32_t *surv_out, int64_t *m_out, double *T_out);

/* PerformSteepestAscent ("terminating when no improvements are possible or a
 * maximum number of flips have been made. No checks for cycling nor tabu lists",
 * P:93-95; 1-flip method of Glover et al. 2002).  For i < m, starting from batch
 * slot s = slots[i] (its f and gains from the last ubqp_eval_batch; gains are computed
 * here if that call did not emit them): repeat  k* = argmax_j Delta_j (lowest j on
 * ties); stop if Delta_k* <= 0 or flips == max_flips; f += Delta_k*; flip x_k*; update
 * Delta.  Outputs per i: f_out int64[m], flips_out int32[m], bits_out uint64[m][W64]
 * (any may be NULL), best_key_out: one int64 = max over i of max_key(f_i, g(s_i))
 * (-1 if m == 0; may be NULL).  The batch itself is not modified.
 * Errors: E_INVALID (slot out of range, m > k_local, max_flips < 0), E_STATE.  Host slots are
 * range-checked before launch; device-resident slots are checked in the kernel, and an
 * out-of-range one yields flips_out[i] = -1 (E_INVALID when flips_out is a host array). */
int ubqp_ascend(ubqp_t h, const int32_t *slots, int64_t m, int32_t max_flips,
                int64_t *f_out, int32_t *flips_out, uint64_t *bits_out,
                int64_t *best_key_out);

/* Path relinking (NEXT-4: Glover's scatter search / path relinking phase, which the
 * paper defers as "solution polishing"; reading R19).  For i < m,
 * from batch slot s = slots[i] (f and gains as for ubqp_ascend) toward the guide
 * y = guides[i mod n_guides] (W64 words each, host or device): D = {j : x_j != y_j};
 * |D| forced steps, each flipping the j in D of largest gain (lowest j on ties, even when
 * the move worsens f), D -= {j}.  Outputs per i: f_out int64[m] = the best strictly
 * interior value (1 <= step < |D|; highest f, earliest step on ties; INT64_MIN if |D| < 2),
 * step_out int32[m] its step (-1 if none), len_out int32[m] = |D|, bits_out
 * uint64[m][W64] that interior solution (the start itself if none), best_key_out = max
 * over i with an interior point of max_key(f_i, g(s_i)) (-1 if none).  Any output may
 * be NULL.  Requires (2n-1)*qmax < 2^21 (E_RANGE).  The batch is not modified.
 * Errors: E_INVALID (slot out of range, m > k_local, n_guides < 1), E_STATE, E_RANGE. */
int ubqp_relink(ubqp_t h, const uint64_t *guides, int64_t n_guides, const int32_t *slots,
                int64_t m, int64_t *f_out, int32_t *step_out, int32_t *len_out,
                uint64_t *bits_out, int64_t *best_key_out);

/* ---------------------------------------------------------------------------------
 * Real-valued Q (a4': "Q ... of real or integer coefficients"; "float or double",
 * P:89).  Two fixed-point images of Q are built at load (readings R20, R22):
 *
 *  - the EVALUATION image (R22) Qw = 2^-w rint(Q 2^w), with
 *        w = max over nonzero Q_ij of min(lsb(Q_ij), 32 - ex(Q_ij)),
 *    lsb(v) the least e making v 2^e an integer and |v| in [2^(ex-1), 2^ex): every coefficient
 *    is EXACT, or (only possible for float64 input) at least 2^31 units of 2^-w, i.e. within
 *    2^-32 |Q_ij|.  A float32 Q is always exact.  rint(Q 2^w) is stored as L <= 10 int8 planes
 *    of balanced base-128 digits, each run through the exact int8 tensor-core evaluation;
 *    f~ = x^t rint(Q 2^w) x is formed exactly (int128) and f = 2^-w f~ is rounded once to
 *    binary64.  Error bound for every accepted Q and every x (S = {i : x_i = 1}):
 *        |f - x^t Q x| <= 2^-32 sum_{i,j in S} |Q_ij| + 2^-53 |x^t Q x|
 *                      <= 2^-32 |S| s(x) + 2^-53 |x^t Q x|,   s(x) = sqrt(sum_{i,j in S} Q_ij^2)
 *    (Cauchy-Schwarz), so with |S| <= 16384: <= 3.9e-6 s(x) + 1.2e-16 |x^t Q x|, inside the
 *    north_star tolerance 1e-5 max(|f|, s(x)) (reading R3).  For float32 Q the first term
 *    vanishes: f is x^t Q x correctly rounded.  A Q needing more than 10 limbs (a dynamic
 *    range max|Q| / min|Q_ij != 0| beyond about 2^36 with float64 significands) is rejected
 *    with UBQP_E_RANGE.
 *  - the WALK image (R20) Qt = rint(Q 2^e) (half-even), e the largest integer with
 *    max|Q| 2^e <= 2^27 - 1 (ubqp_query UBQP_Q_REAL_EXP): the steepest ascent runs exactly on
 *    it (int64 gains), so its flips are those of O7 on Qt; the returned f is then evaluated on
 *    the evaluation image (bound above).
 * ------------------------------------------------------------------------------ */
enum { UBQP_F32 = 1, UBQP_F64 = 2 };

/* statistics of a real-Q batch on the evaluation image, f~_k = f_k 2^exp exactly:
 * sum f~ and max f~ as two's-complement int128 (hi:lo), count; max = INT128_MIN (hi =
 * INT64_MIN, lo = 0) if the batch is empty.  48 bytes. */
typedef struct {
    int64_t sum_hi;
    uint64_t sum_lo;
    int64_t count;
    int64_t max_hi;
    uint64_t max_lo;
    int32_t exp;           /* w of the evaluation image: f = 2^-exp f~ */
    int32_t reserved;      /* 0 */
} ubqp_stats_real;

/* Load a real-valued symmetric Q (row-major n*n float32 or float64, host or device).
 * Errors: E_NOT_SYMMETRIC, E_RANGE (non-finite coefficient, or more than 10 evaluation limbs
 * needed), E_INVALID, E_NOMEM.  Replaces any earlier Q.  Batch generation calls work
 * unchanged; integer-only calls return E_STATE.  Synchronises. */
int ubqp_load_Q_real(ubqp_t h, int32_t n, int dtype, const void *Q, int64_t k_max);

/* Evaluate the batch against the real Q (evaluation image, error bound above): f_out
 * double[k_local] (may be NULL), stats_out (may be NULL).  One tensor-core launch over the
 * L limb planes with the exact int128 combine and the statistics folded in-kernel. */
int ubqp_eval_batch_real(ubqp_t h, double *f_out, ubqp_stats_real *stats_out);

/* Screen the last real batch: T = mean + lambda (max_value - mean) (binary64, no
 * contraction); survivors {k : f_k > T} ascending.  Synchronises. */
int ubqp_screen_real(ubqp_t h, double lambda, double mean, double max_value, int32_t *surv_out,
                     int64_t *m_out, double *T_out);

/* Steepest ascent for real-valued Q (reading R20): ubqp_ascend's walk
 * (gains P:53; k* = argmax Delta, lowest j on ties; stop at Delta_k* <= 0
 * or max_flips) run exactly in int64 on the walk image Qt = rint(Q 2^e) (e =
 * ubqp_query(UBQP_Q_REAL_EXP)).  Starts: batch slots slots[i] of the last
 * ubqp_eval_batch_real (their int64 gains are formed here from the four walk-image int8 limb
 * planes).  Outputs per i (any may be NULL): f_out double[m] = f of the local optimum on the
 * EVALUATION image (re-evaluated on the tensor cores; within the bound above of x^t Q x),
 * fint_out int64[m] = x^t Qt x (the walk image, exact), flips_out int32[m], bits_out
 * uint64[m][W64].  Every returned x is a 1-flip local optimum of Qt unless flips = max_flips;
 * for the real Q its gains are then <= (2|S| + 1) 2^-(e+1).  The batch is not modified.
 * Memory: int64 gains of k_max * n_pad words on first use.
 * Errors: E_STATE (no real Q / no evaluated real batch), E_INVALID, E_NOMEM, E_RANGE. */
int ubqp_ascend_real(ubqp_t h, const int32_t *slots, int64_t m, int32_t max_flips,
                     double *f_out, int64_t *fint_out, int32_t *flips_out, uint64_t *bits_out);

/* Wait for all work queued on the handle's stream. */
int ubqp_sync(ubqp_t h);

/* Introspection (read-only): n, n_pad, W64, k_max, k_local, kernels launched so far, the
 * stream, the walk-image exponent e (R20), 1 if a real Q is loaded, the evaluation-image
 * exponent w and limb count L (R22; integer Q: 0 and 1), the off-diagonal nonzeros of an
 * integer Q, 1 if its sparse rows (fixed-stride ELL rows, NEXT-3) were built (off-diagonal density <= 0.25),
 * the sharding block B, and the kernel of the last ubqp_ascend (0 none yet, 1 dense CTA, 2 sparse,
 * 3 dense warp per solution, 4 dense multi-warp; see UBQP_OPT_ASCENT). */
enum { UBQP_Q_N = 0, UBQP_Q_NPAD = 1, UBQP_Q_W64 = 2, UBQP_Q_KMAX = 3, UBQP_Q_KLOCAL = 4,
       UBQP_Q_LAUNCHES = 5, UBQP_Q_STREAM = 6, UBQP_Q_REAL_EXP = 7, UBQP_Q_IS_REAL = 8,
       UBQP_Q_EVAL_EXP = 9, UBQP_Q_EVAL_LIMBS = 10, UBQP_Q_NNZ = 11, UBQP_Q_SPARSE_ROWS = 12,
       UBQP_Q_SHARD_BLOCK = 13, UBQP_Q_ASCENT_LAST = 14 };
int ubqp_query(ubqp_t h, int what, int64_t *value);

/* Kernel selection (results never depend on it; every choice is exact):
 *   UBQP_OPT_ASCENT     0 = automatic (a dense kernel at every density, as measured fastest: the
 *                       warp-per-solution ascent for 3584 < n_pad <= 7168 and for 1537-2048 and
 *                       2561-3072, the CTA ascent for the other n_pad <= 3584, the multi-warp
 *                       ascent above 7168; the sparse-row kernel measured slower at densities
 *                       0.02-0.2, DESIGN.md §7.4'), 1 = dense CTA ascent (two or more warps per
 *                       solution, byte masks), 2 = sparse-row ascent (NEXT-3; E_STATE if the sparse
 *                       rows were not built), 3 = dense warp-per-solution ascent (E_RANGE if
 *                       n_pad > 7168), 4 = dense multi-warp ascent (2-4 warps per solution, the
 *                       keys of kernel 3; every n).  Used by ubqp_ascend.
 *   UBQP_OPT_EVAL_PAIR  1 = CTA-pair (cta_group::2) evaluation (default), 0 = single CTA.
 *   UBQP_OPT_EVAL_TRI   1 = f-only evaluations use the lower triangle of Q (default), 0 = full.
 *   UBQP_OPT_SHARD_BLOCK  B in [1, 4096], the sharding block (see Sharding; default 2); set it
 *                       before generating a batch.
 * Errors: E_INVALID (unknown option or value). */
enum { UBQP_OPT_ASCENT = 0, UBQP_OPT_EVAL_PAIR = 1, UBQP_OPT_EVAL_TRI = 2, UBQP_OPT_SHARD_BLOCK = 3 };
int ubqp_set_option(ubqp_t h, int what, int64_t value);

#ifdef __cplusplus
}
#endif

#endif /* UBQP_H */
