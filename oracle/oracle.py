"""ctypes wrapper around ``oracle/ubqp_oracle.c`` plus the O8 round loop.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
passage of PAPER.md (P:n) / SPEC.md (S:n) it follows and the SURVEY.md §8(c)
definition (O1..O10) restated in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "ubqp_oracle.c"
_LIB = _HERE / "liboracle_ubqp.so"
_lib = None

__all__ = [
    "build_oracle", "xQx", "eval_batch", "gains", "splitmix_word", "random_solutions",
    "glover_params", "diversify", "blend", "pool_update", "max_key", "stats", "threshold", "screen", "ascend",
    "first_derivative_start", "relink", "polish", "run_rounds", "xQx_real", "eval_batch_real", "first_derivative_start_real",
    "real_image", "ascend_real", "run_rounds_real", "gains_real", "batch_sum_exact", "global_index", "shard_count",
]


def build_oracle(force: bool = False) -> Path:
    """Compile the oracle with plain -O2 (no intrinsics, no fast-math, no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-pthread", str(_SRC), "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(str(_LIB))
        P = ctypes.c_void_p
        i64, i32, u64, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        lib.oracle_eval_batch.argtypes = [i32, P, i64, P, P, i32]
        lib.oracle_eval.argtypes = [i32, P, P]
        lib.oracle_eval.restype = i64
        lib.oracle_gains.argtypes = [i32, P, P, P]
        lib.oracle_splitmix_word.argtypes = [u64, i64, i64, i64]
        lib.oracle_splitmix_word.restype = u64
        lib.oracle_random.argtypes = [i32, u64, i64, i32, i32, i32, P]
        lib.oracle_glover_params.argtypes = [i64, i32, P, P, P]
        lib.oracle_diversify.argtypes = [i32, P, i64, i64, i32, i32, i32, P]
        lib.oracle_blend.argtypes = [i32, P, P, i64, i64, i64, i32, i32, i32, P]
        lib.oracle_max_key.argtypes = [i64, i64]
        lib.oracle_max_key.restype = i64
        lib.oracle_stats.argtypes = [i64, P, i32, i32, i32, P]
        lib.oracle_threshold.argtypes = [dbl, i64, i64, i64]
        lib.oracle_threshold.restype = dbl
        lib.oracle_screen.argtypes = [i64, P, dbl, P]
        lib.oracle_screen.restype = i64
        lib.oracle_ascend_batch.argtypes = [i32, P, i64, P, P, P, i32, i32]
        lib.oracle_first_derivative_start.argtypes = [i32, P, P]
        lib.oracle_relink_batch.argtypes = [i32, P, i64, P, P, P, i64, P, P, P, P, P, i32]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _Q(Q) -> np.ndarray:
    Q = np.ascontiguousarray(Q, dtype=np.int32)
    assert Q.ndim == 2 and Q.shape[0] == Q.shape[1]
    return Q


def _X(X, n) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.uint8)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    assert X.shape[1] == n
    return X


# O1 -- f(x) = x^t Q x (P:24 eq. (P))
def xQx(Q, x) -> int:
    Q = _Q(Q)
    x = _X(x, Q.shape[0])
    return int(_L().oracle_eval(Q.shape[0], _p(Q), _p(x)))


def eval_batch(Q, X, nthreads: int = 1) -> np.ndarray:
    """O1 over a batch ("evaluate ... 1000 samples")."""
    Q = _Q(Q)
    n = Q.shape[0]
    X = _X(X, n)
    f = np.zeros(X.shape[0], dtype=np.int64)
    _L().oracle_eval_batch(n, _p(Q), X.shape[0], _p(X), _p(f), int(nthreads))
    return f


# O2 -- Delta_i = (1-2x_i)(Q_ii + 2 sum_{j!=i} Q_ij x_j)
def gains(Q, x) -> np.ndarray:
    Q = _Q(Q)
    n = Q.shape[0]
    x = _X(x, n)
    d = np.zeros(n, dtype=np.int64)
    _L().oracle_gains(n, _p(Q), _p(x), _p(d))
    return d


# O3 -- random solutions from SplitMix64 (R12)
def splitmix_word(seed: int, g: int, W64: int, w: int) -> int:
    return int(_L().oracle_splitmix_word(seed & (2**64 - 1), g, W64, w))


# O10 -- sharding: slot i on rank r <-> g = (r + floor(i/B) world) B + (i mod B)
def global_index(i: int, rank: int, world: int, block: int = 1) -> int:
    return (rank + (i // block) * world) * block + i % block


def shard_count(rank: int, K: int, world: int, block: int = 1) -> int:
    """number of g in [0, K) that O10 assigns to `rank`"""
    full, rem = divmod(K, world * block)
    return full * block + min(block, max(0, rem - rank * block))


def random_solutions(n: int, seed: int, k_local: int, rank: int = 0, world: int = 1, block: int = 1) -> np.ndarray:
    X = np.zeros((k_local, n), dtype=np.uint8)
    _L().oracle_random(n, seed & (2**64 - 1), k_local, rank, world, block, _p(X))
    return X


# O4 -- Glover diversification generator (R11)
def glover_params(t: int, n: int):
    h, q, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    _L().oracle_glover_params(t, n, ctypes.byref(h), ctypes.byref(q), ctypes.byref(c))
    return h.value, q.value, c.value


def diversify(seed_x, t0: int, k_local: int, rank: int = 0, world: int = 1, block: int = 1) -> np.ndarray:
    seed_x = np.ascontiguousarray(seed_x, dtype=np.uint8).reshape(-1)
    n = seed_x.shape[0]
    X = np.zeros((k_local, n), dtype=np.uint8)
    _L().oracle_diversify(n, _p(seed_x), t0, k_local, rank, world, block, _p(X))
    return X


# O4b -- blend of the incumbent with parent g mod P on the Glover mask (R11b)
def blend(seed_x, parents, t0: int, k_local: int, rank: int = 0, world: int = 1, block: int = 1) -> np.ndarray:
    seed_x = np.ascontiguousarray(seed_x, dtype=np.uint8).reshape(-1)
    n = seed_x.shape[0]
    parents = np.ascontiguousarray(parents, dtype=np.uint8).reshape(-1, n)
    if parents.shape[0] < 1:
        raise ValueError("blend needs at least one parent")
    X = np.zeros((k_local, n), dtype=np.uint8)
    _L().oracle_blend(n, _p(seed_x), _p(parents), parents.shape[0], t0, k_local, rank, world, block, _p(X))
    return X


def pool_update(pool: list, pool_cap: int, inc_x, improved_from, round_best):
    """Parent pool of the blend policy (R11b): distinct local optima other than the
    incumbent, oldest first, at most pool_cap.  After a round, the replaced incumbent
    (improved_from) or else the round's best ascended solution joins the pool unless it
    equals the incumbent or is already pooled."""
    cand = improved_from if improved_from is not None else round_best
    if cand is None:
        return pool
    cand = np.asarray(cand, dtype=np.uint8)
    if np.array_equal(cand, inc_x) or any(np.array_equal(cand, p) for p in pool):
        return pool
    pool = pool + [cand.copy()]
    return pool[-pool_cap:]


# O5 -- stats {sum, count, max_key} (R14)
def max_key(f: int, g: int) -> int:
    return int(_L().oracle_max_key(f, g))


def stats(f, rank: int = 0, world: int = 1, block: int = 1) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.int64)
    out = np.zeros(4, dtype=np.int64)
    _L().oracle_stats(f.shape[0], _p(f), rank, world, block, _p(out))
    return out


# O6 -- T(lambda) = Mean + lambda (Max - Mean); survivors f > T ascending
def threshold(lam: float, mean_sum: int, mean_count: int, max_value: int) -> float:
    return float(_L().oracle_threshold(float(lam), int(mean_sum), int(mean_count), int(max_value)))


def screen(f, T: float) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.int64)
    s = np.zeros(max(1, f.shape[0]), dtype=np.int32)
    m = _L().oracle_screen(f.shape[0], _p(f), float(T), _p(s))
    return s[:m].copy()


# O7 -- steepest ascent (R9)
def ascend(Q, X, f, max_flips: int, nthreads: int = 1):
    """Returns (X_final uint8 [m][n], f_final int64 [m], flips int32 [m]); inputs untouched."""
    Q = _Q(Q)
    n = Q.shape[0]
    X = _X(X, n).copy()
    f = np.ascontiguousarray(f, dtype=np.int64).copy()
    flips = np.zeros(X.shape[0], dtype=np.int32)
    _L().oracle_ascend_batch(n, _p(Q), X.shape[0], _p(X), _p(f), _p(flips), int(max_flips),
                             int(nthreads))
    return X, f, flips


# O11 -- path relinking from X0 toward guides (R19)
def relink(Q, X0, f0, guides, nthreads: int = 1, with_path: bool = False):
    """Returns (Xbest uint8 [m][n], fbest int64 [m] (INT64_MIN: none), sbest int32 [m]
    (-1: none), length |D| int32 [m][, path int32 [m][n] flip order]); guide of row i is
    guides[i mod len(guides)]."""
    Q = _Q(Q)
    n = Q.shape[0]
    X0 = _X(X0, n)
    Y = _X(guides, n)
    m = X0.shape[0]
    f0 = np.ascontiguousarray(f0, dtype=np.int64)
    Xb = np.zeros_like(X0)
    fb = np.zeros(m, np.int64)
    sb = np.zeros(m, np.int32)
    ln = np.zeros(m, np.int32)
    path = np.full((m, n), -1, np.int32) if with_path else None
    rc = _L().oracle_relink_batch(n, _p(Q), m, _p(X0), _p(f0), _p(Y), Y.shape[0], _p(Xb), _p(fb), _p(sb),
                                  _p(ln), _p(path) if with_path else None, int(nthreads))
    if rc:
        raise ValueError("oracle_relink_batch: bad arguments")
    return (Xb, fb, sb, ln, path) if with_path else (Xb, fb, sb, ln)


# first-derivative start
def first_derivative_start(Q) -> np.ndarray:
    Q = _Q(Q)
    x = np.zeros(Q.shape[0], dtype=np.uint8)
    _L().oracle_first_derivative_start(Q.shape[0], _p(Q), _p(x))
    return x


# polish phase over an elite set (NEXT-4; R19): relink every ordered pair, ascend the interior
def polish(Q, elite, max_flips: int, nthreads: int = 1):
    """elite uint8 [E][n].  Every ordered pair (a, b), a != b, in row-major order is relinked
    from elite[a] toward elite[b] (O11); the best interior points (pairs with one) are
    ascended (O7) in pair order; returns (f, x) of the best result (highest f, then the
    earliest pair) or None when no pair has an interior point."""
    Q = _Q(Q)
    n = Q.shape[0]
    E = _X(elite, n)
    pairs = [(a, b) for a in range(E.shape[0]) for b in range(E.shape[0]) if a != b]
    if not pairs:
        return None
    X0 = np.stack([E[a] for a, _ in pairs])
    Y = np.stack([E[b] for _, b in pairs])
    Xb, fb, sb, _ = relink(Q, X0, eval_batch(Q, X0, nthreads), Y, nthreads)
    idx = np.flatnonzero(sb >= 0)
    if idx.size == 0:
        return None
    Xa, fa, _ = ascend(Q, Xb[idx], fb[idx], max_flips, nthreads)
    best = max(range(idx.size), key=lambda i: max_key(int(fa[i]), i))
    return int(fa[best]), Xa[best].copy()


# O8 -- batched rounds of Figure 2 (R5, R6, R13)
def run_rounds(Q, K: int, rounds: int, lam: float, max_flips: int, sample_seed: int,
               world: int = 1, nthreads: int = 1, div: str = "glover", pool_cap: int = 8,
               polish_end: bool = False, trace: list | None = None, block: int = 1):
    """Round 0: K random starts (O3, seed ``sample_seed``) -> pinned (mean_sum, mean_count)
    ("the mean is the average xQx value derived during sampling").  Incumbent =
    first-derivative start.  Round r >= 1: diversify from the incumbent with
    t0 = (r-1)*K ("Diversify(x, best_xQx, i, ...)"), evaluate, Max = max(incumbent,
    batch max) (R6), screen, ascend survivors, replace the incumbent iff the
    best ascended f is strictly greater, ties -> lowest g (R8, R14).
    ``world``/``block`` shard every batch (O10); results must not depend on them.
    ``div`` "blend": once the parent pool (pool_update) is non-empty, rounds blend the
    incumbent with pool[g mod P] (O4b) instead of O4.  ``polish_end``: after the last
    round, polish(pool + [incumbent]) (O11 + O7); a strictly better result is recorded as
    round ``rounds + 1``.  ``trace`` (a list) receives one dict per round: t0, the batch f,
    Max, T, the survivors (global g), the ascended (g, f) pairs, the round's best (f, g, x).
    Returns (best_value, best_x, trajectory[list of (round, best_value)])."""
    Q = _Q(Q)
    n = Q.shape[0]

    def shards(make):
        return [make(r) for r in range(world)]

    f0 = [eval_batch(Q, Xr, nthreads) for Xr in shards(
        lambda r: random_solutions(n, sample_seed, shard_count(r, K, world, block), r, world, block))]
    mean_sum = int(sum(int(fr.sum()) for fr in f0))
    mean_count = K
    inc_x = first_derivative_start(Q)
    inc_f = xQx(Q, inc_x)
    if lam == "paper":
        # P:55 lambda = Max/Mean = Starting_solution/Mean; SPEC S:244 clamp to (0, 1], 0.5 fallback
        m = mean_sum / mean_count
        lam = 0.5 if (m <= 0 or inc_f <= 0) else min(1.0, max(1e-6, inc_f / m))
    traj = [(0, inc_f)]
    pool = []
    for rnd in range(1, rounds + 1):
        t0 = (rnd - 1) * K
        best_key, best = -1, None
        if div == "blend" and pool:
            P = np.stack(pool)
            Xs = shards(lambda r: blend(inc_x, P, t0, shard_count(r, K, world, block), r, world, block))
        else:
            Xs = shards(lambda r: diversify(inc_x, t0, shard_count(r, K, world, block), r, world, block))
        fs = [eval_batch(Q, Xr, nthreads) for Xr in Xs]
        batch_max = max(int(fr.max()) for fr in fs if fr.size)
        T = threshold(lam, mean_sum, mean_count, max(inc_f, batch_max))
        tr = {"round": rnd, "t0": t0, "mean_sum": mean_sum, "mean_count": mean_count,
              "max_value": max(inc_f, batch_max), "T": T, "survivors": [], "ascended": []}
        for r in range(world):
            s = screen(fs[r], T)
            tr["survivors"] += [global_index(int(v), r, world, block) for v in s]
            if s.size == 0:
                continue
            Xa, fa, _ = ascend(Q, Xs[r][s], fs[r][s], max_flips, nthreads)
            for i, slot in enumerate(s):
                key = max_key(int(fa[i]), global_index(int(slot), r, world, block))
                tr["ascended"].append((global_index(int(slot), r, world, block), int(fa[i])))
                if key > best_key:
                    best_key, best = key, (int(fa[i]), Xa[i].copy())
        if trace is not None:
            tr["survivors"].sort()
            tr["ascended"].sort()
            fg = {}
            for r in range(world):
                for i, v in enumerate(fs[r]):
                    fg[global_index(i, r, world, block)] = int(v)
            tr["f"] = [fg[g] for g in range(K)]
            tr["best"] = None if best is None else (best[0], (1 << 22) - 1 - (best_key & ((1 << 22) - 1)),
                                                     best[1].copy())
            trace.append(tr)
        improved_from = None
        if best is not None and best[0] > inc_f:
            improved_from = inc_x
            inc_f, inc_x = best
            traj.append((rnd, inc_f))
        if div == "blend" or polish_end:
            pool = pool_update(pool, pool_cap, inc_x, improved_from,
                               None if best is None else best[1])
    if polish_end:
        res = polish(Q, np.stack(pool + [inc_x]), max_flips, nthreads)
        if res is not None and res[0] > inc_f:
            inc_f, inc_x = res
            traj.append((rounds + 1, inc_f))
    return inc_f, inc_x, traj


# O9 -- real Q: f = sum of Q_ij over i, j with x_i = x_j = 1, correctly rounded ("real or
# integer coefficients"; "float or double").  math.fsum is exactly rounded.
def xQx_real(Q, x) -> float:
    import math
    Q = np.asarray(Q, dtype=np.float64)
    x = np.asarray(x).reshape(-1).astype(bool)
    S = np.flatnonzero(x)
    return math.fsum(Q[np.ix_(S, S)].ravel().tolist())


def eval_batch_real(Q, X) -> np.ndarray:
    X = np.asarray(X)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    return np.array([xQx_real(Q, x) for x in X], dtype=np.float64)


def first_derivative_start_real(Q) -> np.ndarray:
    """x_i = 1 iff sum_j Q_ij > 0, row sums exactly rounded."""
    import math
    Q = np.asarray(Q, dtype=np.float64)
    return np.array([1 if math.fsum(row.tolist()) > 0 else 0 for row in Q], dtype=np.uint8)


# O9b -- real-Q ascent (reading R20): the walk runs exactly on the load-time
# fixed-point image Qt = rint(Q 2^e) (round half to even), e the largest integer with
# max|Q| 2^e <= 2^27 - 1 (the 28-bit range of four balanced base-128 int8 limbs, a4');
# f = 2^-e f~ with f~ = x^t Qt x.  Written from that definition, independently of the
# library's load routine.
def real_image(Q):
    """(Qt int64 [n][n], e)"""
    Q = np.asarray(Q, dtype=np.float64)
    amax = float(np.abs(Q).max()) if Q.size else 0.0
    e = 0
    if amax > 0:
        lim = float(2**27 - 1)
        e = 0
        while np.ldexp(amax, e) > lim:
            e -= 1
        while np.ldexp(amax, e + 1) <= lim:
            e += 1
    return np.rint(np.ldexp(Q, e)).astype(np.int64), e


def ascend_real(Q, X, max_flips: int, nthreads: int = 1):
    """Steepest ascent (O7) on the image Qt of a real Q (R20): returns (X_final, f~ int64,
    f = 2^-e f~ float64, flips, e)."""
    Qt, e = real_image(Q)
    X = np.asarray(X, dtype=np.uint8)
    f0 = eval_batch(Qt.astype(np.int32), X, nthreads)
    Xa, fa, fl = ascend(Qt.astype(np.int32), X, f0, max_flips, nthreads)
    return Xa, fa, np.ldexp(fa.astype(np.float64), -e), fl, e


# O2 on a real Q: Delta_j = f(x xor e_j) - f(x) = (1 - 2 x_j)(Q_jj + 2 sum_{i != j, x_i = 1} Q_ij)
# (S:164), each gain the exactly rounded sum of its terms (math.fsum; +-2 Q_ij is exact
# in binary64).  Independent of any fixed-point image.
def gains_real(Q, x) -> np.ndarray:
    import math
    Q = np.asarray(Q, dtype=np.float64)
    x = np.asarray(x).reshape(-1).astype(bool)
    S = np.flatnonzero(x)
    out = np.empty(Q.shape[0], dtype=np.float64)
    for j in range(Q.shape[0]):
        d = -1.0 if x[j] else 1.0
        terms = [d * Q[j, j]] + [2.0 * d * Q[i, j] for i in S if i != j]
        out[j] = math.fsum(terms)
    return out


def batch_sum_exact(Q, X):
    """sum_k x_k^t Q x_k as an exact rational (fractions.Fraction): sum_ij Q_ij c_ij with the
    integer co-occurrence counts c = X^t X (a library matmul of 0/1 matrices)."""
    from fractions import Fraction
    Q = np.asarray(Q, dtype=np.float64)
    X = np.asarray(X, dtype=np.int64)
    C = X.T @ X
    tot = Fraction(0)
    for q, c in zip(Q.ravel().tolist(), C.ravel().tolist()):
        if q != 0.0 and c:
            tot += Fraction(q) * c
    return tot


# O8 on a real Q (R20, R22): the batched rounds of run_rounds where every objective value is
# the exactly rounded x^t Q x (O9) and each survivor's walk is O7 on the walk image Qt (O9b)
def run_rounds_real(Q, K: int, rounds: int, lam: float, max_flips: int, sample_seed: int,
                    world: int = 1, nthreads: int = 1, block: int = 1):
    """Round 0: K random starts (O3); Mean = the exact rational mean of their objective values,
    rounded once to binary64 (the pinned sampling mean; R5).  Incumbent = the
    first-derivative start on the exactly rounded row sums, value O9.  Round r >= 1:
    Glover diversification with t0 = (r-1)K (O4); f = O9 of each; Max = max(incumbent, batch
    max) (R6); T = Mean + lam (Max - Mean) in binary64; survivors f > T; each
    survivor walks O7 on Qt = rint(Q 2^e) (R20) and its final x is valued by O9; the incumbent
    is replaced iff the best value is strictly greater, ties to the lowest g (R8, R14).
    Returns (best f, best x, trajectory [(round, f)], e)."""
    Q = np.asarray(Q, dtype=np.float64)
    Qt, e = real_image(Q)
    Qi = Qt.astype(np.int32)
    n = Q.shape[0]
    from fractions import Fraction
    total = Fraction(0)
    for r in range(world):
        total += batch_sum_exact(Q, random_solutions(n, sample_seed, shard_count(r, K, world, block), r, world, block))
    mean = float(total / K)
    inc_x = first_derivative_start_real(Q)
    inc_f = xQx_real(Q, inc_x)
    traj = [(0, inc_f)]
    for rnd in range(1, rounds + 1):
        t0 = (rnd - 1) * K
        Xs = [diversify(inc_x, t0, shard_count(r, K, world, block), r, world, block) for r in range(world)]
        fs = [eval_batch_real(Q, Xr) for Xr in Xs]
        bmax = max(float(fr.max()) for fr in fs if fr.size)
        maxv = max(inc_f, bmax)
        T = mean + lam * (maxv - mean)
        best = None
        for r in range(world):
            s = np.flatnonzero(fs[r] > T)
            if s.size == 0:
                continue
            Xa, _, _ = ascend(Qi, Xs[r][s], eval_batch(Qi, Xs[r][s], nthreads), max_flips, nthreads)
            for i, slot in enumerate(s):
                cand = (xQx_real(Q, Xa[i]), -global_index(int(slot), r, world, block))
                if best is None or cand > best[0]:
                    best = (cand, Xa[i].copy())
        if best is not None and best[0][0] > inc_f:
            inc_f, inc_x = best[0][0], best[1]
            traj.append((rnd, inc_f))
    return inc_f, inc_x, traj, e
