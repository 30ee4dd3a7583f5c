"""Pins of the CPU oracle against what the paper and the mathematics fix (not against itself).

Every oracle function (O1..O8) is checked here against an independent fact:
SPEC worked examples (tests/golden/spec_examples.json), closed forms, brute-force
enumeration on tiny inputs, library routines (numpy matmul), identities of symmetric
quadratic forms, the SplitMix64 known answers and Glover's own illustration.
"""
import itertools
import json
import math
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import oracle
from inputs import generate_Q, pack_bits, unpack_bits

GOLD = Path(__file__).resolve().parent / "golden"
SPEC = json.loads((GOLD / "spec_examples.json").read_text())


def _Qn(name):
    return np.array(SPEC[name], dtype=np.int32)


def _all_x(n):
    return np.array(list(itertools.product([0, 1], repeat=n)), dtype=np.uint8)[:, ::-1].copy()


# ---------------------------------------------------------------- O1 eval
def test_spec_eval_examples():
    for e in SPEC["eval"]:
        assert oracle.xQx(_Qn(e["Q"]), e["x"]) == e["f"], e["cite"]
    for e in SPEC["eval_batch"]:
        assert oracle.eval_batch(_Qn(e["Q"]), e["X"]).tolist() == e["f"], e["cite"]


def test_eval_closed_forms():
    rng = np.random.default_rng(11)
    for n in (1, 2, 7, 33, 64, 65, 130):
        Q = generate_Q(n, 0.7, -100, 100, seed=int(rng.integers(1 << 30)))
        zero = np.zeros(n, np.uint8)
        ones = np.ones(n, np.uint8)
        assert oracle.xQx(Q, zero) == 0                              # f(0) = 0
        assert oracle.xQx(Q, ones) == int(Q.astype(np.int64).sum())  # f(1) = sum Q
        E = np.eye(n, dtype=np.uint8)
        assert oracle.eval_batch(Q, E).tolist() == np.diag(Q).astype(np.int64).tolist()  # f(e_i)=Q_ii


def test_eval_matches_library_matmul_and_complement_identity():
    rng = np.random.default_rng(12)
    for n in (3, 50, 129):
        Q = generate_Q(n, 0.5, -100, 100, seed=int(rng.integers(1 << 30)))
        X = rng.integers(0, 2, size=(40, n)).astype(np.uint8)
        f = oracle.eval_batch(Q, X, nthreads=3)
        Q64 = Q.astype(np.int64)
        ref = np.einsum("ki,ij,kj->k", X.astype(np.int64), Q64, X.astype(np.int64))
        assert f.tolist() == ref.tolist()
        # complement: f(1-x) = sum Q - 2 rowsum^T x + f(x)  (symmetric Q)
        fc = oracle.eval_batch(Q, 1 - X)
        rs = Q64.sum(axis=1)
        assert fc.tolist() == (Q64.sum() - 2 * X.astype(np.int64) @ rs + f).tolist()


def test_eval_brute_force_global_optimum_spec():
    Q3 = _Qn("Q3")
    X = _all_x(3)
    f = oracle.eval_batch(Q3, X)
    assert f.max() == 4 and X[f.argmax()].tolist() == [1, 0, 1]    # S:133 global max
    # exhaustive average == closed-form expectation
    assert Fraction(int(f.sum()), len(f)) == Fraction(-1, 2)


def test_eval_thread_count_invariance():
    Q = generate_Q(100, 0.5, -10, 10, seed=5)
    X = np.random.default_rng(5).integers(0, 2, size=(1000, 100)).astype(np.uint8)
    a = oracle.eval_batch(Q, X, 1)
    for t in (2, 8):
        assert np.array_equal(a, oracle.eval_batch(Q, X, t))


# ---------------------------------------------------------------- O2 gains
def test_spec_gain_examples():
    for e in SPEC["gains"]:
        assert oracle.gains(_Qn(e["Q"]), e["x"]).tolist() == e["Delta"], e["cite"]


def test_gains_equal_brute_force_flip_differences():
    rng = np.random.default_rng(13)
    for n in (1, 2, 5, 17, 64):
        Q = generate_Q(n, 0.6, -100, 100, seed=int(rng.integers(1 << 30)))
        for _ in range(5):
            x = rng.integers(0, 2, size=n).astype(np.uint8)
            f = oracle.xQx(Q, x)
            flipped = np.tile(x, (n, 1)) ^ np.eye(n, dtype=np.uint8)
            brute = oracle.eval_batch(Q, flipped) - f                 # f(x xor e_i) - f(x)
            assert oracle.gains(Q, x).tolist() == brute.tolist()
            # Appendix-A identity with Y = Qx from numpy: Delta = Q_ii + 2(1-2x)Y
            Y = Q.astype(np.int64) @ x.astype(np.int64)
            assert oracle.gains(Q, x).tolist() == (np.diag(Q) + 2 * (1 - 2 * x.astype(np.int64)) * Y).tolist()


# ---------------------------------------------------------------- O3 random bits
def test_splitmix64_known_answers():
    for line in (GOLD / "splitmix64_kat.txt").read_text().splitlines():
        if line.startswith("#") or not line.strip():
            continue
        w, v = line.split()
        assert oracle.splitmix_word(0, 0, 3, int(w)) == int(v, 16)


def test_random_solution_bits_layout_and_balance():
    n = 130
    X = oracle.random_solutions(n, 77, 64)
    W = (n + 63) // 64
    for g in (0, 5, 63):
        for j in (0, 63, 64, 129):
            assert X[g, j] == (oracle.splitmix_word(77, g, W, j // 64) >> (j % 64)) & 1
    big = oracle.random_solutions(257, 3, 2000)
    p = big.mean()
    assert abs(p - 0.5) < 4 * math.sqrt(0.25 / big.size)


def test_random_sharding_is_cyclic():
    n, K = 70, 23
    full = oracle.random_solutions(n, 9, K)
    for world in (2, 3, 4):
        for r in range(world):
            part = oracle.random_solutions(n, 9, len(range(r, K, world)), r, world)
            assert np.array_equal(part, full[r::world])


def test_block_sharding_partitions_the_batch():
    """O10 with block B: rank r holds g = (r + floor(i/B) world) B + (i mod B); written out by
    hand for K = 11, world = 3, B = 2: rank 0 -> 0 1 6 7, rank 1 -> 2 3 8 9, rank 2 -> 4 5 10"""
    want = {0: [0, 1, 6, 7], 1: [2, 3, 8, 9], 2: [4, 5, 10]}
    for r, gs in want.items():
        assert oracle.shard_count(r, 11, 3, 2) == len(gs)
        assert [oracle.global_index(i, r, 3, 2) for i in range(len(gs))] == gs
    n = 50
    full = oracle.random_solutions(n, 4, 101)
    seed = np.random.default_rng(2).integers(0, 2, size=n).astype(np.uint8)
    dfull = oracle.diversify(seed, 7, 101)
    for world in (1, 2, 3, 8):
        for B in (1, 2, 3, 16):
            seen = []
            for r in range(world):
                k = oracle.shard_count(r, 101, world, B)
                gs = [oracle.global_index(i, r, world, B) for i in range(k)]
                seen += gs
                assert np.array_equal(oracle.random_solutions(n, 4, k, r, world, B), full[gs])
                assert np.array_equal(oracle.diversify(seed, 7, k, r, world, B), dfull[gs])
            assert sorted(seen) == list(range(101))


def test_sampled_mean_matches_expectation():
    """E f = sum_i Q_ii/2 + sum_{i!=j} Q_ij/4 under iid Bernoulli(1/2) bits."""
    hits = 0
    for s in range(20):
        Q = generate_Q(50, 0.5, -10, 10, seed=1000 + s)
        f = oracle.eval_batch(Q, oracle.random_solutions(50, s, 10000), nthreads=4)
        Q64 = Q.astype(np.int64)
        E = np.trace(Q64) / 2 + (Q64.sum() - np.trace(Q64)) / 4
        se = f.std(ddof=1) / math.sqrt(f.size)
        hits += abs(f.mean() - E) <= 3 * se
    assert hits >= 18


# ---------------------------------------------------------------- O4 Glover diversification
def test_glover_illustration_from_zero_seed():
    n = 10
    for line in (GOLD / "glover_n10.txt").read_text().splitlines():
        if line.startswith("#") or not line.strip():
            continue
        h, q, c, bits = line.split()
        h, q, c = int(h), int(q), int(c)
        t = h * (h - 1) + 2 * (q - 1) + c              # position of (h,q,c) in the enumeration
        assert oracle.glover_params(t, n) == (h, q, c)
        x = oracle.diversify(np.zeros(n, np.uint8), t, 1)[0]
        assert "".join(map(str, x.tolist())) == bits


def test_glover_index_map_enumerates_all_triples_in_order():
    n = 39
    expect = [(h, q, c) for h in range(1, n + 1) for q in range(1, h + 1) for c in (0, 1)]
    assert len(expect) == n * (n + 1)
    got = [oracle.glover_params(t, n) for t in range(n * (n + 1))]
    assert got == expect
    assert oracle.glover_params(n * (n + 1) + 5, n) == expect[5]   # wraps mod n(n+1)


def test_glover_hamming_distances_and_duplicates():
    rng = np.random.default_rng(14)
    n = 97
    seed = rng.integers(0, 2, size=n).astype(np.uint8)
    K = 600
    X = oracle.diversify(seed, 0, K)
    for t in range(K):
        h, q, c = oracle.glover_params(t, n)
        size = (n - q) // h + 1                       # |M(h,q)| = floor((n-q)/h) + 1
        dist = int((X[t] != seed).sum())
        assert dist == (size if c == 0 else n - size)
    assert np.array_equal(X[1], seed)                # t = 1 (h=1, q=1, c=1) is the seed itself
    assert np.array_equal(X[4], X[3]) and np.array_equal(X[5], X[2])  # (2,2,c) == (2,1,1-c)


def test_glover_sharding_is_cyclic():
    n, K = 40, 31
    seed = np.random.default_rng(1).integers(0, 2, size=n).astype(np.uint8)
    full = oracle.diversify(seed, 17, K)
    for world in (2, 5):
        for r in range(world):
            assert np.array_equal(oracle.diversify(seed, 17, len(range(r, K, world)), r, world),
                                  full[r::world])


# ---------------------------------------------------------------- O4b blend (R11b)
def test_blend_hand_worked_example():
    n = 10
    seed = np.zeros(n, np.uint8)
    parent = np.array([1, 1, 1, 1, 1, 0, 0, 0, 0, 0], np.uint8)
    for line in (GOLD / "blend_n10.txt").read_text().splitlines():
        if line.startswith("#") or not line.strip():
            continue
        t, h, q, c, bits = line.split()
        assert oracle.glover_params(int(t), n) == (int(h), int(q), int(c))
        x = oracle.blend(seed, parent[None, :], int(t), 1)[0]
        assert "".join(map(str, x.tolist())) == bits, line


def test_blend_with_complement_parent_is_glover():
    # parent = NOT seed: the child flips exactly the mask, i.e. O4 (pinned to Glover's
    # printed illustration above) -- a wrong mask, shift or complement rule fails here
    rng = np.random.default_rng(21)
    for n in (10, 37, 130):
        seed = rng.integers(0, 2, size=n).astype(np.uint8)
        for t0 in (0, 7, n * (n + 1) - 3):
            a = oracle.blend(seed, (1 - seed)[None, :], t0, 150)
            b = oracle.diversify(seed, t0, 150)
            assert np.array_equal(a, b), (n, t0)


def test_blend_identity_and_shortest_path_property():
    rng = np.random.default_rng(22)
    n = 83
    seed = rng.integers(0, 2, size=n).astype(np.uint8)
    assert np.array_equal(oracle.blend(seed, seed[None, :], 0, 40), np.tile(seed, (40, 1)))
    parents = rng.integers(0, 2, size=(3, n)).astype(np.uint8)
    K = 400
    X = oracle.blend(seed, parents, 11, K)
    for g in range(K):
        p = parents[g % 3]
        x = X[g]
        # the child lies on a shortest seed-parent path and keeps every agreed bit
        assert int((x != seed).sum()) + int((x != p).sum()) == int((seed != p).sum())
        assert np.array_equal(x[seed == p], seed[seed == p])
        h, q, c = oracle.glover_params(11 + g, n)
        inm = np.zeros(n, bool)
        inm[q - 1::h] = True
        take = ~inm if c else inm
        assert int((x != seed).sum()) == int((take & (seed != p)).sum())


def test_blend_sharding_is_cyclic():
    n, K = 50, 29
    rng = np.random.default_rng(23)
    seed = rng.integers(0, 2, size=n).astype(np.uint8)
    parents = rng.integers(0, 2, size=(4, n)).astype(np.uint8)
    full = oracle.blend(seed, parents, 5, K)
    for world in (2, 3):
        for r in range(world):
            assert np.array_equal(oracle.blend(seed, parents, 5, len(range(r, K, world)), r, world),
                                  full[r::world])


def test_pool_update_rules():
    a, b, c, inc = (np.array(v, np.uint8) for v in ([1, 0], [0, 1], [1, 1], [0, 0]))
    pool = oracle.pool_update([], 2, inc, None, a)           # round best joins
    assert len(pool) == 1 and np.array_equal(pool[0], a)
    assert len(oracle.pool_update(pool, 2, inc, None, inc)) == 1   # equal to the incumbent
    assert len(oracle.pool_update(pool, 2, inc, None, a)) == 1     # already pooled
    pool = oracle.pool_update(pool, 2, c, b, c)              # improved: the old incumbent b joins
    assert [p.tolist() for p in pool] == [[1, 0], [0, 1]]
    pool = oracle.pool_update(pool, 2, inc, None, c)         # capacity: oldest leaves
    assert [p.tolist() for p in pool] == [[0, 1], [1, 1]]


# ---------------------------------------------------------------- O11 path relinking (R19)
def test_relink_hand_worked_q3():
    Q = _Qn("Q3")
    for line in (GOLD / "relink_q3.txt").read_text().splitlines():
        if line.startswith("#") or not line.strip():
            continue
        x0, y, path, fb, sb, xb = line.split()
        x0 = np.array([int(c) for c in x0], np.uint8)
        y = np.array([int(c) for c in y], np.uint8)
        Xb, f, s, ln, P = oracle.relink(Q, x0, [oracle.xQx(Q, x0)], y, with_path=True)
        assert P[0][:ln[0]].tolist() == [int(v) for v in path.split(",")], line
        assert (int(f[0]), int(s[0]), "".join(map(str, Xb[0].tolist()))) == (int(fb), int(sb), xb), line


def _brute_walk(Q, x0, y):
    """the walk by brute-force objective evaluation of every candidate move (O1 only)"""
    x = x0.copy()
    D = [j for j in range(len(x)) if x0[j] != y[j]]
    fs, path = [], []
    while D:
        best = None
        for j in D:                                   # ascending j: strict > keeps the lowest
            x[j] ^= 1
            v = oracle.xQx(Q, x)
            x[j] ^= 1
            if best is None or v > best[0]:
                best = (v, j)
        x[best[1]] ^= 1
        D.remove(best[1])
        fs.append(best[0])
        path.append(best[1])
    return fs, path


def test_relink_equals_brute_force_walk():
    rng = np.random.default_rng(41)
    for trial in range(30):
        n = int(rng.integers(2, 14))
        Q = generate_Q(n, 0.6, -20, 20, seed=1000 + trial)
        X0 = rng.integers(0, 2, size=(4, n)).astype(np.uint8)
        Y = rng.integers(0, 2, size=(3, n)).astype(np.uint8)
        f0 = oracle.eval_batch(Q, X0)
        Xb, fb, sb, ln, P = oracle.relink(Q, X0, f0, Y, with_path=True)
        for i in range(4):
            y = Y[i % 3]
            fs, path = _brute_walk(Q, X0[i], y)
            assert ln[i] == len(path) and P[i][:ln[i]].tolist() == path
            if len(path) < 2:
                assert sb[i] == -1 and np.array_equal(Xb[i], X0[i])
                continue
            inner = fs[:-1]
            s = int(np.argmax(inner))                 # first maximum = earliest step
            assert (int(fb[i]), int(sb[i])) == (inner[s], s + 1)
            assert oracle.xQx(Q, Xb[i]) == fb[i]
            assert int((Xb[i] != X0[i]).sum()) == sb[i] and int((Xb[i] != y).sum()) == ln[i] - sb[i]
            if fs:
                assert fs[-1] == oracle.xQx(Q, y)     # the walk ends at the guide


def test_relink_zero_Q_flips_in_index_order():
    n = 9
    Q = np.zeros((n, n), np.int32)
    x0 = np.zeros(n, np.uint8)
    y = np.array([1, 0, 1, 1, 0, 0, 1, 0, 1], np.uint8)
    Xb, fb, sb, ln, P = oracle.relink(Q, x0, [0], y, with_path=True)
    assert P[0][:5].tolist() == [0, 2, 3, 6, 8] and (fb[0], sb[0]) == (0, 1)


# ---------------------------------------------------------------- O5 stats
def test_stats_sum_count_and_key_order():
    rng = np.random.default_rng(15)
    f = rng.integers(-10**9, 10**9, size=300)
    f[[3, 77, 200]] = 10**9 + 5                     # ties on the max -> lowest g wins
    for world, rank in ((1, 0), (3, 2)):
        s = oracle.stats(f, rank, world)
        assert s[0] == int(f.sum()) and s[1] == f.size
        g = rank + np.arange(f.size) * world
        best = max(zip(f.tolist(), (-g).tolist()))   # highest f, then lowest g
        key = s[2]
        assert (key >> 22) - (1 << 40) == best[0]
        assert (1 << 22) - 1 - (key & ((1 << 22) - 1)) == -best[1]


def test_max_key_is_monotone():
    assert oracle.max_key(5, 0) > oracle.max_key(4, 0) > oracle.max_key(4, 1)
    assert oracle.max_key(-(1 << 40) + 1, (1 << 22) - 1) >= 0


# ---------------------------------------------------------------- O6 screen
def test_spec_threshold_examples():
    for e in SPEC["threshold"]:
        assert oracle.threshold(e["lambda"], e["mean"], 1, e["max"]) == e["T"], e["cite"]


def test_screen_strict_and_ascending():
    f = np.array([5, 150, 151, 149, 200, 150, -3], dtype=np.int64)
    T = oracle.threshold(0.5, 100, 1, 200)
    assert T == 150.0
    assert oracle.screen(f, T).tolist() == [2, 4]     # f == T fails ("exceeds"; R8)
    assert oracle.screen(f, oracle.threshold(1.0, 100, 1, 200)).tolist() == []  # lambda=1: T=Max


def test_screen_against_exact_rational_threshold():
    rng = np.random.default_rng(16)
    for _ in range(200):
        s, c = int(rng.integers(-10**12, 10**12)), int(rng.integers(1, 10**6))
        mx = int(rng.integers(-10**9, 10**9))
        lam = float(rng.random())
        T = oracle.threshold(lam, s, c, mx)
        mean = Fraction(s, c)
        exact = mean + Fraction(lam) * (mx - mean)
        assert abs(Fraction(T) - exact) <= abs(exact) * Fraction(1, 2**50) + Fraction(1, 2**40)


# ---------------------------------------------------------------- O7 ascent
def test_spec_ascent_examples():
    for e in SPEC["steepest_ascent"]:
        Q = _Qn(e["Q"])
        x0 = np.array([e["start"]], np.uint8)
        X, f, flips = oracle.ascend(Q, x0, [oracle.xQx(Q, x0)], max_flips=100)
        assert X[0].tolist() == e["x"] and f[0] == e["f"] and flips[0] == e["flips"], e["cite"]
    e = SPEC["apply_flip"][0]
    Q = _Qn(e["Q"])
    X, f, flips = oracle.ascend(Q, np.array([e["x"]], np.uint8), [oracle.xQx(Q, e["x"])], 1)
    assert X[0].tolist() == e["x_after"] and f[0] == e["f_after"]
    assert oracle.gains(Q, X[0]).tolist() == e["Delta_after"], e["cite"]


def _brute_ascent(Q, x, max_flips):
    """Steepest ascent by brute force over all 1-flip neighbours, using only O1 values."""
    x = x.copy()
    n = len(x)
    flips = 0
    while flips < max_flips:
        f = oracle.xQx(Q, x)
        nb = np.tile(x, (n, 1)) ^ np.eye(n, dtype=np.uint8)
        fn = oracle.eval_batch(Q, nb)
        k = int(np.argmax(fn))                  # numpy argmax: first (lowest) index on ties
        if fn[k] - f <= 0:
            break
        x[k] ^= 1
        flips += 1
    return x, oracle.xQx(Q, x), flips


def test_ascent_equals_brute_force_neighbourhood_search():
    rng = np.random.default_rng(17)
    for n in (1, 2, 6, 13, 40):
        Q = generate_Q(n, 0.8, -100, 100, seed=int(rng.integers(1 << 30)))
        X0 = rng.integers(0, 2, size=(12, n)).astype(np.uint8)
        f0 = oracle.eval_batch(Q, X0)
        for mf in (3, 10 * n):
            X, f, flips = oracle.ascend(Q, X0, f0, mf, nthreads=2)
            for k in range(len(X0)):
                bx, bf, bfl = _brute_ascent(Q, X0[k], mf)
                assert X[k].tolist() == bx.tolist() and f[k] == bf and flips[k] == bfl


def test_ascent_local_optimality_and_value_consistency():
    rng = np.random.default_rng(18)
    for n in (50, 200):
        Q = generate_Q(n, 0.5, -100, 100, seed=int(rng.integers(1 << 30)))
        X0 = rng.integers(0, 2, size=(25, n)).astype(np.uint8)
        X, f, flips = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), 10 * n)
        assert np.array_equal(f, oracle.eval_batch(Q, X))
        for k in range(len(X)):
            if flips[k] < 10 * n:
                assert oracle.gains(Q, X[k]).max() <= 0      # 1-flip local optimum


# ---------------------------------------------------------------- first-derivative start
def test_first_derivative_start_spec():
    for e in SPEC["first_derivative_start"]:
        x = oracle.first_derivative_start(_Qn(e["Q"]))
        assert x.tolist() == e["x"] and oracle.xQx(_Qn(e["Q"]), x) == e["f"], e["cite"]


# ---------------------------------------------------------------- O8 rounds, O10 sharding
def test_rounds_reach_spec_optimum():
    best, x, traj = oracle.run_rounds(_Qn("Q3"), K=12, rounds=2, lam=0.5, max_flips=30, sample_seed=1)
    assert best == SPEC["run_optimum"][0]["best"]


def test_rounds_recover_exhaustive_optimum_desk_scale():
    hits = 0
    for s in range(20):
        Q = generate_Q(12, 0.5, -10, 10, seed=500 + s)
        opt = int(oracle.eval_batch(Q, _all_x(12)).max())
        best, x, traj = oracle.run_rounds(Q, K=156, rounds=2, lam=0.3, max_flips=120, sample_seed=s)
        assert best == oracle.xQx(Q, x) and best <= opt
        vals = [v for _, v in traj]
        assert all(b > a for a, b in zip(vals, vals[1:]))   # strictly increasing
        hits += best == opt
    assert hits >= 18


@pytest.mark.parametrize("world", [2, 3])
def test_rounds_independent_of_world_size(world):
    Q = generate_Q(60, 0.5, -100, 100, seed=99)
    a = oracle.run_rounds(Q, K=50, rounds=3, lam=0.4, max_flips=600, sample_seed=3, world=1)
    b = oracle.run_rounds(Q, K=50, rounds=3, lam=0.4, max_flips=600, sample_seed=3, world=world)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_blend_rounds_improve_and_are_world_invariant():
    Q = generate_Q(60, 0.5, -100, 100, seed=98)
    a = oracle.run_rounds(Q, K=50, rounds=4, lam=0.4, max_flips=600, sample_seed=3, div="blend")
    b = oracle.run_rounds(Q, K=50, rounds=4, lam=0.4, max_flips=600, sample_seed=3, world=3, div="blend")
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert a[0] == oracle.xQx(Q, a[1])
    vals = [v for _, v in a[2]]
    assert all(y > x for x, y in zip(vals, vals[1:]))


def test_polish_pairs_and_result_consistency():
    rng = np.random.default_rng(51)
    n = 40
    Q = generate_Q(n, 0.5, -50, 50, seed=51)
    E = rng.integers(0, 2, size=(4, n)).astype(np.uint8)
    f, x = oracle.polish(Q, E, 10 * n)
    assert f == oracle.xQx(Q, x)
    g = oracle.gains(Q, x)
    assert g.max() <= 0                               # an ascended point: 1-flip local optimum
    # brute force over the pairs: the best of ascending each pair's best interior point
    cands = []
    for a in range(4):
        for b in range(4):
            if a == b:
                continue
            Xb, fb, sb, _ = oracle.relink(Q, E[a], [oracle.xQx(Q, E[a])], E[b])
            if sb[0] >= 0:
                Xa, fa, _ = oracle.ascend(Q, Xb, fb, 10 * n)
                cands.append(int(fa[0]))
    assert f == max(cands)
    assert oracle.polish(Q, E[:1], 10 * n) is None    # no pairs
    assert oracle.polish(Q, np.stack([E[0], E[0]]), 10 * n) is None   # |D| = 0


def test_rounds_with_polish_keep_invariants():
    Q = generate_Q(60, 0.5, -100, 100, seed=97)
    a = oracle.run_rounds(Q, K=40, rounds=3, lam=0.4, max_flips=600, sample_seed=5, polish_end=True)
    b = oracle.run_rounds(Q, K=40, rounds=3, lam=0.4, max_flips=600, sample_seed=5, world=2, polish_end=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert a[0] == oracle.xQx(Q, a[1])
    vals = [v for _, v in a[2]]
    assert all(y > x for x, y in zip(vals, vals[1:]))


# ---------------------------------------------------------------- input generator + layout
def test_generator_symmetry_density_determinism():
    Q = generate_Q(100, 0.1, -100, 100, seed=1)
    assert np.array_equal(Q, Q.T) and np.array_equal(Q, generate_Q(100, 0.1, -100, 100, seed=1))
    iu = np.triu_indices(100)
    frac = (Q[iu] != 0).mean()
    assert abs(frac - 0.1) < 0.03
    assert np.all(generate_Q(5, 1.0, 1, 1, seed=3) == 1)


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(2)
    for n in (1, 63, 64, 65, 130):
        X = rng.integers(0, 2, size=(7, n)).astype(np.uint8)
        B = pack_bits(X)
        assert B.shape == (7, (n + 63) // 64)
        assert np.array_equal(unpack_bits(B, n), X)
        j = n - 1
        assert ((B[:, j >> 6] >> np.uint64(j & 63)) & np.uint64(1)).astype(np.uint8).tolist() == X[:, j].tolist()


# ---------------------------------------------------------------- O9 real Q
def test_real_oracle_reduces_to_integer_oracle():
    """On integer-valued float Q the exactly rounded sum is the exact integer xQx (O1)."""
    rng = np.random.default_rng(19)
    Q = generate_Q(60, 0.5, seed=3)
    X = rng.integers(0, 2, size=(20, 60)).astype(np.uint8)
    assert np.array_equal(oracle.eval_batch_real(Q.astype(np.float64), X),
                          oracle.eval_batch(Q, X).astype(np.float64))
    assert np.array_equal(oracle.first_derivative_start_real(Q.astype(np.float64)),
                          oracle.first_derivative_start(Q))


def test_real_oracle_closed_forms_and_exact_rounding():
    from inputs import generate_Q_real
    Q = generate_Q_real(40, 1.0, seed=5)
    n = 40
    assert oracle.xQx_real(Q, np.zeros(n)) == 0.0
    for i in (0, 17, 39):
        assert oracle.xQx_real(Q, np.eye(n)[i]) == Q[i, i]
    # exact rounding: compare against the exact rational sum
    x = np.random.default_rng(1).integers(0, 2, size=n)
    S = np.flatnonzero(x)
    exact = sum(Fraction(float(v)) for v in Q[np.ix_(S, S)].ravel())
    assert oracle.xQx_real(Q, x) == float(exact)


def test_paper_lambda_policy_spec_examples():
    """(mean 100, start 200) -> 1.0; (mean -0.5, start 2) -> 0.5; (100, 100) -> 1.0."""
    from paper_1706_00037_b200.multistart import paper_lambda
    assert paper_lambda(100.0, 200) == 1.0
    assert paper_lambda(-0.5, 2) == 0.5
    assert paper_lambda(100.0, 100) == 1.0
    assert paper_lambda(400.0, 100) == 0.25


# ---------------------------------------------------------------- O9b real-Q ascent image (R20)
def test_real_image_scale_rule_and_rounding():
    def one(v):
        return np.array([[v]], dtype=np.float64)
    assert oracle.real_image(one(1.0))[1] == 26          # 2^26 <= 2^27 - 1 < 2^27
    assert oracle.real_image(one(0.75))[1] == 27         # 0.75 * 2^27 fits, 0.75 * 2^28 does not
    assert oracle.real_image(one(100.0))[1] == 20        # 100 * 2^20 = 104857600 <= 134217727
    Qt, e = oracle.real_image(np.array([[2**27 - 1, 2.5], [2.5, 3.5]]))
    assert e == 0 and Qt.tolist() == [[2**27 - 1, 2], [2, 4]]   # round half to even


def test_real_ascent_reduces_to_integer_ascent():
    # integer-valued real Q with max |Q| = 100: the image is Q * 2^20 exactly, so the walk is
    # the integer walk and f~ = 2^20 f (ties the reading to the pinned integer oracle)
    Q = generate_Q(60, 0.5, -100, 100, seed=61).astype(np.int32)
    Q[0, 0] = 100
    X = oracle.random_solutions(60, 8, 40)
    Xa, fa, ff, fl, e = oracle.ascend_real(Q.astype(np.float64), X, 600)
    Xi, fi, fli = oracle.ascend(Q, X, oracle.eval_batch(Q, X), 600)
    assert e == 20 and np.array_equal(Xa, Xi) and np.array_equal(fl, fli)
    assert np.array_equal(fa, fi * 2**20) and np.array_equal(ff, fi.astype(np.float64))


def test_real_ascent_value_within_rounding_bound():
    rng = np.random.default_rng(62)
    n = 80
    A = rng.uniform(-100, 100, size=(n, n))
    Q = np.triu(A) + np.triu(A, 1).T
    Xa, fa, ff, fl, e = oracle.ascend_real(Q, oracle.random_solutions(n, 9, 20), 800)
    for x, f in zip(Xa, ff):
        S = int(x.sum())
        assert abs(f - oracle.xQx_real(Q, x)) <= S * S * 2.0 ** (-(e + 1)) + 1e-9


def test_real_rounds_integer_Q_reduce_to_integer_rounds_and_world_invariance():
    # integer-valued real Q: every O9 value is the integer O1 value and the walk image is 2^20 Q
    # (max |Q| = 100), so every decision equals the integer round loop's
    Q = generate_Q(60, 0.5, -100, 100, seed=71).astype(np.int32)
    Q[0, 0] = 100
    a = oracle.run_rounds(Q, K=50, rounds=3, lam=0.4, max_flips=600, sample_seed=3)
    b = oracle.run_rounds_real(Q.astype(np.float64), K=50, rounds=3, lam=0.4, max_flips=600, sample_seed=3)
    assert b[3] == 20 and b[0] == a[0] and np.array_equal(b[1], a[1])
    assert b[2] == a[2]
    rng = np.random.default_rng(72)
    A = rng.uniform(-10, 10, size=(45, 45))
    Qr = np.triu(A) + np.triu(A, 1).T
    c = oracle.run_rounds_real(Qr, K=40, rounds=3, lam=0.3, max_flips=500, sample_seed=4)
    d = oracle.run_rounds_real(Qr, K=40, rounds=3, lam=0.3, max_flips=500, sample_seed=4, world=3)
    assert c[0] == d[0] and np.array_equal(c[1], d[1]) and c[2] == d[2]
    assert c[0] == oracle.xQx_real(Qr, c[1])
    assert [v for _, v in c[2]] == sorted(v for _, v in c[2]) and len(set(v for _, v in c[2])) == len(c[2])


def test_real_gains_brute_force_exact():
    """gains_real is the exactly rounded f(x xor e_j) - f(x): checked with exact rationals
    (fractions) on values that are not representable in a short fixed point."""
    from fractions import Fraction
    rng = np.random.default_rng(81)
    n = 9
    A = rng.standard_normal((n, n)) * np.exp2(rng.integers(-30, 30, size=(n, n)))
    Q = np.triu(A) + np.triu(A, 1).T
    for t in range(6):
        x = rng.integers(0, 2, size=n).astype(np.uint8)

        def fx(y):
            S = np.flatnonzero(y)
            return sum((Fraction(Q[i, j]) for i in S for j in S), Fraction(0))

        g = oracle.gains_real(Q, x)
        f0 = fx(x)
        for j in range(n):
            y = x.copy()
            y[j] ^= 1
            assert g[j] == float(fx(y) - f0), (t, j)


def test_batch_sum_exact_matches_fraction_sums():
    from fractions import Fraction
    rng = np.random.default_rng(82)
    n, K = 7, 13
    A = rng.uniform(-1, 1, size=(n, n)) * 1e-3 + 1e6
    Q = np.triu(A) + np.triu(A, 1).T
    X = rng.integers(0, 2, size=(K, n)).astype(np.uint8)
    want = sum((Fraction(Q[i, j]) for x in X for i in np.flatnonzero(x) for j in np.flatnonzero(x)), Fraction(0))
    assert oracle.batch_sum_exact(Q, X) == want


# ---------------------------------------------------------------- O8 hand-worked trace
def _read_rounds_golden():
    g = {"Q": [], "sample": [], "rounds": {}}
    for line in (GOLD / "rounds_n5.txt").read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        tok = line.split()
        key = tok[0]
        if key == "Q":
            g["Q"].append([int(v) for v in tok[1:]])
        elif key == "sample":
            g["sample"].append(([int(c) for c in tok[1]], int(tok[2])))
        elif key in ("K", "n_rounds", "sample_seed", "mean_sum", "mean_count"):
            g[key] = int(tok[1])
        elif key == "lambda":
            g[key] = float(tok[1])
        elif key == "start":
            g["start"] = ([int(c) for c in tok[1]], int(tok[2]))
        else:
            r = int(tok[1])
            d = g["rounds"].setdefault(r, {})
            if key == "round":
                d["t0"] = int(tok[3])
            elif key in ("f", "survivors"):
                d[key] = [int(v) for v in tok[2:]]
            elif key == "max_value":
                d[key] = int(tok[2])
            elif key == "ascended":
                d[key] = [tuple(int(v) for v in p.split(":")) for p in tok[2:]]
            elif key == "best":
                d[key] = (int(tok[2]), int(tok[3]), [int(c) for c in tok[4]])
            elif key == "incumbent":
                d[key] = (int(tok[2]), [int(c) for c in tok[3]])
    return g


def test_rounds_hand_worked_trace():
    """O8 against a hand-worked n = 5 trace (tests/golden/rounds_n5.txt): t0 = (r-1)K, the
    pinned sampling mean, Max = max(incumbent, batch max), ties to the lowest g, strict
    update -- each a reading the trace distinguishes from its plausible alternative."""
    g = _read_rounds_golden()
    Q = np.array(g["Q"], dtype=np.int32)
    n, K = Q.shape[0], g["K"]
    S = oracle.random_solutions(n, g["sample_seed"], K)
    for (x, fv), row in zip(g["sample"], S):
        assert row.tolist() == x and oracle.xQx(Q, row) == fv
    assert sum(fv for _, fv in g["sample"]) == g["mean_sum"] and K == g["mean_count"]
    assert oracle.first_derivative_start(Q).tolist() == g["start"][0]
    trace = []
    best, bx, traj = oracle.run_rounds(Q, K, g["n_rounds"], g["lambda"], 50, g["sample_seed"], trace=trace)
    assert len(trace) == g["n_rounds"]
    inc = g["start"]
    for tr in trace:
        want = g["rounds"][tr["round"]]
        assert tr["t0"] == want["t0"]
        assert (tr["mean_sum"], tr["mean_count"]) == (g["mean_sum"], g["mean_count"])
        assert tr["f"] == want["f"] and tr["max_value"] == want["max_value"]
        mean = g["mean_sum"] / g["mean_count"]
        assert tr["T"] == mean + g["lambda"] * (want["max_value"] - mean)
        assert tr["survivors"] == want["survivors"] and tr["ascended"] == want["ascended"]
        bf, bg, bxx = tr["best"]
        assert (bf, bg, bxx.tolist()) == want["best"]
        if bf > inc[1]:
            inc = (bxx.tolist(), bf)
        assert (inc[1], inc[0]) == want["incumbent"]
    assert best == inc[1] and bx.tolist() == inc[0]
    assert traj == [(0, g["start"][1]), (1, 42)]
