"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Integer Q => every comparison is exact (north_star "bit-exact").
Sizes span several tiles and ragged tails: n in {1..129, 500, 1100, 2500} crosses the
128-byte K block, the 256-column N tile and the 64-bit word; K crosses the 128-row M
tile.  Full-size (n = 7000, K = 262144) runs compare sampled rows.
"""
import numpy as np
import pytest

import oracle
from inputs import generate_Q, pack_bits, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, UbqpError, ubqp_stats  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402
from paper_1706_00037_b200.ubqp import ASCENT_AUTO, ASCENT_DENSE, ASCENT_WARP, OPT_ASCENT  # noqa: E402

build_lib()

NS = [1, 2, 3, 31, 50, 63, 64, 65, 127, 128, 129, 257, 500, 1100, 2500]


@pytest.fixture(scope="module")
def dev():
    return Ubqp(0)


def _handle_with(Q, k_max):
    u = Ubqp(0)
    u.load_Q(Q, k_max)
    return u


def _batch(u, K, n):
    B = np.zeros((max(K, 1), u.W64), dtype=np.uint64)
    u.get_batch(B)
    return unpack_bits(B[:K], n)


@pytest.mark.parametrize("n", NS)
def test_random_batch_bits(n):
    Q = generate_Q(n, 0.5, seed=n)
    K = 300
    u = _handle_with(Q, K)
    u.random(1234 + n, K)
    assert np.array_equal(_batch(u, K, n), oracle.random_solutions(n, 1234 + n, K))


@pytest.mark.parametrize("n", NS)
def test_glover_batch_bits(n):
    Q = generate_Q(n, 0.5, seed=n)
    K = 333
    rng = np.random.default_rng(n)
    seed_x = rng.integers(0, 2, size=n).astype(np.uint8)
    u = _handle_with(Q, K)
    for t0 in (0, 5 * n * (n + 1) + 17):
        u.diversify(pack_bits(seed_x)[0], t0, K)
        assert np.array_equal(_batch(u, K, n), oracle.diversify(seed_x, t0, K)), t0


@pytest.mark.parametrize("n", NS)
def test_blend_batch_bits(n):
    """O4b blend (R11b) bit-exact, host and device parents, P in {1, 3, > K}, sharded."""
    Q = generate_Q(n, 0.5, seed=n)
    K = 333
    rng = np.random.default_rng(100 + n)
    seed_x = rng.integers(0, 2, size=n).astype(np.uint8)
    u = _handle_with(Q, K)
    for P in (1, 3, 400):
        parents = rng.integers(0, 2, size=(P, n)).astype(np.uint8)
        pb = pack_bits(parents)
        for t0 in (0, 3 * n * (n + 1) + 11):
            u.blend(pack_bits(seed_x)[0], pb, P, t0, K)
            assert np.array_equal(_batch(u, K, n), oracle.blend(seed_x, parents, t0, K)), (P, t0)
        pd = torch.from_numpy(pb.view(np.int64)).cuda()
        for world in (1, 3):
            for r in range(world):
                kl = oracle.shard_count(r, K, world, 2)          # the library's default block B = 2
                u.blend(pack_bits(seed_x)[0], pd, P, 9, kl, r, world)
                torch.cuda.synchronize()
                assert np.array_equal(_batch(u, kl, n), oracle.blend(seed_x, parents, 9, kl, r, world, 2)), (P, r)


def test_blend_complement_parent_equals_glover_and_errors():
    n, K = 777, 500
    Q = generate_Q(n, 0.5, seed=3)
    rng = np.random.default_rng(5)
    seed_x = rng.integers(0, 2, size=n).astype(np.uint8)
    u = _handle_with(Q, K)
    u.blend(pack_bits(seed_x)[0], pack_bits((1 - seed_x)[None, :]), 1, 40, K)
    a = _batch(u, K, n)
    u.diversify(pack_bits(seed_x)[0], 40, K)
    assert np.array_equal(a, _batch(u, K, n))
    with pytest.raises(UbqpError):
        u.blend(pack_bits(seed_x)[0], pack_bits(seed_x[None, :]), 0, 0, K)


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("density", [0.1, 1.0])
def test_eval_f_and_stats(n, density):
    Q = generate_Q(n, density, seed=7 * n + 1)
    K = 1 if n == 1 else 389                       # 4 M tiles, ragged
    u = _handle_with(Q, 512)
    u.random(99, K)
    f = np.zeros(K, dtype=np.int64)
    st = ubqp_stats()
    u.eval_batch(0, f, st)
    X = oracle.random_solutions(n, 99, K)
    ref = oracle.eval_batch(Q, X, nthreads=8)
    assert np.array_equal(f, ref)
    ost = oracle.stats(ref)
    assert (st.sum, st.count, st.max_key, st.reserved) == tuple(int(v) for v in ost)


@pytest.mark.parametrize("n", [1, 3, 65, 129, 500, 1100])
def test_eval_gains(n):
    Q = generate_Q(n, 0.7, seed=n + 3)
    K = 150
    u = _handle_with(Q, K)
    u.random(5, K)
    f = np.zeros(K, dtype=np.int64)
    u.eval_batch(UBQP_EMIT_GAINS, f)
    G = np.zeros((K, n), dtype=np.int32)
    u.get_gains(0, K, G)
    X = oracle.random_solutions(n, 5, K)
    for k in range(0, K, 7 if n > 500 else 1):
        assert np.array_equal(G[k].astype(np.int64), oracle.gains(Q, X[k])), k
    assert np.array_equal(f, oracle.eval_batch(Q, X, nthreads=8))


def test_eval_device_pointers_torch():
    n, K = 700, 600
    Q = generate_Q(n, 0.3, seed=11)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(torch.from_numpy(Q).cuda(), K)
    bits = torch.from_numpy(pack_bits(oracle.random_solutions(n, 8, K)).view(np.int64)).cuda()
    u.set_batch(bits, K)
    f = torch.zeros(K, dtype=torch.int64, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    u.eval_batch(0, f, st)
    torch.cuda.synchronize()
    ref = oracle.eval_batch(Q, oracle.random_solutions(n, 8, K), nthreads=8)
    assert np.array_equal(f.cpu().numpy(), ref)
    assert st.cpu().tolist() == oracle.stats(ref).tolist()


@pytest.mark.parametrize("lam", [0.0, 0.25, 0.5, 0.9, 1.0, -0.3])
def test_screen(lam):
    n, K = 300, 5000
    Q = generate_Q(n, 0.5, seed=21)
    u = _handle_with(Q, K)
    u.random(3, K)
    f = np.zeros(K, dtype=np.int64)
    st = ubqp_stats()
    u.eval_batch(0, f, st)
    maxv = (st.max_key >> 22) - (1 << 40)
    surv = np.zeros(K, dtype=np.int32)
    m, T = u.screen(lam, st.sum, st.count, maxv, surv)
    To = oracle.threshold(lam, st.sum, st.count, maxv)
    assert T == To
    assert np.array_equal(surv[:m], oracle.screen(f, To))


def test_screen_boundary_equal_fails():
    n = 2
    Q = np.array([[1, 2], [2, -3]], dtype=np.int32)
    u = _handle_with(Q, 4)
    u.set_batch(pack_bits(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], np.uint8)), 4)
    f = np.zeros(4, dtype=np.int64)
    u.eval_batch(0, f)
    assert f.tolist() == [0, 1, 2, -3]
    surv = np.zeros(4, dtype=np.int32)
    m, T = u.screen(0.5, 0, 1, 2, surv)           # T = 1: f = 1 does not pass ("exceeds")
    assert T == 1.0 and surv[:m].tolist() == [2]


@pytest.mark.parametrize("n", [1, 2, 3, 50, 129, 500, 1100, 2500])
@pytest.mark.parametrize("max_flips", [0, 3, 100000])
@pytest.mark.parametrize("kernel", [ASCENT_AUTO, ASCENT_DENSE, ASCENT_WARP])
def test_ascend(n, max_flips, kernel):
    Q = generate_Q(n, 0.8, seed=31 + n)
    K = 64 if n >= 1100 else 200
    u = _handle_with(Q, K)
    u.set_option(OPT_ASCENT, kernel)
    u.random(17, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(0, K, 3, dtype=np.int32)[::-1].copy()   # unordered subset
    m = len(slots)
    f_o = np.zeros(m, np.int64)
    fl_o = np.zeros(m, np.int32)
    b_o = np.zeros((m, u.W64), np.uint64)
    key = np.zeros(1, np.int64)
    u.ascend(slots, m, max_flips, f_o, fl_o, b_o, key)
    X0 = oracle.random_solutions(n, 17, K)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), max_flips, nthreads=8)
    assert np.array_equal(unpack_bits(b_o, n), Xr)
    assert np.array_equal(f_o, fr)
    assert np.array_equal(fl_o, flr)
    best = max(oracle.max_key(int(fr[i]), int(slots[i])) for i in range(m))
    assert key[0] == best


def test_ascend_computes_missing_gains_and_empty():
    n, K = 300, 100
    Q = generate_Q(n, 0.5, seed=2)
    u = _handle_with(Q, K)
    u.random(4, K)
    u.eval_batch(0)                               # no gains: ascend must compute them
    f_o = np.zeros(K, np.int64)
    u.ascend(np.arange(K, dtype=np.int32), K, 10 * n, f_o)
    X0 = oracle.random_solutions(n, 4, K)
    _, fr, _ = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), 10 * n, nthreads=8)
    assert np.array_equal(f_o, fr)
    key = np.zeros(1, np.int64)
    u.ascend(np.zeros(1, np.int32), 0, 10, best_key_out=key)
    assert key[0] == -1


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("block", [1, 2, 5])
def test_sharding_matches_single_rank(world, block):
    """O10: rank r holds g = (r + floor(i/B) world) B + (i mod B); every rank's f and stats
    come from the global batch, and they partition it"""
    from paper_1706_00037_b200.ubqp import OPT_SHARD_BLOCK, Q_SHARD_BLOCK
    n, K = 400, 1000
    Q = generate_Q(n, 0.5, seed=5)
    seed_x = np.random.default_rng(1).integers(0, 2, size=n).astype(np.uint8)
    full = oracle.eval_batch(Q, oracle.diversify(seed_x, 3, K), nthreads=8)
    u = _handle_with(Q, K)
    assert u.query(Q_SHARD_BLOCK) == 2
    u.set_option(OPT_SHARD_BLOCK, block)
    tot = 0
    best = -1
    seen = []
    for r in range(world):
        kr = oracle.shard_count(r, K, world, block)
        gs = [oracle.global_index(i, r, world, block) for i in range(kr)]
        seen += gs
        u.diversify(pack_bits(seed_x)[0], 3, kr, r, world)
        f = np.zeros(kr, np.int64)
        st = ubqp_stats()
        u.eval_batch(0, f, st)
        assert np.array_equal(f, full[gs])
        assert st.max_key == oracle.stats(full[gs], r, world, block)[2]
        tot += st.sum
        best = max(best, st.max_key)
    assert sorted(seen) == list(range(K))
    ost = oracle.stats(full)
    assert tot == ost[0] and best == ost[2]


def test_first_derivative_start():
    for n in (3, 64, 65, 1000):
        Q = generate_Q(n, 0.5, seed=n)
        u = _handle_with(Q, 4)
        b = np.zeros(u.W64, np.uint64)
        u.first_derivative(b)
        assert np.array_equal(unpack_bits(b, n)[0], oracle.first_derivative_start(Q))


def test_errors():
    u = Ubqp(0)
    with pytest.raises(UbqpError) as e:
        u.eval_batch(0)
    assert e.value.code == 4                       # E_STATE
    Q = np.array([[1, 2], [3, 1]], np.int32)
    with pytest.raises(UbqpError) as e:
        u.load_Q(Q, 4)
    assert e.value.code == 2                       # E_NOT_SYMMETRIC
    with pytest.raises(UbqpError) as e:
        u.load_Q(np.array([[200]], np.int32), 4)
    assert e.value.code == 3                       # E_RANGE
    u.load_Q(np.array([[5]], np.int32), 4)
    with pytest.raises(UbqpError):
        u.random(0, 5)                             # k_local > k_max
    u.random(0, 0)
    st = ubqp_stats()
    u.eval_batch(0, None, st)
    assert st.count == 0 and st.max_key == -1


def test_errors_of_every_call():
    """Return codes of the C-ABI (include/ubqp.h "Errors"): each call rejects bad arguments
    with its documented code and leaves the handle usable."""
    u = Ubqp(0)
    n = 70
    Q = generate_Q(n, 0.5, seed=8)
    codes = []

    def err(fn, *a):
        with pytest.raises(UbqpError) as e:
            fn(*a)
        codes.append(e.value.code)
        return e.value.code

    assert err(u.diversify, np.zeros(2, np.uint64), 0, 4) == 4           # no Q: E_STATE
    assert err(u.load_Q, Q, 0) == 1                                    # k_max < 1
    assert err(u.load_Q, Q, (1 << 22) + 1) == 1                        # k_max > 2^22
    u.load_Q(Q, 64)
    seed = pack_bits(oracle.first_derivative_start(Q))[0]
    assert err(u.diversify, seed, -1, 8) == 1                          # t0 < 0
    assert err(u.diversify, seed, (1 << 62) + 1, 8) == 1               # t0 > 2^62
    assert err(u.blend, seed, pack_bits(np.zeros((1, n), np.uint8)), 1, -5, 8) == 1
    assert err(u.diversify, seed, 0, 8, 3, 2) == 1                     # rank >= world
    u.diversify(seed, 0, 8)
    assert err(u.ascend, np.arange(8, dtype=np.int32), 8, 10) == 4     # not evaluated: E_STATE
    u.eval_batch(UBQP_EMIT_GAINS)
    surv = np.zeros(8, np.int32)
    assert err(u.screen, float("nan"), 1, 1, 1, surv) == 1             # non-finite lambda
    assert err(u.screen, 0.5, 1, 0, 1, surv) == 4                      # mean_count <= 0
    assert err(u.ascend, np.arange(9, dtype=np.int32), 9, 10) == 1     # m > k_local
    assert err(u.ascend, np.arange(8, dtype=np.int32), 8, -1) == 1     # max_flips < 0
    assert err(u.get_gains, 5, 10, np.zeros((10, n), np.int32)) == 1   # slots past k_local
    u.ascend(np.arange(8, dtype=np.int32), 8, 10)                      # still usable
    assert err(u.ascend_real, np.arange(8, dtype=np.int32), 8, 10) == 4  # integer Q loaded
    assert err(u.eval_batch_real) == 4
    u.close()


# ------------------------------------------------------------------ full-size, sampled
@pytest.mark.parametrize("n,K,kind", [(5000, 1000, "random"), (7000, 1000, "random"),
                                      (7000, 262144, "glover")])
def test_full_size_sampled(n, K, kind):
    Q = generate_Q(n, 1.0, seed=4)
    u = _handle_with(Q, K)
    if kind == "random":
        u.random(4, K)
        Xs = lambda idx: oracle.random_solutions(n, 4, K)[idx]   # noqa: E731
    else:
        b = np.zeros(u.W64, np.uint64)
        u.first_derivative(b)
        seed_x = unpack_bits(b, n)[0]
        u.diversify(b, 0, K)
        Xs = lambda idx: np.stack([oracle.diversify(seed_x, int(i), 1)[0] for i in idx])  # noqa: E731
    f = np.zeros(K, np.int64)
    st = ubqp_stats()
    u.eval_batch(0, f, st)
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([[0, 1, K - 1], rng.integers(0, K, 61)]))
    assert np.array_equal(f[idx], oracle.eval_batch(Q, Xs(idx), nthreads=8))
    assert st.sum == int(f.sum()) and st.count == K


@pytest.mark.parametrize("n", [5000, 7000, 9000, 12000])
@pytest.mark.parametrize("kernel", [ASCENT_AUTO, ASCENT_DENSE])
def test_ascend_full_size(n, kernel):
    """Automatic kernel (warp per solution up to n_pad = 7168, CTA above) and the CTA
    kernel's default shapes 64x5 (n=5000), 64x7 (n=7000), 96x6 (n=9000), 128x6 (n=12000),
    exact against the oracle."""
    Q = generate_Q(n, 1.0, seed=4)
    K = 24
    u = _handle_with(Q, K)
    u.set_option(OPT_ASCENT, kernel)
    b = np.zeros(u.W64, np.uint64)
    u.first_derivative(b)
    x0 = unpack_bits(b, n)[0]
    u.diversify(b, 600, K)                     # Glover solutions near the first-derivative start
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(K, dtype=np.int32)
    f_o = np.zeros(K, np.int64)
    fl_o = np.zeros(K, np.int32)
    b_o = np.zeros((K, u.W64), np.uint64)
    u.ascend(slots, K, 10 * n, f_o, fl_o, b_o)
    X0 = oracle.diversify(x0, 600, K)
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), 10 * n, nthreads=8)
    assert np.array_equal(f_o, fr) and np.array_equal(fl_o, flr)
    assert np.array_equal(unpack_bits(b_o, n), Xr)


@pytest.mark.parametrize("shape", ["32,5", "32,7", "64,5", "64,7", "96,5", "96,6", "128,5", "160,7"])
def test_ascend_forced_shapes(shape, monkeypatch):
    n, K = 2500, 40
    Q = generate_Q(n, 0.5, seed=8)
    u = _handle_with(Q, K)
    u.set_option(OPT_ASCENT, ASCENT_DENSE)       # the shapes of the CTA kernel
    u.random(9, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    monkeypatch.setenv("UBQP_ASC_CFG", shape)
    f_o = np.zeros(K, np.int64)
    b_o = np.zeros((K, u.W64), np.uint64)
    u.ascend(np.arange(K, dtype=np.int32), K, 100000, f_o, None, b_o)
    X0 = oracle.random_solutions(n, 9, K)
    Xr, fr, _ = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), 100000, nthreads=8)
    assert np.array_equal(f_o, fr) and np.array_equal(unpack_bits(b_o, n), Xr)


@pytest.mark.parametrize("n,K,rounds,lam", [(50, 1000, 3, 0.5), (300, 2000, 2, 0.3), (1100, 600, 2, 0.7)])
def test_multistart_rounds_match_oracle(n, K, rounds, lam):
    """The composed product round (MultiStart: sampling mean, first-derivative incumbent,
    diversify/eval/screen/ascend/best record; O8) against the oracle's run_rounds."""
    from paper_1706_00037_b200.multistart import MultiStart
    Q = generate_Q(n, 0.1 if n == 50 else 0.5, seed=n)
    ms = MultiStart(Q, K, lam=lam, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=7)
    obest, ox, otraj = oracle.run_rounds(Q, K, rounds, lam, 10 * n, sample_seed=7, nthreads=8)
    assert best == obest and traj == otraj
    got = unpack_bits(bits.cpu().numpy().view(np.uint64), n)[0]
    assert np.array_equal(got, ox)


@pytest.mark.parametrize("n", [1, 2, 3, 31, 64, 65, 129, 500, 1100, 2500])
def test_relink_matches_oracle(n):
    """O11 path relinking (NEXT-4, R19) bit-exact: best interior value, its step, |D|, the
    interior solution and the best key; host and device guides, several guides."""
    Q = generate_Q(n, 0.5, seed=300 + n)
    rng = np.random.default_rng(n)
    K = 150
    X0 = rng.integers(0, 2, size=(K, n)).astype(np.uint8)
    G = rng.integers(0, 2, size=(3, n)).astype(np.uint8)
    slots = np.arange(K, dtype=np.int32)[::-1].copy()   # list order differs from slot order
    X0[slots[3]] = G[0]                             # list entry 3 -> guide 0: |D| = 0
    X0[slots[4]] = G[1]
    X0[slots[4]][0] ^= 1                            # list entry 4 -> guide 1: |D| = 1
    u = _handle_with(Q, K)
    u.set_batch(pack_bits(X0), K)
    f0 = np.zeros(K, np.int64)
    u.eval_batch(UBQP_EMIT_GAINS, f0)
    Xs = X0[slots]
    ob, of, os_, ol = oracle.relink(Q, Xs, f0[slots], G, nthreads=8)
    for guides in (pack_bits(G), torch.from_numpy(pack_bits(G).view(np.int64)).cuda()):
        f = np.zeros(K, np.int64)
        st = np.zeros(K, np.int32)
        ln = np.zeros(K, np.int32)
        b = np.zeros((K, u.W64), np.uint64)
        key = np.zeros(1, np.int64)
        u.relink(guides, 3, slots, K, f, st, ln, b, key)
        assert np.array_equal(ln, ol) and np.array_equal(st, os_) and np.array_equal(f, of)
        assert np.array_equal(unpack_bits(b, n), ob)
        has = os_ >= 0
        want = max((oracle.max_key(int(of[i]), int(slots[i])) for i in np.flatnonzero(has)), default=-1)
        assert int(key[0]) == want


def test_relink_range_and_errors():
    n = 9000                                        # (2n-1)*qmax >= 2^21 at qmax = 127
    Q = np.zeros((n, n), np.int32)
    Q[0, 0] = 127
    u = _handle_with(Q, 4)
    u.random(1, 4)
    u.eval_batch(UBQP_EMIT_GAINS)
    g = np.zeros((1, u.W64), np.uint64)
    with pytest.raises(UbqpError):
        u.relink(g, 1, np.arange(4, dtype=np.int32), 4)
    Q2 = generate_Q(100, 0.5, seed=1)
    u2 = _handle_with(Q2, 4)
    u2.random(1, 4)
    u2.eval_batch(UBQP_EMIT_GAINS)
    with pytest.raises(UbqpError):
        u2.relink(np.zeros((1, u2.W64), np.uint64), 0, np.arange(4, dtype=np.int32), 4)
    with pytest.raises(UbqpError):
        u2.relink(np.zeros((1, u2.W64), np.uint64), 1, np.array([0, 9], np.int32), 2)


@pytest.mark.parametrize("n", [1, 2, 200, 257, 513, 2500])
def test_symmetric_and_full_eval_agree(n, monkeypatch):
    """f-only evaluations use the triangular GEMM (NEXT-1); UBQP_FULL_EVAL=1 forces the full
    one; UBQP_EVAL_2SM=0 the single-CTA kernel.  All must equal the oracle exactly."""
    Q = generate_Q(n, 0.6, seed=n + 40)
    K = 300
    X = oracle.random_solutions(n, 21, K)
    ref = oracle.eval_batch(Q, X, nthreads=8)
    for pair in ("1", "0"):                       # CTA-pair (cta_group::2) and single-CTA kernels
        monkeypatch.setenv("UBQP_EVAL_2SM", pair)
        for full in ("0", "1"):
            monkeypatch.setenv("UBQP_FULL_EVAL", full)
            u = _handle_with(Q, K)
            u.random(21, K)
            f = np.zeros(K, np.int64)
            st = ubqp_stats()
            u.eval_batch(0, f, st)
            assert np.array_equal(f, ref), (pair, full)
            assert st.max_key == oracle.stats(ref)[2]
            if n <= 513:
                u.eval_batch(UBQP_EMIT_GAINS, f)
                G = np.zeros((K, n), np.int32)
                u.get_gains(0, K, G)
                for k in (0, K // 2, K - 1):
                    assert np.array_equal(G[k].astype(np.int64), oracle.gains(Q, X[k])), (pair, k)


def test_bench_round_full_size():
    """The exact bench step (config 4: n = 7000, K = 262144 Glover, lambda = 0.5, max_flips =
    10n): sampled survivors are ascended by the oracle and compared exactly; for ALL survivors
    the outputs are checked by properties at full size: f equals an independent re-evaluation
    of the returned bits, and every returned solution is a 1-flip local optimum (all gains
    <= 0, recomputed by the eval kernel) unless it used max_flips."""
    from paper_1706_00037_b200.multistart import MultiStart
    from inputs import CONFIGS
    cfg = CONFIGS[4]
    n, K = cfg["n"], cfg["K"]
    Q = generate_Q(n, cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, K, lam=cfg["lam"], max_flips=cfg["max_flips"])
    x0_bits, f0 = ms.first_derivative()
    res = ms.round(x0_bits, 0, f0)
    m = res.m
    assert m > 1000
    surv = ms.surv[:m].cpu().numpy()
    f_asc = ms.f_asc[:m].cpu().numpy()
    flips = ms.flips[:m].cpu().numpy()
    bits = ms.bits[:m].cpu().numpy().view(np.uint64)
    # sampled exact comparison with the oracle
    x0 = unpack_bits(x0_bits.cpu().numpy().view(np.uint64), n)[0]
    rng = np.random.default_rng(3)
    pick = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 10)]))
    X0 = np.stack([oracle.diversify(x0, int(surv[i]), 1)[0] for i in pick])
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), cfg["max_flips"], nthreads=8)
    assert np.array_equal(f_asc[pick], fr) and np.array_equal(flips[pick], flr)
    assert np.array_equal(unpack_bits(bits[pick], n), Xr)
    # full-size properties through an independent evaluation of the returned solutions
    u = _handle_with(Q, m)
    u.set_batch(bits.copy(), m)
    f_re = torch.zeros(m, dtype=torch.int64, device="cuda")
    u.eval_batch(UBQP_EMIT_GAINS, f_re)
    torch.cuda.synchronize()
    assert np.array_equal(f_re.cpu().numpy(), f_asc)
    chunk = 16384
    G = torch.empty((chunk, n), dtype=torch.int32, device="cuda")
    for s0 in range(0, m, chunk):
        c = min(chunk, m - s0)
        u.get_gains(s0, c, G[:c])
        torch.cuda.synchronize()
        gmax = G[:c].max(dim=1).values.cpu().numpy()
        capped = flips[s0:s0 + c] >= cfg["max_flips"]
        assert np.all((gmax <= 0) | capped)


def test_multistart_paper_lambda_matches_oracle():
    from paper_1706_00037_b200.multistart import MultiStart
    n, K = 200, 1500
    Q = generate_Q(n, 0.5, seed=77)
    ms = MultiStart(Q, K, lam=0.5, max_flips=10 * n)
    best, bits, traj = ms.run(3, sample_seed=9, lam_policy="paper")
    obest, ox, otraj = oracle.run_rounds(Q, K, 3, "paper", 10 * n, sample_seed=9, nthreads=8)
    assert best == obest and traj == otraj


@pytest.mark.parametrize("n,K,rounds,lam", [(60, 400, 5, 0.4), (300, 2000, 4, 0.3)])
def test_multistart_blend_matches_oracle(n, K, rounds, lam):
    """Figure-2 driver with blend diversification (NEXT-2, R11b) against the oracle."""
    from paper_1706_00037_b200.multistart import MultiStart
    Q = generate_Q(n, 0.5, seed=200 + n)
    ms = MultiStart(Q, K, lam=lam, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=4, div="blend")
    obest, ox, otraj = oracle.run_rounds(Q, K, rounds, lam, 10 * n, sample_seed=4, nthreads=8, div="blend")
    assert best == obest and traj == otraj
    assert np.array_equal(unpack_bits(bits.cpu().numpy().view(np.uint64), n)[0], ox)


@pytest.mark.parametrize("n,E", [(40, 4), (700, 9), (2500, 5)])
def test_polish_matches_oracle(n, E):
    from paper_1706_00037_b200.multistart import MultiStart
    Q = generate_Q(n, 0.5, seed=400 + n)
    rng = np.random.default_rng(n)
    El = rng.integers(0, 2, size=(E, n)).astype(np.uint8)
    El[1] = El[0]                                   # a pair with |D| = 0 both ways
    ms = MultiStart(Q, 64, lam=0.5, max_flips=10 * n)
    got = ms.polish(torch.from_numpy(pack_bits(El).view(np.int64)).cuda())
    want = oracle.polish(Q, El, 10 * n, nthreads=8)
    assert got[0] == want[0]
    assert np.array_equal(unpack_bits(got[1].cpu().numpy().view(np.uint64)[None, :], n)[0], want[1])


@pytest.mark.parametrize("n,K,rounds,div", [(60, 400, 4, "glover"), (300, 1500, 3, "blend")])
def test_multistart_polish_matches_oracle(n, K, rounds, div):
    from paper_1706_00037_b200.multistart import MultiStart
    Q = generate_Q(n, 0.5, seed=500 + n)
    ms = MultiStart(Q, K, lam=0.4, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=6, div=div, polish_end=True)
    obest, ox, otraj = oracle.run_rounds(Q, K, rounds, 0.4, 10 * n, sample_seed=6, nthreads=8, div=div,
                                         polish_end=True)
    assert best == obest and traj == otraj
    assert np.array_equal(unpack_bits(bits.cpu().numpy().view(np.uint64), n)[0], ox)


@pytest.mark.parametrize("n", [16384])
def test_limits_max_n_and_coefficients(n):
    """The documented limits: n = 16384 (largest ascent shape 160x7) with every coefficient
    at +127 or -127, where |Y| = n*127, |Delta| = (2n-1)*127 (keys 256*Delta ~ 1.07e9, next to
    the int32 edge) and f = 127 n^2 exercise every overflow bound of include/ubqp.h."""
    rng = np.random.default_rng(5)
    sign = np.where(rng.random((n, n)) < 0.5, -1, 1).astype(np.int32)
    Q = 127 * np.triu(sign)
    Q = Q + np.triu(Q, 1).T                                  # symmetric, all entries +-127
    Qp = np.full((n, n), 127, dtype=np.int32)               # all +127: ascent from 0 flips everything
    for QQ, name in ((Qp, "plus"), (Q, "mixed")):
        u = _handle_with(QQ, 4)
        X = np.zeros((4, n), np.uint8)
        X[1] = 1
        X[2:] = rng.integers(0, 2, size=(2, n))
        u.set_batch(pack_bits(X), 4)
        f = np.zeros(4, np.int64)
        u.eval_batch(UBQP_EMIT_GAINS, f)
        fo = oracle.eval_batch(QQ, X, nthreads=8)
        assert np.array_equal(f, fo), name
        if name == "plus":
            assert f[1] == 127 * n * n
        slots = np.array([0, 2], np.int32)
        fa = np.zeros(2, np.int64)
        fl = np.zeros(2, np.int32)
        ba = np.zeros((2, u.W64), np.uint64)
        u.ascend(slots, 2, 10 * n, fa, fl, ba)
        Xr, fr, flr = oracle.ascend(QQ, X[slots], fo[slots], 10 * n, nthreads=2)
        assert np.array_equal(fa, fr) and np.array_equal(fl, flr), name
        assert np.array_equal(unpack_bits(ba, n), Xr), name
        u.close()
