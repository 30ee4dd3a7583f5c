"""GPU parity of the multi-warp steepest ascent (ascend_warp.cu ascend_mw_kernel, UBQP_OPT_ASCENT
= 4: 2 or 3 warps per solution, one cross-warp argmax exchange per step) against the oracle's O7
(plain C steepest ascent, lowest index on ties) and word for word against the CTA
kernel (UBQP_OPT_ASCENT = 1): final bits, f, flip counts, best key.

Sizes cross the 1024-variable chunk of two warps (512 per warp), the padded-row guard (the two-
warp chunk past q_ld at n = 1 and n = 1100), the largest two-warp shape (n_pad = 14336) and the
three-warp shapes (n_pad in (14336, 16384]).
"""
import numpy as np
import pytest

import oracle
from inputs import generate_Q, pack_bits, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402
from paper_1706_00037_b200.ubqp import ASCENT_DENSE, ASCENT_MW, OPT_ASCENT, Q_ASCENT_LAST  # noqa: E402

build_lib()


def _run(u, slots, max_flips, kernel):
    m = len(slots)
    u.set_option(OPT_ASCENT, kernel)
    f = np.zeros(max(m, 1), np.int64)
    fl = np.zeros(max(m, 1), np.int32)
    b = np.zeros((max(m, 1), u.W64), np.uint64)
    key = np.zeros(1, np.int64)
    u.ascend(slots, m, max_flips, f, fl, b, key)
    return f[:m], fl[:m], b[:m], int(key[0])


@pytest.mark.parametrize("n", [1, 2, 17, 511, 512, 513, 1023, 1024, 1025, 1100, 2049, 4100, 7000,
                               9000, 10240, 12001, 13312, 14336, 14337, 15360, 16384])
def test_mw_ascent_matches_oracle(n):
    dens = 1.0 if n >= 2500 else 0.6
    Q = generate_Q(n, dens, seed=301 + n)
    K = 6 if n >= 9000 else (24 if n >= 2500 else 96)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(17 + n, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(K, dtype=np.int32)[::-1].copy()
    f, fl, b, key = _run(u, slots, 10 * n, ASCENT_MW)
    assert u.query(Q_ASCENT_LAST) == ASCENT_MW
    few = slots[:3] if n >= 9000 else slots
    X0 = oracle.random_solutions(n, 17 + n, K)[few]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), 10 * n, nthreads=8)
    sel = np.arange(len(few))
    assert np.array_equal(f[sel], fr)
    assert np.array_equal(fl[sel], flr)
    assert np.array_equal(unpack_bits(b[sel], n), Xr)
    if len(few) == K:
        assert key == max(oracle.max_key(int(fr[i]), int(slots[i])) for i in range(K))
    f2, fl2, b2, key2 = _run(u, slots, 10 * n, ASCENT_DENSE)
    assert np.array_equal(f, f2) and np.array_equal(fl, fl2) and np.array_equal(b, b2) and key == key2
    u.close()


@pytest.mark.parametrize("max_flips", [0, 1, 2, 7, 50])
def test_mw_ascent_flip_limit(max_flips):
    n, K = 3000, 32
    Q = generate_Q(n, 0.8, seed=6)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(4, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(0, K, 2, dtype=np.int32)
    f, fl, b, _ = _run(u, slots, max_flips, ASCENT_MW)
    X0 = oracle.random_solutions(n, 4, K)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), max_flips, nthreads=8)
    assert np.array_equal(f, fr) and np.array_equal(fl, flr)
    assert np.array_equal(unpack_bits(b, n), Xr)
    u.close()


@pytest.mark.parametrize("n", [14336, 16384])
def test_mw_ascent_extreme_coefficients(n):
    """Largest two- and three-warp shapes with every coefficient at +127 (from x = 0 every step
    flips the next variable in index order: ties everywhere, and Delta climbs to 254 n - 127 =
    4.16e6 at n = 16384, next to the multi-warp key offset 2^22) and at random +-127."""
    rng = np.random.default_rng(13)
    for name in ("plus", "mixed"):
        if name == "plus":
            QQ = np.full((n, n), 127, dtype=np.int32)
        else:
            QQ = np.triu(np.where(rng.random((n, n), dtype=np.float32) < 0.5, -127, 127).astype(np.int32))
            QQ += np.triu(QQ, 1).T
        u = Ubqp(0)
        u.load_Q(QQ, 2)
        X = np.zeros((2, n), np.uint8)
        X[1] = rng.integers(0, 2, size=n)
        u.set_batch(pack_bits(X), 2)
        fo = oracle.eval_batch(QQ, X, nthreads=8)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = np.array([0, 1], np.int32)
        f, fl, b, _ = _run(u, slots, 10 * n, ASCENT_MW)
        Xr, fr, flr = oracle.ascend(QQ, X[slots], fo[slots], 10 * n, nthreads=2)
        assert np.array_equal(f, fr) and np.array_equal(fl, flr), name
        assert np.array_equal(unpack_bits(b, n), Xr), name
        u.close()
        del QQ


def test_mw_ascent_invalid_slots():
    n, K = 3000, 16
    Q = generate_Q(n, 0.5, seed=9)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(1, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = torch.tensor([3, -1, K, 5], dtype=torch.int32, device="cuda")
    u.set_option(OPT_ASCENT, ASCENT_MW)
    f = torch.zeros(4, dtype=torch.int64, device="cuda")
    fl = torch.zeros(4, dtype=torch.int32, device="cuda")
    b = torch.zeros((4, u.W64), dtype=torch.int64, device="cuda")
    u.ascend(slots, 4, 10 * n, f, fl, b)
    torch.cuda.synchronize()
    f, fl, b = f.cpu().numpy(), fl.cpu().numpy(), b.cpu().numpy().view(np.uint64)
    assert fl[1] == -1 and fl[2] == -1 and f[1] == 0 and f[2] == 0
    X0 = oracle.random_solutions(n, 1, K)[[3, 5]]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), 10 * n, nthreads=2)
    assert f[0] == fr[0] and f[3] == fr[1] and fl[0] == flr[0] and fl[3] == flr[1]
    assert np.array_equal(unpack_bits(b[[0, 3]], n), Xr)
    u.close()


hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=int(__import__("os").environ.get("UBQP_HYPO_EXAMPLES", 30)), deadline=None)
@given(n=st.integers(1, 16384), density=st.sampled_from([0.02, 0.3, 1.0]), qmax=st.sampled_from([1, 3, 100, 127]),
       seed=st.integers(0, 2**31 - 1), max_flips=st.sampled_from([0, 1, 17, 10**6]))
def test_mw_ascent_random(n, density, qmax, seed, max_flips):
    """Randomised: the multi-warp kernel word for word against the CTA kernel on a batch and
    against O7 (oracle) on one start, over the two- and three-warp shapes."""
    K = 8
    Q = generate_Q(n, density, -qmax, qmax, seed=seed)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(seed, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(K, dtype=np.int32)
    f, fl, b, key = _run(u, slots, max_flips, ASCENT_MW)
    f2, fl2, b2, key2 = _run(u, slots, max_flips, ASCENT_DENSE)
    assert np.array_equal(f, f2) and np.array_equal(fl, fl2) and np.array_equal(b, b2) and key == key2
    few = slots[:1]
    X0 = oracle.random_solutions(n, seed, K)[few]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), max_flips, nthreads=8)
    assert np.array_equal(f[few], fr) and np.array_equal(fl[few], flr)
    assert np.array_equal(unpack_bits(b[few], n), Xr)
    u.close()
