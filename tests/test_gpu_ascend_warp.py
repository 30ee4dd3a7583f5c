"""GPU parity of the warp-per-solution steepest ascent (ascend_warp.cu, UBQP_OPT_ASCENT = 3)
against the oracle's O7 (plain C steepest ascent, lowest index on ties) and
against the CTA kernel (UBQP_OPT_ASCENT = 1), exactly: final bits, f, flip counts, best key.

Sizes cross the kernel's 512-variable chunk (16 per lane), the 64-bit word and the largest
register shape (n_pad = 7168, 14 chunks); coefficients at +-127 at n = 7168 put |Delta| at
254 n - 127 = 1.82e6, next to the key offset 2^21 of the sign-folded keys.
"""
import numpy as np
import pytest

import oracle
from inputs import generate_Q, pack_bits, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, UbqpError  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402
from paper_1706_00037_b200.ubqp import (ASCENT_AUTO, ASCENT_DENSE, ASCENT_WARP, OPT_ASCENT,  # noqa: E402
                                        Q_ASCENT_LAST)

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


@pytest.mark.parametrize("n", [1, 2, 3, 16, 17, 31, 33, 64, 100, 255, 511, 512, 513, 1023, 1025,
                               1536, 2500, 3583, 3584, 4097, 5000, 6656, 6657, 7000, 7168])
def test_warp_ascent_matches_oracle(n):
    dens = 1.0 if n >= 2500 else 0.6
    Q = generate_Q(n, dens, seed=101 + n)
    K = 24 if n >= 2500 else 96
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(7 + n, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(K, dtype=np.int32)[::-1].copy()
    f, fl, b, key = _run(u, slots, 10 * n, ASCENT_WARP)
    assert u.query(Q_ASCENT_LAST) == ASCENT_WARP
    X0 = oracle.random_solutions(n, 7 + n, K)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), 10 * n, nthreads=8)
    assert np.array_equal(f, fr)
    assert np.array_equal(fl, flr)
    assert np.array_equal(unpack_bits(b, n), Xr)
    assert key == max(oracle.max_key(int(fr[i]), int(slots[i])) for i in range(K))
    # the CTA kernel agrees word for word (padding bits included)
    f2, fl2, b2, key2 = _run(u, slots, 10 * n, ASCENT_DENSE)
    assert u.query(Q_ASCENT_LAST) == ASCENT_DENSE
    _run(u, slots[:1], 1, ASCENT_AUTO)                # automatic: include/ubqp.h UBQP_OPT_ASCENT
    n_pad = -(-n // 128) * 128
    nch = -(-n_pad // 512)
    assert u.query(Q_ASCENT_LAST) == (ASCENT_WARP if n_pad <= 7168 and (nch >= 8 or nch in (4, 6)) else ASCENT_DENSE)
    assert np.array_equal(f, f2) and np.array_equal(fl, fl2) and np.array_equal(b, b2) and key == key2
    u.close()


@pytest.mark.parametrize("max_flips", [0, 1, 2, 7, 50])
def test_warp_ascent_flip_limit(max_flips):
    n, K = 1100, 64
    Q = generate_Q(n, 0.8, seed=5)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(3, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(0, K, 2, dtype=np.int32)
    f, fl, b, _ = _run(u, slots, max_flips, ASCENT_WARP)
    X0 = oracle.random_solutions(n, 3, K)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0), max_flips, nthreads=8)
    assert np.array_equal(f, fr) and np.array_equal(fl, flr)
    assert np.array_equal(unpack_bits(b, n), Xr)
    u.close()


def test_warp_ascent_extreme_coefficients():
    """n = 7168 (the largest warp shape, no padding) with every coefficient at +-127 and with
    all +127 (the ascent from x = 0 flips every variable)."""
    n = 7168
    rng = np.random.default_rng(11)
    sign = np.where(rng.random((n, n)) < 0.5, -1, 1).astype(np.int32)
    Qm = 127 * np.triu(sign)
    Qm = Qm + np.triu(Qm, 1).T
    Qp = np.full((n, n), 127, dtype=np.int32)
    for QQ, name in ((Qp, "plus"), (Qm, "mixed")):
        u = Ubqp(0)
        u.load_Q(QQ, 3)
        X = np.zeros((3, n), np.uint8)
        X[1] = 1
        X[2] = rng.integers(0, 2, size=n)
        u.set_batch(pack_bits(X), 3)
        fo = oracle.eval_batch(QQ, X, nthreads=8)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = np.array([0, 2], np.int32)
        f, fl, b, _ = _run(u, slots, 10 * n, ASCENT_WARP)
        Xr, fr, flr = oracle.ascend(QQ, X[slots], fo[slots], 10 * n, nthreads=2)
        assert np.array_equal(f, fr) and np.array_equal(fl, flr), name
        assert np.array_equal(unpack_bits(b, n), Xr), name
        u.close()


def test_warp_ascent_invalid_slots_and_range():
    n, K = 600, 16
    Q = generate_Q(n, 0.5, seed=9)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(1, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    # invalid slots are reachable only through a device slot array (host arrays are validated)
    slots = torch.tensor([3, -1, K, 5], dtype=torch.int32, device="cuda")
    u.set_option(OPT_ASCENT, ASCENT_WARP)
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
    # n_pad > 7168: the warp kernel is out of range (E_RANGE); automatic selection uses the multi-warp kernel
    n = 7169
    Q = generate_Q(n, 0.01, seed=1)
    u = Ubqp(0)
    u.load_Q(Q, 2)
    u.random(1, 2)
    u.eval_batch(UBQP_EMIT_GAINS)
    u.set_option(OPT_ASCENT, ASCENT_WARP)
    with pytest.raises(UbqpError) as e:
        u.ascend(np.arange(2, dtype=np.int32), 2, 10)
    assert e.value.code == 3
    u.set_option(OPT_ASCENT, ASCENT_AUTO)
    u.ascend(np.arange(2, dtype=np.int32), 2, 10)
    assert u.query(Q_ASCENT_LAST) == 4
    u.close()


hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=int(__import__("os").environ.get("UBQP_HYPO_EXAMPLES", 40)), deadline=None)
@given(n=st.integers(1, 7168), density=st.sampled_from([0.02, 0.3, 1.0]), qmax=st.sampled_from([1, 3, 100, 127]),
       seed=st.integers(0, 2**31 - 1), max_flips=st.sampled_from([0, 1, 17, 10**6]))
def test_warp_ascent_random(n, density, qmax, seed, max_flips):
    """Randomised: the warp kernel against O7 (oracle) on a few starts, and word for word
    against the CTA kernel on the whole batch, over every chunk count NCH = 1..14."""
    K = 12
    Q = generate_Q(n, density, -qmax, qmax, seed=seed)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(seed, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(K, dtype=np.int32)
    f, fl, b, key = _run(u, slots, max_flips, ASCENT_WARP)
    f2, fl2, b2, key2 = _run(u, slots, max_flips, ASCENT_DENSE)
    assert np.array_equal(f, f2) and np.array_equal(fl, fl2) and np.array_equal(b, b2) and key == key2
    few = slots[:3] if n > 3000 else slots
    X0 = oracle.random_solutions(n, seed, K)[few]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), max_flips, nthreads=8)
    assert np.array_equal(f[few], fr) and np.array_equal(fl[few], flr)
    assert np.array_equal(unpack_bits(b[few], n), Xr)
    u.close()
