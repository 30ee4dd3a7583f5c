"""Randomised GPU parity (hypothesis): arbitrary sizes, densities, coefficient ranges, seeds,
lambda and max_flips; every output of eval / screen / ascent must equal the oracle exactly.
UBQP_HYPO_EXAMPLES=N raises the example count of every test, UBQP_HYPO_NMAX the largest n
(long soak runs over every ascent shape)."""
import os

import numpy as np
import pytest

import oracle
from inputs import generate_Q, pack_bits, unpack_bits

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import given, settings, strategies as st  # noqa: E402

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, ubqp_stats  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402

build_lib()


@settings(max_examples=int(os.environ.get("UBQP_HYPO_EXAMPLES", 120)), deadline=None)
@given(n=st.integers(1, int(os.environ.get("UBQP_HYPO_NMAX", 700))), K=st.integers(1, 700), density=st.sampled_from([0.05, 0.3, 1.0]),
       qmax=st.sampled_from([1, 7, 100, 127]), seed=st.integers(0, 2**31 - 1),
       lam=st.floats(-0.5, 1.5), max_flips=st.sampled_from([0, 1, 5, 10**6]),
       glover=st.booleans())
def test_round_matches_oracle(n, K, density, qmax, seed, lam, max_flips, glover):
    Q = generate_Q(n, density, -qmax, qmax, seed=seed)
    u = Ubqp(0)
    u.load_Q(Q, K)
    if glover:
        x0 = oracle.first_derivative_start(Q)
        u.diversify(pack_bits(x0)[0], seed % (n * (n + 1)), K)
        X = oracle.diversify(x0, seed % (n * (n + 1)), K)
    else:
        u.random(seed, K)
        X = oracle.random_solutions(n, seed, K)
    f = np.zeros(K, np.int64)
    stt = ubqp_stats()
    u.eval_batch(UBQP_EMIT_GAINS if seed & 1 else 0, f, stt)
    fo = oracle.eval_batch(Q, X, nthreads=8)
    assert np.array_equal(f, fo)
    so = oracle.stats(fo)
    assert (stt.sum, stt.count, stt.max_key) == (int(so[0]), int(so[1]), int(so[2]))
    maxv = (stt.max_key >> 22) - (1 << 40)
    surv = np.zeros(K, np.int32)
    m, T = u.screen(lam, stt.sum, stt.count, maxv, surv)
    To = oracle.threshold(lam, stt.sum, stt.count, maxv)
    assert T == To
    s = oracle.screen(fo, To)
    assert np.array_equal(surv[:m], s)
    if m:
        fa = np.zeros(m, np.int64)
        fl = np.zeros(m, np.int32)
        ba = np.zeros((m, u.W64), np.uint64)
        key = np.zeros(1, np.int64)
        u.ascend(surv[:m].copy(), m, max_flips, fa, fl, ba, key)
        Xr, fr, flr = oracle.ascend(Q, X[s], fo[s], max_flips, nthreads=8)
        assert np.array_equal(fa, fr) and np.array_equal(fl, flr)
        assert np.array_equal(unpack_bits(ba, n), Xr)
        assert key[0] == max(oracle.max_key(int(fr[i]), int(s[i])) for i in range(m))
    u.close()


@settings(max_examples=int(os.environ.get("UBQP_HYPO_EXAMPLES", 60)), deadline=None)
@given(n=st.integers(1, int(os.environ.get("UBQP_HYPO_NMAX", 600))), K=st.integers(1, 300), P=st.integers(1, 9), qmax=st.sampled_from([1, 50, 127]),
       seed=st.integers(0, 2**31 - 1), t0=st.integers(0, 10**6))
def test_blend_and_relink_match_oracle(n, K, P, qmax, seed, t0):
    """O4b blend bits and O11 relinking outputs on arbitrary shapes (R11b, R19)."""
    Q = generate_Q(n, 0.5, -qmax, qmax, seed=seed)
    rng = np.random.default_rng(seed)
    s0 = rng.integers(0, 2, size=n).astype(np.uint8)
    par = rng.integers(0, 2, size=(P, n)).astype(np.uint8)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.blend(pack_bits(s0)[0], pack_bits(par), P, t0, K)
    B = np.zeros((K, u.W64), np.uint64)
    u.get_batch(B)
    X = oracle.blend(s0, par, t0, K)
    assert np.array_equal(unpack_bits(B, n), X)
    f0 = np.zeros(K, np.int64)
    u.eval_batch(UBQP_EMIT_GAINS, f0)
    f = np.zeros(K, np.int64)
    stp = np.zeros(K, np.int32)
    ln = np.zeros(K, np.int32)
    b = np.zeros((K, u.W64), np.uint64)
    u.relink(pack_bits(par), P, np.arange(K, dtype=np.int32), K, f, stp, ln, b)
    ob, of, os_, ol = oracle.relink(Q, X, f0, par, nthreads=8)
    assert np.array_equal(ln, ol) and np.array_equal(stp, os_) and np.array_equal(f, of)
    assert np.array_equal(unpack_bits(b, n), ob)
    u.close()


@settings(max_examples=int(os.environ.get("UBQP_HYPO_EXAMPLES", 40)), deadline=None)
@given(n=st.integers(1, int(os.environ.get("UBQP_HYPO_NMAX", 500))), K=st.integers(1, 120), scale=st.sampled_from([1e-3, 1.0, 37.5, 1e6]),
       seed=st.integers(0, 2**31 - 1), f32=st.booleans(), max_flips=st.sampled_from([0, 3, 10**6]))
def test_real_ascent_matches_oracle(n, K, scale, seed, f32, max_flips):
    """R20 real-Q ascent on arbitrary shapes and coefficient scales."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-scale, scale, size=(n, n))
    Q = np.triu(A) + np.triu(A, 1).T
    if f32:
        Q = Q.astype(np.float32)
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(seed, K)
    u.eval_batch_real()
    fi = np.zeros(K, np.int64)
    fl = np.zeros(K, np.int32)
    b = np.zeros((K, u.W64), np.uint64)
    u.ascend_real(np.arange(K, dtype=np.int32), K, max_flips, None, fi, fl, b)
    Xa, fa, ff, ofl, e = oracle.ascend_real(Q.astype(np.float64), oracle.random_solutions(n, seed, K), max_flips,
                                            nthreads=8)
    assert e == u.real_exp
    assert np.array_equal(fi, fa) and np.array_equal(fl, ofl) and np.array_equal(unpack_bits(b, n), Xa)
    u.close()
