"""Randomised GPU parity (hypothesis): arbitrary sizes, densities, coefficient ranges, seeds,
lambda and max_flips; every output of eval / screen / ascent must equal the oracle exactly."""
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


@settings(max_examples=120, deadline=None)
@given(n=st.integers(1, 700), K=st.integers(1, 700), density=st.sampled_from([0.05, 0.3, 1.0]),
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
