"""GPU parity of the sparse-row ascent (Beasley-shaped "linear and
quadratic density = 0.1" instances) against the oracle's steepest ascent O7, bit for bit
(final x, f, flips, best key), and against the dense register ascent on the same inputs.
Densities 0.02..0.2, n up to 7000, ragged n (segments of 32 variables), max_flips limits."""
import numpy as np
import pytest

import oracle
from inputs import generate_Q, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, UbqpError  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402
from paper_1706_00037_b200.ubqp import (ASCENT_AUTO, ASCENT_DENSE, ASCENT_SPARSE, OPT_ASCENT,  # noqa: E402
                                        Q_NNZ, Q_SPARSE_ROWS)

build_lib()


def _run(u, slots, m, max_flips, W64):
    f = np.zeros(m, np.int64)
    fl = np.zeros(m, np.int32)
    b = np.zeros((m, W64), np.uint64)
    key = np.zeros(1, np.int64)
    u.ascend(slots, m, max_flips, f, fl, b, key)
    return f, fl, b, key[0]


@pytest.mark.parametrize("n,density", [(2, 0.2), (31, 0.2), (33, 0.1), (64, 0.1), (65, 0.05), (500, 0.05),
                                       (500, 0.1), (500, 0.2), (1111, 0.1), (2500, 0.1), (2500, 0.02), (7000, 0.1)])
@pytest.mark.parametrize("max_flips", [0, 5, 10**6])
def test_sparse_ascent_matches_oracle(n, density, max_flips):
    Q = generate_Q(n, density, seed=200 + n)
    K = 40 if n >= 2500 else 160
    u = Ubqp(0)
    u.load_Q(Q, K)
    assert u.query(Q_SPARSE_ROWS) == 1
    assert u.query(Q_NNZ) == int(np.count_nonzero(Q) - np.count_nonzero(np.diag(Q)))
    u.set_option(OPT_ASCENT, ASCENT_SPARSE)
    u.random(n + 3, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(0, K, 2, dtype=np.int32)[::-1].copy()
    m = len(slots)
    f, fl, b, key = _run(u, slots, m, max_flips, u.W64)
    X0 = oracle.random_solutions(n, n + 3, K)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), max_flips, nthreads=8)
    assert np.array_equal(unpack_bits(b, n), Xr)
    assert np.array_equal(f, fr) and np.array_equal(fl, flr)
    assert key == max(oracle.max_key(int(fr[i]), int(slots[i])) for i in range(m))
    # the dense register kernel walks the same path
    u.set_option(OPT_ASCENT, ASCENT_DENSE)
    f2, fl2, b2, key2 = _run(u, slots, m, max_flips, u.W64)
    assert np.array_equal(f2, f) and np.array_equal(fl2, fl) and np.array_equal(b2, b) and key2 == key


def test_sparse_ascent_all_coefficients_extreme():
    """every nonzero at +-127 (the int8 range) and ties everywhere: lowest-index argmax"""
    n, K = 900, 64
    rng = np.random.default_rng(5)
    Q = generate_Q(n, 0.1, seed=9)
    Q = (np.sign(Q) * 127).astype(np.int32)
    Q[rng.integers(0, n, 20), rng.integers(0, n, 20)] = 0
    Q = np.triu(Q) + np.triu(Q, 1).T
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.set_option(OPT_ASCENT, ASCENT_SPARSE)
    u.random(1, K)
    u.eval_batch(0)                                    # gains formed by the ascent call
    slots = np.arange(K, dtype=np.int32)
    f, fl, b, key = _run(u, slots, K, 10 * n, u.W64)
    X0 = oracle.random_solutions(n, 1, K)
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=8), 10 * n, nthreads=8)
    assert np.array_equal(unpack_bits(b, n), Xr) and np.array_equal(f, fr) and np.array_equal(fl, flr)


def test_sparse_selection_and_errors():
    n, K = 600, 16
    dense = generate_Q(n, 1.0, seed=1)
    u = Ubqp(0)
    u.load_Q(dense, K)
    assert u.query(Q_SPARSE_ROWS) == 0                 # density > 0.25: no CSR rows
    u.set_option(OPT_ASCENT, ASCENT_SPARSE)
    u.random(2, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    with pytest.raises(UbqpError) as e:
        u.ascend(np.arange(K, dtype=np.int32), K, 100)
    assert e.value.code == 4
    with pytest.raises(UbqpError) as e:
        u.set_option(OPT_ASCENT, 5)
    assert e.value.code == 1
    # automatic selection gives the same results either way
    sp = generate_Q(n, 0.1, seed=2)
    u.load_Q(sp, K)
    u.set_option(OPT_ASCENT, ASCENT_AUTO)
    u.random(3, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    r_auto = _run(u, np.arange(K, dtype=np.int32), K, 10 * n, u.W64)
    u.set_option(OPT_ASCENT, ASCENT_DENSE)
    r_dense = _run(u, np.arange(K, dtype=np.int32), K, 10 * n, u.W64)
    assert all(np.array_equal(a, b) for a, b in zip(r_auto[:3], r_dense[:3])) and r_auto[3] == r_dense[3]


def test_sparse_invalid_device_slot_reports_minus_one():
    n, K = 300, 8
    Q = generate_Q(n, 0.1, seed=3)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.set_option(OPT_ASCENT, ASCENT_SPARSE)
    u.random(2, K)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = torch.tensor([0, 99, 3], dtype=torch.int32, device="cuda")
    fl = torch.zeros(3, dtype=torch.int32, device="cuda")
    u.ascend(slots, 3, 100, None, fl)
    torch.cuda.synchronize()
    assert fl[1].item() == -1 and fl[0].item() >= 0 and fl[2].item() >= 0
