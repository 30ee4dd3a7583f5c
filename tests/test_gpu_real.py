"""GPU parity of the real-valued Q path (SURVEY §8(a) a4'): int8 limb planes on the tensor
cores, exact integer combine, against the exactly rounded oracle O9.

Tolerance (R3, north_star "within a relative 1e-5 for floating-point Q"):
    |f_gpu - f_ref| <= 1e-5 * max(|f_ref|, s_k),  s_k = sqrt(sum_{i,j in S} Q_ij^2),
and the tighter analytic bound of the 28-bit fixed point (include/ubqp.h):
    |f_gpu - f_ref| <= |S|^2 * 2^-(e+1) + |f_ref| * 2^-52.
"""
import numpy as np
import pytest

import oracle
from inputs import generate_Q, generate_Q_real, pack_bits, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import Ubqp, UbqpError, ubqp_stats_real  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402

build_lib()


def _check(Q, X, f, e):
    Q = np.asarray(Q, dtype=np.float64)
    for k in range(X.shape[0]):
        S = np.flatnonzero(X[k])
        ref = oracle.xQx_real(Q, X[k])
        sk = float(np.sqrt((Q[np.ix_(S, S)] ** 2).sum())) if S.size else 0.0
        err = abs(f[k] - ref)
        assert err <= 1e-5 * max(abs(ref), sk), (k, f[k], ref)
        assert err <= S.size ** 2 * 2.0 ** (-(e + 1)) + abs(ref) * 2.0 ** -52 + 1e-300, (k, err)


@pytest.mark.parametrize("n", [1, 3, 65, 300, 1100, 2500])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_eval_real(n, dtype):
    Q = generate_Q_real(n, 0.7, seed=n, dtype=dtype)
    K = 40 if n >= 1100 else 150
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(n + 1, K)
    f = np.zeros(K, np.float64)
    st = ubqp_stats_real()
    u.eval_batch_real(f, st)
    X = oracle.random_solutions(n, n + 1, K)
    _check(Q, X, f, u.real_exp)
    # integer-image stats are exact: sum of f * 2^e equals the int128 sum
    fint = [int(round(v * 2.0 ** u.real_exp)) for v in f]
    assert st.count == K and st.sum_fint == sum(fint) and st.max_fint == max(fint)


def test_real_equals_integer_path_on_integer_Q():
    n, K = 500, 300
    Q = generate_Q(n, 0.5, seed=12)
    u = Ubqp(0)
    u.load_Q_real(Q.astype(np.float64), K)
    u.random(3, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    assert np.array_equal(f, oracle.eval_batch(Q, oracle.random_solutions(n, 3, K), nthreads=8).astype(np.float64))


def test_real_screen_and_first_derivative():
    n, K = 400, 2000
    Q = generate_Q_real(n, 0.5, seed=4)
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    b = np.zeros(u.W64, np.uint64)
    u.first_derivative(b)
    assert np.array_equal(unpack_bits(b, n)[0], oracle.first_derivative_start_real(Q))
    u.diversify(b, 0, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    mean, mx = float(f.mean()), float(f.max())
    surv = np.zeros(K, np.int32)
    for lam in (0.0, 0.5, 0.9):
        m, T = u.screen_real(lam, mean, mx, surv)
        assert T == mean + lam * (mx - mean)
        assert surv[:m].tolist() == np.flatnonzero(f > T).tolist()


def test_real_errors():
    u = Ubqp(0)
    with pytest.raises(UbqpError) as e:
        u.load_Q_real(np.array([[1.0, 2.0], [2.5, 1.0]]), 4)
    assert e.value.code == 2
    with pytest.raises(UbqpError) as e:
        u.load_Q_real(np.array([[np.nan]]), 4)
    assert e.value.code == 3
    u.load_Q_real(np.array([[1.5]]), 4)
    u.random(0, 1)
    with pytest.raises(UbqpError) as e:
        u.eval_batch(0)                       # integer-only entry point
    assert e.value.code == 4
    f = np.zeros(1)
    u.eval_batch_real(f)
    assert f[0] in (0.0, 1.5)


@pytest.mark.parametrize("n", [7000])
def test_real_full_size_sampled(n):
    Q = generate_Q_real(n, 1.0, seed=4, dtype=np.float32)
    K = 4096
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(4, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    idx = np.array([0, 1, 777, K - 1])
    X = oracle.random_solutions(n, 4, K)[idx]
    _check(Q, X, f[idx], u.real_exp)


@pytest.mark.parametrize("n", [1, 2, 65, 300, 1100, 2500])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ascend_real_matches_oracle(n, dtype):
    """R20: the real-Q walk on the fixed-point image is bit-exact against the oracle's walk
    on its own image (x, flips, f~), f = 2^-e f~ exactly, and f is within R3 of fsum."""
    Q = generate_Q_real(n, 0.7, seed=100 + n, dtype=dtype)
    K = 24 if n >= 1100 else 96
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(n + 5, K)
    u.eval_batch_real()
    X0 = oracle.random_solutions(n, n + 5, K)
    slots = np.arange(K, dtype=np.int32)[::-1].copy()
    f = np.zeros(K, np.float64)
    fi = np.zeros(K, np.int64)
    fl = np.zeros(K, np.int32)
    b = np.zeros((K, u.W64), np.uint64)
    u.ascend_real(slots, K, 10 * n, f, fi, fl, b)
    Xa, fa, ff, ofl, e = oracle.ascend_real(Q.astype(np.float64), X0[slots], 10 * n, nthreads=8)
    assert e == u.real_exp
    assert np.array_equal(unpack_bits(b, n), Xa) and np.array_equal(fl, ofl) and np.array_equal(fi, fa)
    assert np.array_equal(f, ff)
    _check(Q, Xa, f, e)


def test_ascend_real_integer_Q_equals_integer_ascent_and_device_outputs():
    n, K = 700, 200
    Q = generate_Q(n, 0.5, seed=13)
    Q[0, 0] = 100
    ui = Ubqp(0)
    ui.load_Q(Q, K)
    ui.random(4, K)
    ui.eval_batch(1)
    fo = np.zeros(K, np.int64)
    flo = np.zeros(K, np.int32)
    bo = np.zeros((K, ui.W64), np.uint64)
    ui.ascend(np.arange(K, dtype=np.int32), K, 10 * n, fo, flo, bo)
    ur = Ubqp(0)
    ur.load_Q_real(Q.astype(np.float64), K)
    ur.random(4, K)
    ur.eval_batch_real()
    assert ur.real_exp == 20
    sl = torch.arange(K, dtype=torch.int32, device="cuda")
    f = torch.zeros(K, dtype=torch.float64, device="cuda")
    fi = torch.zeros(K, dtype=torch.int64, device="cuda")
    fl = torch.zeros(K, dtype=torch.int32, device="cuda")
    b = torch.zeros((K, ur.W64), dtype=torch.int64, device="cuda")
    ur.ascend_real(sl, K, 10 * n, f, fi, fl, b)
    torch.cuda.synchronize()
    assert np.array_equal(fl.cpu().numpy(), flo) and np.array_equal(b.cpu().numpy().view(np.uint64), bo)
    assert np.array_equal(fi.cpu().numpy(), fo * 2**20) and np.array_equal(f.cpu().numpy(), fo.astype(np.float64))


def test_ascend_real_errors():
    u = Ubqp(0)
    Q = generate_Q(50, 0.5, seed=1)
    u.load_Q(Q, 8)
    u.random(1, 8)
    u.eval_batch(0)
    with pytest.raises(UbqpError):                  # integer Q loaded
        u.ascend_real(np.arange(8, dtype=np.int32), 8, 100)
    ur = Ubqp(0)
    ur.load_Q_real(Q.astype(np.float64), 8)
    ur.random(1, 8)
    with pytest.raises(UbqpError):                  # not evaluated yet
        ur.ascend_real(np.arange(8, dtype=np.int32), 8, 100)
    ur.eval_batch_real()
    with pytest.raises(UbqpError):
        ur.ascend_real(np.array([0, 8], np.int32), 2, 100)


def test_real_top_limb_at_64():
    """Regression: max|Q| just below a power of two puts |rint(Q 2^e)| above the balanced
    4-digit range (63 * (1 + 128 + 128^2 + 128^3)); the top limb must then hold 64."""
    Q = np.array([[0.999, -0.5, 0.25], [-0.5, -0.9999, 0.125], [0.25, 0.125, 0.75]])
    K = 8
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    assert u.real_exp == 27
    X = np.array([[1, 1, 1], [1, 0, 0], [0, 1, 0], [1, 0, 1], [0, 1, 1], [1, 1, 0], [0, 0, 1], [0, 0, 0]], np.uint8)
    u.set_batch(pack_bits(X), K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    Qt, e = oracle.real_image(Q)
    ft = oracle.eval_batch(Qt.astype(np.int32), X)
    assert np.array_equal(f, np.ldexp(ft.astype(np.float64), -e))
    fi = np.zeros(K, np.int64)
    u.ascend_real(np.arange(K, dtype=np.int32), K, 100, None, fi)
    Xa, fa, _, _, _ = oracle.ascend_real(Q, X, 100)
    assert np.array_equal(fi, fa)


@pytest.mark.parametrize("n,K,rounds,lam", [(60, 400, 3, 0.4), (500, 2000, 3, 0.3)])
def test_multistart_real_matches_oracle(n, K, rounds, lam):
    """Figure-2 rounds on a real Q (R20) against oracle.run_rounds_real: trajectory of exact
    f~ values and the final solution."""
    from paper_1706_00037_b200.multistart import MultiStartReal
    rng = np.random.default_rng(n)
    A = rng.uniform(-50, 50, size=(n, n))
    Q = np.triu(A) + np.triu(A, 1).T
    ms = MultiStartReal(Q, K, lam=lam, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=5)
    ob, ox, otraj, e = oracle.run_rounds_real(Q, K, rounds, lam, 10 * n, sample_seed=5, nthreads=8)
    assert ms.e == e and best == ob and traj == otraj
    assert np.array_equal(unpack_bits(bits.cpu().numpy().view(np.uint64)[None, :], n)[0], ox)
