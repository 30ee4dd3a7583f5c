"""GPU parity of the real-valued Q path (SURVEY §8(a) a4'; readings R3, R20, R22).

Evaluation (R22): the evaluation image is exact for float32 Q, so f must equal the exactly
rounded oracle O9 (math.fsum) BIT FOR BIT; for float64 Q every coefficient is within 2^-32 of
itself, so (include/ubqp.h)
    |f_gpu - x^t Q x| <= 2^-32 sum_{i,j in S} |Q_ij| + 2^-53 |x^t Q x|
and in particular the north_star tolerance (R3)
    |f_gpu - f_ref| <= 1e-5 * max(|f_ref|, s_k),  s_k = sqrt(sum_{i,j in S} Q_ij^2).
The adversarial cases of the round-1 review (correlated rounding: a two-valued float64 Q, a
wide-range float32 Q, a wide-range float64 Q) are included.

Ascent (R20): the walk on the 28-bit walk image is bit-exact against the oracle's walk O9b
(bits, flips, f~); independently of any image, every returned x is a 1-flip local optimum of
the REAL Q up to the walk image's quantisation, (2|S| + 1) 2^-(e+1), by the oracle's exact
real gains (gains_real), and its reported f obeys the evaluation bound above.
"""
import math

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


def _check(Q, X, f, exact=False):
    """R3 and the R22 bound for every row; exact=True (float32 Q): f == fsum bit for bit."""
    Q = np.asarray(Q, dtype=np.float64)
    for k in range(X.shape[0]):
        S = np.flatnonzero(X[k])
        ref = oracle.xQx_real(Q, X[k])
        if exact:
            assert f[k] == ref, (k, f[k], ref)
            continue
        sub = Q[np.ix_(S, S)]
        sk = float(np.sqrt((sub ** 2).sum())) if S.size else 0.0
        err = abs(f[k] - ref)
        assert err <= 1e-5 * max(abs(ref), sk), (k, f[k], ref, sk)
        assert err <= 2.0 ** -32 * math.fsum(np.abs(sub).ravel().tolist()) + 2.0 ** -52 * abs(ref) + 1e-300, (k, err)


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
    _check(Q, X, f, exact=dtype == np.float32)
    assert st.count == K and st.exp == u.eval_exp and 1 <= u.eval_limbs <= 10
    if dtype == np.float32:
        # the int128 statistics are exact: sum f~ = 2^w * (exact rational batch sum), max likewise
        from fractions import Fraction
        tot = oracle.batch_sum_exact(Q, X) * (Fraction(2) ** st.exp)
        assert tot.denominator == 1 and st.sum_fint == tot.numerator
        assert math.ldexp(float(st.max_fint), -st.exp) == max(f)


def test_real_equals_integer_path_on_integer_Q():
    n, K = 500, 300
    Q = generate_Q(n, 0.5, seed=12)
    u = Ubqp(0)
    u.load_Q_real(Q.astype(np.float64), K)
    assert u.eval_exp == 0 and u.eval_limbs == 1          # integers |q| <= 100: one exact plane
    u.random(3, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    assert np.array_equal(f, oracle.eval_batch(Q, oracle.random_solutions(n, 3, K), nthreads=8).astype(np.float64))


def _two_valued(n, seed):
    """float64 entries in {+0.3, -0.7} with P(+0.3) = 0.7: zero mean, every entry rounded the
    same way in any fixed point (correlated rounding errors)"""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n)
    v = np.where(rng.random(iu.size) < 0.7, 0.3, -0.7)
    Q = np.zeros((n, n))
    Q[iu, ju] = v
    Q[ju, iu] = v
    return Q


def _wide_range(n, seed, dtype):
    """one coefficient 100, the rest (m + 1/2) 2^-20 with |.| < 8: 28 bits cannot hold both"""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n)
    m = rng.integers(-8 * 2**20, 8 * 2**20 - 1, size=iu.size)
    v = (m.astype(np.float64) + 0.5) * 2.0 ** -20
    Q = np.zeros((n, n))
    Q[iu, ju] = v
    Q[ju, iu] = v
    Q[0, 0] = 100.0
    return Q.astype(dtype)


@pytest.mark.parametrize("case", ["two_valued_f64_n7000", "wide_range_f32_n7000", "wide_range_f64_n1000"])
def test_eval_real_adversarial_rounding(case):
    """The inputs that broke the 28-bit image of round 1 (2.3x, 35.7x and 4.8x the R3 bound)."""
    if case == "two_valued_f64_n7000":
        n, Q, exact = 7000, _two_valued(7000, 1), False
    elif case == "wide_range_f32_n7000":
        n, Q, exact = 7000, _wide_range(7000, 2, np.float32), True
    else:
        n, Q, exact = 1000, _wide_range(1000, 3, np.float64), True   # (m + 1/2) 2^-20 is exact in binary64
    K = 256
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(11, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    X = oracle.random_solutions(n, 11, K)
    idx = np.array([0, 1, 100, 129, 200, K - 1])
    _check(Q, X[idx], f[idx], exact=exact)
    if case.startswith("wide"):
        assert u.eval_exp == 21                             # lsb 2^-21 of (m + 1/2) 2^-20


def test_eval_real_rejects_excess_dynamic_range():
    u = Ubqp(0)
    with pytest.raises(UbqpError) as e:
        u.load_Q_real(np.array([[1e30, 1e-30], [1e-30, 1.0]]), 4)
    assert e.value.code == 3
    with pytest.raises(UbqpError) as e:
        u.load_Q_real(np.array([[2.0 ** 100, 0.0], [0.0, 2.0 ** -100]], np.float32), 4)
    assert e.value.code == 3
    # the widest accepted range: |V| <= 126 * 128^9 with 32 significant bits
    u.load_Q_real(np.array([[2.0 ** 30, 0.0], [0.0, 2.0 ** -8]]), 4)
    assert u.eval_limbs <= 10


def test_real_screen_and_first_derivative():
    n, K = 400, 2000
    Q = generate_Q_real(n, 0.5, seed=4, dtype=np.float32)
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


def test_real_full_size_sampled():
    n = 7000
    Q = generate_Q_real(n, 1.0, seed=4, dtype=np.float32)
    K = 4096
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(4, K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    idx = np.array([0, 1, 255, 256, 777, 2048 + 129, K - 1])
    X = oracle.random_solutions(n, 4, K)[idx]
    _check(Q, X, f[idx], exact=True)


def _local_opt_real(Q, X, flips, max_flips, e):
    """every x not stopped by max_flips: all exact real gains <= (2|S| + 1) 2^-(e+1)"""
    for x, fl in zip(X, flips):
        if fl == max_flips:
            continue
        g = oracle.gains_real(Q, x)
        tol = (2 * int(x.sum()) + 1) * 2.0 ** -(e + 1)
        assert g.max() <= tol, (g.max(), tol)


@pytest.mark.parametrize("n", [1, 2, 65, 300, 1100, 2500])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ascend_real_matches_oracle(n, dtype):
    """R20 walk bit-exact against O9b (x, flips, f~); f on the evaluation image vs O9; local
    optimality of the real Q by exact gains."""
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
    Xa, fa, _, ofl, e = oracle.ascend_real(Q.astype(np.float64), X0[slots], 10 * n, nthreads=8)
    assert e == u.real_exp
    assert np.array_equal(unpack_bits(b, n), Xa) and np.array_equal(fl, ofl) and np.array_equal(fi, fa)
    _check(Q, Xa, f, exact=dtype == np.float32)
    sel = slice(None) if n <= 300 else slice(0, 4)
    _local_opt_real(np.asarray(Q, np.float64), Xa[sel], fl[sel], 10 * n, e)


@pytest.mark.parametrize("case", ["two_valued_f64", "wide_range_f32"])
def test_ascend_real_adversarial_local_optimality(case):
    n = 600
    Q = _two_valued(n, 7) if case == "two_valued_f64" else _wide_range(n, 8, np.float32)
    K = 32
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    u.random(9, K)
    u.eval_batch_real()
    f = np.zeros(K, np.float64)
    fl = np.zeros(K, np.int32)
    b = np.zeros((K, u.W64), np.uint64)
    u.ascend_real(np.arange(K, dtype=np.int32), K, 10 * n, f, None, fl, b)
    X = unpack_bits(b, n)
    _check(Q, X, f, exact=case == "wide_range_f32")
    _local_opt_real(np.asarray(Q, np.float64), X[:8], fl[:8], 10 * n, u.real_exp)


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
    4-digit range of the walk image (63 * (1 + 128 + 128^2 + 128^3)); the top limb holds 64."""
    Q = np.array([[0.999, -0.5, 0.25], [-0.5, -0.9999, 0.125], [0.25, 0.125, 0.75]])
    K = 8
    u = Ubqp(0)
    u.load_Q_real(Q, K)
    assert u.real_exp == 27
    X = np.array([[1, 1, 1], [1, 0, 0], [0, 1, 0], [1, 0, 1], [0, 1, 1], [1, 1, 0], [0, 0, 1], [0, 0, 0]], np.uint8)
    u.set_batch(pack_bits(X), K)
    f = np.zeros(K, np.float64)
    u.eval_batch_real(f)
    _check(Q, X, f)
    fi = np.zeros(K, np.int64)
    u.ascend_real(np.arange(K, dtype=np.int32), K, 100, None, fi)
    Xa, fa, _, _, _ = oracle.ascend_real(Q, X, 100)
    assert np.array_equal(fi, fa)


@pytest.mark.parametrize("n,K,rounds,lam", [(60, 400, 3, 0.4), (300, 800, 3, 0.3)])
def test_multistart_real_matches_oracle(n, K, rounds, lam):
    """Figure-2 rounds on a float32-valued real Q against oracle.run_rounds_real: the values
    are exactly rounded on both sides, so trajectory and final solution agree exactly."""
    from paper_1706_00037_b200.multistart import MultiStartReal
    rng = np.random.default_rng(n)
    A = rng.uniform(-50, 50, size=(n, n)).astype(np.float32)
    Q = (np.triu(A) + np.triu(A, 1).T).astype(np.float64)
    ms = MultiStartReal(Q, K, lam=lam, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=5)
    ob, ox, otraj, e = oracle.run_rounds_real(Q, K, rounds, lam, 10 * n, sample_seed=5, nthreads=8)
    assert ms.e == e and best == ob and traj == otraj
    assert np.array_equal(unpack_bits(bits.cpu().numpy().view(np.uint64)[None, :], n)[0], ox)
