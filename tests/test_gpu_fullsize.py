"""Full-size parity at the bench configuration (config 4: n = 7000 dense, K = 262144 Glover
solutions from the first-derivative start; SURVEY §8(d) "sampled (>= 1024 g) for configs 4-5")
and microbench A at n = 7000 ("full equality ... m <= 1024 subset at n = 7000"),
every sampled value compared exactly with the ORACLE (not with the library itself).

Rows are sampled so that every 256-row CTA-pair tile of the evaluation contributes one row,
cycling over both CTAs of the pair and all four TMEM lane quarters (the epilogue warp that
drains the row) -- a tile, quarter or CTA-rank indexing slip anywhere shows up.
"""
import os

import numpy as np
import pytest

import oracle
from inputs import CONFIGS, generate_Q, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, ubqp_stats  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402

build_lib()
THREADS = os.cpu_count() or 8


def _tile_rows(K, per_tile=1):
    """one row per 256-row pair tile: CTA rank, lane quarter and lane vary with the tile"""
    rows = []
    for t in range((K + 255) // 256):
        for r in range(per_tile):
            k = t * per_tile + r
            off = (k % 2) * 128 + ((k // 2) % 4) * 32 + (k * 7) % 32
            row = t * 256 + off
            if row < K:
                rows.append(row)
    return np.array(sorted(set(rows + [K - 1])), dtype=np.int64)


@pytest.fixture(scope="module")
def cfg4():
    cfg = CONFIGS[4]
    n, K = cfg["n"], cfg["K"]
    Q = generate_Q(n, cfg["density"], seed=cfg["seed_Q"])
    u = Ubqp(0)
    u.load_Q(Q, K)
    b = np.zeros(u.W64, np.uint64)
    u.first_derivative(b)
    x0 = unpack_bits(b, n)[0]
    assert np.array_equal(x0, oracle.first_derivative_start(Q))
    u.diversify(b, 0, K)
    return cfg, Q, u, b, x0


def _glover_rows(x0, rows):
    return np.stack([oracle.diversify(x0, int(g), 1)[0] for g in rows])


def test_config4_f_every_pair_tile(cfg4):
    """f of 1025 rows (every pair tile, all quarters) on the gains launch and on the f-only
    triangular launch, plus the fused statistics."""
    cfg, Q, u, b, x0 = cfg4
    K = cfg["K"]
    rows = _tile_rows(K)
    assert rows.size >= 1024
    fo = oracle.eval_batch(Q, _glover_rows(x0, rows), nthreads=THREADS)
    f = np.zeros(K, np.int64)
    st = ubqp_stats()
    u.eval_batch(UBQP_EMIT_GAINS, f, st)
    assert np.array_equal(f[rows], fo)
    assert st.sum == int(f.sum()) and st.count == K
    g_best = int(np.argmax(f))                       # lowest index among the maxima
    assert st.max_key == oracle.max_key(int(f[g_best]), g_best)
    f2 = np.zeros(K, np.int64)
    st2 = ubqp_stats()
    u.eval_batch(0, f2, st2)                         # f only: the triangular GEMM
    assert np.array_equal(f2, f) and (st2.sum, st2.count, st2.max_key) == (st.sum, st.count, st.max_key)


def test_config4_gain_rows_against_O2(cfg4):
    """64 full gain rows (n = 7000 each) of the config-4 gains launch against O2."""
    cfg, Q, u, b, x0 = cfg4
    K, n = cfg["K"], cfg["n"]
    rows = _tile_rows(K)[:: max(1, (K // 256) // 64)][:64]
    assert rows.size == 64
    u.eval_batch(UBQP_EMIT_GAINS)
    X = _glover_rows(x0, rows)
    G = np.zeros((1, n), np.int32)
    for r, x in zip(rows, X):
        u.get_gains(int(r), 1, G)
        assert np.array_equal(G[0].astype(np.int64), oracle.gains(Q, x)), int(r)


def test_config4_round_1024_survivors_against_oracle():
    """The exact bench step through MultiStart: >= 1024 ascended survivors (spread over the
    survivor list) re-derived by the oracle from their global index (diversify -> eval ->
    steepest ascent) and compared exactly: f, flips, bits; plus the screen and best key."""
    from paper_1706_00037_b200.multistart import MultiStart, key_f
    cfg = CONFIGS[4]
    n, K = cfg["n"], cfg["K"]
    Q = generate_Q(n, cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, K, lam=cfg["lam"], max_flips=cfg["max_flips"])
    x0_bits, f0 = ms.first_derivative()
    res = ms.round(x0_bits, 0, f0)
    m = res.m
    assert m > 100000
    surv = ms.surv[:m].cpu().numpy()
    f_asc = ms.f_asc[:m].cpu().numpy()
    flips = ms.flips[:m].cpu().numpy()
    bits = ms.bits[:m].cpu().numpy().view(np.uint64)
    x0 = unpack_bits(x0_bits.cpu().numpy().view(np.uint64), n)[0]
    assert f0 == oracle.xQx(Q, x0)
    pick = np.unique(np.concatenate([np.linspace(0, m - 1, 1024).astype(np.int64), [int(np.argmax(f_asc))]]))
    X0 = _glover_rows(x0, surv[pick])
    f_start = oracle.eval_batch(Q, X0, nthreads=THREADS)
    # the screen: each sampled survivor passes T, computed by the oracle from the fused stats
    assert np.all(f_start > res.T)
    Xr, fr, flr = oracle.ascend(Q, X0, f_start, cfg["max_flips"], nthreads=THREADS)
    assert np.array_equal(f_asc[pick], fr) and np.array_equal(flips[pick], flr)
    assert np.array_equal(unpack_bits(bits[pick], n), Xr)
    # best record: the key of the round's best survivor
    i = int(np.argmax(f_asc))
    assert key_f(res.best_key) == int(f_asc[i]) == int(fr[np.searchsorted(pick, i)])


def test_microbench_A_subset_n7000():
    """SURVEY §8(d) microbench A at n = 7000 (dense, random starts O3 seed 5, max_flips 10 n):
    1024 of the 8192 starts ascended, full equality with O7."""
    n, m = 7000, 8192
    Q = generate_Q(n, 1.0, seed=5)
    u = Ubqp(0)
    u.load_Q(Q, m)
    u.random(5, m)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = np.arange(0, m, 8, dtype=np.int32)
    k = slots.size
    f = np.zeros(k, np.int64)
    fl = np.zeros(k, np.int32)
    bb = np.zeros((k, u.W64), np.uint64)
    u.ascend(slots, k, 10 * n, f, fl, bb)
    X0 = oracle.random_solutions(n, 5, m)[slots]
    Xr, fr, flr = oracle.ascend(Q, X0, oracle.eval_batch(Q, X0, nthreads=THREADS), 10 * n, nthreads=THREADS)
    assert np.array_equal(f, fr) and np.array_equal(fl, flr) and np.array_equal(unpack_bits(bb, n), Xr)
