"""The in-kernel fold of the evaluation (eval_tc.cu: per-item partials, per-group counters, a
fold warp, self-resetting counters): randomised shapes, both kernels (CTA pair / single CTA),
triangular and full GEMMs, K splits, ranks and shard blocks, and back-to-back launches that
reuse the counters -- f and the statistics must equal the oracle exactly every time."""
import os

import numpy as np
import pytest

import oracle
from inputs import generate_Q

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import given, settings, strategies as st  # noqa: E402

from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, ubqp_stats  # noqa: E402
from paper_1706_00037_b200.build import build_lib  # noqa: E402
from paper_1706_00037_b200.ubqp import OPT_EVAL_PAIR, OPT_EVAL_TRI, OPT_SHARD_BLOCK  # noqa: E402

build_lib()


@settings(max_examples=int(os.environ.get("UBQP_HYPO_EXAMPLES", 60)), deadline=None)
@given(n=st.integers(1, 1300), K=st.integers(1, 1500), pair=st.booleans(), tri=st.booleans(),
       world=st.integers(1, 5), block=st.integers(1, 4), seed=st.integers(0, 2**31 - 1))
def test_fold_matches_oracle(n, K, pair, tri, world, block, seed):
    Q = generate_Q(n, 0.6, seed=seed)
    rank = seed % world
    kl = oracle.shard_count(rank, K, world, block)
    u = Ubqp(0)
    u.set_option(OPT_EVAL_PAIR, int(pair))
    u.set_option(OPT_EVAL_TRI, int(tri))
    u.set_option(OPT_SHARD_BLOCK, block)
    u.load_Q(Q, max(kl, 1))
    u.random(seed, kl, rank, world)
    X = oracle.random_solutions(n, seed, kl, rank, world, block)
    fo = oracle.eval_batch(Q, X, nthreads=8)
    so = oracle.stats(fo, rank, world, block)
    for flags in (0, UBQP_EMIT_GAINS, 0):            # back to back: the counters reset themselves
        f = np.zeros(max(kl, 1), np.int64)
        stt = ubqp_stats()
        u.eval_batch(flags, f, stt)
        assert np.array_equal(f[:kl], fo)
        assert (stt.sum, stt.count, stt.max_key) == (int(so[0]), kl, int(so[2]) if kl else -1)


def test_fold_device_outputs_and_interleaved_handles():
    """device f / stats are written by the kernel; two handles on one stream interleave"""
    n1, n2, K = 700, 333, 2000
    Q1, Q2 = generate_Q(n1, 1.0, seed=1), generate_Q(n2, 0.2, seed=2)
    s = torch.cuda.Stream()
    u1 = Ubqp(0, stream=s.cuda_stream)
    u2 = Ubqp(0, stream=s.cuda_stream)
    u1.load_Q(Q1, K)
    u2.load_Q(Q2, K)
    u1.random(3, K)
    u2.random(4, K)
    f1 = torch.zeros(K, dtype=torch.int64, device="cuda")
    f2 = torch.zeros(K, dtype=torch.int64, device="cuda")
    s1 = torch.zeros(4, dtype=torch.int64, device="cuda")
    s2 = torch.zeros(4, dtype=torch.int64, device="cuda")
    for _ in range(3):
        u1.eval_batch(0, f1, s1)
        u2.eval_batch(UBQP_EMIT_GAINS, f2, s2)
    torch.cuda.synchronize()
    fo1 = oracle.eval_batch(Q1, oracle.random_solutions(n1, 3, K), nthreads=8)
    fo2 = oracle.eval_batch(Q2, oracle.random_solutions(n2, 4, K), nthreads=8)
    assert np.array_equal(f1.cpu().numpy(), fo1) and np.array_equal(f2.cpu().numpy(), fo2)
    assert s1.cpu().tolist()[:3] == oracle.stats(fo1).tolist()[:3]
    assert s2.cpu().tolist()[:3] == oracle.stats(fo2).tolist()[:3]


@pytest.mark.parametrize("n,K,pair", [(2500, 1000, 1), (700, 3000, 1), (300, 200, 0)])
def test_back_to_back_evals_overlap(n, K, pair):
    """Chains of evaluations on one handle with device outputs and no host sync: the CTA-pair
    kernel is launched with programmatic dependent launch (the next evaluation's TMA producer
    and MMA issuer start while the previous one's fold still runs; poll-mode fold at n = 2500,
    K = 1000, counters at K = 3000).  Every f and statistics buffer, the gains of the last
    evaluation and an ascent reading them must equal the oracle."""
    import oracle as O
    from paper_1706_00037_b200.ubqp import ASCENT_AUTO, OPT_ASCENT  # noqa: F401
    Q = generate_Q(n, 0.1 if n == 2500 else 0.7, seed=n + K)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.set_option(OPT_EVAL_PAIR, pair)
    u.load_Q(Q, K)
    u.random(77, K)
    fs = [torch.full((K,), -1, dtype=torch.int64, device="cuda") for _ in range(9)]
    ss = [torch.full((4,), -1, dtype=torch.int64, device="cuda") for _ in range(9)]
    for i in range(9):
        u.eval_batch(UBQP_EMIT_GAINS if i % 3 == 2 else 0, fs[i], ss[i])
    slots = torch.arange(min(K, 64), dtype=torch.int32, device="cuda")
    fa = torch.zeros(len(slots), dtype=torch.int64, device="cuda")
    u.ascend(slots, len(slots), 10 * n, fa)
    torch.cuda.synchronize()
    X = O.random_solutions(n, 77, K)
    fo = O.eval_batch(Q, X, nthreads=8)
    st = O.stats(fo).tolist()[:3]
    for i in range(9):
        assert np.array_equal(fs[i].cpu().numpy(), fo), i
        assert ss[i].cpu().tolist()[:3] == st, i
    g = np.zeros((4, n), np.int32)
    u.get_gains(0, 4, g)
    assert np.array_equal(g, np.stack([O.gains(Q, X[i]) for i in range(4)]))
    _, fr, _ = O.ascend(Q, X[:len(slots)], fo[:len(slots)], 10 * n, nthreads=8)
    assert np.array_equal(fa.cpu().numpy(), fr)
    u.close()


def test_evals_in_cuda_graph():
    """Evaluations captured in a CUDA graph (the programmatic-launch edges between them become
    graph edges) and replayed twice on new batches: f and the statistics equal the oracle.
    (Replays bypass the handle's host-side state, so gains are not read back here.)"""
    import oracle as O
    n, K = 2500, 1000
    Q = generate_Q(n, 0.1, seed=31)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    u = Ubqp(0, stream=s.cuda_stream)
    u.load_Q(Q, K)
    f = [torch.zeros(K, dtype=torch.int64, device="cuda") for _ in range(3)]
    st = [torch.zeros(4, dtype=torch.int64, device="cuda") for _ in range(3)]
    u.random(1, K)
    for i in range(3):                          # warm-up: buffers sized outside the capture
        u.eval_batch(UBQP_EMIT_GAINS if i == 1 else 0, f[i], st[i])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(3):
            u.eval_batch(UBQP_EMIT_GAINS if i == 1 else 0, f[i], st[i])
    for seed in (5, 6):
        u.random(seed, K)
        for t in f + st:
            t.fill_(-7)
        g.replay()
        torch.cuda.synchronize()
        X = O.random_solutions(n, seed, K)
        fo = O.eval_batch(Q, X, nthreads=8)
        for i in range(3):
            assert np.array_equal(f[i].cpu().numpy(), fo), (seed, i)
            assert st[i].cpu().tolist()[:3] == O.stats(fo).tolist()[:3], (seed, i)
    u.close()
    torch.cuda.set_stream(torch.cuda.default_stream())


@pytest.mark.parametrize("n,K", [(16000, 5), (9000, 300), (2500, 1000), (4097, 129)])
@pytest.mark.parametrize("ksplit", ["0", "3", "16"])
def test_fold_balanced_splits_large_n(n, K, ksplit, monkeypatch):
    """f-only launches with fewer tiles than CTA pairs use the balanced K-split table
    (eval_tc.cu eval_shape); at n = 16000 (63 N tiles) it has > 32 entries, so the fold stages
    the partials in two batches.  UBQP_KSPLIT forces uniform splits of every tile (3: uneven
    ranges, 16: clamped by the 256-entry table).  f and the statistics equal the oracle."""
    import subprocess
    import sys
    code = f"""
import numpy as np, oracle
from inputs import generate_Q
from paper_1706_00037_b200 import Ubqp, ubqp_stats
Q = generate_Q({n}, 0.3, seed=7)
u = Ubqp(0)
u.load_Q(Q, {K})
u.random(11, {K})
X = oracle.random_solutions({n}, 11, {K})
fo = oracle.eval_batch(Q, X, nthreads=8)
so = oracle.stats(fo)
for _ in range(2):
    f = np.zeros({K}, np.int64)
    st = ubqp_stats()
    u.eval_batch(0, f, st)
    assert np.array_equal(f, fo)
    assert (st.sum, st.count, st.max_key) == (int(so[0]), {K}, int(so[2]))
print("ok")
"""
    env = dict(os.environ, UBQP_KSPLIT=ksplit)       # read once per process: run in a child
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
