"""The product's N > 1 path on one GPU: two ranks (torch.distributed, gloo) each run
MultiStart on a cyclic shard of the batch; the collectives are host-side, the ranks' kernels
never wait on one another, so this is a functional test of the sharded round (O10), not a
measurement.  Results must equal the single-rank oracle exactly (every output depends on g
only)."""
import os
import socket

import numpy as np
import pytest

import oracle
from inputs import generate_Q, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, K, rounds, lam, div, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1706_00037_b200.multistart import MultiStart
        Q = generate_Q(n, 0.5, seed=900 + n)
        ms = MultiStart(Q, K, lam=lam, max_flips=10 * n, device=0)
        best, bits, traj = ms.run(rounds, sample_seed=3, div=div)
        out[rank] = (best, traj, bits.cpu().numpy().tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,div", [(2, "glover"), (3, "blend")])
def test_sharded_rounds_match_single_rank_oracle(world, div):
    n, K, rounds, lam = 200, 1200, 3, 0.4
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _port(), n, K, rounds, lam, div, out), nprocs=world, join=True)
    Q = generate_Q(n, 0.5, seed=900 + n)
    obest, ox, otraj = oracle.run_rounds(Q, K, rounds, lam, 10 * n, sample_seed=3, nthreads=8, div=div)
    for r in range(world):
        best, traj, bits = out[r]
        assert best == obest and traj == otraj
        got = unpack_bits(np.frombuffer(bits, dtype=np.uint64)[None, :], n)[0]
        assert np.array_equal(got, ox)


def _worker_real(rank, world, port, n, K, rounds, lam, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1706_00037_b200.multistart import MultiStartReal
        rng = np.random.default_rng(n)
        A = rng.uniform(-30, 30, size=(n, n)).astype(np.float32)   # exactly represented (R22)
        Q = (np.triu(A) + np.triu(A, 1).T).astype(np.float64)
        ms = MultiStartReal(Q, K, lam=lam, max_flips=10 * n, device=0)
        best, bits, traj = ms.run(rounds, sample_seed=4)
        out[rank] = (best, traj, bits.cpu().numpy().tobytes())
    finally:
        dist.destroy_process_group()


def test_sharded_real_rounds_match_single_rank_oracle():
    """MultiStartReal (R20, R22) on 2 ranks: int128 stats exchange, best (f, g) record, owner bits."""
    n, K, rounds, lam, world = 150, 900, 3, 0.35, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_real, args=(world, _port(), n, K, rounds, lam, out), nprocs=world, join=True)
    rng = np.random.default_rng(n)
    A = rng.uniform(-30, 30, size=(n, n)).astype(np.float32)
    Q = (np.triu(A) + np.triu(A, 1).T).astype(np.float64)
    ob, ox, otraj, e = oracle.run_rounds_real(Q, K, rounds, lam, 10 * n, sample_seed=4, nthreads=8)
    for r in range(world):
        best, traj, bits = out[r]
        assert best == ob and traj == otraj
        assert np.array_equal(unpack_bits(np.frombuffer(bits, dtype=np.uint64)[None, :], n)[0], ox)
