"""The NCCL exchange path on one GPU: a world-size-1 NCCL process group with
UBQP_FORCE_COLLECTIVES=1 makes MultiStart run every collective of a round (stats all-reduce
SUM/MAX, best-key all-reduce MAX, winner-bits broadcast) through NCCL on the library's stream;
the rounds must equal the oracle's run_rounds exactly (O8).  Multi-GPU NCCL runs need more than
one GPU (not available here); the exchange logic at world sizes 2-8 is covered by the gloo
tests (tests/test_multirank_gloo.py, tests/test_gpu_multirank.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import numpy as np, torch, torch.distributed as dist
import oracle
from inputs import generate_Q, unpack_bits
from paper_1706_00037_b200.multistart import MultiStart
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
assert dist.get_backend() == "nccl"
for n, K, rounds, lam in ((300, 2000, 3, 0.5), (1100, 600, 2, 0.3), (7000, 4096, 2, 0.5)):
    Q = generate_Q(n, 0.5, seed=n)
    ms = MultiStart(Q, K, lam=lam, max_flips=10 * n)
    best, bits, traj = ms.run(rounds, sample_seed=7)
    obest, ox, otraj = oracle.run_rounds(Q, K, rounds, lam, 10 * n, sample_seed=7, nthreads=8)
    assert best == obest and traj == otraj, (n, best, obest)
    assert np.array_equal(unpack_bits(bits.cpu().numpy().view(np.uint64), n)[0], ox)
dist.destroy_process_group()
print("nccl ok")
"""


def test_multistart_rounds_through_nccl():
    env = dict(os.environ, UBQP_FORCE_COLLECTIVES="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29517",
               NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "nccl ok" in r.stdout, (r.stdout[-1000:], r.stderr[-3000:])
