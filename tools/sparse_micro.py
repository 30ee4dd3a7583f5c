"""NEXT-3 microbench: sparse-row vs dense register ascent on Beasley-shaped Q (density d,
P:99) with m = 8192 random starts, full ascent (max_flips 10 n), same box, same inputs.
    python tools/sparse_micro.py [n:density ...]      (default 2500:0.1 7000:0.1 2500:0.02 2500:0.2)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp  # noqa: E402
from paper_1706_00037_b200.ubqp import ASCENT_DENSE, ASCENT_SPARSE, OPT_ASCENT, Q_NNZ  # noqa: E402


def run(n, d, m=8192):
    Q = generate_Q(n, d, seed=2)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, m)
    nnz = u.query(Q_NNZ)
    u.random(5, m)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = torch.arange(m, dtype=torch.int32, device="cuda")
    out = {}
    for name, opt in (("dense", ASCENT_DENSE), ("sparse", ASCENT_SPARSE)):
        u.set_option(OPT_ASCENT, opt)
        flips = torch.zeros(m, dtype=torch.int32, device="cuda")
        fo = torch.zeros(m, dtype=torch.int64, device="cuda")
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            u.ascend(slots, m, 10 * n, fo, flips)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        steps = int(flips.sum().item())
        out[name] = (best, steps, int(fo.sum().item()))
    u.close()
    (td, sd, fd), (ts, ss, fs) = out["dense"], out["sparse"]
    assert sd == ss and fd == fs, "dense and sparse walks differ"
    row = nnz / n                                  # mean off-diagonal nonzeros per row
    print(f"n={n} d={d}: dense {td:8.2f} ms {sd / td / 1e6:6.3f} Gsteps/s | sparse {ts:8.2f} ms "
          f"{ss / ts / 1e6:6.3f} Gsteps/s ({ss * row * 4 / (ts * 1e-3) / 1e12:5.2f} TB/s of CSR entries) "
          f"| speedup {td / ts:5.2f}x  steps={sd}", flush=True)


if __name__ == "__main__":
    torch.cuda.set_stream(torch.cuda.Stream())
    args = sys.argv[1:] or ["2500:0.1", "7000:0.1", "2500:0.02", "2500:0.2", "1000:0.1", "5000:0.05"]
    for a in args:
        n, d = a.split(":")
        run(int(n), float(d))
