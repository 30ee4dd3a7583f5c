"""Time eval (full + gains, f-only) for the single-CTA and CTA-pair kernels at config 4."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp  # noqa: E402

n, K = 7000, 262144
torch.cuda.set_stream(torch.cuda.Stream())
Q = generate_Q(n, 1.0, seed=4)
for pair in ("1", "0"):
    os.environ["UBQP_EVAL_2SM"] = pair
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, K)
    u.random(4, K)
    f = torch.zeros(K, dtype=torch.int64, device="cuda")
    res = {}
    for name, flags in (("gains", UBQP_EMIT_GAINS), ("f_only", 0)):
        for _ in range(3):
            u.eval_batch(flags, f)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            u.eval_batch(flags, f)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        ops = 2.0 * n * n * K if flags else n * (n + 1.0) * K
        res[name] = f"{ms:.3f} ms {ops / ms / 1e9:.0f} TOP/s"
    print("pair" if pair == "1" else "single", res, int(f.sum().item()), flush=True)
    u.close()
    del u
