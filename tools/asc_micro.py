"""SURVEY §8(d) ascent microbench A at n in {2500, 5000, 7000} (8192 random starts, full
ascent): flip steps/s per n and per dense kernel (1 = CTA, 3 = warp per solution, 4 = 2-3 warps per
solution; UBQP_ASC_KERNELS="1,3"; UBQP_ASC_M starts), on the library UBQP_LIB points at (A/B of
kernel variants).
    python tools/asc_micro.py [n ...]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp  # noqa: E402
from paper_1706_00037_b200.ubqp import OPT_ASCENT, Q_ASCENT_LAST  # noqa: E402


def main():
    ns = [int(a) for a in sys.argv[1:]] or [2500, 5000, 7000]
    m = int(os.environ.get("UBQP_ASC_M", 8192))
    st = torch.cuda.Stream()                 # a non-default stream shared with the library
    torch.cuda.set_stream(st)
    for n in ns:
        Q = generate_Q(n, 1.0, seed=5)
        u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
        u.load_Q(Q, m)
        u.random(5, m)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = torch.arange(m, dtype=torch.int32, device="cuda")
        flips = torch.zeros(m, dtype=torch.int32, device="cuda")
        fo = torch.zeros(m, dtype=torch.int64, device="cuda")
        for kern in [int(k) for k in os.environ.get("UBQP_ASC_KERNELS", "1,3").split(",")]:
            if kern == 3 and n > 7168:
                continue            # kernel 0 (automatic) prints the kernel it chose
            u.set_option(OPT_ASCENT, kern)
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                u.ascend(slots, m, 10 * n, fo, flips)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            steps = int(flips.sum().item())
            chose = f" (ran {u.query(Q_ASCENT_LAST)})" if kern == 0 else ""
            print(f"n={n} kernel={kern}{chose}: {best:7.2f} ms  {steps / best / 1e6:6.3f} Gsteps/s  steps={steps} "
                  f"fsum={int(fo.sum().item())}", flush=True)
        u.close()


if __name__ == "__main__":
    main()
