"""One config-4-shaped round on a real-valued Q (R20): n = 7000 dense U(-100, 100) float32,
K = 262144 Glover diversifications of the first-derivative start, lambda 0.5.
    python tools/real_round.py [K]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import generate_Q_real  # noqa: E402
from paper_1706_00037_b200.multistart import MultiStartReal  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    Q = generate_Q_real(7000, 1.0, seed=4, dtype=np.float32)
    ms = MultiStartReal(Q, K, lam=0.5, max_flips=70000)
    mean = ms.sample_mean(5)
    x0, f0 = ms.first_derivative()
    ms.round(x0, 0, f0, mean)                      # warm-up (allocates the int64 gains)
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ms.stream)
        m, T, bf, _ = ms.round(x0, 0, f0, mean)
        e1.record(ms.stream)
        torch.cuda.synchronize()
        print(f"K={K} survivors={m} T={T:.6g} best f={bf * 2.0 ** -ms.e:.6f} "
              f"round {e0.elapsed_time(e1):.1f} ms (wall {1e3 * (time.perf_counter() - t):.1f}) "
              f"-> {K / (e0.elapsed_time(e1) * 1e-3):.0f} evals/s", flush=True)


if __name__ == "__main__":
    main()
