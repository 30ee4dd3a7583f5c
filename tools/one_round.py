"""One round of the hot path on one GPU (for ncu captures): first-derivative start,
Glover diversify, eval + gains, stats, screen, ascend.  Usage:
    python tools/one_round.py [config]      (default: 4 = n 7000, K 262144)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from inputs import CONFIGS, generate_Q  # noqa: E402
from paper_1706_00037_b200.multistart import MultiStart  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "4"
    cfg = CONFIGS[int(key) if key.isdigit() else key]
    Q = generate_Q(cfg["n"], cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, cfg["K"], lam=cfg.get("lam", 0.5), max_flips=cfg.get("max_flips"))
    x0, f0 = ms.first_derivative()
    res = ms.round(x0, 0, f0)
    torch.cuda.synchronize()
    print(f"n={cfg['n']} K={cfg['K']} survivors={res.m} T={res.T:.1f} best={res.best_key >> 22} "
          f"launches={ms.u.launches}")


if __name__ == "__main__":
    main()
