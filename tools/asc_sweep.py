"""Time the ascent kernel of one config-4 round under several (BLOCK, NCH) shapes.
    python tools/asc_sweep.py [config] "128,4" "96,5" ..."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from inputs import CONFIGS, generate_Q  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS  # noqa: E402
from paper_1706_00037_b200.multistart import MultiStart, key_f  # noqa: E402


def main():
    key = sys.argv[1]
    cfg = CONFIGS[int(key) if key.isdigit() else key]
    Q = generate_Q(cfg["n"], cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, cfg["K"], lam=cfg.get("lam", 0.5), max_flips=cfg.get("max_flips"))
    u = ms.u
    x0, f0 = ms.first_derivative()
    u.diversify(x0, 0, ms.k_local)
    u.eval_batch(UBQP_EMIT_GAINS, None, ms.stats)
    s = ms.stats.tolist()
    m, T = u.screen(cfg.get("lam", 0.5), s[0], s[1], max(f0, key_f(s[2])), ms.surv)
    ref = None
    for shape in sys.argv[2:] or ["default"]:
        if shape == "default":
            os.environ.pop("UBQP_ASC_CFG", None)
        else:
            os.environ["UBQP_ASC_CFG"] = shape
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ms.stream)
            u.ascend(ms.surv, m, ms.max_flips, ms.f_asc, ms.flips, ms.bits, ms.key)
            e1.record(ms.stream)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        fl = int(ms.flips[:m].sum().item())
        h = (int(ms.f_asc[:m].sum().item()), fl, int(ms.key.item()))
        ref = ref or h
        print(f"{shape:>8}: {best:8.2f} ms  {fl / best / 1e3:7.1f} Msteps/s  "
              f"{fl * cfg['n'] / best / 1e9:6.2f} TB/s  same={h == ref}", flush=True)


if __name__ == "__main__":
    main()
