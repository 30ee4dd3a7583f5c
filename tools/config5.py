"""BASELINE config 5: the full multi-start loop (Figure 2 as batched rounds)
at n = 7000 with a lambda sweep 0.2..0.8, on the ranks of torch.distributed (1 GPU if run
plainly).  Writes one trajectory CSV per lambda in the SPEC schema (S:369:
elapsed_s,iteration,best_value,percent_of_reference) and a JSON summary.

    python tools/config5.py [--rounds R] [--K K] [--n N] [--out DIR]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200.multistart import MultiStart, key_f, pool_update  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--K", type=int, default=262144)
    ap.add_argument("--n", type=int, default=7000)
    ap.add_argument("--out", default="gpurun_out/config5")
    ap.add_argument("--lams", default="0.2,0.3,0.4,0.5,0.6,0.7,0.8")
    ap.add_argument("--div", default="glover", choices=["glover", "blend"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("UBQP_DIST_BACKEND", "nccl"))
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    Q = generate_Q(args.n, 1.0, seed=4)
    summary = {"n": args.n, "K": args.K, "rounds": args.rounds, "world": world, "div": args.div, "runs": []}
    for lam in [float(v) for v in args.lams.split(",")]:
        ms = MultiStart(Q, args.K, lam=lam, max_flips=10 * args.n, device=local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mean = ms.sample_mean(5)                      # round 0: K random starts, pinned mean
        inc_bits, inc_f = ms.first_derivative()
        rows = [(time.perf_counter() - t0, 0, inc_f)]
        per_round = []
        pool = []
        for r in range(1, args.rounds + 1):
            tr = time.perf_counter()
            parents = torch.stack(pool) if (args.div == "blend" and pool) else None
            res = ms.round(inc_bits, (r - 1) * args.K, inc_f, mean, parents=parents)
            torch.cuda.synchronize()
            per_round.append({"round": r, "survivors_rank0": res.m, "T": res.T,
                              "round_best": key_f(res.best_key) if res.best_key >= 0 else None,
                              "parents": 0 if parents is None else int(parents.shape[0]),
                              "ms": 1e3 * (time.perf_counter() - tr)})
            improved_from = None
            if res.best_key >= 0 and key_f(res.best_key) > inc_f:
                improved_from = inc_bits
                inc_f = key_f(res.best_key)
                inc_bits = res.best_bits.clone()
                rows.append((time.perf_counter() - t0, r, inc_f))
            if args.div == "blend":
                pool = pool_update(pool, 8, inc_bits, improved_from,
                                   res.best_bits if res.best_key >= 0 else None)
        if rank == 0:
            csv = out / f"trajectory_lambda{lam:.1f}.csv"
            csv.write_text("elapsed_s,iteration,best_value,percent_of_reference\n" +
                           "".join(f"{e:.3f},{i},{v},\n" for e, i, v in rows))
            summary["runs"].append({"lambda": lam, "best": inc_f, "trajectory": rows, "per_round": per_round,
                                    "mean_sum": mean[0], "mean_count": mean[1]})
            print(f"div={args.div} lambda={lam:.1f} best={inc_f} improvements={len(rows) - 1} "
                  f"round_best={[p['round_best'] for p in per_round]} "
                  f"surv={[p['survivors_rank0'] for p in per_round]} "
                  f"round_ms={[round(p['ms'], 1) for p in per_round]}", flush=True)
        ms.u.close()
        del ms
    if rank == 0:
        (out / "summary.json").write_text(json.dumps(summary, indent=1))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
