#!/usr/bin/env python
"""Benchmark of the UBQP multi-start hot path on B200 (contract: see DESIGN.md §8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full round of the method (Figure 2) over one batch:
    Glover diversify -> xQx eval + 1-flip gains (tcgen05 int8) -> stats all-reduce ->
    T(lambda) screen -> batched steepest ascent of the survivors -> best record,
on BASELINE.json config 4: n = 7000 dense integer Q (U{-100..100}\\{0}, seed 4),
K = 262144 Glover solutions from the first-derivative start (t0 = 0), lambda = 0.5,
max_flips = 10 n, sharded cyclically over the ranks (strong scaling).
value = K / (step time, max over ranks) in xQx evals/s.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from inputs import CONFIGS, generate_Q  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "xQx evals/sec (full diversify-eval-screen-ascent round)"
UNIT = "evals/s"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


def workload_config(cfg, world, extra=None):
    c = {"workload": cfg["name"], "n": cfg["n"], "density": cfg["density"], "seed_Q": cfg["seed_Q"],
         "K_global": cfg["K"], "K_per_rank": -(-cfg["K"] // world), "lambda": cfg.get("lam"),
         "max_flips": cfg.get("max_flips"), "t0": 0, "Q_coeffs": "U{-100..100}\\{0}",
         "parallelism": f"dp{world} (solutions sharded in blocks of 2 dealt round robin, Q replicated)",
         "l2": "inputs larger than L2 (X8 1.85 GB + gains 7.4 GB per round); Q (49 MB) L2-resident by design"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": "nvml unavailable"}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ oracle (cpu_baseline / reference arm)
def oracle_sample_step(Q, x0, f0, cfg, S, threads):
    """The oracle doing one bounded sample of the workload: the first S slots of the batch
    (eval + screen against the sample's own mean/max + ascent of the survivors)."""
    import oracle
    X = oracle.diversify(x0, 0, S)
    f = oracle.eval_batch(Q, X, threads)
    maxv = max(f0, int(f.max()))
    T = oracle.threshold(cfg["lam"], int(f.sum()), S, maxv)
    s = oracle.screen(f, T)
    _, fa, flips = oracle.ascend(Q, X[s], f[s], cfg["max_flips"], threads)
    return len(s), int(flips.sum())


def cpu_sample_size(Q, x0, f0, cfg, cores, target_s):
    """Size the bounded oracle sample so one step costs about target_s seconds of CPU time."""
    if "UBQP_CPU_SAMPLE" in os.environ:
        return int(os.environ["UBQP_CPU_SAMPLE"])
    S = cores
    t = time.perf_counter()
    oracle_sample_step(Q, x0, f0, cfg, S, cores)
    dt = max(time.perf_counter() - t, 1e-3)
    S = int(S * target_s / dt) // cores * cores
    return max(cores, min(S, cfg["K"]))


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    cores = os.cpu_count() or 1
    Q = generate_Q(cfg["n"], cfg["density"], seed=cfg["seed_Q"])
    x0 = oracle.first_derivative_start(Q)
    f0 = oracle.xQx(Q, x0)
    S = cpu_sample_size(Q, x0, f0, cfg, cores, target_s=8.0)
    for _ in range(args.warmup):
        oracle_sample_step(Q, x0, f0, cfg, S, cores)
    t = time.perf_counter()
    tot_flips = 0
    for _ in range(args.steps):
        _, fl = oracle_sample_step(Q, x0, f0, cfg, S, cores)
        tot_flips += fl
    dt = time.perf_counter() - t
    value = S * args.steps / dt
    sample = (f"first {S} of the {cfg['K']} Glover solutions per step (eval + screen + ascent of "
              f"survivors), {cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": workload_config(cfg, 1, {"sample_per_step": S}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ascent_flips_per_step": tot_flips / args.steps,
    }), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1706_00037_b200 import UBQP_EMIT_GAINS
    from paper_1706_00037_b200.build import build_lib
    from paper_1706_00037_b200.multistart import MultiStart, combine_stats, key_f

    build_lib()
    torch.cuda.set_device(local_rank)
    backend = os.environ.get("UBQP_DIST_BACKEND", "nccl")
    peaks = load_peaks()
    n, K, lam = cfg["n"], cfg["K"], cfg["lam"]
    Q = generate_Q(n, cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, K, lam=lam, max_flips=cfg["max_flips"], device=local_rank)
    u = ms.u
    stream = ms.stream
    x0_bits, f0 = ms.first_derivative()

    ev = {k: torch.cuda.Event(enable_timing=True) for k in
          ("eval0", "eval1", "asc0", "asc1")}
    acc = {"eval": 0.0, "asc": 0.0}

    def step(timed_kernels: bool):
        u.diversify(x0_bits, 0, ms.k_local, rank, world)
        if timed_kernels:
            ev["eval0"].record(stream)
        u.eval_batch(UBQP_EMIT_GAINS, None, ms.stats)
        if timed_kernels:
            ev["eval1"].record(stream)
        combine_stats(ms.stats)
        ssum, scount, skey, _ = ms.stats.tolist()
        maxv = max(f0, key_f(skey))
        m, T = u.screen(lam, ssum, scount, maxv, ms.surv)
        if timed_kernels:
            ev["asc0"].record(stream)
        u.ascend(ms.surv, m, ms.max_flips, ms.f_asc, ms.flips, ms.bits, ms.key)
        if timed_kernels:
            ev["asc1"].record(stream)
        gk = ms.key.clone()
        if world > 1:
            dist.all_reduce(gk, op=dist.ReduceOp.MAX)
        if timed_kernels:
            stream.synchronize()
            acc["eval"] += ev["eval0"].elapsed_time(ev["eval1"])
            acc["asc"] += ev["asc0"].elapsed_time(ev["asc1"])
        return m, int(gk.item())

    for _ in range(args.warmup):
        m, gkey = step(False)
    flips_total = int(ms.flips[:m].sum().item()) if m else 0
    launches0 = u.launches

    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t_start.record(stream)
        marks[0].record(stream)
        for i in range(args.steps):
            m, gkey = step(True)
            marks[i + 1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = u.launches - launches0
    ms_step = t_start.elapsed_time(t_end) / args.steps
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    eval_ms = acc["eval"] / args.steps
    asc_ms = acc["asc"] / args.steps
    t = torch.tensor([ms_step, eval_ms, asc_ms, float(flips_total), float(m)], dtype=torch.float64,
                     device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_step, eval_ms, asc_ms = tmax[0].item(), tmax[1].item(), tmax[2].item()
        flips_all, m_all = tsum[3].item(), tsum[4].item()
    else:
        flips_all, m_all = float(flips_total), float(m)

    # ---- e2e through the C-ABI with host (pinned) buffers, copies inside the timed region
    kl = ms.k_local
    W = ms.W64
    h_seed = torch.empty(W, dtype=torch.int64, pin_memory=True)
    h_seed.copy_(x0_bits.cpu())
    h_stats = torch.empty(4, dtype=torch.int64, pin_memory=True)
    h_surv = torch.empty(max(kl, 1), dtype=torch.int32, pin_memory=True)
    h_f = torch.empty(max(kl, 1), dtype=torch.int64, pin_memory=True)
    h_fl = torch.empty(max(kl, 1), dtype=torch.int32, pin_memory=True)
    h_bits = torch.empty((max(kl, 1), W), dtype=torch.int64, pin_memory=True)
    h_key = torch.empty(1, dtype=torch.int64, pin_memory=True)
    e_steps = args.steps
    d_stats = ms.stats
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    emarks = [torch.cuda.Event(enable_timing=True) for _ in range(e_steps + 1)]
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    emarks[0].record(stream)
    for ei in range(e_steps):
        u.diversify(h_seed, 0, kl, rank, world)
        u.eval_batch(UBQP_EMIT_GAINS, None, h_stats)
        if world > 1:
            d_stats.copy_(h_stats, non_blocking=False)
            combine_stats(d_stats)
            h_stats.copy_(d_stats)
        s = h_stats.tolist()
        m_e, T_e = u.screen(lam, s[0], s[1], max(f0, key_f(s[2])), h_surv)
        u.ascend(h_surv, m_e, ms.max_flips, h_f, h_fl, h_bits, h_key)
        h2d += W * 8 + m_e * 4
        d2h += 32 + m_e * 4 + m_e * (8 + 4 + W * 8) + 8
        emarks[ei + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e_steps
    e2e_median = float(np.median([emarks[i].elapsed_time(emarks[i + 1]) for i in range(e_steps)]))
    te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = te.item()

    if rank != 0:
        return
    value = K / (ms_step * 1e-3)
    # ---- roofline of the dominant kernel (achieved from live CUDA events of this run)
    eval_ops = 2.0 * n * n * K / world                       # per rank per launch (algorithmic)
    eval_tops = eval_ops / (eval_ms * 1e-3) / 1e12
    int8_peak_burst = 2.0 * peaks["bf16_tflops"]             # guide: int8 dense = 2x bf16 nominal
    int8_peak_sust = 2.0 * peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    int8_meas = measure_int8_peak() if not args.no_int8_peak else None
    int8_ok = bool(int8_meas) and "burst_tops" in int8_meas
    int8_peak = int8_meas["burst_tops"] if int8_ok else int8_peak_burst
    asc_bytes = flips_all / world * n                        # one int8 Q row per flip step
    asc_gbs = asc_bytes / (asc_ms * 1e-3) / 1e9 if asc_ms > 0 else 0.0
    traffic = {}
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(cfg["name"], {})
        except Exception:
            traffic = {}
    roof_eval = {"bound": "tensor", "achieved": eval_tops, "peak": int8_peak, "unit": "TOP/s",
                 "frac": eval_tops / int8_peak,
                 "traffic": traffic.get("eval_tc_pair_kernel", traffic.get("eval_tc_kernel")),
                 "kernel": "eval_tc_pair_kernel (+stats)", "ms": eval_ms,
                 "peak_note": ("measured cuBLASLt int8 GEMM (torch._int_mm 8192^3, best of 10) on this GPU"
                               if int8_ok else "int8 = 2 x bf16 " + peaks["_source"]),
                 "int8_measured": int8_meas,
                 "frac_of_2x_bf16_burst": eval_tops / int8_peak_burst,
                 "frac_of_2x_bf16_sustained": eval_tops / int8_peak_sust,
                 "frac_of_spec_4500": eval_tops / 4500.0}
    from paper_1706_00037_b200.ubqp import Q_ASCENT_LAST
    asc_kind = {1: "ascend_kernel", 2: "ascend_sparse_kernel", 3: "ascend_warp_kernel", 4: "ascend_mw_kernel"}.get(
        u.query(Q_ASCENT_LAST), "ascend_kernel")
    roof_asc = {"bound": "hbm", "achieved": asc_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": asc_gbs / peaks["hbm_gbs"], "traffic": traffic.get(asc_kind),
                "kernel": asc_kind, "ms": asc_ms, "steps_per_s": flips_all / (asc_ms * 1e-3) if asc_ms else 0,
                "algorithmic_bytes": "n bytes (one int8 Q row) per flip step"}
    # Q (49 MB int8) is L2-resident, so the byte roofline above overstates the headroom.
    # The issue-pipe view: every variable update of a flip step needs one
    # FMA-heavy instruction (IDP.2A: byte extract + signed multiply-add, the minimum for an exact
    # integer update) and at least half an ALU instruction for the running argmax; both pipes
    # retire 16 lanes/cycle per SMSP (rt_SMSP = 2, B300_MICROARCH "Pipe rates"; ncu on B200:
    # IDP.2A counts on pipe_fmaheavy), so a dense ascent caps at 148 x 4 x 16 variable updates
    # per SM clock whatever its argmax bookkeeping.  Kernel-specific caps are reported beside it:
    # the CTA kernel issues 1.25 ALU instructions per variable, the warp kernel 1.0 (ALU) + 1.0
    # (FMA-heavy).
    sm_mhz = clk.summary().get("sm_mhz") or 1965.0
    alu_peak = 148 * 4 * 16 * sm_mhz * 1e6
    kernel_ops = {"ascend_kernel": 1.25, "ascend_warp_kernel": 1.0}.get(asc_kind, 1.0)
    upd = flips_all / world * n / (asc_ms * 1e-3) if asc_ms else 0.0
    roof_asc_alu = {"bound": "alu", "achieved": upd, "peak": alu_peak, "unit": "variable updates/s",
                    "frac": upd / alu_peak, "traffic": traffic.get(asc_kind), "kernel": asc_kind,
                    "ms": asc_ms, "steps_per_s": roof_asc["steps_per_s"], "sm_mhz": sm_mhz,
                    "peak_derivation": "148 SMs x 4 SMSP x 16 lanes/cycle of the FMA-heavy pipe (one IDP.2A per "
                                       "variable update, the minimum exact integer update; B300_MICROARCH pipe "
                                       "rates, ncu pipe_fmaheavy) at the sampled SM clock; the ALU argmax "
                                       "bookkeeping (>= 0.5 instructions per variable) runs on its own pipe",
                    "kernel_cap": {"instructions_per_variable_on_busiest_pipe": kernel_ops,
                                   "peak": alu_peak / kernel_ops, "frac": upd * kernel_ops / alu_peak},
                    # tools/pipebench.cu (profiles/r02_pipebench.log): a 1:1 IDP.2A + VIMNMX3 mix, the
                    # warp kernel's per-variable pair, issues 2.563 warp instructions per SM cycle at 32
                    # warps/SM -- 41 variable updates per SM cycle, the measured ceiling of that mix
                    "measured_mix_ceiling": {"var_updates_per_sm_cycle": 2.563 / 2 * 32,
                                             "peak": 148 * 2.563 / 2 * 32 * sm_mhz * 1e6,
                                             "frac": upd / (148 * 2.563 / 2 * 32 * sm_mhz * 1e6),
                                             "source": "tools/pipebench.cu, profiles/r02_pipebench.log"},
                    "algorithmic_work": "n variable updates (gain + running argmax) per flip step",
                    "why_not_hbm": "Q (49 MB int8) is L2-resident (ncu L2 hit 99.5%); the byte view is hbm_view",
                    "hbm_view": dict(roof_asc)}
    roof_asc["alu_view"] = {k: v for k, v in roof_asc_alu.items() if k != "hbm_view"}
    # the dominant kernel's roofline: the ascent against the ALU pipe (its real bound)
    dominant = roof_asc_alu if asc_ms >= eval_ms else roof_eval
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": float(np.median(step_ms)),
        "ms_per_step_minmax": [min(step_ms), max(step_ms)], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "dtype_detail": "int8 x int8 -> int32 tensor-core eval, int32 gains / int64 f in the ascent",
        "config": workload_config(cfg, world, {"dist_backend": backend if world > 1 else None}),
        "roofline": dominant,
        "roofline_eval": roof_eval, "roofline_ascent": roof_asc,
        "eval_only_evals_per_s": K / (eval_ms * 1e-3),
        "survivors_per_step": m_all, "flip_steps_per_step": flips_all,
        "e2e": {"value": K / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d // e_steps,
                "d2h_bytes_per_step": d2h // e_steps, "ms_per_step": e2e_ms, "ms_per_step_median": e2e_median,
                "steps": e_steps,
                "path": "C-ABI with pinned host buffers (seed in; stats, survivors, ascent outputs out)"},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        # the cpu_baseline leg is the one place the main arm runs the oracle: its timing, and
        # a sampled exact parity check of the timed step's survivors (before anything else
        # reuses the step's buffers)
        parity = None if args.no_parity else sampled_parity(cfg, Q, x0_bits, ms, m, rank, world)
        out["cpu_baseline"] = cpu_baseline(cfg, Q)
        out["cpu_baseline"].update(cpu_baseline_split())
        if parity is not None:
            out["cpu_baseline"]["parity"] = parity
    if world == 1 and not args.no_projection:
        ms._bench_ms_step = ms_step
        out["shard_projection"] = shard_projection(ms, x0_bits, f0, cfg, ms_step)
    if world == 1 and not args.no_table1:
        out["table1_eval_1000"] = table1_eval(local_rank)
        out["config1_round"] = config1_round(local_rank)
        out["real_q_eval"] = real_q_eval(local_rank)
        out["real_q_ascent"] = real_q_ascent(local_rank)
        out["f_only_eval"] = f_only_eval(local_rank, cfg, Q)
        out["ascent_microbench"] = ascent_microbench(local_rank)
        out["relink_microbench"] = relink_microbench(local_rank)
        out["sparse_ascent"] = sparse_ascent_microbench(local_rank, peaks)
    print(json.dumps(out), flush=True)


def shard_projection(ms, x0_bits, f0, cfg, ms_step_1gpu):
    """Multi-GPU readiness on one GPU: rank r of G holds the cyclic shard
    g = r + i G (K_r = K / G); each shard's round (diversify -> eval + gains -> screen against the
    GLOBAL T -> ascend) is timed on this B200 for every r, G in {2, 4, 8}.  The projected G-GPU
    step is the slowest shard (max over r) -- a projection, not a measurement of G GPUs: the
    three per-round collectives (~tens of microseconds over NVLink) are not included."""
    import torch

    from paper_1706_00037_b200 import UBQP_EMIT_GAINS
    from paper_1706_00037_b200.multistart import key_f
    u, stream, K = ms.u, ms.stream, cfg["K"]
    # the global statistics of the batch (identical for every sharding)
    u.diversify(x0_bits, 0, K, 0, 1)
    u.eval_batch(0, None, ms.stats)
    ssum, scount, skey, _ = ms.stats.tolist()
    maxv = max(f0, key_f(skey))
    from paper_1706_00037_b200.ubqp import OPT_SHARD_BLOCK, shard_count
    out = {"what": "per-rank shard rounds (O10 sharding, blocks of B consecutive g dealt round robin) timed one "
                   "after another on one B200; the projected G-GPU step is the slowest shard; collectives not "
                   "included", "ms_1gpu": ms_step_1gpu}
    slots_per_wave = 148 * 8                                  # warp-ascent solutions resident at n = 7000
    for B, G in ((1, 2), (1, 8), (2, 2), (2, 4), (2, 8)):
        u.set_option(OPT_SHARD_BLOCK, B)
        per = []
        surv = []
        for r in range(G):
            kr = shard_count(r, K, G, B)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            u.diversify(x0_bits, 0, kr, r, G)
            u.eval_batch(UBQP_EMIT_GAINS, None, ms.stats)
            m, _ = u.screen(cfg["lam"], ssum, scount, maxv, ms.surv)
            u.ascend(ms.surv, m, ms.max_flips, ms.f_asc, ms.flips, ms.bits, ms.key)
            e1.record(stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
            surv.append(m)
        mx = max(per)
        out[f"G{G}" + ("_cyclic" if B == 1 else "")] = {"block": B, "per_rank_ms": per, "max_ms": mx, "mean_ms": float(np.mean(per)),
                        "imbalance": mx / float(np.mean(per)), "survivors_per_rank": surv,
                        "ascent_waves": max(surv) / slots_per_wave,
                        "projected_evals_per_s": K / (mx * 1e-3),
                        "projected_speedup": ms_step_1gpu / mx}
    u.set_option(OPT_SHARD_BLOCK, 2)
    try:
        out["exchange_nccl_world1"] = nccl_exchange_cost(ms)
    except Exception as e:                                    # keep the bench line on any failure
        out["exchange_nccl_world1"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    return out


def nccl_exchange_cost(ms, reps: int = 200):
    """The per-round exchange of MultiStart (stats all-reduce SUM + MAX, best-key all-reduce MAX,
    winner-bits broadcast) through NCCL on a world-size-1 process group on this GPU
    (UBQP_FORCE_COLLECTIVES semantics): the launch/synchronisation cost of the collectives on the
    library's stream.  A lower bound for G GPUs (no NVLink transfer at world size 1)."""
    import os
    import sys

    import torch
    import torch.distributed as dist

    from paper_1706_00037_b200 import multistart as msmod
    if dist.is_initialized():
        return {"skipped": "a process group is already initialised"}
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    # the bench prints ONE JSON line on stdout: keep NCCL's banner (written to fd 1) off it
    saved_debug = os.environ.get("NCCL_DEBUG")
    os.environ["NCCL_DEBUG"] = "WARN"

    def quiet(fn):                                            # run fn with fd 1 on /dev/null
        sys.stdout.flush()
        fd1, null = os.dup(1), os.open(os.devnull, os.O_WRONLY)
        os.dup2(null, 1)
        try:
            fn()
        finally:
            os.dup2(fd1, 1)
            os.close(fd1)
            os.close(null)

    def init():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", torch.cuda.current_device()))
        dist.barrier()
    try:
        quiet(init)
    finally:
        if saved_debug is None:
            os.environ.pop("NCCL_DEBUG", None)
        else:
            os.environ["NCCL_DEBUG"] = saved_debug
    force = msmod.FORCE_COLLECTIVES
    msmod.FORCE_COLLECTIVES = True
    try:
        stats = ms.stats.clone()
        key = torch.zeros(1, dtype=torch.int64, device=stats.device)
        row = ms.bits[0].contiguous()
        for _ in range(10):
            msmod.combine_stats(stats)
            msmod.combine_best(key, row)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            msmod.combine_stats(stats)
            msmod.combine_best(key, row)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
    finally:
        msmod.FORCE_COLLECTIVES = force
        quiet(dist.destroy_process_group)
    return {"us_per_round": us, "backend": "nccl", "world": 1,
            "what": "combine_stats + combine_best (3 all-reduces, 1 broadcast, their host reads) per round",
            "fraction_of_step": us * 1e-3 / ms_step_hint(ms)}


def ms_step_hint(ms):
    return getattr(ms, "_bench_ms_step", 216.0)


def cpu_baseline_split():
    """BASELINE.md's CPU baseline recipe: the oracle's evaluation single-threaded and on all
    host cores at n in {2500 (density 0.1), 5000, 7000}, and its steepest ascent
    single-threaded on 64 microbench-A starts (n = 7000, random O3 seed 5, max_flips 10 n)."""
    import platform

    import oracle
    cores = os.cpu_count() or 1
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    res = {"nproc": cores, "cpu_model": model, "machine": platform.machine(),
           "oracle_build": "gcc -O2 -std=c11 -ffp-contract=off -pthread (oracle/oracle.py build_oracle)",
           "eval_single_thread": {}, "eval_all_cores": {}}
    for n, d, sq, k1 in ((2500, 0.1, 2, 32), (5000, 1.0, 3, 8), (7000, 1.0, 4, 4)):
        Q = generate_Q(n, d, seed=sq)
        X = oracle.random_solutions(n, sq, max(k1, cores) * 2)
        t = time.perf_counter()
        oracle.eval_batch(Q, X[:k1], 1)
        dt1 = time.perf_counter() - t
        t = time.perf_counter()
        oracle.eval_batch(Q, X, cores)
        dtn = time.perf_counter() - t
        res["eval_single_thread"][f"n{n}"] = {"evals_per_s": k1 / dt1, "sample": k1}
        res["eval_all_cores"][f"n{n}"] = {"evals_per_s": X.shape[0] / dtn, "sample": int(X.shape[0]),
                                          "threads": cores}
    n = 7000
    Q = generate_Q(n, 1.0, seed=5)
    X = oracle.random_solutions(n, 5, 64)
    f = oracle.eval_batch(Q, X, cores)
    t = time.perf_counter()
    _, _, fl = oracle.ascend(Q, X, f, 10 * n, 1)
    dt = time.perf_counter() - t
    res["ascent_single_thread"] = {"n": n, "starts": 64, "flip_steps": int(fl.sum()),
                                   "steps_per_s": float(fl.sum()) / dt, "seconds": dt}
    return res


def sparse_ascent_microbench(device, peaks):
    """NEXT-3: the sparse-row ascent vs the dense register ascent on Beasley-shaped Q (density
    0.1, the b2500 shape) and n = 7000 density 0.1: 8192 random starts, full ascent
    (identical walks).  Algorithmic bytes of the sparse kernel: 4 bytes per off-diagonal
    nonzero of row k* per step (L2-resident rows)."""
    import torch

    from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp
    from paper_1706_00037_b200.ubqp import ASCENT_DENSE, ASCENT_SPARSE, OPT_ASCENT, Q_NNZ
    res = {}
    m = 8192
    for n, d in ((2500, 0.1), (7000, 0.1)):
        Q = generate_Q(n, d, seed=2)
        u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
        u.load_Q(Q, m)
        row = u.query(Q_NNZ) / n
        u.random(5, m)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = torch.arange(m, dtype=torch.int32, device="cuda")
        r = {}
        for name, opt in (("dense", ASCENT_DENSE), ("sparse", ASCENT_SPARSE)):
            u.set_option(OPT_ASCENT, opt)
            fl = torch.zeros(m, dtype=torch.int32, device="cuda")
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                u.ascend(slots, m, 10 * n, None, fl)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            steps = int(fl.sum().item())
            r[name] = {"ms": best, "steps": steps, "steps_per_s": steps / (best * 1e-3)}
        r["sparse"]["GB_per_s_rows"] = r["sparse"]["steps"] * row * 4 / (r["sparse"]["ms"] * 1e-3) / 1e9
        r["sparse"]["frac_of_hbm"] = r["sparse"]["GB_per_s_rows"] / peaks["hbm_gbs"]
        r["speedup_sparse_vs_dense"] = r["dense"]["ms"] / r["sparse"]["ms"]
        r["row_nnz_mean"] = row
        res[f"n{n}_d{d}"] = r
        u.close()
    return res


def measure_int8_peak():
    """Measured int8 tensor ceiling: cuBLASLt int8 GEMM 8192^3 (torch._int_mm), best of 10
    (burst) and back to back for 2 s (sustained), timed with CUDA events."""
    import torch
    try:
        n = 8192
        g = torch.Generator(device="cuda").manual_seed(0)
        a = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda", generator=g)
        b = torch.randint(-100, 100, (n, n), dtype=torch.int8, device="cuda", generator=g).t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(10):
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        t = time.time()
        cnt = 0
        e0.record()
        while time.time() - t < 2.0:
            torch._int_mm(a, b)
            cnt += 1
        e1.record()
        torch.cuda.synchronize()
        ops = 2.0 * n ** 3
        return {"burst_tops": ops / best / 1e9, "sustained_tops": ops * cnt / e0.elapsed_time(e1) / 1e9}
    except Exception as exc:                                  # keep the bench line on failure
        return {"error": str(exc)[:200]}


def sampled_parity(cfg, Q, x0_bits, ms, m, rank, world, samples=128):
    """SURVEY §8(d) "sampled (>= 1024 g) for configs 4-5", bounded here to ~1 s of host time
    (tests/test_gpu_fullsize.py checks 1025): survivors of the last timed step (first, last and
    random ones) are re-derived by the oracle from their global index g -- Glover
    diversification, exact f, steepest ascent, on all host cores -- and compared exactly with
    the step's ascent outputs (f, flips, bits)."""
    import oracle
    from inputs import unpack_bits
    from paper_1706_00037_b200.ubqp import global_index
    if m == 0:
        return {"checked": 0}
    n = cfg["n"]
    rng = np.random.default_rng(123)
    pick = sorted({0, m - 1, *rng.integers(0, m, size=max(0, samples - 2)).tolist()})
    surv = ms.surv[:m].cpu().numpy()
    f_gpu = ms.f_asc[:m].cpu().numpy()
    fl_gpu = ms.flips[:m].cpu().numpy()
    b_gpu = unpack_bits(ms.bits[:m].cpu().numpy().view(np.uint64), n)
    x0 = unpack_bits(x0_bits.cpu().numpy().view(np.uint64)[None, :], n)[0]
    cores = os.cpu_count() or 1
    X = np.concatenate([oracle.diversify(x0, cfg.get("t0", 0) + global_index(int(surv[i]), rank, world), 1)
                        for i in pick])
    Xa, fa, fla = oracle.ascend(Q, X, oracle.eval_batch(Q, X, cores), cfg["max_flips"], nthreads=cores)
    ok = sum(int(fa[r] == f_gpu[i] and fla[r] == fl_gpu[i] and np.array_equal(Xa[r], b_gpu[i]))
             for r, i in enumerate(pick))
    return {"checked": len(pick), "exact": ok, "what": "survivors of the last timed step re-derived by the "
            "oracle from g (diversify, eval, ascend): f, flips and bits compared exactly"}


def cpu_baseline(cfg, Q):
    import oracle
    cores = os.cpu_count() or 1
    x0 = oracle.first_derivative_start(Q)
    f0 = oracle.xQx(Q, x0)
    S = cpu_sample_size(Q, x0, f0, cfg, cores, target_s=15.0)
    t = time.perf_counter()
    m, fl = oracle_sample_step(Q, x0, f0, cfg, S, cores)
    dt = time.perf_counter() - t
    return {"value": S / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {S} of the {cfg['K']} Glover solutions (eval + screen + ascent of {m} "
                      f"survivors, {fl} flips), {cores} threads, {dt:.1f} s"}


def config1_round(device):
    """SURVEY §8(d) config 1 (n = 50, density 0.1, K = 1000 Glover solutions from the
    first-derivative seed, lambda = 0.5, max_flips = 500): the whole round, latency-bound
    (everything on-chip).  Reports evals/s and ascent steps/s, no roofline %."""
    import torch

    from paper_1706_00037_b200.multistart import MultiStart
    cfg = CONFIGS[1]
    Q = generate_Q(cfg["n"], cfg["density"], seed=cfg["seed_Q"])
    ms = MultiStart(Q, cfg["K"], lam=cfg["lam"], max_flips=cfg["max_flips"], device=device)
    x0, f0 = ms.first_derivative()
    for _ in range(5):
        ms.round(x0, 0, f0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, steps = 50, 0
    e0.record(ms.stream)
    for _ in range(reps):
        res = ms.round(x0, 0, f0)
        steps += int(ms.flips[:res.m].sum().item()) if res.m else 0
    e1.record(ms.stream)
    torch.cuda.synchronize()
    ms_round = e0.elapsed_time(e1) / reps
    ms.u.close()
    return {"n": cfg["n"], "K": cfg["K"], "ms_per_round": ms_round, "evals_per_s": cfg["K"] / (ms_round * 1e-3),
            "ascent_steps_per_round": steps // reps, "note": "round incl. host syncs of screen/best record"}


def table1_eval(device):
    """Paper Table 1 shape: 1000 random solutions evaluated at n = 2500/5000/7000."""
    import torch

    from paper_1706_00037_b200 import Ubqp
    res = {}
    for n, dens, sq, paper_s in ((2500, 0.1, 2, 0.7), (5000, 1.0, 3, 2.0), (7000, 1.0, 4, 3.5)):
        Q = generate_Q(n, dens, seed=sq)
        u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
        u.load_Q(Q, 1000)
        u.random(sq, 1000)
        f = torch.zeros(1000, dtype=torch.int64, device="cuda")
        st = torch.zeros(4, dtype=torch.int64, device="cuda")
        for _ in range(5):
            u.eval_batch(0, f, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            u.eval_batch(0, f, st)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        res[f"n{n}"] = {"us_per_1000_evals": us, "evals_per_s": 1000 / (us * 1e-6),
                        "paper_gtx780ti_s": paper_s, "speedup_vs_paper": paper_s / (us * 1e-6)}
        u.close()
    return res


def f_only_eval(device, cfg, Q):
    """f-only evaluation of the config-4 batch (no gains): the triangular GEMM (SURVEY §8(f)
    NEXT-1), algorithmic work n(n+1) ops per evaluation."""
    import torch

    from paper_1706_00037_b200 import Ubqp
    n, K = cfg["n"], cfg["K"]
    u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, K)
    u.random(4, K)
    f = torch.zeros(K, dtype=torch.int64, device="cuda")
    for _ in range(3):
        u.eval_batch(0, f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        u.eval_batch(0, f)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    u.close()
    return {"n": n, "K": K, "ms": ms, "evals_per_s": K / (ms * 1e-3),
            "algorithmic_tops": n * (n + 1) * K / (ms * 1e-3) / 1e12,
            "note": "n(n+1) ops per evaluation (upper triangle incl. diagonal)"}


def ascent_microbench(device):
    """SURVEY §8(d) microbench A: m = 8192 random starts (SplitMix64 seed 5), dense n in
    {2500, 5000, 7000}, full steepest ascent (max_flips = 10n): flip steps/s."""
    import torch

    from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp
    out = {}
    m = 8192
    for n in (2500, 5000, 7000):
        Q = generate_Q(n, 1.0, seed=5)
        u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
        u.load_Q(Q, m)
        u.random(5, m)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = torch.arange(m, dtype=torch.int32, device="cuda")
        flips = torch.zeros(m, dtype=torch.int32, device="cuda")
        fo = torch.zeros(m, dtype=torch.int64, device="cuda")
        u.ascend(slots, m, 10 * n, fo, flips)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u.ascend(slots, m, 10 * n, fo, flips)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        steps = int(flips.sum().item())
        out[f"n{n}"] = {"ms": ms, "flip_steps": steps, "steps_per_s": steps / (ms * 1e-3),
                        "TB_per_s_qrow": steps * n / (ms * 1e-3) / 1e12}
        u.close()
    return out


def relink_microbench(device):
    """NEXT-4 path relinking (O11): m = 8192 random starts (SplitMix64 seed 5) relinked
    toward 8 random guides (seed 6, i mod 8) at n = 7000 dense: |D| ~ n/2 forced steps
    each, the same per-step work as the ascent (one Q row of n bytes)."""
    import torch

    from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp
    n, m = 7000, 8192
    Q = generate_Q(n, 1.0, seed=5)
    u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, m)
    u.random(6, 8)
    guides = torch.zeros((8, u.W64), dtype=torch.int64, device="cuda")
    u.get_batch(guides)
    u.random(5, m)
    u.eval_batch(UBQP_EMIT_GAINS)
    slots = torch.arange(m, dtype=torch.int32, device="cuda")
    ln = torch.zeros(m, dtype=torch.int32, device="cuda")
    fo = torch.zeros(m, dtype=torch.int64, device="cuda")
    u.relink(guides, 8, slots, m, fo, None, ln)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u.relink(guides, 8, slots, m, fo, None, ln)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    steps = int(ln.sum().item())
    u.close()
    return {"n": n, "m": m, "ms": ms, "steps": steps, "steps_per_s": steps / (ms * 1e-3),
            "TB_per_s_qrow": steps * n / (ms * 1e-3) / 1e12}


def real_q_ascent(device):
    """R20: real-valued Q (n = 7000 dense, U(-100,100) float32), 8192 random starts ascended
    exactly on the fixed-point image (int64 gains, Qt rows int32 = 4 qt_ld bytes per step,
    HBM-resident): flip steps/s and Qt-row GB/s."""
    import torch

    from inputs import generate_Q_real
    from paper_1706_00037_b200 import Ubqp
    n, m = 7000, 8192
    Q = generate_Q_real(n, 1.0, seed=4, dtype=np.float32)
    u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q_real(Q, m)
    u.random(5, m)
    u.eval_batch_real()
    slots = torch.arange(m, dtype=torch.int32, device="cuda")
    fl = torch.zeros(m, dtype=torch.int32, device="cuda")
    u.ascend_real(slots, m, 10 * n, None, None, fl)          # forms the int64 gains
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u.ascend_real(slots, m, 10 * n, None, None, fl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    steps = int(fl.sum().item())
    row_bytes = 4 * n                                         # algorithmic: one int32 Qt row per step
    u.close()
    return {"n": n, "m": m, "ms": ms, "steps": steps, "steps_per_s": steps / (ms * 1e-3),
            "GB_per_s_qt_rows": steps * row_bytes / (ms * 1e-3) / 1e9,
            "note": "Qt (int32, 196 MB) exceeds L2: HBM-bound, vs the measured copy bandwidth"}


def real_q_eval(device):
    """a4': real-valued Q (n = 7000 dense, U(-100,100) float32), 65536 random solutions:
    four int8 limb-plane evaluations + exact combine."""
    import torch

    from inputs import generate_Q_real
    from paper_1706_00037_b200 import Ubqp
    n, K = 7000, 65536
    Q = generate_Q_real(n, 1.0, seed=4, dtype=np.float32)
    u = Ubqp(device, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q_real(Q, K)
    u.random(4, K)
    f = torch.zeros(K, dtype=torch.float64, device="cuda")
    for _ in range(3):
        u.eval_batch_real(f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        u.eval_batch_real(f)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    planes, w = u.eval_limbs, u.eval_exp
    u.close()
    # one triangular (f-only) int8 pass per limb plane: n (n + 1) ops per plane and solution
    return {"n": n, "K": K, "ms": ms, "evals_per_s": K / (ms * 1e-3), "planes": planes, "eval_exp": w,
            "int8_equiv_tops": planes * float(n) * (n + 1) * K / (ms * 1e-3) / 1e12,
            "note": "evaluation image exact for float32 Q (R22): f = x^t Q x correctly rounded; "
                    "one launch over all planes with the int128 combine and stats folded in-kernel"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-table1", action="store_true")
    ap.add_argument("--no-int8-peak", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-projection", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the contract requires >= 3 warm-up steps", file=sys.stderr)
    key = int(args.config) if args.config.isdigit() else args.config
    cfg = dict(CONFIGS[key])
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    # UBQP_DIST_BACKEND=gloo + fewer GPUs than ranks: a functional check of the multi-rank path
    # on one GPU (ranks share a device; only host-side collectives, no kernel waits on a peer).
    backend = os.environ.get("UBQP_DIST_BACKEND", "nccl")
    if world > 1:
        import torch
        import torch.distributed as dist
        local_rank = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
