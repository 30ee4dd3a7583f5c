"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py <round-tag> <launches.csv | -> <rep1.ncu-rep> [<rep2> ...]

Writes profiles/<tag>_summary.md (launch-list shares + per-kernel metrics and stall
reasons) and, when a launch list is given (a config-4 round), updates profiles/traffic.json
(dram bytes per launch, read by bench.py)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "tensor IMMA pipe %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "TC pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run([NCU, "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        kernels.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return kernels


def to_bytes(val, unit):
    return float(val.replace(",", "")) * UNIT_SCALE.get(unit, 1)


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    reps = [Path(p) for p in sys.argv[3:]]
    lines = [f"# ncu summary — {tag}", ""]
    if launches != "-":
        lines += launch_list(Path(launches))
    traffic_p = ROOT / "profiles" / "traffic.json"
    traffic = json.loads(traffic_p.read_text()) if traffic_p.exists() else {}
    lines += kernels_summary(reps, traffic)
    out = ROOT / "profiles" / f"{tag}_summary.md"
    out.write_text("\n".join(lines) + "\n")
    if launches != "-":
        traffic_p.write_text(json.dumps(traffic, indent=1) + "\n")
    print(out)


def launch_list(launches):
    lines = []
    txt = [ln for ln in launches.read_text().splitlines() if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("\n".join(txt))))
    tot = sum(float(r["Metric Value"].replace(",", "")) for r in rows)
    agg = {}
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", ""))
    lines += [f"## Launch list (`{launches.name}`: cold-cache, serialised; compare shares)", "",
              "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name}` | {cnt} | {t / 1e3:.1f} | {100 * t / tot:.2f}% |")
    lines.append("")
    return lines


def kernels_summary(reps, traffic):
    lines = []
    for rep in reps:
        for k in raw(rep):
            kname = k["Kernel Name"][0]
            short = kname.split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            lines += [f"## `{kname[:120]}`  ({rep.name})", "", "| metric | value |", "|---|---|"]
            if "lts__t_bytes.sum" not in k and "lts__t_sectors.sum" in k:   # --set full has sectors
                sv, _ = k["lts__t_sectors.sum"]
                k["lts__t_bytes.sum"] = (f"{float(sv.replace(',', '')) * 32 / 1e9:.6f}", "Gbyte")
            for key, label in METRICS:
                if key in k:
                    v, unit = k[key]
                    lines.append(f"| {label} (`{key}`) | {v} {unit} |")
            stalls = []
            for key, (v, unit) in k.items():
                if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), key.split("stalled_")[1].split("_per_issue")[0]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            lines.append("| top stall reasons (warps per issue) | " +
                         ", ".join(f"{n} {x:.2f}" for x, n in stalls[:6]) + " |")
            lines.append("")
            if "dram__bytes_read.sum" in k:
                rb = to_bytes(*k["dram__bytes_read.sum"])
                wb = to_bytes(*k["dram__bytes_write.sum"])
                traffic.setdefault("cfg4_n7000_K262144_glover", {})[short] = rb + wb
    return lines


if __name__ == "__main__":
    main()
