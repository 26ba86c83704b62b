"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

    python tools/ncu_summary.py <round tag>

Writes profiles/<tag>_ncu_summary.txt (key metrics of each full capture, the
launch-list shares) and profiles/ncu_traffic.json (per-launch DRAM bytes of the
C2 decode kernel, read by bench.py for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
lines = [f"# ncu summaries ({tag}); captures: ncu --set full --clock-control none (cold-cache, serialised)"]
traffic = {}
for rep in sorted(f for f in os.listdir(OUT) if f.endswith(".ncu-rep")):
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    lines.append(f"\n## {rep}: {name[:110]}")
    vals = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            vals[k] = v[i]
            lines.append(f"  {k:78s} {v[i]:>14s} {u[i]}")
    if "decode" in rep and "merge" not in rep:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def nbytes(k):  # each metric in its own unit (ncu picks byte / Kbyte / Mbyte per value)
            return float(vals.get(k, "0").replace(",", "")) * scale.get(u[h.index(k)], 1) if k in h else 0.0
        traffic["decode_c2_dram_bytes_per_launch"] = int(nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"))
        traffic["source"] = f"profiles/{tag}_ncu_summary.txt ({rep}, dram__bytes_read.sum + dram__bytes_write.sum)"
lc = os.path.join(OUT, "launches.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:70]][r[mi]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
    lines.append("\n## launch list (bench.py --steps 40 --warmup 3 --sets 2 --quick; cold-cache serialised durations)")
    for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        d = m["gpu__time_duration.sum"]
        lines.append(f"  {k:70s} n={len(d):4d} mean={sum(d) / len(d) / 1e3:8.2f} us share={sum(d) / tot:6.1%} "
                     f"dram_rd/launch={sum(m['dram__bytes_read.sum']) / len(d) / 1e6:8.2f} MB")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
if os.path.exists(lc):  # the per-launch list itself, one row per launch
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d = launches.setdefault(r[h.index("ID")], {"kernel": r[ki].split("(")[0], "grid": r[h.index("Grid Size")],
                                                       "block": r[h.index("Block Size")]})
            d[r[mi]] = r[vi]
    cols = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_launches.csv"), "w", newline="") as f:
        f.write("# ncu --metrics " + ",".join(cols) + " --clock-control none\n")
        f.write("# command: python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 --quick (tools/gpu_profile.sh)\n")
        w = csv.writer(f)
        w.writerow(["ID", "kernel", "grid", "block"] + cols)
        for i, d in launches.items():
            w.writerow([i, d["kernel"], d["grid"], d["block"]] + [d.get(c, "") for c in cols])
with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
if traffic:
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
print("\n".join(lines))
