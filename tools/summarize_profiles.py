"""Copy the round's measurement artefacts from gpurun_out/ into profiles/.

python tools/summarize_profiles.py ROUND NCU_REP [LAUNCHES_CSV BENCH_JSON]
(defaults gpurun_out/launches_r01.csv, gpurun_out/bench_full.json).  Writes profiles/rROUND_launches_bench.csv, rROUND_kstep_ncu_raw_selected.csv,
kstep_traffic.json and prints the launch table (markdown)."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "launches_r01.csv")
bench = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", "bench_full.json")
prof = os.path.join(ROOT, "profiles")
shutil.copy(launches, os.path.join(prof, f"r{rnd}_launches_bench.csv"))
shutil.copy(bench, os.path.join(prof, f"r{rnd}_bench.json"))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, u, v = rows[0], rows[1], rows[2]
keep = [i for i, k in enumerate(h) if any(s in k for s in (
    "dram__bytes", "gpu__time_duration", "launch__", "sm__warps_active", "issue_active",
    "pipe_fp64", "pipe_alu", "pipe_fma", "inst_executed.sum", "warps_issue_stalled",
    "sm__throughput", "dram_throughput", "lts__t_bytes"))]
with open(os.path.join(prof, f"r{rnd}_kstep_ncu_raw_selected.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["metric", "unit", "value"])
    for i in keep:
        w.writerow([h[i], u[i], v[i]])
val = {k: (float(v[i].replace(",", "")) if v[i] else None) for i, k in enumerate(h)
       if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
unit = {k: u[i] for i, k in enumerate(h) if k in val}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rd = val["dram__bytes_read.sum"] * scale[unit["dram__bytes_read.sum"]]
wr = val["dram__bytes_write.sum"] * scale[unit["dram__bytes_write.sum"]]
def _metric(name):
    return float(v[h.index(name)].replace(",", "")) if name in h else None


json.dump({"grid": [4096, 16384], "kernel": "k_step", "dram_bytes_read": rd,
           "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "fp64_pipe_active_pct": _metric(
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
           "issue_active_pct": _metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "warps_per_sm": _metric("sm__warps_active.avg.per_cycle_active"),
           "registers_per_thread": _metric("launch__registers_per_thread"),
           "algorithmic_bytes_per_launch": 64.0 * 4096 * 16384,
           "source": f"ncu --set full -k regex:k_step -s 3 -c 1, round {rnd} "
                     f"(profiles/r{rnd}_kstep_ncu_raw_selected.csv)"},
          open(os.path.join(prof, "kstep_traffic.json"), "w"), indent=1)
lr = list(csv.reader(open(os.path.join(prof, f"r{rnd}_launches_bench.csv"))))
i = [k for k, r in enumerate(lr) if "Kernel Name" in r][0]
hh = lr[i]
ki, vi = hh.index("Kernel Name"), hh.index("Metric Value")
agg = collections.OrderedDict()
for r in lr[i + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += float(r[vi])
tot = sum(x[1] for x in agg.values())
for k, x in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"| `{k}` | {x[0]} | {x[1] / 1e6:.3f} | {x[1] / x[0] / 1e3:.1f} | {x[1] / tot * 100:.1f}% |")
print("dram per launch", rd + wr)
for i2, k in enumerate(h):
    if k in ("smsp__issue_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
             "smsp__inst_executed.sum", "gpu__time_duration.sum"):
        print(k, v[i2], u[i2])
