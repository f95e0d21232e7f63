"""Refresh the numbers of profiles/r01_summary.md and DESIGN.md section 6 from
gpurun_out/bench_full.json, bench_ref.json, the launch table and the phase
table (tools/summarize_profiles.py and tools/ncu_phases.py outputs).
python tools/refresh_summary.py launch_table.md phases.md ncu_tag"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "gpurun_out", "bench_full.json")))
ref = json.load(open(os.path.join(ROOT, "gpurun_out", "bench_ref.json")))
lt = [l for l in open(sys.argv[1]).read().split("\n") if l.startswith("| `")]
extra = {l.split()[0]: l.split()[1] for l in open(sys.argv[1]).read().split("\n")
         if l and not l.startswith("|")}
phases = open(sys.argv[2]).read().strip()
tag = sys.argv[3]
r = d["roofline"]
tj = json.load(open(os.path.join(ROOT, "profiles", "kstep_traffic.json")))
kmean = float(lt[0].split("|")[4])

p = os.path.join(ROOT, "profiles", "r01_summary.md")
s = open(p).read()


def sub(pattern, repl):
    global s
    s2, n = re.subn(pattern, repl, s, count=1, flags=re.S)
    assert n == 1, pattern
    s = s2


sub(r"- \*\*Clocks:\*\*.*?throttle reasons\.",
    f"- **Clocks:** {d['clocks']['sm_mhz']:.0f} MHz median SM clock (max "
    f"{d['clocks']['sm_max_mhz']:.0f}), {d['clocks']['samples']} samples during the timed "
    "region, no\n  throttle reasons.")
sub(r"\| device throughput \(`value`\) \|[^\n]*",
    f"| device throughput (`value`) | **{d['value']:.3g} cell-updates/s** "
    f"({d['ms_per_step']:.2f} ms/step) |")
sub(r"(\| e2e through `Simulation`[^|]*\|)[^\n]*", rf"\1 {d['e2e']['value']:.3g} cell-updates/s |")
sub(r"(\| CPU baseline: C restatement[^|]*\|)[^\n]*",
    rf"\1 {d['cpu_baseline']['value']:.2g} cell-updates/s |")
sub(r"(\| `--impl reference` arm[^|]*\|)[^\n]*", rf"\1 {ref['value']:.3g} cell-updates/s |")
sub(r"\| target \| ≥ 4\.0e8; value / target = [0-9]+× \|",
    f"| target | ≥ 4.0e8; value / target = {d['value'] / 4e8:.0f}× |")
sub(r"\| paper, Titan Black \|[^\n]*",
    f"| paper, Titan Black | 2.0e7; value / paper = {d['value'] / 2e7:.0f}× |")
sub(r"takes [0-9.]+ ms per launch\n\(CUDA events, `wb_profile_steps`\)\. The ncu launch list gives "
    r"[0-9.]+ ms mean",
    f"takes {r['kernel_ms']:.2f} ms per launch\n(CUDA events, `wb_profile_steps`). The ncu "
    f"launch list gives {kmean / 1e3:.2f} ms mean")
sub(r"- Achieved: .*?i\.e\. \*\*[0-9.]+%\*\*\.",
    f"- Achieved: {r['achieved']:.2f} TFLOP/s against {r['peak']:.1f} TFLOP/s measured DFMA "
    f"peak, i.e. **{100 * r['frac']:.1f}%**.")
sub(r"- ncu \(`kstep_r01\w+`\): FP64 pipe [0-9.]+% active, issue slots [0-9.]+% busy, [0-9.]+ "
    r"warps per SM \([0-9]+\n  registers",
    f"- ncu (`{tag}`): FP64 pipe {tj['fp64_pipe_active_pct']:.1f}% active, issue slots "
    f"{tj['issue_active_pct']:.1f}% busy, {tj['warps_per_sm']:.1f} warps per SM "
    f"({tj['registers_per_thread']:.0f}\n  registers")
sub(r"[0-9.]+e9 warp-instructions per step",
    f"{float(extra['smsp__inst_executed.sum']) / 1e9:.2f}e9 warp-instructions per step")
gb = tj["dram_bytes_per_launch"] / 1e9
sub(r"- ncu `dram__bytes_read \+ write` = \*\*[0-9.]+ GB per launch\*\*, [0-9.]+× the algorithmic",
    f"- ncu `dram__bytes_read + write` = **{gb:.2f} GB per launch**, "
    f"{gb / 4.294967296:.2f}× the algorithmic")
bw = tj["dram_bytes_per_launch"] / (kmean * 1e-6) / 1e9
sub(r"- That is [0-9]+ GB/s, [0-9.]+% of the measured 6451\.8 GB/s\.",
    f"- That is {bw:.0f} GB/s, {100 * bw / 6451.8:.1f}% of the measured 6451.8 GB/s.")
i = s.index("| phase | warp-instructions |")
j = s.index("\n\n", i)
s = s[:i] + phases + s[j:]
lines = s.split("\n")
a = next(k for k, l in enumerate(lines) if l.startswith("| kernel | launches"))
b = a + 2
c = b
while c < len(lines) and lines[c].startswith("| `"):
    c += 1
lines = lines[:b] + lt + lines[c:]
open(p, "w").write("\n".join(lines))

p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
a = s.index("| value (device) |")
b = s.index("Other configurations (`tools/config_sweep.py`")
s = s[:a] + (
    f"| value (device) | **{d['value']:.3g} cell-updates/s** ({d['ms_per_step']:.2f} ms/step, "
    "essentially all of it `k_step`, detection included) |\n"
    f"| e2e (host buffers) | {d['e2e']['value']:.3g} cell-updates/s (the 2 × 2.7 GB PCIe copies "
    "are ~1/3 of the e2e time at K = 20) |\n"
    f"| vs paper | ~{d['value'] / 2e7:.0f}× the paper's 2e7 (Titan Black); "
    f"~{d['value'] / 4e8:.0f}× the ≥4e8 target |\n"
    f"| CPU baseline (16 threads) | {d['cpu_baseline']['value']:.2g} cell-updates/s (reference "
    f"arm {ref['value']:.2g}), i.e. ~{d['value'] / ref['value']:.0f}× device and "
    f"~{d['e2e']['value'] / ref['value']:.0f}× e2e against the reference arm |\n"
    f"| roofline, `k_step` | {r['achieved']:.2f} TF algorithmic FP64 of {r['peak']:.1f} TF "
    f"measured DFMA = {100 * r['frac']:.1f}%; FP64 pipe {tj['fp64_pipe_active_pct']:.0f}%, issue "
    f"{tj['issue_active_pct']:.0f}% active (ncu); DRAM {gb:.2f} GB per launch = "
    f"{gb / 4.294967296:.2f}× the algorithmic 4.29 GB ({100 * bw / 6451.8:.0f}% of HBM) |\n\n") + s[b:]
open(p, "w").write(s)
print("ok")
