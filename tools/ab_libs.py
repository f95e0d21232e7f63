"""A/B timing of several builds of the library on the bench workload (GPU).

    LIBS="base=paper_1806_04960_b200/libwbflow_b200.so,x=tools/exp/lib_x.so|WB_ROWS=32" \
        python tools/ab_libs.py [rounds] [warm,warm,...]

(an entry may carry environment settings after '|').

For every (round, warm-up, library) a fresh process loads that library
(WB_LIB_PATH), advances the C5 slab 4096x16384 `warm` steps, times k_step
alone over 5 steps with CUDA events (wb_profile_steps) and prints the time
and a SHA-256 of the state, which must agree between libraries (the builds
must be bit-identical)."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import ctypes, hashlib, os, sys
sys.path.insert(0, %r)
from paper_1806_04960_b200 import _lib
from paper_1806_04960_b200.scenarios import build_scenario
from paper_1806_04960_b200.timestepper import Simulation
warm = int(sys.argv[1])
sc = build_scenario("wall-impact", (4096, 16384))
sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
sim.run_steps(warm, chunk=min(warm, 16))
md, ms, mt = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
_lib.check(sim._L.wb_profile_steps(sim._h, 5, ctypes.byref(md), ctypes.byref(ms),
                                   ctypes.byref(mt)), "profile")
h = hashlib.sha256(sim.q.tobytes()).hexdigest()[:16]
print(f"RESULT {ms.value:.4f} {h} {sim.work_counters()['replays']}")
""" % ROOT


def main():
    libs = [kv.split("=", 1) for kv in os.environ["LIBS"].split(",")]
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    warms = [int(w) for w in (sys.argv[2] if len(sys.argv) > 2 else "3,300").split(",")]
    res = {}
    for r in range(rounds):
        for w in warms:
            for name, spec in libs:
                path, *envs = spec.split("|")
                env = dict(os.environ, WB_LIB_PATH=os.path.join(ROOT, path))
                env.update(e.split("=", 1) for e in envs)
                out = subprocess.run([sys.executable, "-c", CHILD, str(w)], env=env,
                                     capture_output=True, text=True, timeout=900)
                line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT")]
                if not line:
                    print(f"{name} warm {w}: FAILED\n{out.stderr[-1500:]}", flush=True)
                    continue
                _, ms, h, nrep = line[0].split()
                res.setdefault((w, name), []).append((float(ms), h, int(nrep)))
                print(f"round {r} warm {w:4d} {name:12s} k_step {float(ms):7.3f} ms  q {h}  "
                      f"replays {nrep}", flush=True)
    print("\nsummary (min over rounds):")
    for w in warms:
        hs = {res[(w, n)][0][1] for n, _ in libs if (w, n) in res}
        for n, _ in libs:
            if (w, n) in res:
                print(f"  warm {w:4d} {n:12s} {min(v[0] for v in res[(w, n)]):7.3f} ms")
        print(f"  warm {w:4d} states {'IDENTICAL' if len(hs) == 1 else 'DIFFER: ' + str(hs)}")


if __name__ == "__main__":
    main()
