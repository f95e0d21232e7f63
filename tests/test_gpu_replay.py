"""The exact out-of-line replay path of k_step against the oracle (GPU tests).

k_step evaluates every unit (cell reconstruction, x-face, y-face, update,
flux pair) speculatively with range-gated FastDiv divisions and replays the
unit with IEEE '/' when any operand leaves the proven range
(wb_device.cuh FastDiv).  Two checks:

- the forced-replay build (libwbflow_b200_replay.so, -DWB_FORCE_REPLAY)
  rejects every speculative unit, so *every* unit goes through
  reconstruct_safe / osher_x_safe / osher_romberg_y_safe / update_cell_safe /
  flux_*_safe; the golden cases, the stage arrays and the error path run
  bit-exact against the oracle through it (child pytest process, since the
  library is chosen at import time via WB_LIB_PATH);
- a developed flow (wall-impact 512 x 288, 400 steps) in the product build,
  lockstep with the oracle at every step, where the device replay counter
  shows that replays really fired.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_util import same

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPLAY_LIB = os.path.join(ROOT, "paper_1806_04960_b200", "libwbflow_b200_replay.so")


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_forced_replay_build_is_bitexact(cuda):
    assert os.path.exists(REPLAY_LIB), "run __graft_entry__.build() (builds the replay library)"
    env = dict(os.environ, WB_LIB_PATH=REPLAY_LIB, WB_EXPECT_FORCED_REPLAY="1")
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"),
           os.path.join(ROOT, "tests", "test_gpu_replay.py"), "-k",
           "golden_cases or stage_arrays or error_path or run_until or initial_state "
           "or child_replay_counter"]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    sys.stdout.write(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    # 12 golden cases + 5 stage-array cases + error path + 2 run_until + initial
    # state + the replay-counter check, none skipped
    import re
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 22 and "skipped" not in r.stdout.split("\n")[-2], r.stdout[-2000:]


def test_child_replay_counter(cuda):
    """Runs inside the forced-replay child: every solved unit is a replay."""
    if os.environ.get("WB_EXPECT_FORCED_REPLAY") != "1":
        pytest.skip("only meaningful in the forced-replay child process")
    from paper_1806_04960_b200 import _lib
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    assert _lib.LIB_PATH == REPLAY_LIB
    sc = build_scenario("wall-impact", (64, 36))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.advance()
    wc = sim.work_counters()
    # at least one replay per fluid cell (its reconstruction and update)
    assert wc["replays"] >= 2 * wc["n_fluid"], wc


def test_developed_flow_replays_bitexact(cuda, oracle):
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    oracle.set_threads(os.cpu_count() or 1)
    sc = build_scenario("wall-impact", (512, 288))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    first_replay = None
    for s in range(1, 401):
        dtr = ref.advance()
        dtg = sim.advance()
        assert dtg == dtr, f"dt differs at step {s}"
        assert same(sim.q, ref.q), f"state differs at step {s}"
        if first_replay is None and sim.work_counters()["replays"] > 0:
            first_replay = s
    n = sim.work_counters()["replays"]
    print(f"replays after 400 steps: {n} (first at step {first_replay})")
    assert n > 0, "the developed flow never left the fast division path"
    assert same(sim.dt_log(), np.array(ref.dt_log))
