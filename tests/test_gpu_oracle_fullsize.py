"""Oracle lockstep at BASELINE.json's full sizes, including the benchmarked
shape (GPU tests).

The CPU oracle (oracle/wb_oracle.c, all host threads; pinned to the
unmodified reference by tests/test_oracle_golden.py) runs these grids at
~5e7 cell-updates/s on the GPU box's 16 cores and needs ~540 B per cell of
host memory, so the shapes below fit in a few minutes and < 80 GB:

- C5 slab 4096 x 16384 (the bench.py workload): steps 1-25, i.e. the driver's
  `--warmup 5 --steps 20` window, through the same device loop bench.py
  times (`run_steps`, CUDA-graph chunks) plus per-step `advance()`;
- C3 drop 4096^2: 20 steps, state compared after every step;
- C4 weir 16384 x 8192: 3 steps (skipped if the host lacks the memory).

Every comparison is bit-exact (golden_util.same: identical bit patterns) on
q, t and the dt sequence.
"""
import os

import numpy as np
import pytest

from golden_util import same

pytestmark = pytest.mark.gpu

ORACLE_BYTES_PER_CELL = 560  # q, q_next, 10 stage arrays, profiles, flags + sim.q copies


@pytest.fixture(scope="module")
def Simulation():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_04960_b200.timestepper import Simulation
    return Simulation


@pytest.fixture(scope="module")
def full_oracle(oracle):
    oracle.set_threads(os.cpu_count() or 1)
    return oracle


def _need_host_memory(cells):
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        return
    need = cells * ORACLE_BYTES_PER_CELL
    if avail < need:
        pytest.skip(f"host memory {avail / 2**30:.0f} GiB < {need / 2**30:.0f} GiB needed")


def _pair(Simulation, oracle, name, res):
    from paper_1806_04960_b200.scenarios import build_scenario
    _need_host_memory(res[0] * res[1])
    sc = build_scenario(name, res)
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    return sc, sim, ref


def _step_both(sim, ref, n):
    for s in range(n):
        dtr = ref.advance()
        dtg = sim.advance()
        assert dtg == dtr, f"dt differs at step {ref.step_count}: {dtg!r} vs {dtr!r}"
        assert same(sim.q, ref.q), f"state differs at step {ref.step_count}"


def test_c5_slab_bench_window(Simulation, full_oracle):
    """The bench workload, wall-impact x-slab 4096 x 16384: steps 1-5 with
    advance() (state compared every step), then steps 6-25 through the device
    loop bench.py times; q, t and all 25 dt values equal the oracle's."""
    sc, sim, ref = _pair(Simulation, full_oracle, "wall-impact", (4096, 16384))
    _step_both(sim, ref, 5)
    ref.run_steps(20)
    sim.run_steps(20, chunk=10)
    assert sim.step_count == ref.step_count == 25
    assert sim.t == ref.t
    assert same(sim.dt_log(), np.array(ref.dt_log))
    assert same(sim.q, ref.q)
    wc = sim.work_counters()
    assert wc["y_faces"] > 0 and wc["n_second_order"] > 0


def test_c3_drop_20_steps(Simulation, full_oracle):
    sc, sim, ref = _pair(Simulation, full_oracle, "drop", (4096, 4096))
    _step_both(sim, ref, 20)
    assert sim.t == ref.t


def test_c4_weir_3_steps(Simulation, full_oracle):
    sc, sim, ref = _pair(Simulation, full_oracle, "weir", (16384, 8192))
    ref.run_steps(3)
    sim.run_steps(3)
    assert sim.t == ref.t
    assert same(sim.dt_log(), np.array(ref.dt_log))
    assert same(sim.q, ref.q)
