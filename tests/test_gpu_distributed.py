"""The NCCL multi-GPU driver on a single GPU (world size 1, GPU test): the
aliased reduction vector, the all-reduce and the step pipeline of
distributed.DistributedSimulation reproduce the single-handle Simulation."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("overlap,graphs,halo", [(False, False, "collective"),
                                                 (False, True, "collective"),
                                                 (True, True, "collective"),
                                                 (True, True, "peer"),
                                                 (False, True, "peer")])
def test_nccl_world1_matches_simulation(overlap, graphs, halo):
    """NCCL world 1 (halo exchange skipped, all-reduce real): plain and
    overlapped steps, eager and CUDA-graph-captured chunks, equal the
    single-domain Simulation bit for bit; run_until twice and a later
    advance() keep stepping (a reached target does not stick)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    from paper_1806_04960_b200.distributed import (DeviceSlab, DistributedSimulation,
                                                   slab_bounds, stored_range)
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda:0"))
    try:
        res = (300, 160)
        i0, i1 = slab_bounds(res[0], 1, 0)
        lo, hi = stored_range(res[0], i0, i1)
        sc = build_scenario("wall-impact", res, columns=(lo, hi))
        be = DeviceSlab(sc.grid, sc.params, sc.q0, lo, sc.boundary, 0.45, i0, i1, 0)
        dsim = DistributedSimulation(be, sc.grid, overlap=overlap, graphs=graphs, halo=halo)
        assert dsim.halo == halo
        dsim.run_steps(25, check_every=8)
        assert dsim.use_graphs == graphs  # the capture worked
        full = build_scenario("wall-impact", res)
        sim = Simulation(full.grid, full.params, full.q0, full.boundary)
        sim.run_steps(25)
        assert dsim.step_count == 25 and dsim.t == sim.t
        assert np.array_equal(be.owned_state(), sim.q)
        t_end = dsim.t + 5 * sim.stats.dt
        dsim.run_until(t_end)
        sim.run_until(t_end)
        assert dsim.t == sim.t and np.array_equal(be.owned_state(), sim.q)
        t_end2 = dsim.t + 3 * sim.stats.dt
        dsim.run_until(t_end2)
        sim.run_until(t_end2)
        dt_d, dt_s = dsim.advance(), sim.advance()
        assert dt_d == dt_s and dsim.step_count == sim.step_count
        assert dsim.t == sim.t and np.array_equal(be.owned_state(), sim.q)
        dsim.run_steps(8, check_every=8)
        sim.run_steps(8)
        assert np.array_equal(be.owned_state(), sim.q)
    finally:
        dist.destroy_process_group()


def _gloo_worker(rank, world, port, scen, res, steps, out, overlap, halo="collective"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_1806_04960_b200.distributed import (DeviceSlab, DistributedSimulation,
                                                   slab_bounds, stored_range)
    from paper_1806_04960_b200.errors import SimulationError
    from paper_1806_04960_b200.scenarios import build_scenario
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    i0, i1 = slab_bounds(res[0], world, rank)
    lo, hi = stored_range(res[0], i0, i1)
    sc = build_scenario(scen, res, columns=(lo, hi))
    be = DeviceSlab(sc.grid, sc.params, sc.q0, lo, sc.boundary, 0.45, i0, i1, 0)
    dsim = DistributedSimulation(be, sc.grid, overlap=overlap, halo=halo)
    assert dsim.halo == halo  # peer: CUDA IPC between the two processes worked
    err = None
    try:
        dsim.run_steps(steps, check_every=7)
    except SimulationError as e:
        err = (str(e), e.step, e.cell)
    np.savez(os.path.join(out, f"rank{rank}.npz"), q=be.owned_state(), t=dsim.t,
             step=dsim.step_count, err=np.array(repr(err)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scen,res,steps,overlap,halo", [
    ("wall-impact", (300, 160), 25, True, "collective"),
    ("wall-impact", (300, 160), 25, False, "collective"),
    ("dambreak-dry", (200, 100), 400, True, "collective"),
    ("wall-impact", (900, 96), 25, True, "peer"),
    ("wall-impact", (300, 160), 25, False, "peer"),
    ("dambreak-dry", (200, 100), 400, True, "peer")])
def test_device_slabs_two_processes_gloo(scen, res, steps, overlap, halo):
    """The full multi-process driver (torch.distributed, two ranks, device
    slabs on cuda:0, collectives staged through host memory by gloo) against
    the single-handle Simulation: same state, t and step; on the dry dambreak
    the same abort (step 309, cell (98, 37)) on both ranks.  halo="peer":
    the boundary columns go straight into the other process's buffers (CUDA
    IPC), ordered by the host-staged all-reduce."""
    import tempfile
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_04960_b200.errors import SimulationError
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    out = tempfile.mkdtemp()
    mp.spawn(_gloo_worker, args=(2, _port(), scen, res, steps, out, overlap, halo), nprocs=2,
             join=True)
    parts = [np.load(os.path.join(out, f"rank{r}.npz")) for r in range(2)]
    full = build_scenario(scen, res)
    sim = Simulation(full.grid, full.params, full.q0, full.boundary)
    err = None
    try:
        sim.run_steps(steps)
    except SimulationError as e:
        err = (str(e), e.step, e.cell)
    for p in parts:
        assert str(p["err"]) == repr(err)
        assert float(p["t"]) == sim.t and int(p["step"]) == sim.step_count
    assert np.array_equal(np.concatenate([p["q"] for p in parts], axis=0), sim.q)
    if scen == "dambreak-dry":
        assert err is not None and err[1] == 309 and err[2] == (98, 37)
