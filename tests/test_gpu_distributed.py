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


def test_nccl_world1_matches_simulation():
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
        dsim = DistributedSimulation(be, sc.grid)
        dsim.run_steps(25, check_every=8)
        full = build_scenario("wall-impact", res)
        sim = Simulation(full.grid, full.params, full.q0, full.boundary)
        sim.run_steps(25)
        assert dsim.step_count == 25 and dsim.t == sim.t
        assert np.array_equal(be.owned_state(), sim.q)
        t_end = dsim.t + 5 * sim.stats.dt
        dsim.run_until(t_end)
        sim.run_until(t_end)
        assert dsim.t == sim.t and np.array_equal(be.owned_state(), sim.q)
    finally:
        dist.destroy_process_group()
