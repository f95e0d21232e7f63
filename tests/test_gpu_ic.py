"""Device-side initial conditions: the
column-equilibrium scenarios built by wb_init_column_equilibrium equal the
host builder bit for bit, and the runs from them equal the runs from an
uploaded host state (GPU tests)."""
import numpy as np
import pytest

from golden_util import same

pytestmark = pytest.mark.gpu

CASES = [("dambreak-dry", (200, 100)), ("dambreak-wet", (400, 40)),
         ("dambreak-step-dry", (400, 40)), ("dambreak-step-wet", (400, 40)),
         ("weir", (600, 84)), ("wall-impact", (256, 144)), ("lake", (512, 256)),
         ("equilibrium-flat", (100, 100)), ("equilibrium-obstacle", (100, 100))]


@pytest.fixture(scope="module")
def Simulation():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_04960_b200.timestepper import Simulation
    return Simulation


@pytest.mark.parametrize("name,res", CASES)
def test_device_ic_equals_host(Simulation, name, res):
    from paper_1806_04960_b200.scenarios import build_scenario
    host = build_scenario(name, res)
    dev_sc = build_scenario(name, res, host_state=False)
    assert dev_sc.q0 is None and dev_sc.ic is not None
    sim_d = Simulation.from_scenario(dev_sc)
    assert same(sim_d.q, host.q0)
    sim_h = Simulation(host.grid, host.params, host.q0, host.boundary)
    for _ in range(5):
        assert sim_d.advance() == sim_h.advance()
    assert same(sim_d.q, sim_h.q) and sim_d.t == sim_h.t


def test_device_ic_bench_slab(Simulation):
    """The bench workload (C5 slab 4096 x 16384) built on the device equals the
    host build (2.7 GB, compared via the device download)."""
    from paper_1806_04960_b200.scenarios import build_scenario
    host = build_scenario("wall-impact", (4096, 16384))
    sim_d = Simulation.from_scenario(build_scenario("wall-impact", (4096, 16384),
                                                    host_state=False))
    assert same(sim_d.q, host.q0)


@pytest.mark.parametrize("name,res", [("wall-impact", (300, 160)), ("weir", (330, 60))])
def test_device_ic_slabs(Simulation, name, res):
    """x-slabs whose columns are built on the device (what bench.py's N > 1
    path does) hold the same state as host-built, uploaded slabs."""
    import torch
    from test_gpu_slabs import _slabs
    a = _slabs(torch, name, res, 3, device_ic=True)
    b = _slabs(torch, name, res, 3)
    for x, y in zip(a, b):
        assert same(x.owned_state(), y.owned_state())
