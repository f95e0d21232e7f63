"""Multi-rank x-slab driver (paper_1806_04960_b200.distributed) over gloo on
the CPU, with the oracle as the slab backend (oracle.OracleSlab mirrors the
device status machine).  Checks that the host logic of the multi-GPU path --
slab bounds, halo exchange, the MAX-allreduced [error key, CFL rate] vector,
commit/stop decisions and error reporting -- reproduces the single-domain run
bit for bit, including the reference's abort step and cell."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scen, res, steps, out, run_until, overlap=False):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch.distributed as dist
    import oracle as orc
    from paper_1806_04960_b200.distributed import (DistributedSimulation, slab_bounds,
                                                   stored_range)
    from paper_1806_04960_b200.errors import SimulationError
    from paper_1806_04960_b200.scenarios import build_scenario
    orc.set_threads(1)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    nx = res[0]
    i0, i1 = slab_bounds(nx, world, rank)
    lo, hi = stored_range(nx, i0, i1)
    sc = build_scenario(scen, res, columns=(lo, hi))
    be = orc.OracleSlab(sc.grid, sc.params, sc.q0, lo, sc.boundary, 0.45, i0, i1)
    sim = DistributedSimulation(be, sc.grid, overlap=overlap)
    err = None
    try:
        if run_until is not None:
            sim.run_until(run_until)
        else:
            sim.run_steps(steps, check_every=5)
    except SimulationError as e:
        err = (str(e), e.step, e.cell)
    np.savez(os.path.join(out, f"rank{rank}.npz"), q=be.owned_state(), i0=i0, i1=i1,
             t=sim.t, step=sim.step_count, err=np.array(repr(err)))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, scen, res, steps=None, run_until=None, overlap=False):
    out = tempfile.mkdtemp()
    mp.spawn(_worker, args=(world, _free_port(), scen, res, steps, out, run_until, overlap),
             nprocs=world, join=True)
    parts = [np.load(os.path.join(out, f"rank{r}.npz")) for r in range(world)]
    q = np.concatenate([p["q"] for p in parts], axis=0)
    return q, parts


def _reference(oracle, scen, res, steps=None, run_until=None):
    from paper_1806_04960_b200.scenarios import build_scenario
    sc = build_scenario(scen, res)
    sim = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    err = None
    try:
        if run_until is not None:
            sim.run_until(run_until)
        else:
            sim.run_steps(steps)
    except oracle.OracleError as e:
        err = (str(e), e.step, e.cell)
    return sim, err


@pytest.mark.parametrize("world,overlap", [(2, False), (3, False), (2, True), (3, True)])
def test_slabs_bitexact(oracle, world, overlap):
    q, parts = _run(world, "wall-impact", (61, 32), steps=12, overlap=overlap)
    ref, err = _reference(oracle, "wall-impact", (61, 32), steps=12)
    assert err is None
    assert np.array_equal(q, ref.q)
    for p in parts:
        assert float(p["t"]) == ref.t and int(p["step"]) == 12


def test_slabs_run_until(oracle):
    q, parts = _run(2, "perturbed-lake", (40, 32), run_until=0.004)
    ref, err = _reference(oracle, "perturbed-lake", (40, 32), run_until=0.004)
    assert np.array_equal(q, ref.q)
    assert float(parts[0]["t"]) == ref.t and int(parts[1]["step"]) == ref.step_count


@pytest.mark.slow
def test_slabs_error_path(oracle):
    """200x100 dry dambreak: the reference aborts at step 309, cell (98, 37);
    split over 2 ranks at column 100 the distributed run reports the same
    error on every rank and keeps the state of step 309."""
    q, parts = _run(2, "dambreak-dry", (200, 100), steps=400)
    ref, err = _reference(oracle, "dambreak-dry", (200, 100), steps=400)
    assert err is not None
    for p in parts:
        assert str(p["err"]) == repr(err)
        assert int(p["step"]) == ref.step_count
    assert np.array_equal(q, ref.q)


def test_slab_bounds():
    from paper_1806_04960_b200.distributed import slab_bounds, stored_range
    for nx, w in ((61, 3), (4096 * 8, 8), (10, 4)):
        b = [slab_bounds(nx, w, r) for r in range(w)]
        assert b[0][0] == 0 and b[-1][1] == nx
        assert all(b[k][1] == b[k + 1][0] for k in range(w - 1))
        assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
    assert stored_range(100, 0, 50) == (0, 52)
    assert stored_range(100, 50, 100) == (48, 100)
