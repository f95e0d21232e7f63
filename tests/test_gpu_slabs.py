"""x-slab device path on one GPU (GPU test).

Several DeviceSlab handles (i_begin/i_end subsets of one grid, each on its own
stream) are stepped in one process; the collectives of the multi-GPU driver
are emulated on the host (MAX of the reduction vectors, halo buffers copied
between neighbours), never by kernels that wait on each other.  The owned
columns must match the single-domain oracle bit for bit, including the error
stop of the 200x100 dambreak at step 309."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _slabs(torch, scen, res, world, device_ic=False):
    from paper_1806_04960_b200.distributed import DeviceSlab, slab_bounds, stored_range
    from paper_1806_04960_b200.scenarios import build_scenario
    out = []
    for r in range(world):
        i0, i1 = slab_bounds(res[0], world, r)
        lo, hi = stored_range(res[0], i0, i1)
        sc = build_scenario(scen, res, columns=(lo, hi), host_state=not device_ic)
        out.append(DeviceSlab(sc.grid, sc.params, sc.q0, lo, sc.boundary, 0.45, i0, i1, 0,
                              ic=sc.ic if device_ic else None))
    return out


def _reduce(torch, slabs):
    torch.cuda.synchronize()
    red = torch.stack([s.red for s in slabs]).max(dim=0).values
    for s in slabs:
        s.red.copy_(red)
    torch.cuda.synchronize()


def _halo(torch, slabs):
    for s in slabs:
        with s.stream_ctx():
            s.pack_halo()
    torch.cuda.synchronize()
    W = len(slabs)
    half = slabs[0].send.numel() // 2
    for r, s in enumerate(slabs):
        if r > 0:
            s.recv[:half].copy_(slabs[r - 1].send[half:])
        if r < W - 1:
            s.recv[half:].copy_(slabs[r + 1].send[:half])
    torch.cuda.synchronize()
    for r, s in enumerate(slabs):
        s.unpack_halo(r > 0, r < W - 1)
    torch.cuda.synchronize()


def _exchange(torch, slabs):
    torch.cuda.synchronize()
    W = len(slabs)
    half = slabs[0].send.numel() // 2
    for r, s in enumerate(slabs):
        if r > 0:
            s.recv[:half].copy_(slabs[r - 1].send[half:])
        if r < W - 1:
            s.recv[half:].copy_(slabs[r + 1].send[:half])
    torch.cuda.synchronize()


def _set_peers(slabs):
    """Halo over peer memory between the slabs (same GPU, direct pointers)."""
    W = len(slabs)
    for r, s in enumerate(slabs):
        s.set_peers(slabs[r - 1].peer_desc() if r > 0 else None,
                    slabs[r + 1].peer_desc() if r < W - 1 else None)


def _run(torch, slabs, steps, overlap=False, peer=False):
    """Drive the slabs like distributed.DistributedSimulation: either
    step_local -> all-reduce -> finalize -> halo exchange, or the overlapped
    step_begin (edge strips + pack on the edge stream, interior strips on the
    main stream) -> exchange -> unpack_halo_next -> step_end -> all-reduce ->
    finalize."""
    for s in slabs:
        s.prepare_local()
        s.prepare_pack()
    _reduce(torch, slabs)
    for s in slabs:
        s.prepare_unpack()
    for s in slabs:
        assert s.check_prepare()[1] == 0
    W = len(slabs)
    for _ in range(steps):
        if peer:
            # edges + peer halo stores, interior; the emulated all-reduce (a
            # device synchronisation) orders the stores before the next step
            for s in slabs:
                if overlap:
                    s.step_begin_peer(None, None, 0)
                    s.step_end()
                else:
                    s.step_local(None, None, 0)
                    s.push_halo_next()
            _reduce(torch, slabs)
            for s in slabs:
                s.finalize()
        elif overlap:
            for s in slabs:
                s.step_begin(None, None, 0)
            _exchange(torch, slabs)
            for r, s in enumerate(slabs):
                s.unpack_halo_next(r > 0, r < W - 1)
            for s in slabs:
                s.step_end()
            _reduce(torch, slabs)
            for s in slabs:
                s.finalize()
        else:
            for s in slabs:
                s.step_local(None, None, 0)
            _reduce(torch, slabs)
            for s in slabs:
                s.finalize()
            _halo(torch, slabs)
        st = [s.status() for s in slabs]
        if st[0]["stop"] > 0:
            return [s.last_error() for s in slabs]
    return None


@pytest.mark.parametrize("world", [2, 3])
def test_device_slabs_bitexact(torch_cuda, oracle, world):
    from paper_1806_04960_b200.scenarios import build_scenario
    res = (131, 70)
    slabs = _slabs(torch_cuda, "wall-impact", res, world)
    assert _run(torch_cuda, slabs, 15) is None
    q = np.concatenate([s.owned_state() for s in slabs], axis=0)
    sc = build_scenario("wall-impact", res)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref.run_steps(15)
    assert np.array_equal(q, ref.q)
    assert all(s.status()["t"] == ref.t for s in slabs)


def test_device_slabs_error_stop(torch_cuda):
    slabs = _slabs(torch_cuda, "dambreak-dry", (200, 100), 2)
    errs = _run(torch_cuda, slabs, 400)
    assert errs is not None
    for code, key, step, _ in errs:
        assert (code, divmod(key, 100), step) == (4, (98, 37), 309)


@pytest.mark.parametrize("world", [2, 3])
def test_device_slabs_overlapped_bitexact(torch_cuda, oracle, world):
    """Overlapped step with a real edge/interior split (>= 3 column strips
    per slab at 64-thread CTAs) against the oracle."""
    from paper_1806_04960_b200.scenarios import build_scenario
    res = (400 * world, 96)
    slabs = _slabs(torch_cuda, "wall-impact", res, world)
    assert _run(torch_cuda, slabs, 12, overlap=True) is None
    q = np.concatenate([s.owned_state() for s in slabs], axis=0)
    sc = build_scenario("wall-impact", res)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref.run_steps(12)
    assert np.array_equal(q, ref.q)
    assert all(s.status()["t"] == ref.t for s in slabs)


def test_device_slabs_overlapped_error_stop(torch_cuda):
    slabs = _slabs(torch_cuda, "dambreak-dry", (200, 100), 2)
    errs = _run(torch_cuda, slabs, 400, overlap=True)
    assert errs is not None
    for code, key, step, _ in errs:
        assert (code, divmod(key, 100), step) == (4, (98, 37), 309)


@pytest.mark.parametrize("world,overlap", [(2, True), (3, True), (3, False)])
def test_device_slabs_peer_halo_bitexact(torch_cuda, oracle, world, overlap):
    """Halo over peer memory: each slab's step stores its boundary columns
    straight into the neighbours' halo (k_push_halo), with a real edge /
    interior split; bit-identical to the single-domain oracle."""
    from paper_1806_04960_b200.scenarios import build_scenario
    res = (400 * world, 96)
    slabs = _slabs(torch_cuda, "wall-impact", res, world)
    _set_peers(slabs)
    assert _run(torch_cuda, slabs, 12, overlap=overlap, peer=True) is None
    q = np.concatenate([s.owned_state() for s in slabs], axis=0)
    sc = build_scenario("wall-impact", res)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref.run_steps(12)
    assert np.array_equal(q, ref.q)
    assert all(s.status()["t"] == ref.t for s in slabs)


def test_device_slabs_peer_halo_error_stop(torch_cuda):
    slabs = _slabs(torch_cuda, "dambreak-dry", (200, 100), 2)
    _set_peers(slabs)
    errs = _run(torch_cuda, slabs, 400, overlap=True, peer=True)
    assert errs is not None
    for code, key, step, _ in errs:
        assert (code, divmod(key, 100), step) == (4, (98, 37), 309)


def test_device_slabs_peer_halo_fused_chain(torch_cuda, oracle):
    """Slabs of two column strips (no edge/interior split) with long columns
    (ny >= 2048: the detection is chained inside the step kernel): the edge
    launch is the whole step, and its last row segment stores the halo
    columns' detection into the neighbours along with the state."""
    from paper_1806_04960_b200.scenarios import build_scenario
    res = (200, 2048)
    slabs = _slabs(torch_cuda, "wall-impact", res, 2)
    _set_peers(slabs)
    assert _run(torch_cuda, slabs, 10, overlap=True, peer=True) is None
    q = np.concatenate([s.owned_state() for s in slabs], axis=0)
    sc = build_scenario("wall-impact", res)
    ref = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    ref.run_steps(10)
    assert np.array_equal(q, ref.q)


def test_device_slabs_peer_halo_gamma7_matches_collective(torch_cuda):
    """gamma != 1 (pow; the 64-thread gamma != 1 edge kernel stores the halo
    into the peers): slabs with the peer-memory halo equal, bit for bit, the
    same slabs with the packed halo exchange (the arithmetic is the same; only
    the halo transport differs), and the single-handle Simulation."""
    import numpy as np
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    res = (400, 32)
    a = _slabs(torch_cuda, "tait7", res, 2)
    b = _slabs(torch_cuda, "tait7", res, 2)
    _set_peers(a)
    assert _run(torch_cuda, a, 6, overlap=True, peer=True) is None
    assert _run(torch_cuda, b, 6, overlap=True) is None
    qa = np.concatenate([s.owned_state() for s in a], axis=0)
    qb = np.concatenate([s.owned_state() for s in b], axis=0)
    assert np.array_equal(qa.view(np.uint64), qb.view(np.uint64))
    sc = build_scenario("tait7", res)
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.run_steps(6)
    assert np.array_equal(qa.view(np.uint64), sim.q.view(np.uint64))
