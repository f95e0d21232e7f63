"""Cost of the overlapped (edge/interior split) step against the plain step
on one GPU: the multi-rank driver at world size 1 over NCCL, C5 slab.
python tools/overlap_bench.py [steps]"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from paper_1806_04960_b200.distributed import (DeviceSlab, DistributedSimulation,  # noqa: E402
                                               slab_bounds, stored_range)
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda:0"))
res = (4096, 16384)
i0, i1 = slab_bounds(res[0], 1, 0)
lo, hi = stored_range(res[0], i0, i1)
sc = build_scenario("wall-impact", res, columns=(lo, hi))
import hashlib  # noqa: E402
digests = set()
for rnd in range(2):
    for overlap, graphs in ((False, False), (True, False), (False, True), (True, True)):
        be = DeviceSlab(sc.grid, sc.params, sc.q0, lo, sc.boundary, 0.45, i0, i1, 0)
        sim = DistributedSimulation(be, sc.grid, overlap=overlap, graphs=graphs)
        sim.run_steps(3)
        sim.enqueue_steps(steps)  # captures the graph (graphs=True) outside the timing
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(be.stream)
        sim.enqueue_steps(steps)
        e1.record(be.stream)
        torch.cuda.synchronize()
        st = sim._sync()
        sim._check(st)
        digests.add(hashlib.sha256(be.owned_state().tobytes()).hexdigest()[:16])
        print(f"overlap={overlap} graphs={graphs and sim.use_graphs}: "
              f"{e0.elapsed_time(e1) / steps:.3f} ms/step", flush=True)
        del sim, be
        torch.cuda.empty_cache()
print("states", "IDENTICAL" if len(digests) == 1 else f"DIFFER {digests}")
dist.destroy_process_group()
