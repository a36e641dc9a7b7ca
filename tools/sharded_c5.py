"""Config 5 column-sharded over torchrun ranks (NCCL exchange when each rank has
its own GPU, else gloo callbacks), vs the 1-GPU engine.  Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2005_01182_b200 import Solver, workloads as W
from paper_2005_01182_b200.sharded import column_span, init_exchange, solve_sharded
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
dist.init_process_group("gloo")
ndev = torch.cuda.device_count()
dev = local % ndev
torch.cuda.set_device(dev)
key = os.environ.get("CFG", "c5")
c = W.CONFIGS[key].make(); n = c.shape[0]
cb, nc = column_span(n, world, rank)
slab = torch.from_numpy(np.ascontiguousarray(c[:, cb:cb + nc])).cuda()
s = Solver(dev)
mode = "nccl" if ndev >= world else "group"
init_exchange(s, mode)
dist.barrier(); t0 = time.perf_counter()
r2c, u, v, tot, st = solve_sharded(s, slab, n, cb, 1)
dist.barrier(); t = time.perf_counter() - t0
single = None
if rank == 0 and world == 1:
    s2 = Solver(dev); dc = torch.from_numpy(c).cuda()
    rr = torch.empty(n, dtype=torch.int32, device="cuda"); uu = torch.empty(n, dtype=torch.int64, device="cuda")
    vv = torch.empty_like(uu); tt = torch.empty(1, dtype=torch.int64, device="cuda")
    for _ in range(2): st1 = s2.solve_into(dc, n, n, 1, rr, uu, vv, tt)
    single = {"seconds": st1.seconds, "same_cost": int(tt.item()) == tot}
if rank == 0:
    print(json.dumps({"config": key, "world": world, "exchange": mode, "sharded_seconds": t,
                      "rounds": st["rounds"], "epochs": st["phases"], "dual_steps": st["dual_steps"],
                      "total_cost": tot, "one_gpu_engine": single}), flush=True)
dist.destroy_process_group()
