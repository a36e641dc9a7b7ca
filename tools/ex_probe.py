"""Config-4 solve time before/after other work in the same process (why the
bench's c4 extra reads slower than a fresh process)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2005_01182_b200 import Solver
s = Solver(0)
one = lambda tag: print(tag, {k: round(v["solve_ms"], 1) for k, v in bench.extras_single(s).items() if k == "c4"}, flush=True)
one("fresh")
x = torch.empty(1 << 28, dtype=torch.int32, device="cuda"); x.fill_(1); del x
one("after 1 GiB torch alloc+fill+free")
torch.cuda.empty_cache()
one("after empty_cache")
bench.extras_c5(s, 6554.2)
one("after c5")
torch.cuda.empty_cache()
one("after c5 + empty_cache")
