import os, sys; sys.path.insert(0, os.getcwd())
from paper_2005_01182_b200 import Solver, workloads as W
s = Solver(0)
c = W.CONFIGS["c1"].make(); o = s.auction(c, True); print("c1", o["bids"], o["seconds"])
