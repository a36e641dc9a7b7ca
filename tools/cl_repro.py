import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2005_01182_b200 import Solver
from paper_2005_01182_b200.api import OPT_ENGINE, OPT_MAX_CTAS
s = Solver(0); s.set_option(OPT_ENGINE, 11); s.set_option(OPT_MAX_CTAS, int(os.environ.get("G", "4")))
n = int(os.environ.get("N", "300"))
c = np.random.default_rng(5).integers(0, int(os.environ.get("HI", "2")), size=(n, n)).astype(np.int32)
r = s.solve(c, int(os.environ.get("SEED", "0")))
print("ok", r.total_cost)
