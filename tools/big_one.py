"""One global-tier PERTURB argmin launch (for ncu): python tools/big_one.py wide|long [M]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402

specs = {"wide": lambda: synth.random_dag(5, 900, avg_deg=1.5),
         "long": lambda: synth.random_dag(11, 3200, avg_deg=1.2, max_in=3, window=40)}
name = sys.argv[1]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = pp.Dfg(specs[name]())
base = np.zeros(g.K, dtype=np.uint8)
for r in range(3):
    out = g.search_range(M, pp.GEN_PERTURB, 1 + r, 8, base, 0, 4_000_000)
torch.cuda.synchronize()
print(name, M, g.tier, pp.u64(out))
