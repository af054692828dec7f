"""Is the EFT seed a local optimum?  (for GNMT and
BigLSTM at M = 2 no PERTURB candidate ever beats the seed.)

For each paper-shaped DFG and M, every placement at Hamming distance 1 and 2
from the EFT-greedy placement — K·(M−1) and
C(K,2)·(M−1)² placements — is evaluated exactly through pp_eval_placements,
and the best neighbour's makespan is compared with the seed's.  If none is
better the seed is 2-opt locally optimal under op moves, which is what a
PERTURB search at small τ explores.  One JSON line per case.

  python tools/local_opt.py [--models gnmt,biglstm] [--Ms 2,4,8]
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402


def neighbours(p0, M, dist, chunk=1 << 16):
    """Batches (uint8 [n, K] on the GPU) of the placements at Hamming distance
    `dist` ∈ {1, 2} from p0."""
    K = len(p0)
    base = torch.as_tensor(p0, dtype=torch.uint8, device="cuda")
    rows = []

    def flush():
        nonlocal rows
        if rows:
            idx = torch.as_tensor(np.array(rows, dtype=np.int64), device="cuda")
            t = base.repeat(len(rows), 1)
            for c in range(dist):
                t[torch.arange(len(rows), device="cuda"), idx[:, 2 * c]] = idx[:, 2 * c + 1].to(torch.uint8)
            rows = []
            return t
        return None

    if dist == 1:
        it = ((i, v) for i in range(K) for v in range(M) if v != p0[i])
    else:
        it = ((i, a, j, b) for i, j in itertools.combinations(range(K), 2)
              for a in range(M) if a != p0[i] for b in range(M) if b != p0[j])
    for x in it:
        rows.append(x)
        if len(rows) == chunk:
            yield flush()
    t = flush()
    if t is not None:
        yield t


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="inception_v3,gnmt,biglstm")
    ap.add_argument("--Ms", default="2,4,8")
    a = ap.parse_args()
    for model in a.models.split(","):
        g = pp.Dfg(getattr(synth, model)())
        for M in map(int, a.Ms.split(",")):
            p0 = g.eft_place(M)
            seed_mk = int(pp.u64(g.eval_placements(M, torch.as_tensor(p0[None], device="cuda")))[0])
            out = {"model": model, "K": g.K, "M": M, "seed_ps": seed_mk}
            for dist in (1, 2):
                best, n, better = None, 0, 0
                for t in neighbours(p0, M, dist):
                    v = pp.u64(g.eval_placements(M, t))
                    n += len(v)
                    better += int((v < seed_mk).sum())
                    m = int(v.min())
                    best = m if best is None else min(best, m)
                out[f"d{dist}_count"] = n
                out[f"d{dist}_best_ps"] = best
                out[f"d{dist}_improving"] = better
            out["locally_optimal_2opt"] = out["d1_improving"] == 0 and out["d2_improving"] == 0
            print(json.dumps(out), flush=True)
        g.close()
