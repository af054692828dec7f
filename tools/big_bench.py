"""Global-state tier: device time of a PERTURB argmin range
on DFGs beyond shared memory, and on the paper-shaped DFGs with the tier
forced (PP_TIER=global) next to their shared-memory tier.  One JSON line per
case: placements/s, the INT32-issue roofline fraction (bench.py's algorithmic
count), and L2-resident state bytes.

  python tools/big_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402
from bench import alg_counts  # noqa: E402

PEAK = 148 * 128 * 1.965e9   # int32 issue, as bench.py


def timed(g, M, count, reps=3):
    base = np.zeros(g.K, dtype=np.uint8)
    g.search_range(M, pp.GEN_PERTURB, 1, 8, base, 0, count)   # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        out = g.search_range(M, pp.GEN_PERTURB, 2 + r, 8, base, 0, count)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, pp.u64(out)


if __name__ == "__main__":
    cases = [("random_wide_K900", synth.random_dag(5, 900, avg_deg=1.5), None),
             ("random_long_K3200", synth.random_dag(11, 3200, avg_deg=1.2, max_in=3, window=40), None),
             ("random_long_K12000", synth.random_dag(12, 12000, avg_deg=1.2, max_in=3, window=40), None)]
    for name in ("inception_v3", "gnmt", "biglstm"):
        spec = getattr(synth, name)()
        cases += [(name, spec, "shared"), (name, spec, "global")]
    for name, spec, tier in cases:
        if tier == "global":
            os.environ["PP_TIER"] = "global"
        else:
            os.environ.pop("PP_TIER", None)
        ops, _ = alg_counts(spec)
        budgets = ["4096", "64"] if tier != "shared" else [None]
        for mb in budgets:   # PP_BIG_STATE_MB: scratch cap on resident warps (A/B)
            if mb:
                os.environ["PP_BIG_STATE_MB"] = mb
            g = pp.Dfg(spec)
            for M in (2, 4):
                count = max(1_000_000, int(4e11 / ops))
                ms, out = timed(g, M, count)
                rate = count / (ms / 1e3)
                print(json.dumps({"dfg": name, "K": g.K, "W": g.W, "image_bytes": g.image_bytes,
                                  "tier": "global" if g.tier == pp.TIER_GLOBAL else "shared", "state_mb": mb,
                                  "M": M, "count": count, "ms": ms, "placements_per_s": rate,
                                  "frac": rate * ops / PEAK, "best": [int(out[0]), int(out[1])]}), flush=True)
            g.close()
        os.environ.pop("PP_BIG_STATE_MB", None)
    os.environ.pop("PP_TIER", None)
