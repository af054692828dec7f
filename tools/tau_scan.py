"""Search effectiveness vs the PERTURB flip threshold τ.

For each paper-shaped DFG and M: the EFT seed's makespan (candidate 0 of
round 0), then T_M after `rounds` × `count` PERTURB candidates at several τ,
with the improvement over the seed.  One JSON line per case.

  python tools/tau_scan.py [--count 10000000] [--rounds 10] [--taus 1,2,3,4,8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=10_000_000)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--taus", default="1,2,3,4,6,8,16")
    ap.add_argument("--models", default="inception_v3,gnmt,biglstm")
    ap.add_argument("--Ms", default="2,4,8")
    ap.add_argument("--seed", type=int, default=13257)
    a = ap.parse_args()
    for model in a.models.split(","):
        g = pp.Dfg(getattr(synth, model)())
        for M in map(int, a.Ms.split(",")):
            base = g.eft_place(M)
            seed_mk = g.search_best(M, pp.GEN_PERTURB, a.seed, 1, rounds=1, tau=8, base=base).best_makespan_ps
            for tau in map(int, a.taus.split(",")):
                t = time.perf_counter()
                r = g.search_best(M, pp.GEN_PERTURB, a.seed, a.count, rounds=a.rounds, tau=tau, base=base)
                dt = time.perf_counter() - t
                print(json.dumps({"model": model, "K": g.K, "M": M, "tau": tau, "flips_per_cand": g.K * tau / 256,
                                  "seed_ps": seed_mk, "T_M_ps": r.best_makespan_ps, "best_round": r.best_round,
                                  "best_index": r.best_index, "improve": 1 - r.best_makespan_ps / seed_mk,
                                  "su_seed": g.t1 / seed_mk, "su": g.t1 / r.best_makespan_ps,
                                  "rate_gps": r.evaluated / dt / 1e9}), flush=True)
        g.close()
