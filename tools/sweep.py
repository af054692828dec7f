"""BASELINE config 5: the full end-to-end projection sweep on one GPU.

For each paper-shaped DFG (Inception-V3, GNMT, BigLSTM): a PERTURB search for
M ∈ {2, 4, 8} (rounds × count candidates each, seeded with the EFT placement)
gives T_M (T_1 = ΣΔ needs no search); for GNMT and BigLSTM — which the paper
split by pipelining — the GPipe search (§8(f) f3, stage cuts ×
m ∈ {1..32}) gives a second T_M, and the projection takes the better of the
two.  Then the projection over M ∈ {1, 2, 4, 8} × N = 1..N_max with the
16-knot epochs curve (reading R13) in EQ5 and TIME modes, and the crossover.
Prints one JSON line per model plus a summary line.

  python tools/sweep.py [--count 1000000] [--rounds 10] [--nmax 1024]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402

MODELS = ["inception_v3", "gnmt", "biglstm"]
MS = [1, 2, 4, 8]
PIPELINED = ("gnmt", "biglstm")
MICRO = [1, 2, 4, 8, 16, 32]


def run(count, rounds, nmax, seed=13257, tau=8):
    out = []
    total = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    ev0.record()
    for model in MODELS:
        g = pp.Dfg(getattr(synth, model)())
        T = [g.t1]
        su, su_pipe = {}, {}
        for M in MS[1:]:
            r = g.search_best(M, pp.GEN_PERTURB, seed, count, rounds=rounds, tau=tau, base=g.eft_place(M))
            t_m = r.best_makespan_ps
            total += r.evaluated
            su[M] = g.t1 / t_m
            if model in PIPELINED and M <= 4:          # M = 8 spans 10^13 stage splits
                p = g.pipeline_search(M, MICRO)
                total += p["candidates"]
                su_pipe[M] = g.t1 / p["makespan_ps"]
                t_m = min(t_m, p["makespan_ps"])
            T.append(t_m)
        res = {"model": model, "K": g.K, "T_ps": dict(zip(MS, T)), "su_mp_placement": su,
               "su_mp_pipeline": su_pipe, "su_mp": {M: g.t1 / t for M, t in zip(MS[1:], T[1:])}}
        for mode, name in ((0, "EQ5"), (1, "TIME")):
            sc = synth.sweep_scenario(model, g.t1, g.grad_bytes, ar_mode=mode)
            cells = pp.project_e2e(sc, MS, T, nmax)
            x = pp.crossover(cells, MS, nmax)
            res[name] = {"n_star": x.n_star, "m_at_n_star": x.m_at_n_star, "n_star_M": dict(zip(MS, x.n_star_M)),
                         "persistent_M": dict(zip(MS, x.persistent_M)), "n_star_vs_best_dp": x.n_star_vs_best_dp,
                         "best_m_at_pow2": {N: x.best_m[N - 1] for N in (8, 16, 32, 64, 128, 256, 512, 1024) if N <= nmax}}
        out.append(res)
        g.close()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    return out, total, ms, time.perf_counter() - t_wall


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--nmax", type=int, default=1024)
    a = ap.parse_args()
    run(10_000, 1, a.nmax)          # warm-up (module load, attributes)
    out, total, ms, wall = run(a.count, a.rounds, a.nmax)
    for r in out:
        print(json.dumps(r))
    print(json.dumps({"config": "BASELINE config 5 full sweep", "placements": total, "gpu_ms": ms,
                      "placements_per_s": total / (ms / 1e3), "wall_s": wall,
                      "cells": len(MODELS) * len(MS) * a.nmax * 2}))
