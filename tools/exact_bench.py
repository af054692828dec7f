"""Throughput of the exact-schedule branch and bound
against the oracle's enumeration, on toy-12 and seeded random DAGs.

    python tools/exact_bench.py            # one line per case, JSON
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402


def case(name, spec, M, n):
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, min(n, 64))   # warm-up (module load, tables)
    g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    os.environ["PP_NO_SYM"] = "1"
    g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    os.environ.pop("PP_NO_SYM", None)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    best, idx, unresolved = g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    e.record()
    torch.cuda.synchronize()
    gpu_s = s.elapsed_time(e) / 1e3
    # the same search without the relabelling-class reduction (§12b)
    os.environ["PP_NO_SYM"] = "1"
    s.record()
    best_u, idx_u, _ = g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    e.record()
    torch.cuda.synchronize()
    os.environ.pop("PP_NO_SYM", None)
    unreduced_s = s.elapsed_time(e) / 1e3
    mk, _ = g.eval_exact_generated(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    torch.cuda.synchronize()
    s.record()
    mk, ex = g.eval_exact_generated(M, pp.GEN_GRAY, 0, 0, None, 0, n)
    e.record()
    torch.cuda.synchronize()
    eval_s = s.elapsed_time(e) / 1e3
    # the oracle on a time-bounded prefix (about 10 s), then GPU parity on it
    t = time.perf_counter()
    oracle_n, ob = 0, (O.INFEASIBLE, 0)
    while oracle_n < n and time.perf_counter() - t < 10.0:
        m = od.exact_pi(M, O.gen(len(spec["fwd_ps"]), M, O.GEN_GRAY, 0, 0, None, oracle_n))
        if m < ob[0]:
            ob = (m, oracle_n)
        oracle_n += 1
    cpu_s = time.perf_counter() - t
    sub = g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, oracle_n)
    inorder = g.search_best(M, pp.GEN_GRAY, 0, n).best_makespan_ps
    print(json.dumps({
        "case": name, "K": len(spec["fwd_ps"]), "M": M, "candidates": n,
        "exact_best_ps": best, "index": idx, "unresolved": unresolved, "in_order_best_ps": inorder,
        "search_exact_s": gpu_s, "search_exact_unreduced_s": unreduced_s,
        "symmetry_speedup": unreduced_s / gpu_s, "same_as_unreduced": (best, idx) == (best_u, idx_u),
        "eval_exact_s": eval_s,
        "search_exact_per_s": n / gpu_s, "eval_exact_per_s": n / eval_s,
        "oracle_per_s": oracle_n / cpu_s, "oracle_sample": oracle_n,
        "oracle_prefix_parity": sub[:2] == ob,
    }), flush=True)


def main():
    case("toy12", synth.toy12(), 2, 2**12)
    case("toy12", synth.toy12(), 3, 3**12)
    case("random_dag_K14", synth.random_dag(5, 14, window=4), 2, 2**14)
    case("random_dag_K16", synth.random_dag(6, 16, window=4), 2, 2**16)
    case("random_dag_K10", synth.random_dag(7, 10, window=4), 4, 4**10)


if __name__ == "__main__":
    main()
