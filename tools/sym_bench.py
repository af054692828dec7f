"""Exhaustive GRAY search with and without the relabelling-class reduction
(DESIGN.md §12b): device time of pp_search_best over the
whole M^K space, reduced (default) vs unreduced (PP_NO_SYM=1), and both
results.  One JSON line per case.

  python tools/sym_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402


def timed(g, M, space, reps):
    g.search_best(M, pp.GEN_GRAY, 0, space)      # warm-up (module load, NP choice)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = g.search_best(M, pp.GEN_GRAY, 0, space)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


def classes(K, M):
    prev = [1] * (M + 2)
    for _ in range(1, K):
        prev = [0] + [m * prev[m] + (prev[m + 1] if m < M else 0) for m in range(1, M + 1)] + [0]
    return prev[1]


if __name__ == "__main__":
    cases = [("toy12", synth.toy12(), M) for M in (2, 3, 4)]
    r16 = synth.random_dag(1616, 16, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)
    cases += [("random_K16", r16, M) for M in (2, 3, 4)]
    # M = 2 spaces large enough that the launch is not latency-bound (2^24, 2^28)
    for K in (24, 28):
        cases.append((f"random_K{K}", synth.random_dag(1600 + K, K, avg_deg=1.6, max_cost=10**6, max_bytes=10**6), 2))
    for name, spec, M in cases:
        g = pp.Dfg(spec)
        K = g.K
        space = M ** K
        reps = 20 if space < 10**7 else 3
        os.environ.pop("PP_NO_SYM", None)
        t_sym, r_sym = timed(g, M, space, reps)
        os.environ["PP_NO_SYM"] = "1"
        t_full, r_full = timed(g, M, space, max(1, reps // 3))
        os.environ.pop("PP_NO_SYM", None)
        n_cls = classes(K, M)
        print(json.dumps({"dfg": name, "K": K, "M": M, "space": space, "classes": n_cls,
                          "space_over_classes": space / n_cls, "ms_reduced": t_sym, "ms_full": t_full,
                          "speedup": t_full / t_sym, "same_result": (r_sym.best_makespan_ps, r_sym.best_index) ==
                          (r_full.best_makespan_ps, r_full.best_index),
                          "best_ps": r_sym.best_makespan_ps, "best_index": r_sym.best_index,
                          "placements_per_s_effective": space / (t_sym / 1e3)}), flush=True)
        g.close()
