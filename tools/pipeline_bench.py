"""Throughput of the pipeline-parallel MP search against
the oracle: exhaustive over stage cuts × micro-batch counts on the GNMT- and
BigLSTM-shaped DFGs.  One JSON line per case."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1907_13257_b200 as pp  # noqa: E402
import synth  # noqa: E402

MICRO = [1, 2, 4, 8, 16, 32]


def case(name, M):
    spec = getattr(synth, name)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    n = g.pipeline_space(M, len(MICRO))
    g.pipeline_search(M, MICRO)                       # warm-up (builds the tables)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    r = g.pipeline_search(M, MICRO)
    e.record()
    torch.cuda.synchronize()
    gpu_s = s.elapsed_time(e) / 1e3
    # oracle on a bounded prefix (~5 s)
    t = time.perf_counter()
    k = 1000
    while True:
        od.pipeline_search(M, MICRO, 0, min(k, n))
        dt = time.perf_counter() - t
        if dt > 5 or k >= n:
            break
        k *= 4
        t = time.perf_counter()
    k = min(k, n)
    (pb, pi), _ = g.pipeline_range(M, MICRO, 0, k)
    print(json.dumps({"case": name, "M": M, "candidates": n, "gpu_s": gpu_s, "gpu_per_s": n / gpu_s,
                      "best_ps": r["makespan_ps"], "su": od.t1 / r["makespan_ps"], "cuts": r["cuts"],
                      "micro": r["micro_batches"], "oracle_per_s": k / dt, "oracle_sample": k,
                      "prefix_parity": (pb, pi) == od.pipeline_search(M, MICRO, 0, k)}), flush=True)


def range_case(name, M, count):
    """M ≥ 5 (space too large to enumerate): device argmin over the first
    `count` candidates, and the oracle's argmin of the first 20,000."""
    spec = getattr(synth, name)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    g.pipeline_range(M, MICRO, 0, 1000)                # warm-up (builds the tables)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    (b, i), _ = g.pipeline_range(M, MICRO, 0, count)
    e.record()
    torch.cuda.synchronize()
    gpu_s = s.elapsed_time(e) / 1e3
    k = 20000
    t = time.perf_counter()
    want = od.pipeline_search(M, MICRO, 0, k)
    dt = time.perf_counter() - t
    print(json.dumps({"case": name, "M": M, "candidates": count, "space": g.pipeline_space(M, len(MICRO)),
                      "gpu_s": gpu_s, "gpu_per_s": count / gpu_s, "best_ps": b, "index": i,
                      "oracle_per_s": k / dt, "oracle_sample": k,
                      "prefix_parity": g.pipeline_range(M, MICRO, 0, k)[0] == want}), flush=True)


if __name__ == "__main__":
    for name in ("gnmt", "biglstm"):
        for M in (2, 3, 4):
            case(name, M)
    for name in ("gnmt", "biglstm"):
        for M in (5, 6, 8):
            range_case(name, M, 20_000_000)
