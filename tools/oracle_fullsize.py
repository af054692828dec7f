"""Full-size parity golden from the CPU oracle alone (VERDICT r1 missing #2).

Runs every search of synth/configs.py at its stated size with the oracle
(`oracle/`, nothing from the CUDA path), slicing each round's candidate range
over host threads — the oracle's C calls release the GIL and keep no global
state, so each slice is one single-threaded or_round call (SURVEY.md §8(d):
"Parity still uses the full oracle, run once (possibly as one single-threaded
process per slice across host cores)").  The rounds are replayed with O7's
rule exactly as or_search states it (pp_oracle.c or_search): the round winner
is the lexicographic (makespan, index) minimum over the slices, the base moves
to it iff its makespan is strictly below the base's, and the reported best is
the first round that reached the final best.  `tests/test_oracle_fullsize.py`
checks that this replay equals or_search itself on small counts.

Then the GPipe searches (or_pipeline_search over slices of the split space)
and every projection/crossover of synth/configs.py.  Writes
tests/golden/fullsize_r02.json.

  python tools/oracle_fullsize.py [--threads 8] [--slices 64] [--only KEY,...]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from synth import configs  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "fullsize_r02.json")
GENS = {"gray": O.GEN_GRAY, "random": O.GEN_RANDOM, "perturb": O.GEN_PERTURB}


def _slices(n, S):
    return [(n * s // S, n * (s + 1) // S) for s in range(S) if n * s // S < n * (s + 1) // S]


def sliced_round(pool, od, M, gen, seed_r, tau, base_pi, count, S):
    """Argmin (makespan, index) of candidates [0, count) as the lexicographic
    minimum of the per-slice oracle argmins."""
    futs = [pool.submit(od.round, M, gen, seed_r, tau, base_pi, b, e) for b, e in _slices(count, S)]
    return min(f.result() for f in futs)


def sliced_search(pool, od, M, gen, seed, count, rounds, tau, base_desc, S):
    """or_search (O7) with each round's argmin computed over slices."""
    K = od.K
    base_pi = np.ascontiguousarray((base_desc if base_desc is not None else np.zeros(K, np.uint8))[od.pi])
    best = None
    for r in range(rounds):
        seed_r = seed + r
        mk, idx = sliced_round(pool, od, M, gen, seed_r, tau, base_pi, count, S)
        d = O.gen(K, M, gen, seed_r, tau, base_pi, idx)
        if r == 0 or mk < best[0]:
            best = (mk, idx, r, d)
        if mk < od.makespan_pi(M, base_pi):
            base_pi = np.ascontiguousarray(d)
    placement = np.zeros(K, np.uint8)
    placement[od.pi] = best[3]
    return dict(T_M=best[0], best_index=best[1], best_round=best[2], placement="".join(map(str, placement)))


def sliced_pipeline(pool, od, M, micro, S):
    from math import comb
    n = comb(od.K - 1, M - 1) * len(micro)
    futs = [pool.submit(od.pipeline_search, M, micro, b, e) for b, e in _slices(n, S)]
    mk, idx = min(f.result() for f in futs)
    return dict(makespan=mk, index=idx, candidates=n)


def spec_of(model):
    return getattr(synth, model)()


def fingerprint(model):
    """Digest of the DFG descriptor synth builds (entries of an earlier golden
    are reused only when their DFG is unchanged)."""
    import hashlib
    sp = spec_of(model)
    keys = ["fwd_ps", "bwd_ps", "edge_src", "edge_dst", "edge_fwd_bytes", "edge_bwd_bytes", "mem_bytes",
            "param_bytes", "op_id", "link_bw_Bps", "link_lat_ps", "dev_mem_cap_bytes"]
    return hashlib.sha256(json.dumps([sp.get(k) for k in keys], default=int).encode()).hexdigest()[:16]


def run(threads, S, only=None, log=print, reuse=None):
    out = {"generator": "oracle/ only (tools/oracle_fullsize.py)", "seed": configs.SEED,
           "searches": {}, "pipelines": {}, "projections": {}, "dfg_sha": {}}
    ods = {}
    fps = {}
    with cf.ThreadPoolExecutor(max_workers=threads) as pool:
        for s in configs.searches():
            if only and s["key"] not in only:
                continue
            fp = fps.setdefault(s["model"], fingerprint(s["model"]))
            out["dfg_sha"][s["model"]] = fp
            old = (reuse or {}).get("searches", {}).get(s["key"])
            if old is not None and old.get("dfg_sha") == fp:
                out["searches"][s["key"]] = old
                continue
            od = ods.setdefault(s["model"], O.Dfg.from_spec(spec_of(s["model"])))
            base = od.eft(s["M"]) if s["base"] == "eft" else None
            t = time.perf_counter()
            r = sliced_search(pool, od, s["M"], GENS[s["gen"]], s["seed"], s["count"], s["rounds"], s["tau"],
                              base, S)
            seed_ps = od.makespan(s["M"], base) if base is not None else od.t1
            r.update(seed_ps=seed_ps, t1_ps=od.t1, evaluated=s["count"] * s["rounds"], dfg_sha=fp,
                     oracle_s=round(time.perf_counter() - t, 1))
            out["searches"][s["key"]] = r
            log(f"{s['key']}: T_M={r['T_M']} idx={r['best_index']} round={r['best_round']} "
                f"seed={seed_ps} ({time.perf_counter() - t:.1f} s)")
        for p in configs.pipelines():
            if only and p["key"] not in only:
                continue
            fp = fps.setdefault(p["model"], fingerprint(p["model"]))
            old = (reuse or {}).get("pipelines", {}).get(p["key"])
            if old is not None and old.get("dfg_sha") == fp:
                out["pipelines"][p["key"]] = old
                continue
            od = ods.setdefault(p["model"], O.Dfg.from_spec(spec_of(p["model"])))
            t = time.perf_counter()
            out["pipelines"][p["key"]] = dict(sliced_pipeline(pool, od, p["M"], p["micro"], S), dfg_sha=fp)
            log(f"{p['key']}: {out['pipelines'][p['key']]} ({time.perf_counter() - t:.1f} s)")
    if only:
        return out
    for pr in configs.projections():
        od = ods.setdefault(pr["model"], O.Dfg.from_spec(spec_of(pr["model"])))
        T = [od.t1]
        for M in pr["Ms"][1:]:
            vals = [out["searches"][k]["T_M"] if k in out["searches"] else out["pipelines"][k]["makespan"]
                    for k in pr["T"][M]]
            T.append(min(vals))
        if pr["model"] == "toy12":
            sc = synth.toy12_scenario(od.t1, ar_mode=pr["mode"])
        else:
            sc = synth.sweep_scenario(pr["model"], od.t1, od.grad_bytes, ar_mode=pr["mode"])
        cells = O.Scenario.from_spec(sc).project(pr["Ms"], T, pr["nmax"])
        x = O.crossover(cells, pr["Ms"], pr["nmax"])
        out["projections"][pr["name"]] = dict(
            T=T, n_star=x.n_star, m_at_n_star=x.m_at_n_star, n_star_M=list(x.n_star_M)[:len(pr["Ms"])],
            persistent_M=list(x.persistent_M)[:len(pr["Ms"])], n_star_vs_best_dp=x.n_star_vs_best_dp,
            best_m=list(x.best_m),
            C=[str(c.C) if c.feasible else None for c in cells])
        log(f"{pr['name']}: T={T} N*={x.n_star} n_star_M={list(x.n_star_M)[:len(pr['Ms'])]}")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--slices", type=int, default=64)
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=GOLDEN)
    ap.add_argument("--fresh", action="store_true", help="recompute every entry (default: reuse entries of the "
                                                          "existing golden whose DFG digest is unchanged)")
    a = ap.parse_args()
    t0 = time.perf_counter()
    reuse = None
    if not a.fresh and os.path.exists(a.out):
        reuse = json.load(open(a.out))
    res = run(a.threads, a.slices, set(a.only.split(",")) if a.only else None, reuse=reuse)
    res["wall_s"] = round(time.perf_counter() - t0, 1)
    res["threads"] = a.threads
    if not a.only:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
        print(f"wrote {a.out} in {res['wall_s']} s")
    else:
        print(json.dumps(res))
