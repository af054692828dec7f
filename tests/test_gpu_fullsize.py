"""Parity at BASELINE.json's full sizes (VERDICT r1 missing #2, SURVEY.md
§8(d) "Parity still uses the full oracle, run once").

Every search, GPipe search and projection of synth/configs.py — configs 1–5
at their stated sizes plus config 5 at the bench's 10 × 10^7 — runs on the GPU
through the C ABI and must equal tests/golden/fullsize_r02.json value for
value.  That file is written by tools/oracle_fullsize.py from `oracle/` alone
(the oracle's rounds sliced over host threads; the slicing is checked against
or_search itself in tests/test_oracle_fullsize.py), so no expected value comes
from the CUDA path.

Compared per search: T_M, the winning index and round, the winning placement
and T_1; per GPipe search: makespan and index; per projection: every cell's
C (feasible cells) and feasibility, N*, the M at N*, N*_M, persistence,
N* vs the best DP and the best M at every N.  The searches run in the launch
configuration bench.py times (pp_search_best, default NP rule, EFT base from
pp_eft_place).  A sampled element-by-element block of the bench config's
round 0 is kept as well.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import synth
from synth import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_r02.json")))
GENS = {"gray": pp.GEN_GRAY, "random": pp.GEN_RANDOM, "perturb": pp.GEN_PERTURB}


@pytest.fixture(scope="module")
def gpu():
    dfgs, res, pipes = {}, {}, {}
    for s in configs.searches():
        g = dfgs.get(s["model"]) or dfgs.setdefault(s["model"], pp.Dfg(getattr(synth, s["model"])()))
        base = g.eft_place(s["M"]) if s["base"] == "eft" else None
        res[s["key"]] = g.search_best(s["M"], GENS[s["gen"]], s["seed"], s["count"], rounds=s["rounds"],
                                      tau=s["tau"], base=base)
    for p in configs.pipelines():
        pipes[p["key"]] = dfgs[p["model"]].pipeline_search(p["M"], p["micro"])
    yield dfgs, res, pipes
    for g in dfgs.values():
        g.close()


@pytest.mark.parametrize("key", [s["key"] for s in configs.searches()])
def test_search_equals_oracle_golden(gpu, key):
    _, res, _ = gpu
    r, want = res[key], GOLDEN["searches"][key]
    assert (r.best_makespan_ps, r.best_index, r.best_round) == (want["T_M"], want["best_index"], want["best_round"])
    assert "".join(map(str, r.placement)) == want["placement"]
    assert r.t1_ps == want["t1_ps"] and r.evaluated == want["evaluated"]


@pytest.mark.parametrize("key", [p["key"] for p in configs.pipelines()])
def test_pipeline_equals_oracle_golden(gpu, key):
    _, _, pipes = gpu
    want = GOLDEN["pipelines"][key]
    assert (pipes[key]["makespan_ps"], pipes[key]["index"], pipes[key]["candidates"]) == \
           (want["makespan"], want["index"], want["candidates"])


@pytest.mark.parametrize("pr", configs.projections(), ids=lambda p: p["name"])
def test_projection_and_crossover_equal_oracle_golden(gpu, pr):
    dfgs, res, pipes = gpu
    want = GOLDEN["projections"][pr["name"]]
    g = dfgs[pr["model"]]
    T = [g.t1] + [min(res[k].best_makespan_ps if k in res else pipes[k]["makespan_ps"] for k in pr["T"][M])
                  for M in pr["Ms"][1:]]
    assert T == want["T"]
    if pr["model"] == "toy12":
        sc = synth.toy12_scenario(g.t1, ar_mode=pr["mode"])
    else:
        sc = synth.sweep_scenario(pr["model"], g.t1, g.grad_bytes, ar_mode=pr["mode"])
    cells = pp.project_e2e(sc, pr["Ms"], T, pr["nmax"])
    got = pp.cells_to_numpy(cells).reshape(-1)
    gotC = [str((int(c["C_hi"]) << 64) | int(c["C_lo"])) if int(c["feasible"]) else None for c in got]
    assert gotC == want["C"]
    x = pp.crossover(cells, pr["Ms"], pr["nmax"])
    assert (x.n_star, x.m_at_n_star, list(x.n_star_M), list(x.persistent_M), x.n_star_vs_best_dp, list(x.best_m)) == \
           (want["n_star"], want["m_at_n_star"], want["n_star_M"], want["persistent_M"], want["n_star_vs_best_dp"],
            want["best_m"])


def test_bench_round0_block_element_by_element():
    """A 4,096-candidate block of the bench config's round 0 at a random
    offset, each candidate's makespan against the oracle's."""
    M, count = 2, 10_000_000
    spec = synth.inception_v3()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    base = g.eft_place(M)
    assert np.array_equal(base, od.eft(M))
    base_pi = np.ascontiguousarray(base[od.pi])
    lo = int(np.random.default_rng(2).integers(0, count - 4096))
    got = pp.u64(g.eval_generated(M, pp.GEN_PERTURB, configs.SEED, configs.TAU, base_pi, lo, 4096))
    want = np.array([od.makespan_pi(M, O.gen(od.K, M, O.GEN_PERTURB, configs.SEED, configs.TAU, base_pi, i))
                     for i in range(lo, lo + 4096)], dtype=np.uint64)
    assert np.array_equal(got, want)
    g.close()
