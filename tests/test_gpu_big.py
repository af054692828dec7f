"""GPU parity of the global-state tier (pp.h pp_dfg_get_tier):
DFGs whose image exceeds the 96 KB shared-memory image or whose per-lane
state ((W + 1 + M) slots) leaves fewer than 4 resident warps per SM run
search_big_kernel — image read from HBM, lane state in a global scratch.
Every value is compared bit for bit with the CPU oracle (integer ps, zero
tolerance), as in test_gpu_parity.py."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402


def _specs():
    # producers anywhere in a 900-op DAG: W in the hundreds (state overflow)
    wide = synth.random_dag(5, 900, avg_deg=1.5)
    # 3200 ops with a producer window of 40: W small, image ≈ 250 KB (image overflow)
    long_ = synth.random_dag(11, 3200, avg_deg=1.2, max_in=3, window=40)
    # memory-capped variant of the wide DAG (R7): binding for M ≥ 2
    capped = dict(wide)
    rng = np.random.default_rng(3)
    capped["mem_bytes"] = [int(x) for x in rng.integers(1, 1000, size=len(wide["fwd_ps"]))]
    capped["dev_mem_cap_bytes"] = int(sum(capped["mem_bytes"]) * 0.6)
    return {"wide": wide, "long": long_, "capped": capped}


SPECS = _specs()


@pytest.fixture(scope="module")
def big():
    out = {}
    for name, spec in SPECS.items():
        out[name] = (pp.Dfg(spec), O.Dfg.from_spec(spec))
    return out


def _cands(od, M, gen, seed_r, tau, base_pi, idx):
    return np.array([od.makespan_pi(M, O.gen(od.K, M, gen, seed_r, tau, base_pi, int(i))) for i in idx],
                    dtype=np.uint64)


def test_tier_selection(big):
    g, _ = big["wide"]
    assert g.W >= 300 and g.tier == pp.TIER_GLOBAL
    g, _ = big["long"]
    assert g.image_bytes > 96 * 1024 and g.tier == pp.TIER_GLOBAL
    assert pp.Dfg(synth.inception_v3()).tier == pp.TIER_SHARED


@pytest.mark.parametrize("name", ["wide", "long", "capped"])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 8])
def test_generated_candidates(big, name, M):
    """Every candidate of RANDOM and PERTURB ranges (several warps and a
    ragged tail) equals the oracle's makespan."""
    g, od = big[name]
    count = 32 * 9 + 13
    rng = np.random.default_rng(M)
    base = rng.integers(0, M, size=g.K, dtype=np.uint8)
    for gen, ogen, seed, tau, b, begin in [(pp.GEN_RANDOM, O.GEN_RANDOM, 7 + M, 0, None, 0),
                                           (pp.GEN_PERTURB, O.GEN_PERTURB, 99, 40, base, 0),
                                           (pp.GEN_PERTURB, O.GEN_PERTURB, 5, 256, base, 1000)]:
        cnt = count   # (GRAY needs M^K ≤ 2^63: covered by test_forced_global_tier_gray)
        got = pp.u64(g.eval_generated(M, gen, seed, tau, b, begin, cnt))
        want = _cands(od, M, ogen, seed, tau, b, range(begin, begin + cnt))
        assert np.array_equal(got, want), (name, M, gen)


@pytest.mark.parametrize("name", ["wide", "long", "capped"])
@pytest.mark.parametrize("M", [2, 4, 8])
def test_range_argmin(big, name, M):
    """The device argmin (warp → CTA → last CTA, dynamic tiles) equals the
    oracle's (makespan, index) over a range larger than one grid pass."""
    g, od = big[name]
    base = np.zeros(g.K, dtype=np.uint8)
    for gen, ogen, tau in [(pp.GEN_PERTURB, O.GEN_PERTURB, 24), (pp.GEN_RANDOM, O.GEN_RANDOM, 0)]:
        b = base if gen == pp.GEN_PERTURB else None
        r = pp.u64(g.search_range(M, gen, 31, tau, b, 17, 17 + 6000))
        want = od.round(M, ogen, 31, tau, b, 17, 17 + 6000)
        assert (int(r[0]), int(r[1])) == want, (name, M, gen)


@pytest.mark.parametrize("M", [2, 3, 8])
def test_explicit_rows(big, M):
    """pp_eval_placements on the global tier, including rows with values ≥ M
    (reported infeasible, neighbours unaffected) and the memory cap."""
    for name in ("wide", "capped", "long"):
        g, od = big[name]
        rng = np.random.default_rng(50 + M)
        count = 300
        pl = rng.integers(0, M, size=(count, g.K), dtype=np.uint8)
        pl[0] = 0
        bad = rng.choice(count - 1, 20, replace=False) + 1
        pl[bad, rng.integers(0, g.K, size=20)] = M + 3
        got = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
        for i in range(count):
            want = pp.INFEASIBLE if i in set(bad.tolist()) else od.makespan(M, pl[i])
            assert int(got[i]) == want, (name, M, i)


@pytest.mark.parametrize("name", ["wide", "long"])
def test_search_best_rounds(big, name):
    """The multi-round PERTURB search (base ← strictly better round winner)
    on the global tier equals the oracle's search, trajectory included."""
    g, od = big[name]
    for M in (2, 4):
        r = g.search_best(M, pp.GEN_PERTURB, 2024, 4000, rounds=3, tau=16)
        o = od.search(M, O.GEN_PERTURB, 2024, 4000, rounds=3, tau=16)
        assert (r.best_makespan_ps, r.best_index, r.best_round, r.evaluated) == \
               (o.best_makespan_ps, o.best_index, o.best_round, o.evaluated), (name, M)
        assert np.array_equal(r.placement, o.placement)


@pytest.mark.parametrize("dfg", ["toy12", "inception_v3", "gnmt", "biglstm"])
def test_forced_global_tier_paper_dfgs(dfg, monkeypatch):
    """PP_TIER=global runs the paper-shaped DFGs (which fit in shared memory)
    on the global tier: identical search results, and the exhaustive GRAY
    search takes the plain Gray order instead of the symmetry reduction."""
    monkeypatch.setenv("PP_TIER", "global")
    spec = getattr(synth, dfg)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.tier == pp.TIER_GLOBAL
    if dfg == "toy12":
        r = g.search_best(2, pp.GEN_GRAY, 0, 4096)
        o = od.search(2, O.GEN_GRAY, 0, 4096)
    else:
        r = g.search_best(2, pp.GEN_PERTURB, 77, 5000, rounds=2, tau=8)
        o = od.search(2, O.GEN_PERTURB, 77, 5000, rounds=2, tau=8)
    assert (r.best_makespan_ps, r.best_index, r.best_round) == (o.best_makespan_ps, o.best_index, o.best_round)
    assert np.array_equal(r.placement, o.placement)
    got = pp.u64(g.eval_generated(4, pp.GEN_RANDOM, 3, 0, None, 0, 200))
    assert np.array_equal(got, _cands(od, 4, O.GEN_RANDOM, 3, 0, None, range(200)))


@pytest.mark.parametrize("M", [2, 3, 4, 5, 8])
def test_forced_global_tier_gray(M, monkeypatch):
    """GRAY candidates (small K only: M^K ≤ 2^63) on the global tier, every
    makespan of a range with a ragged tail, and the exhaustive search."""
    monkeypatch.setenv("PP_TIER", "global")
    spec = synth.random_dag(2020 + M, 20, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.tier == pp.TIER_GLOBAL
    begin, cnt = 777, 32 * 7 + 5
    got = pp.u64(g.eval_generated(M, pp.GEN_GRAY, 0, 0, None, begin, cnt))
    assert np.array_equal(got, _cands(od, M, O.GEN_GRAY, 0, 0, None, range(begin, begin + cnt)))
    space = min(M ** g.K, 60_000)
    r = pp.u64(g.search_range(M, pp.GEN_GRAY, 0, 0, None, 0, space))
    assert (int(r[0]), int(r[1])) == od.round(M, O.GEN_GRAY, 0, 0, None, 0, space)


@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
def test_u64_time_range_runs_global_tier(M):
    """A DFG whose time bound is ≥ 2^49 ps needs the tagged-u64 arithmetic,
    which only the global tier runs: every candidate and the
    range argmin equal the oracle's."""
    spec = synth.random_dag(4900 + M, 120, avg_deg=1.5, max_cost=10**15, max_bytes=10**9, bw=10**9)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.tier == pp.TIER_GLOBAL
    assert od.t1 >= 1 << 49
    base = np.random.default_rng(M).integers(0, M, size=g.K, dtype=np.uint8)
    for gen, ogen in [(pp.GEN_RANDOM, O.GEN_RANDOM), (pp.GEN_PERTURB, O.GEN_PERTURB)]:
        got = pp.u64(g.eval_generated(M, gen, 11, 64, base, 3, 300))
        assert np.array_equal(got, _cands(od, M, ogen, 11, 64, base, range(3, 303))), gen
        r = pp.u64(g.search_range(M, gen, 12, 64, base, 0, 5000))
        assert (int(r[0]), int(r[1])) == od.round(M, ogen, 12, 64, base, 0, 5000)


def test_forced_global_tier_other_entry_points(monkeypatch):
    """The exact search (its in-order incumbent runs on the global tier), the
    EFT seed and the GPipe search of a DFG loaded on the global tier equal the
    oracle's."""
    monkeypatch.setenv("PP_TIER", "global")
    spec = synth.toy12()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.tier == pp.TIER_GLOBAL
    for M, end in ((2, 600), (3, 400)):
        ex = g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, end)
        assert ex[:2] == od.round_exact(M, O.GEN_GRAY, 0, 0, None, 0, end), M
        assert np.array_equal(g.eft_place(M), od.eft(M))
        pr = g.pipeline_search(M, [1, 2, 4])
        assert (pr["makespan_ps"], pr["index"]) == od.pipeline_search(M, [1, 2, 4])
