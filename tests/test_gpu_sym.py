"""the symmetry-reduced exhaustive GRAY search.

An exhaustive GRAY search (count = M^K) on the uniform link model evaluates
one placement per device-relabelling class (restricted-growth strings) and
reports each class by its smallest Gray index (search_kernel.cuh RgsGen,
gray_min_index).  The (makespan, Gray index, placement) must equal the
oracle's plain search over all M^K placements (O5, O7) — for the in-order
schedule and for the exact schedule — and the unreduced kernel's
(PP_NO_SYM=1)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402


def _cases():
    out = [("toy12", synth.toy12())]
    for K, seed in ((6, 1), (9, 2), (11, 3), (13, 4)):
        out.append((f"rand{K}", synth.random_dag(700 + seed, K, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)))
    # a memory cap (the same on every device, so still symmetric)
    spec = synth.random_dag(777, 10, avg_deg=1.5, max_cost=10**6, max_bytes=10**6)
    spec["mem_bytes"] = [int(x) for x in np.random.default_rng(5).integers(1, 100, size=10)]
    spec["dev_mem_cap_bytes"] = int(sum(spec["mem_bytes"]) * 0.55)   # feasible for M ≥ 2, binding
    out.append(("cap10", spec))
    # equal ops and no communication: many classes tie, so the Gray tie-break decides
    out.append(("indep8", synth.independent(8, 5, 7)))
    return out


CASES = _cases()


@pytest.mark.parametrize("name,spec", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("M", [2, 3, 4, 5, 8])
def test_exhaustive_gray_equals_oracle(name, spec, M, monkeypatch):
    K = len(spec["fwd_ps"])
    space = M ** K
    if space > 2 * 10**9:
        pytest.skip("GPU time of the unreduced search")
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    if space > 3 * 10**6:
        # beyond the oracle's time: the reduced search must equal the unreduced
        # GPU search (itself oracle-checked on smaller spaces), and the winner's
        # makespan must be the oracle's for the placement its Gray index names
        r = g.search_best(M, pp.GEN_GRAY, 0, space)
        monkeypatch.setenv("PP_NO_SYM", "1")
        r0 = g.search_best(M, pp.GEN_GRAY, 0, space)
        assert (r.best_makespan_ps, r.best_index) == (r0.best_makespan_ps, r0.best_index), (name, M)
        assert np.array_equal(r.placement, r0.placement)
        d = O.gen(K, M, O.GEN_GRAY, 0, 0, None, r.best_index)
        assert od.makespan_pi(M, d) == r.best_makespan_ps
        g.close()
        return
    want = od.search(M, O.GEN_GRAY, 0, space)
    for np_ in ("1", "2", "4"):
        monkeypatch.setenv("PP_NP", np_)
        r = g.search_best(M, pp.GEN_GRAY, 0, space)
        assert (r.best_makespan_ps, r.best_index, r.best_round) == \
               (want.best_makespan_ps, want.best_index, want.best_round), (np_, name, M)
        assert np.array_equal(r.placement, want.placement)
        # the device-side range argmin over the whole space takes the same path
        b = pp.u64(g.search_range(M, pp.GEN_GRAY, 0, 0, None, 0, space))
        assert (int(b[0]), int(b[1])) == (want.best_makespan_ps, want.best_index)
    monkeypatch.setenv("PP_NO_SYM", "1")
    r = g.search_best(M, pp.GEN_GRAY, 0, space)
    assert (r.best_makespan_ps, r.best_index) == (want.best_makespan_ps, want.best_index)
    g.close()


def test_toy12_m4_full_space():
    """toy-12 at M = 4: 4^12 = 16.8 M placements, 0.70 M classes."""
    spec = synth.toy12()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    want = od.search(4, O.GEN_GRAY, 0, 4**12)
    r = g.search_best(4, pp.GEN_GRAY, 0, 4**12)
    assert (r.best_makespan_ps, r.best_index) == (want.best_makespan_ps, want.best_index)
    assert np.array_equal(r.placement, want.placement)
    g.close()


def test_partial_range_is_not_reduced():
    """A prefix of the Gray space is not closed under relabelling: it runs the
    plain kernel (and matches the oracle)."""
    spec = synth.toy12()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    for end in (1000, 3**12 - 1):
        b = pp.u64(g.search_range(3, pp.GEN_GRAY, 0, 0, None, 0, end))
        assert (int(b[0]), int(b[1])) == od.round(3, O.GEN_GRAY, 0, 0, None, 0, end)
    g.close()


@pytest.mark.parametrize("K,M", [(5, 3), (6, 3), (6, 4), (7, 2), (5, 5)])
def test_exact_search_reduced_equals_oracle(K, M):
    spec = synth.random_dag(900 + K * 10 + M, K, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    want = od.round_exact(M, O.GEN_GRAY, 0, 0, None, 0, M ** K)
    got = g.search_exact(M, pp.GEN_GRAY, 0, 0, None, 0, M ** K)
    assert got[:2] == want and got[2] == 0
    g.close()


def test_hardware_graph_is_not_reduced():
    """Device pairs differ on a hardware graph, so relabelling changes
    makespans: the full space runs unreduced and still equals the oracle."""
    from synth import hw as H
    spec = synth.random_dag(31, 7, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)
    spec["hw"] = H.ring(4)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    want = od.search(4, O.GEN_GRAY, 0, 4**7)
    r = g.search_best(4, pp.GEN_GRAY, 0, 4**7)
    assert (r.best_makespan_ps, r.best_index) == (want.best_makespan_ps, want.best_index)
    g.close()
