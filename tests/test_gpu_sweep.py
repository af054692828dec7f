"""BASELINE config 5 at reduced candidate counts: the GPU sweep (searches for
M ∈ {2,4,8} on the three paper-shaped DFGs, projection over M ∈ {1,2,4,8} ×
N = 1..1024 with 16 knots in EQ5 and TIME modes, crossover) equals the
oracle's, value for value."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402

MS = [1, 2, 4, 8]


@pytest.mark.parametrize("model", ["inception_v3", "gnmt", "biglstm"])
def test_full_sweep_matches_oracle(model):
    spec = getattr(synth, model)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    T, To = [g.t1], [od.t1]
    for M in MS[1:]:
        r = g.search_best(M, pp.GEN_PERTURB, 5, 3_000, rounds=3, tau=8)
        o = od.search(M, O.GEN_PERTURB, 5, 3_000, rounds=3, tau=8)
        assert (r.best_makespan_ps, r.best_index, r.best_round) == (o.best_makespan_ps, o.best_index, o.best_round)
        T.append(r.best_makespan_ps)
        To.append(o.best_makespan_ps)
    for mode in (0, 1):
        sc = synth.sweep_scenario(model, g.t1, g.grad_bytes, ar_mode=mode)
        cells = pp.cells_to_numpy(pp.project_e2e(sc, MS, T, 1024))
        oc = O.Scenario.from_spec(sc).project(MS, To, 1024)
        got = np.array([[int(c["C_lo"]), int(c["C_hi"]), int(c["feasible"])] for c in cells.reshape(-1)])
        want = np.array([[c.C_lo, c.C_hi, c.feasible] for c in oc])
        assert np.array_equal(got, want)
        x = pp.crossover(pp.project_e2e(sc, MS, T, 1024), MS, 1024)
        ox = O.crossover(oc, MS, 1024)
        assert (x.n_star, x.m_at_n_star, x.n_star_M, x.persistent_M, x.n_star_vs_best_dp, x.best_m) == \
               (ox.n_star, ox.m_at_n_star, ox.n_star_M, ox.persistent_M, ox.n_star_vs_best_dp, ox.best_m)
