"""GPU parity of the projection cells and the crossover (exact u128 values)."""
import random

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402
from tests.test_oracle_projection import _rand_scenario  # noqa: E402


def _compare(sc, Ms, TM, Nmax):
    cells = pp.project_e2e(sc, Ms, TM, Nmax)
    got = pp.cells_to_numpy(cells)
    oc = O.Scenario.from_spec(sc).project(Ms, TM, Nmax)
    for m in range(len(Ms)):
        for N in range(1, Nmax + 1):
            c, o = got[m, N - 1], oc[m * Nmax + N - 1]
            assert (int(c["C_lo"]), int(c["C_hi"]), int(c["step_ps"]), int(c["steps"]), int(c["uepochs"]),
                    int(c["feasible"]), int(c["accum"])) == \
                   (o.C_lo, o.C_hi, o.step_ps, o.steps, o.uepochs, o.feasible, o.accum), (m, N)
    if 1 in Ms:
        x = pp.crossover(cells, Ms, Nmax)
        ox = O.crossover(oc, Ms, Nmax)
        assert (x.n_star, x.m_at_n_star, x.n_star_M, x.persistent_M, x.n_star_vs_best_dp, x.best_m) == \
               (ox.n_star, ox.m_at_n_star, ox.n_star_M, ox.persistent_M, ox.n_star_vs_best_dp, ox.best_m)
        return x
    return None


@pytest.mark.parametrize("fx", [synth.inception_fixture, synth.biglstm_fixture, synth.gnmt_fixture])
def test_paper_fixtures(fx):
    sc, Ms, TM, Nmax = fx()
    x = _compare(sc, Ms, TM, Nmax)
    assert x.n_star == {synth.inception_fixture: 54, synth.biglstm_fixture: 22, synth.gnmt_fixture: 214}[fx]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("model", ["inception_v3", "gnmt", "biglstm"])
def test_sweep_scenarios(model, mode):
    # BASELINE config 5 shape: M ∈ {1,2,4,8}, N = 1..1024, 16 knots, AR on
    t1 = 200 * 10**9
    sc = synth.sweep_scenario(model, t1, 10**8, ar_mode=mode)
    _compare(sc, [1, 2, 4, 8], [t1, 150 * 10**9, 140 * 10**9, 139 * 10**9], 1024)


@pytest.mark.parametrize("seed", range(8))
def test_random_scenarios(seed):
    rng = random.Random(seed)
    sc = _rand_scenario(rng, ar_mode=seed % 2, ar_on=seed % 3 != 0)
    t1 = sc["t1_ps"]
    Ms = [1, 2, 4, 8][:rng.randint(2, 4)]
    rng.shuffle(Ms)
    TM = [t1 if M == 1 else rng.randint(t1 // M, t1) for M in Ms]
    _compare(sc, Ms, TM, rng.choice([1, 7, 256, 1000, 4097]))


def test_projection_errors_match():
    sc = dict(synth.inception_fixture()[0])
    with pytest.raises(pp.PPError) as e:
        pp.project_e2e(dict(sc, knot_G=[64, 64]), [1], [1], 4)
    assert e.value.code == -1
    cells = pp.project_e2e(sc, [2, 4], [10, 10], 8)
    with pytest.raises(pp.PPError) as e:
        pp.crossover(cells, [2, 4], 8)   # no DP baseline
    assert e.value.code == -1
    # u128 overflow: huge T_M and epochs
    big = dict(sc, knot_uepochs=[2**62] * 9, t1_ps=2**63)
    with pytest.raises(pp.PPError) as e:
        pp.project_e2e(big, [1], [2**63], 4)
    assert e.value.code == -3
    with pytest.raises(O.OracleError) as e2:
        O.Scenario.from_spec(big).project([1], [2**63], 4)
    assert e2.value.code == -3


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("model", ["inception_v3", "gnmt", "biglstm"])
def test_accumulation_axis_and_shards(model, mode):
    # a ∈ {1, 2, 4, 8, 16} per cell and placement-aware
    # all-reduce shards from the EFT placements of the paper-shaped DFG
    spec = getattr(synth, model)()
    g = pp.Dfg(spec)
    Ms = [1, 2, 4, 8]
    shards = [[g.grad_bytes] + [0] * 7] + [g.shard_bytes(M, g.eft_place(M)) for M in Ms[1:]]
    assert all(sum(r) == g.grad_bytes for r in shards)
    t1 = g.t1
    sc = synth.sweep_scenario(model, t1, g.grad_bytes, ar_mode=mode)
    sc = dict(sc, accum=[1, 2, 4, 8, 16], shard_bytes=shards)
    x = _compare(sc, Ms, [t1, t1 * 3 // 4, t1 * 2 // 3, t1 * 3 // 5], 1024)
    assert x is not None
