"""GPU parity of the EFT-greedy base seed: eft_kernel
against the oracle's or_eft, bit for bit (device per op)."""
import random

import numpy as np
import pytest

import oracle as O
import synth
from synth import hw as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402


@pytest.mark.parametrize("name", ["toy12", "inception_v3", "gnmt", "biglstm"])
def test_paper_dfgs(name):
    spec = getattr(synth, name)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    for M in range(1, 9):
        assert np.array_equal(g.eft_place(M), od.eft(M)), M


@pytest.mark.parametrize("topo", ["cube_mesh", "two_nodes"])
def test_hardware_graphs(topo):
    hw = H.hybrid_cube_mesh() if topo == "cube_mesh" else H.two_nodes(4)
    for name in ("inception_v3", "gnmt"):
        spec = dict(getattr(synth, name)(), hw=hw)
        g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
        for M in (2, 4, 8):
            assert np.array_equal(g.eft_place(M), od.eft(M)), (name, M)


@pytest.mark.parametrize("seed", range(8))
def test_random_dags_with_caps(seed):
    rng = random.Random(seed)
    K, M = rng.randint(1, 200), rng.randint(1, 8)
    spec = synth.random_dag(1400 + seed, K, window=12)
    spec["mem_bytes"] = [rng.randint(0, 100) for _ in range(K)]
    spec["dev_mem_cap_bytes"] = rng.choice([0, 60 * K // M + 100, 30 * K // M + 50])
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    try:
        want = od.eft(M)
    except O.OracleError:
        with pytest.raises(pp.PPError):
            g.eft_place(M)
        return
    assert np.array_equal(g.eft_place(M), want)


def test_eft_base_then_perturb_search():
    spec = synth.inception_v3()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    base = g.eft_place(2)
    r = g.search_best(2, pp.GEN_PERTURB, 7, 20_000, rounds=3, tau=8, base=base)
    o = od.search(2, O.GEN_PERTURB, 7, 20_000, rounds=3, tau=8, base=base)
    assert (r.best_makespan_ps, r.best_index, r.best_round) == (o.best_makespan_ps, o.best_index, o.best_round)
    assert r.best_makespan_ps <= od.makespan(2, base)
