"""GPU parity on the general hardware graph: the CUDA
path loaded with pp_load_dfg_hw against the oracle's or_prepare_hw, bit for
bit (integer ps)."""
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

TOPOS = {
    "cube_mesh": H.hybrid_cube_mesh,
    "switch8": lambda: H.switch(8),
    "ring8": lambda: H.ring(8),
    "two_nodes": lambda: H.two_nodes(4),
}


def _pair(spec, hw):
    s = dict(spec, hw=hw)
    return pp.Dfg(s), O.Dfg.from_spec(s)


def _oracle_candidates(od, M, gen, seed_r, tau, base_pi, idx):
    return np.array([od.makespan_pi(M, O.gen(od.K, M, gen, seed_r, tau, base_pi, int(i))) for i in idx],
                    dtype=np.uint64)


@pytest.mark.parametrize("topo", list(TOPOS))
@pytest.mark.parametrize("name", ["inception_v3", "gnmt", "biglstm"])
def test_eval_placements_paper_dfgs(name, topo):
    g, od = _pair(getattr(synth, name)(), TOPOS[topo]())
    rng = np.random.default_rng(len(name) + len(topo))
    for M in (2, 3, 4, 8):
        count = 600 + 29
        pl = rng.integers(0, M, size=(count, g.K), dtype=np.uint8)
        got = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
        want = np.array([od.makespan(M, row) for row in pl], dtype=np.uint64)
        assert np.array_equal(got, want), (name, topo, M)


@pytest.mark.parametrize("gen", [O.GEN_GRAY, O.GEN_RANDOM, O.GEN_PERTURB])
@pytest.mark.parametrize("M", [2, 3, 5, 8])
def test_eval_generated_cube_mesh(gen, M):
    if gen == O.GEN_GRAY:   # a DFG small enough for the Gray space (M^K ≤ 2^63)
        import math
        spec = synth.random_dag(40 + M, min(40, int(62 / math.log2(M))), max_bytes=10**7, window=8)
    else:
        spec = synth.inception_v3()
    g, od = _pair(spec, H.hybrid_cube_mesh())
    rng = np.random.default_rng(M * 7 + gen)
    base = rng.integers(0, M, size=g.K, dtype=np.uint8)
    seed = int(rng.integers(0, 2**63))
    for begin, count in ((0, 1000), (10**9 + 5, 61)):
        got = pp.u64(g.eval_generated(M, gen, seed, 40, base, begin, count))
        want = _oracle_candidates(od, M, gen, seed, 40, base, range(begin, begin + count))
        assert np.array_equal(got, want)


@pytest.mark.parametrize("np_", [1, 2, 4])
def test_search_perturb_rounds_every_np(np_, monkeypatch):
    monkeypatch.setenv("PP_NP", str(np_))
    g, od = _pair(synth.gnmt(), H.two_nodes(4))
    for M in (2, 4, 8):
        base = np.random.default_rng(M).integers(0, M, size=g.K, dtype=np.uint8)
        r = g.search_best(M, pp.GEN_PERTURB, 3 + M, 6000, rounds=3, tau=10, base=base)
        o = od.search(M, O.GEN_PERTURB, 3 + M, 6000, rounds=3, tau=10, base=base)
        assert (r.best_makespan_ps, r.best_index, r.best_round, r.evaluated) == \
               (o.best_makespan_ps, o.best_index, o.best_round, o.evaluated)
        assert np.array_equal(r.placement, o.placement)


@pytest.mark.parametrize("seed", range(10))
def test_fuzz_random_dags_random_hw(seed):
    rng = random.Random(seed)
    nd = rng.randint(2, 8)
    hw = H.random_hw(seed, nd, nr=rng.randint(0, 3), extra_links=rng.randint(0, 6),
                     cap=rng.choice([0, 0, 10**4]))
    spec = synth.random_dag(900 + seed, rng.randint(1, 90), max_bytes=10**7, window=10)
    spec["mem_bytes"] = [rng.randint(0, 3000) for _ in spec["fwd_ps"]]
    g, od = _pair(spec, hw)
    M = rng.randint(1, nd)
    n = 777
    pl = np.random.default_rng(seed).integers(0, M, size=(n, g.K), dtype=np.uint8)
    got = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
    want = np.array([od.makespan(M, row) for row in pl], dtype=np.uint64)
    assert np.array_equal(got, want)
    try:
        o = od.search(M, O.GEN_RANDOM, seed, 3001)
    except O.OracleError as e:                 # every candidate over the memory cap
        assert e.code == -5
        with pytest.raises(pp.PPError):
            g.search_best(M, pp.GEN_RANDOM, seed, 3001)
        return
    r = g.search_best(M, pp.GEN_RANDOM, seed, 3001)
    assert (r.best_makespan_ps, r.best_index) == (o.best_makespan_ps, o.best_index)


def test_full_mesh_matches_uniform_link_path():
    spec = synth.inception_v3()
    uni = pp.Dfg(spec)
    g = pp.Dfg(dict(spec, hw=H.full_mesh(4, bw=spec["link_bw_Bps"], lat=spec["link_lat_ps"])))
    pl = np.random.default_rng(1).integers(0, 4, size=(2000, g.K), dtype=np.uint8)
    t = torch.as_tensor(pl, device="cuda")
    assert np.array_equal(pp.u64(g.eval_placements(4, t)), pp.u64(uni.eval_placements(4, t)))


def test_errors():
    spec = synth.toy12()
    g = pp.Dfg(dict(spec, hw=H.ring(3)))
    with pytest.raises(pp.PPError):                      # M > num_devices
        g.search_best(4, pp.GEN_RANDOM, 0, 100)
    bad = dict(H.ring(3), link_a=[0], link_b=[1], link_bw_Bps=[1], link_lat_ps=[0])
    with pytest.raises(pp.PPError):                      # device 2 unreachable
        pp.Dfg(dict(spec, hw=bad))
    slow = H.ring(2, bw=1, lat=0)                         # 1 B/s: times ≥ 2^49 ps
    with pytest.raises(pp.PPError):
        pp.Dfg(dict(spec, hw=slow))
