"""Pins of the oracle's schedule (O4), π (O2), edge cost (O3) and search (O7).

Everything here is checked against something other than the oracle itself:
worked examples (tests/golden/schedule_pins.json, each cited), closed forms,
invariants, and the independent longest-path brute force in tests/brute.py.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

import oracle as O
import synth
from tests import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_pins.json")))


def _diamond(p):
    return synth.diamond(fwd=p["fwd"], bwd=p["bwd"], fwd_bytes=p["fwd_bytes"], bwd_bytes=p["bwd_bytes"])


def test_K1_split_diamond_starts():
    p = GOLD["K1_split_diamond"]
    d = O.Dfg.from_spec(_diamond(p))
    mk, f, _ = d.schedule(2, p["placement"])
    assert list(f) == p["starts"]
    assert mk == p["makespan"]
    p2 = GOLD["K1b_colocated_diamond"]
    assert d.makespan(2, p2["placement"]) == p2["makespan"]


@pytest.mark.parametrize("key", ["K2_diamond_exhaustive", "K3_diamond_fwd_bwd"])
def test_K2_K3_diamond_search(key):
    p = GOLD[key]
    spec = _diamond(p)
    d = O.Dfg.from_spec(spec)
    r = d.search(p["M"], O.GEN_GRAY, 0, 2**4)
    assert r.best_makespan_ps == p["best"]
    assert r.t1_ps == p["t1"] == d.t1
    if "optima" in p:
        assert list(r.placement) in p["optima"]
        best, opt = brute.exhaustive(spec, 2)
        assert best == p["best"] and sorted(map(list, opt)) == sorted(p["optima"])


def test_K4_chain_huge_comm():
    p = GOLD["K4_chain_huge_comm"]
    spec = synth.chain(2, p["fwd"], p["bwd"], p["fwd_bytes"])
    spec["edge_bwd_bytes"] = [p["bwd_bytes"]]
    d = O.Dfg.from_spec(spec)
    assert d.search(2, O.GEN_GRAY, 0, 4).best_makespan_ps == p["best"]
    assert d.makespan(2, p["split_placement"]) == p["split_makespan"]


def test_K5_star():
    p = GOLD["K5_star"]
    spec = synth.star(p["leaves"], p["delta"], p["delta"])
    d = O.Dfg.from_spec(spec)
    r = d.search(p["M"], O.GEN_GRAY, 0, 2**(p["leaves"] + 1))
    assert r.best_makespan_ps == p["best"]


def test_edge_cost_values():
    p = GOLD["edge_costs"]
    for nbytes, ps in p["cases"]:
        assert O.edge_cost(nbytes, p["bw"], p["lat"]) == ps


def test_K8_toy12_exhaustive():
    p = GOLD["K8_toy12"]
    spec = synth.toy12()
    d = O.Dfg.from_spec(spec)
    assert d.t1 == p["t1"]
    r = d.search(p["M"], O.GEN_GRAY, 0, p["count"])
    assert r.best_makespan_ps == p["best"]
    assert r.best_index == p["gray_index"]
    assert list(r.placement) == p["placement"]
    # independent re-derivation: longest-path brute force + textbook Gray list
    best, opt = brute.exhaustive(spec, 2)
    assert best == p["best"] and len(opt) == p["n_optima"]
    gi, pl = brute.gray_first_index(spec, 2, best)
    assert gi == p["gray_index"] and pl == p["placement"]


# ------------------------------------------------------------ closed forms
@pytest.mark.parametrize("seed", range(6))
def test_K6_chain_su_is_one(seed):
    rng = random.Random(seed)
    K = rng.randint(2, 7)
    spec = synth.chain(K, [rng.randint(1, 50) for _ in range(K)], [rng.randint(0, 90) for _ in range(K)],
                       rng.randint(0, 40), lat=rng.randint(0, 5))
    d = O.Dfg.from_spec(spec)
    for M in (2, 3):
        r = d.search(M, O.GEN_GRAY, 0, M**K)
        assert r.best_makespan_ps == d.t1 == sum(spec["fwd_ps"]) + sum(spec["bwd_ps"])


@pytest.mark.parametrize("K,M", [(4, 2), (6, 2), (6, 3), (8, 4), (8, 2)])
def test_K7_independent_ops_su_is_M(K, M):
    d = O.Dfg.from_spec(synth.independent(K, 4, 5))
    r = d.search(M, O.GEN_GRAY, 0, M**K)
    assert r.best_makespan_ps == (K // M) * 9
    assert d.t1 == K * 9


def test_all_on_one_device_is_t1():
    for name in ("toy12", "inception_v3", "gnmt", "biglstm"):
        spec = getattr(synth, name)()
        d = O.Dfg.from_spec(spec)
        assert d.makespan(2, [0] * d.K) == d.t1 == sum(spec["fwd_ps"]) + sum(spec["bwd_ps"])
        assert d.makespan(4, [3] * d.K) == d.t1


# -------------------------------------------------------------- π (Kahn)
def test_pi_ascending_id_ties():
    # Kahn with ties by ascending id; ids deliberately not 0..K-1
    spec = synth.diamond()
    spec["op_id"] = [40, 7, 3, 90]
    d = O.Dfg.from_spec(spec)
    assert list(d.pi) == [0, 2, 1, 3]
    for seed in range(20):
        s = synth.random_dag(seed, 30)
        assert list(O.Dfg.from_spec(s).pi) == brute.kahn_by_id(30, s["op_id"], s["edge_src"], s["edge_dst"])


def test_validation_errors():
    base = synth.diamond()
    bad = dict(base, edge_src=[0, 0, 1, 3], edge_dst=[1, 2, 3, 1])     # cycle 1->3->1
    with pytest.raises(O.OracleError) as e:
        O.Dfg.from_spec(bad)
    assert e.value.code == -2 and "cycle" in str(e.value)
    with pytest.raises(O.OracleError) as e:
        O.Dfg.from_spec(dict(base, edge_dst=[1, 2, 3, 9]))
    assert e.value.code == -1
    with pytest.raises(O.OracleError) as e:
        O.Dfg.from_spec(dict(base, edge_dst=[1, 2, 3, 2], edge_src=[0, 0, 1, 2]))
    assert e.value.code == -1
    with pytest.raises(O.OracleError) as e:
        O.Dfg.from_spec(dict(base, op_id=[1, 2, 2, 3]))
    assert e.value.code == -1
    with pytest.raises(O.OracleError) as e:
        O.Dfg.from_spec(dict(base, fwd_ps=[2**60, 2**60, 8, 2]))
    assert e.value.code == -3


# ------------------------------------------------ K16: brute-force equality
@pytest.mark.parametrize("seed", range(40))
def test_K16_small_dags_exhaustive_equals_brute(seed):
    rng = random.Random(1000 + seed)
    K = rng.randint(1, 7)
    M = rng.choice([2, 3]) if K <= 6 else 2
    spec = synth.random_dag(seed, K, avg_deg=1.6, max_cost=60, max_bytes=80, lat_max=9)
    if seed % 5 == 0:
        spec["mem_bytes"] = [rng.randint(0, 10) for _ in range(K)]
        spec["dev_mem_cap_bytes"] = rng.randint(10, 40)
    d = O.Dfg.from_spec(spec)
    best, _ = brute.exhaustive(spec, M)
    if best == (1 << 64) - 1:
        with pytest.raises(O.OracleError) as e:
            d.search(M, O.GEN_GRAY, 0, M**K)
        assert e.value.code == -5
        return
    r = d.search(M, O.GEN_GRAY, 0, M**K)
    assert r.best_makespan_ps == best
    gi, pl = brute.gray_first_index(spec, M, best)
    assert r.best_index == gi and list(r.placement) == pl


@pytest.mark.parametrize("seed", range(12))
def test_random_placements_equal_longest_path(seed):
    rng = random.Random(seed)
    K = rng.randint(20, 120)
    spec = synth.random_dag(50 + seed, K, avg_deg=2.0)
    d = O.Dfg.from_spec(spec)
    for _ in range(10):
        M = rng.randint(1, 8)
        pl = [rng.randrange(M) for _ in range(K)]
        assert d.makespan(M, pl) == brute.longest_path_makespan(spec, M, pl)


def test_paper_shaped_placements_equal_longest_path():
    rng = random.Random(7)
    for name in ("toy12", "gnmt", "biglstm", "inception_v3"):
        spec = getattr(synth, name)()
        d = O.Dfg.from_spec(spec)
        for M in (2, 4, 8):
            pl = [rng.randrange(M) for _ in range(d.K)]
            assert d.makespan(M, pl) == brute.longest_path_makespan(spec, M, pl)
