"""Pins of the oracle's general hardware graph: edge cost
= delay of the cheapest route (PAPER.md:424–462 routing constraints and
Δ_e = Σ_l C_el·(D(e)/B(l) + L(l))).

Checked against worked examples (tests/golden/hw_pins.json), closed forms on
named topologies, the uniform-link model (a full mesh must reproduce it), and
the independent Floyd–Warshall + longest-path brute force in tests/brute.py.
"""
import itertools
import json
import os
import random

import pytest

import oracle as O
import synth
from synth import hw as H
from tests import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hw_pins.json")))


def _pair(nbytes, hw):
    """Two ops joined by one edge of `nbytes` in both directions."""
    spec = synth.chain(2, [10, 10], [10, 10], nbytes)
    spec["edge_bwd_bytes"] = [nbytes]
    spec["hw"] = hw
    return spec


@pytest.mark.parametrize("key", ["H1_direct_link", "H2_via_router"])
def test_spec_shortest_route_examples(key):
    p = GOLD[key]
    d = O.Dfg.from_spec(_pair(p["payload"], p["hw"]))
    assert d.hw_edge_cost(0, 0, 1) == p["delay_ps"]
    assert d.hw_edge_cost(0, 1, 0, bwd=True) == p["delay_ps"]
    # split placement: F0 | cut | F1, B1 | cut | B0 on a 2-op chain
    assert d.makespan(2, [0, 1]) == 10 + p["delay_ps"] + 10 + 10 + p["delay_ps"] + 10


def test_same_device_costs_nothing():
    p = GOLD["H3_same_device"]
    d = O.Dfg.from_spec(_pair(p["payload"], H.ring(4, bw=10**6, lat=10**6)))
    for a in range(4):
        assert d.hw_edge_cost(0, a, a) == p["delay_ps"]
        assert d.makespan(4, [a, a]) == 40


@pytest.mark.parametrize("nd", [3, 4, 6, 8])
def test_ring_hops_closed_form(nd):
    bw, lat, nbytes = 10**6, 777, 5
    d = O.Dfg.from_spec(_pair(nbytes, H.ring(nd, bw=bw, lat=lat)))
    hop = 5 * 10**6 + lat
    for a in range(nd):
        for b in range(nd):
            k = min((a - b) % nd, (b - a) % nd)
            assert d.hw_edge_cost(0, a, b) == k * hop


def test_switch_and_two_nodes_closed_form():
    nbytes = 3
    d = O.Dfg.from_spec(_pair(nbytes, H.switch(4, bw=10**6, lat=100)))
    for a, b in itertools.permutations(range(4), 2):
        assert d.hw_edge_cost(0, a, b) == 2 * (3 * 10**6 + 100)
    hw = H.two_nodes(per_node=2, bw=10**6, lat=100, ib_bw=10**5, ib_lat=1000)
    d = O.Dfg.from_spec(_pair(nbytes, hw))
    intra = 2 * (3 * 10**6 + 100)
    inter = intra + 3 * 10**7 + 1000
    assert d.hw_edge_cost(0, 0, 1) == intra and d.hw_edge_cost(0, 2, 3) == intra
    assert d.hw_edge_cost(0, 0, 2) == inter and d.hw_edge_cost(0, 3, 1) == inter


def test_cheapest_route_depends_on_payload():
    # a low-latency thin link vs a high-latency fat link between d0 and d1
    # (via a router): small payloads take the thin link, large the fat one
    hw = {"num_devices": 2, "num_routers": 1, "link_a": [0, 0, 2], "link_b": [1, 2, 1],
          "link_bw_Bps": [10**6, 10**9, 10**9], "link_lat_ps": [0, 10**6, 10**6]}
    small = O.Dfg.from_spec(_pair(1, hw)).hw_edge_cost(0, 0, 1)
    large = O.Dfg.from_spec(_pair(10**4, hw)).hw_edge_cost(0, 0, 1)
    assert small == 10**6                              # thin: 1 B / 1e6 B/s
    assert large == 2 * (10**4 * 10**3 + 10**6)        # fat: two hops


@pytest.mark.parametrize("nd", [2, 3, 5, 8])
def test_full_mesh_equals_uniform_link(nd):
    bw, lat = 7 * 10**9, 12345
    for seed in range(3):
        spec = synth.random_dag(100 + seed, 30, bw=bw, lat_max=0, window=8)
        spec["link_lat_ps"] = lat
        uni = O.Dfg.from_spec(spec)
        spec_hw = dict(spec, hw=H.full_mesh(nd, bw=bw, lat=lat))
        hwd = O.Dfg.from_spec(spec_hw)
        rng = random.Random(seed)
        for _ in range(40):
            pl = [rng.randrange(nd) for _ in range(30)]
            assert hwd.makespan(nd, pl) == uni.makespan(nd, pl)


@pytest.mark.parametrize("seed", range(6))
def test_route_costs_match_floyd_warshall(seed):
    nd = 2 + seed % 6
    hw = H.random_hw(seed, nd, nr=seed % 3, extra_links=seed)
    spec = synth.random_dag(seed, 12, window=6)
    spec["hw"] = hw
    d = O.Dfg.from_spec(spec)
    bb = spec.get("edge_bwd_bytes") or spec["edge_fwd_bytes"]
    for e in range(len(spec["edge_src"])):
        df = brute.route_delays(hw, spec["edge_fwd_bytes"][e])
        db = brute.route_delays(hw, bb[e])
        for a in range(nd):
            for b in range(nd):
                assert d.hw_edge_cost(e, a, b) == df[a][b]
                assert d.hw_edge_cost(e, a, b, bwd=True) == db[a][b]


@pytest.mark.parametrize("seed", range(8))
def test_makespan_matches_longest_path(seed):
    nd = 2 + seed % 7
    hw = [H.ring(nd), H.switch(nd), H.random_hw(seed, nd, nr=1 + seed % 2, extra_links=2)][seed % 3]
    spec = synth.random_dag(50 + seed, 25, max_bytes=10**6, window=6)
    spec["hw"] = hw
    d = O.Dfg.from_spec(spec)
    rng = random.Random(seed)
    for _ in range(25):
        M = rng.randint(1, nd)
        pl = [rng.randrange(M) for _ in range(25)]
        assert d.makespan(M, pl) == brute.longest_path_makespan(spec, M, pl)


def test_exhaustive_search_matches_brute_force():
    spec = synth.random_dag(7, 7, max_bytes=10**6, window=4)
    spec["hw"] = H.ring(3, bw=10**9, lat=10**5)
    d = O.Dfg.from_spec(spec)
    best, opt = brute.exhaustive(spec, 3)
    r = d.search(3, O.GEN_GRAY, 0, 3**7)
    assert r.best_makespan_ps == best
    assert tuple(int(x) for x in r.placement) in opt


def test_hybrid_cube_mesh_classes():
    # direct pairs cost one hop at bw or 2·bw; the rest two hops
    d = O.Dfg.from_spec(_pair(10**3, H.hybrid_cube_mesh(bw=10**9, lat=0)))
    one, dbl = 10**6, 5 * 10**5
    assert d.hw_edge_cost(0, 0, 1) == one and d.hw_edge_cost(0, 0, 3) == dbl
    assert d.hw_edge_cost(0, 0, 4) == dbl
    assert d.hw_edge_cost(0, 0, 5) == dbl + one          # 0 → 4 → 5 (or 0 → 1 → 5)
    assert d.hw_edge_cost(0, 1, 7) == dbl + one          # 1 → 5 → 7 (or 1 → 3 → 7)
    # symmetric
    for a, b in itertools.permutations(range(8), 2):
        assert d.hw_edge_cost(0, a, b) == d.hw_edge_cost(0, b, a)


def test_memory_cap_applies():
    spec = synth.chain(3, [1, 1, 1], [1, 1, 1], 1)
    spec["mem_bytes"] = [10, 10, 10]
    spec["hw"] = H.ring(3, cap=15)
    d = O.Dfg.from_spec(spec)
    assert d.makespan(3, [0, 0, 1]) == 2**64 - 1
    assert d.makespan(3, [0, 1, 2]) < 2**64 - 1


def test_errors():
    spec = _pair(8, {"num_devices": 3, "num_routers": 0, "link_a": [0], "link_b": [1],
                     "link_bw_Bps": [1], "link_lat_ps": [0]})
    with pytest.raises(O.OracleError):              # device 2 unreachable
        O.Dfg.from_spec(spec)
    d = O.Dfg.from_spec(_pair(8, H.ring(3)))
    with pytest.raises(O.OracleError):              # M > num_devices
        d.search(4, O.GEN_GRAY, 0, 16)
    with pytest.raises(O.OracleError):              # zero bandwidth
        O.Dfg.from_spec(_pair(8, dict(H.ring(3), link_bw_Bps=[1, 0, 1])))
