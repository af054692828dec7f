"""Pins of the oracle's exact schedule (reading R22 in
DESIGN.md §12): the makespan-optimal schedule of a fixed placement.

Checked against SPEC.md's exact_schedule / brute_force_place worked examples,
a hand-built case where in-order issue loses, the independent disjunctive-graph
brute force (tests/brute.py::exact_makespan: all per-device orders, longest
path), and bounds that hold for any schedule.
"""
import itertools
import random

import numpy as np
import pytest

import oracle as O
import synth
from synth import hw as H
from tests import brute


def test_spec_single_device_chain_equals_list_schedule():
    # SPEC.md:165 "any single-device chain → same as list_schedule"
    spec = synth.chain(4, [2, 8, 3, 5], [1, 1, 1, 1], 100)
    d = O.Dfg.from_spec(spec)
    assert d.makespan_exact(1, [0] * 4) == d.makespan(1, [0] * 4) == 2 + 8 + 3 + 5 + 4
    assert d.makespan_exact(2, [0] * 4) == 22


def test_spec_split_diamond_is_14():
    # SPEC.md:166 "diamond split as above → makespan 14 (list schedule already optimal)"
    spec = synth.diamond(fwd=[2, 8, 8, 2], bwd=[0, 0, 0, 0], fwd_bytes=1, bwd_bytes=0)
    d = O.Dfg.from_spec(spec)
    assert d.makespan_exact(2, [0, 0, 1, 0]) == d.makespan(2, [0, 0, 1, 0]) == 14
    assert d.makespan_exact(2, [0, 0, 0, 0]) == 20          # SPEC.md:159 serial sum


def test_in_order_issue_loses_hand_case():
    # a (id 0, 10 ps) and b (id 1, 1 ps) on device 0, c (id 2, 10 ps) on device 1,
    # edge b → c free.  π = (a, b, c): in order a runs first and c starts at 11,
    # finishing at 21; the optimum runs b first: b [0,1], a [1,11], c [1,11] → 11.
    spec = {"fwd_ps": [10, 1, 10], "bwd_ps": [0, 0, 0], "edge_src": [1], "edge_dst": [2],
            "edge_fwd_bytes": [0], "link_bw_Bps": 10**12, "link_lat_ps": 0}
    d = O.Dfg.from_spec(spec)
    assert d.makespan(2, [0, 0, 1]) == 21
    assert d.makespan_exact(2, [0, 0, 1]) == 11
    assert brute.exact_makespan(spec, 2, [0, 0, 1]) == 11


def test_spec_star_two_devices():
    # SPEC.md:241 "star graph 0→{1,2,3,4}, Δ all equal, zero comm cost, 2 devices
    # → makespan = Δ0 + 2Δ (two leaves per device)"
    spec = synth.star(4, 10, 10, nbytes=0, lat=0)        # 0 bytes, 0 latency: free edges
    d = O.Dfg.from_spec(spec)
    best, idx = d.round_exact(2, O.GEN_GRAY, 0, 0, None, 0, 2**5)
    assert best == 10 + 2 * 10


def test_spec_brute_force_place_examples():
    # SPEC.md:235 1 vertex (Δ=10), 2 devices → 10
    d = O.Dfg.from_spec(synth.chain(1, [10], [0], 0))
    assert d.round_exact(2, O.GEN_GRAY, 0, 0, None, 0, 2) == (10, 0)
    # SPEC.md:236 chain 0(5)→1(5), delay 1000 → co-located, 10 (split costs 1010)
    spec = synth.chain(2, [5, 5], [0, 0], 1000)
    spec["edge_bwd_bytes"] = [0]
    spec["link_bw_Bps"], spec["link_lat_ps"] = 10**12, 0
    d = O.Dfg.from_spec(spec)
    assert d.makespan_exact(2, [0, 1]) == 1010
    assert d.round_exact(2, O.GEN_GRAY, 0, 0, None, 0, 4) == (10, 0)
    # SPEC.md:237 diamond on 2 devices, unit cross delay: SPEC says 14, but its
    # 16 placements include (0,0,1,1) at 13 (tests/golden/schedule_pins.json K2,
    # SURVEY.md §8(c) K2); the exact schedule cannot beat 13 either: device 1
    # runs v2 (8) and v3 (2) after v0's output arrives at 3; the brute force
    # over all 16 placements and all per-device orders agrees.
    spec = synth.diamond(fwd=[2, 8, 8, 2], bwd=[0, 0, 0, 0], fwd_bytes=1, bwd_bytes=0)
    assert O.Dfg.from_spec(spec).round_exact(2, O.GEN_GRAY, 0, 0, None, 0, 16)[0] == 13
    assert min(brute.exact_makespan(spec, 2, pl) for pl in itertools.product(range(2), repeat=4)) == 13


@pytest.mark.parametrize("seed", range(12))
def test_matches_disjunctive_brute_force(seed):
    rng = random.Random(seed)
    K = rng.randint(1, 4)
    M = rng.choice([2, 2, 3])
    spec = synth.random_dag(700 + seed, K, max_cost=20, max_bytes=30, bw=10**12, lat_max=5)
    d = O.Dfg.from_spec(spec)
    for pl in itertools.product(range(M), repeat=K):
        assert d.makespan_exact(M, pl) == brute.exact_makespan(spec, M, pl), pl


@pytest.mark.parametrize("seed", range(4))
def test_matches_brute_force_on_hardware_graph(seed):
    spec = synth.random_dag(800 + seed, 4, max_cost=10**6, max_bytes=10**6, window=3)
    spec["hw"] = H.ring(3, bw=10**9, lat=10**5)
    d = O.Dfg.from_spec(spec)
    rng = random.Random(seed)
    for _ in range(6):
        pl = [rng.randrange(3) for _ in range(4)]
        assert d.makespan_exact(3, pl) == brute.exact_makespan(spec, 3, pl)


@pytest.mark.parametrize("seed", range(10))
def test_bounds_and_invariants(seed):
    rng = random.Random(seed)
    K = rng.randint(3, 7)
    M = rng.randint(2, 4)
    spec = synth.random_dag(900 + seed, K, max_cost=50, max_bytes=80, bw=10**12, lat_max=10)
    d = O.Dfg.from_spec(spec)
    assert d.makespan_exact(1, [0] * K) == d.t1                         # one device: the serial sum
    for _ in range(8):
        pl = [rng.randrange(M) for _ in range(K)]
        ex, lo = d.makespan_exact(M, pl), d.makespan(M, pl)
        assert ex <= lo                                                 # SPEC.md:167 dominance
        work = max(sum(spec["fwd_ps"][k] + spec["bwd_ps"][k] for k in range(K) if pl[k] == m)
                   for m in range(M))
        assert ex >= work                                               # one op at a time per device
        perm = list(range(M))
        rng.shuffle(perm)
        assert d.makespan_exact(M, [perm[x] for x in pl]) == ex         # identical devices
    # the exact search is no worse than the in-order search
    n = min(M**K, 300)
    assert d.round_exact(M, O.GEN_GRAY, 0, 0, None, 0, n)[0] <= d.round(M, O.GEN_GRAY, 0, 0, None, 0, n)[0]


def test_memory_cap():
    spec = synth.chain(3, [1, 1, 1], [1, 1, 1], 1)
    spec["mem_bytes"] = [10, 10, 10]
    spec["dev_mem_cap_bytes"] = 15
    d = O.Dfg.from_spec(spec)
    assert d.makespan_exact(3, [0, 0, 1]) == O.INFEASIBLE
    assert d.makespan_exact(3, [0, 1, 2]) < O.INFEASIBLE
