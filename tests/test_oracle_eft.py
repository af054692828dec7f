"""Pins of the oracle's EFT-greedy base seed (SPEC.md:245–253
heuristic_place; reading R23 in DESIGN.md §13)."""
import random

import numpy as np
import pytest

import oracle as O
import synth
from synth import hw as H


def test_spec_single_device():
    # SPEC.md:250 "any single-device hardware graph → all vertices on that device"
    d = O.Dfg.from_spec(synth.toy12())
    assert not d.eft(1).any()


def test_spec_diamond_bounds_and_hand_value():
    # SPEC.md:251 "diamond fixture → makespan ≤ 20 and ≥ 14"; by hand: v0 → d0
    # [0,2]; v1: d0 ends 10, d1 ends 2+1+8 = 11 → d0; v2: d0 ends 18, d1 ends 11
    # → d1; v3: d0 ends max(12, 10)+2 = 14, d1 ends max(11, 11)+2 = 13 → d1.
    spec = synth.diamond(fwd=[2, 8, 8, 2], bwd=[0, 0, 0, 0], fwd_bytes=1, bwd_bytes=0)
    d = O.Dfg.from_spec(spec)
    pl = d.eft(2)
    assert list(pl) == [0, 0, 1, 1]
    assert d.makespan(2, pl) == 13           # = the optimum (K2); SPEC's 14 bound is loose
    assert 13 <= d.makespan(2, pl) <= 20


@pytest.mark.parametrize("M", [2, 3, 4, 8])
def test_independent_equal_ops_round_robin(M):
    # every op can start at once; the least-loaded device (smallest on ties) wins
    K = 3 * M + 1
    d = O.Dfg.from_spec(synth.independent(K, 5, 7))
    assert list(d.eft(M)) == [p % M for p in range(K)]


def test_chain_with_huge_comm_stays_whole():
    spec = synth.chain(6, 10, 10, 10**6)          # 1 µs per edge ≫ 10 ps ops
    assert not O.Dfg.from_spec(spec).eft(4).any()


def test_memory_cap_forces_spreading_and_reports_infeasible():
    spec = synth.chain(3, [1, 1, 1], [1, 1, 1], 1)
    spec["mem_bytes"] = [10, 10, 10]
    spec["dev_mem_cap_bytes"] = 15
    d = O.Dfg.from_spec(spec)
    assert list(d.eft(3)) == [0, 1, 2]
    with pytest.raises(O.OracleError):
        d.eft(2)


@pytest.mark.parametrize("seed", range(8))
def test_greedy_choice_is_locally_optimal(seed):
    # With the placement of ops before p fixed, the in-order forward schedule
    # (or_schedule_ex, pinned separately) gives op p's finish on each device;
    # EFT's device must achieve the minimum, ties to the smaller device.
    rng = random.Random(seed)
    K, M = rng.randint(4, 20), rng.randint(2, 5)
    spec = synth.random_dag(1300 + seed, K, window=5)
    if seed % 2:
        spec["hw"] = H.random_hw(seed, M, nr=1, extra_links=2)
    d = O.Dfg.from_spec(spec)
    pl = d.eft(M)
    pi = list(d.pi)
    for p in range(K):
        k = pi[p]
        fins = []
        for m in range(M):
            alt = pl.copy()
            alt[k] = m
            for q in range(p + 1, K):        # later ops do not affect op p's forward
                alt[pi[q]] = 0
            _, f, _ = d.schedule(M, alt)
            fins.append(int(f[k]) + spec["fwd_ps"][k])
        assert fins[pl[k]] == min(fins)
        assert pl[k] == fins.index(min(fins))


def test_seed_beats_all_zero_base_on_paper_dfgs():
    for name in ("inception_v3", "gnmt", "biglstm"):
        d = O.Dfg.from_spec(getattr(synth, name)())
        for M in (2, 4):
            assert d.makespan(M, d.eft(M)) < d.t1
