"""Pins of the oracle's gradient-accumulation axis and placement-aware
all-reduce shards (PAPER.md:251 delayed gradient update;
readings R24/R25 in DESIGN.md §13)."""
import numpy as np
import pytest

import oracle as O
import synth

# D = 1000 items, B = 10, a flat E(G) = 10^6 µ-epochs on G ∈ [10, 10^6];
# all-reduce of S = 1000 B at 1.5·10^12 B/s over W = 4: ⌈2·3·1000·10^12 /
# (4·1.5·10^12)⌉ = 1000 ps, no latency.
FLAT = dict(dataset_items=1000, mini_batch=10, knot_G=[10, 10**6], knot_uepochs=[10**6, 10**6],
            grad_bytes=1000, t1_ps=100, bw_intra_Bps=1_500_000_000_000, lat_intra_ps=0,
            bw_inter_Bps=1_500_000_000_000, lat_inter_ps=0, node_size=8)


@pytest.mark.parametrize("mode", [0, 1])
def test_hand_case_best_accumulation(mode):
    # N = 4, M = 1 (W = 4), T_M = T_1 = 100: C(a) = (100a + 1000)·⌈1000/(40a)⌉·10^6
    #   a = 1: 1100·25 = 27500;  a = 4: 1400·7 = 9800;  a = 16: 2600·2 = 5200;
    #   a = 64: 7400·1 = 7400   → a = 16
    sc = O.Scenario(**FLAT, ar_mode=mode, accum=[1, 4, 16, 64])
    c = sc.project([1], [100], 4)[3]
    assert (c.feasible, c.accum, c.step_ps, c.steps, c.uepochs) == (1, 16, 2600, 2, 10**6)
    assert (c.C_hi << 64 | c.C_lo) == 5200 * 10**6
    # without the axis the cell is the a = 1 value
    c1 = O.Scenario(**FLAT, ar_mode=mode).project([1], [100], 4)[3]
    assert (c1.accum, c1.C_lo) == (1, 27500 * 10**6)


def test_accum_one_is_the_default_on_paper_scenarios():
    for name in ("inception_v3", "gnmt", "biglstm"):
        spec = synth.sweep_scenario(name, 10**9, 10**8)
        a = O.Scenario.from_spec(spec).project([1, 2, 4], [10**9, 6 * 10**8, 4 * 10**8], 256)
        b = O.Scenario(**spec, accum=[1]).project([1, 2, 4], [10**9, 6 * 10**8, 4 * 10**8], 256)
        assert [(x.C_lo, x.C_hi, x.feasible) for x in a] == [(x.C_lo, x.C_hi, x.feasible) for x in b]


def test_more_factors_never_hurt():
    spec = synth.sweep_scenario("gnmt", 10**9, 10**9)
    small = O.Scenario(**spec, accum=[1, 2]).project([1, 2], [10**9, 6 * 10**8], 128)
    big = O.Scenario(**spec, accum=[1, 2, 4, 8]).project([1, 2], [10**9, 6 * 10**8], 128)
    for x, y in zip(small, big):
        if x.feasible:
            assert y.feasible and (y.C_hi << 64 | y.C_lo) <= (x.C_hi << 64 | x.C_lo)


def test_shards_take_the_slowest_device():
    # M = 2, N = 8: W = 4 workers; AR(4, S_d) = S_d ps with this link
    base = dict(FLAT, accum=None)
    full = O.Scenario(**base, ar_mode=1).project([2], [100], 8)[7]
    assert full.step_ps == 100 + 1000
    halves = O.Scenario(**base, ar_mode=1, shard_bytes=[[500, 500, 0, 0, 0, 0, 0, 0]]).project([2], [100], 8)[7]
    assert halves.step_ps == 100 + 500
    skew = O.Scenario(**base, ar_mode=1, shard_bytes=[[300, 700, 0, 0, 0, 0, 0, 0]]).project([2], [100], 8)[7]
    assert skew.step_ps == 100 + 700


def test_shard_bytes_of_a_placement():
    spec = synth.chain(4, 10, 10, 1)
    spec["param_bytes"] = [1, 20, 300, 4000]
    d = O.Dfg.from_spec(spec)
    assert d.shard_bytes(2, [0, 1, 1, 0]) == [4001, 320, 0, 0, 0, 0, 0, 0]
    assert sum(d.shard_bytes(3, [2, 0, 1, 2])) == d.grad_bytes


def test_invalid_accum():
    with pytest.raises(O.OracleError):
        O.Scenario(**FLAT, accum=[1, 0]).project([1], [100], 4)
