"""Pins of the oracle's projection: ring AR (O8), E(G) (O9), cells (O10) and
crossover (O11), against the paper's printed numbers (tests/golden/
projection_pins.json), closed forms and exact invariants."""
import json
import os
import random
from fractions import Fraction

import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "projection_pins.json")))


def _fixture(fn):
    sc, Ms, TM, Nmax = fn()
    S = O.Scenario.from_spec(sc)
    cells = S.project(Ms, TM, Nmax)
    return S, Ms, TM, Nmax, cells


def _ratio(cells, Nmax, N, m_dp=0, m_hy=1, N_hy=None):
    return Fraction(O.cell_C(cells, m_dp, N, Nmax), O.cell_C(cells, m_hy, N_hy or N, Nmax))


def test_K9_ring_allreduce_closed_form():
    p = GOLD["K9_ring_allreduce"]
    S = O.Scenario(dataset_items=1, mini_batch=1, knot_G=[1], knot_uepochs=[1], grad_bytes=p["S"],
                   t1_ps=1, bw_intra_Bps=p["bw"], lat_intra_ps=p["alpha"], node_size=8)
    assert S.ar(p["n"], p["n"]) == p["expected"]
    assert S.ar(1, 1) == 0
    # tier: 8 workers on 16 devices cross nodes -> inter tier, which is off here (bw 0)
    assert S.ar(8, 16) == 0


def test_ring_allreduce_limits():
    S = O.Scenario(dataset_items=1, mini_batch=1, knot_G=[1], knot_uepochs=[1], grad_bytes=10**9,
                   t1_ps=1, bw_intra_Bps=10**11, lat_intra_ps=0, bw_inter_Bps=10**10,
                   lat_inter_ps=0, node_size=8)
    # 2(n-1)/n -> 2: bandwidth term approaches 2*S/BW from below, never above
    lim = 2 * 10**9 * 10**12 // 10**11
    prev = 0
    for n in range(2, 9):
        a = S.ar(n, n)
        assert prev < a <= lim
        prev = a
    assert S.ar(2, 2) == 10**9 * 10**12 // 10**11          # n = 2: exactly S/BW
    assert S.ar(16, 16) > S.ar(8, 8)                       # slower inter-node tier


def test_epochs_interpolation_and_range():
    S = O.Scenario(dataset_items=10, mini_batch=1, knot_G=[2, 4, 8], knot_uepochs=[10, 20, 21],
                   grad_bytes=0, t1_ps=1)
    assert S.epochs(2) == 10 and S.epochs(4) == 20 and S.epochs(8) == 21
    assert S.epochs(3) == 15
    assert S.epochs(5) == 20   # floor(20*3/4 + 21*1/4) = floor(20.25)
    assert S.epochs(1) is None and S.epochs(9) is None


def test_K10_inception_paper_ratios():
    g = GOLD["K10_inception"]
    S, Ms, TM, Nmax, cells = _fixture(synth.inception_fixture)
    for N, (a, b) in g["ratios"].items():
        assert _ratio(cells, Nmax, int(N)) == Fraction(a, b)
    assert float(_ratio(cells, Nmax, 64)) == pytest.approx(1.155)
    assert float(_ratio(cells, Nmax, 256)) == pytest.approx(1.265)
    for N in g["hybrid_loses_at"]:
        assert _ratio(cells, Nmax, N) < 1
    pow2 = [N for N in (2, 4, 8, 16, 32, 64, 128, 256) if _ratio(cells, Nmax, N) > 1]
    assert pow2[0] == g["pow2_crossover"] and pow2 == [64, 128, 256]
    x = O.crossover(cells, Ms, Nmax)
    assert x.n_star == g["all_N_crossover"] and x.n_star_M == [0, g["all_N_crossover"]]
    assert x.persistent_M == [0, 1]
    assert x.m_at_n_star == 2
    assert x.n_star_vs_best_dp == g["n_star_vs_best_dp"]


def test_K11_biglstm_paper_ratios():
    g = GOLD["K11_biglstm"]
    S, Ms, TM, Nmax, cells = _fixture(synth.biglstm_fixture)
    assert _ratio(cells, Nmax, 32) == Fraction(*g["ratio_32"])
    # hybrid 16x2 (N = 32) vs DP's best scale, which is N = 16
    dp = {N: O.cell_C(cells, 0, N, Nmax) for N in range(1, 33)}
    best_N = min(dp, key=lambda n: (dp[n], n))
    assert best_N == g["best_dp_N"]
    assert Fraction(dp[best_N], O.cell_C(cells, 1, 32, Nmax)) == Fraction(*g["ratio_vs_best_dp"])
    c11 = O.cell_C(cells, 0, 1, Nmax)
    assert Fraction(c11, dp[32]) == Fraction(*g["dp_speedup_32"])
    assert Fraction(c11, O.cell_C(cells, 1, 32, Nmax)) == Fraction(*g["hybrid_speedup_32"])
    # Eq. 6 margin SU^2 - 2*E_16/E_32 = 1.22 - 2/3.2 = 0.595
    e16, e32 = cells[15].uepochs, cells[31].uepochs
    assert Fraction(122, 100) - 2 * Fraction(e16, e32) == Fraction(595, 1000)
    x = O.crossover(cells, Ms, Nmax)
    assert x.n_star == g["all_N_crossover"]
    assert x.n_star_vs_best_dp == g["n_star_vs_best_dp"]
    assert x.persistent_M == [0, 1]


def test_K12_gnmt_paper_ratio():
    g = GOLD["K12_gnmt"]
    S, Ms, TM, Nmax, cells = _fixture(synth.gnmt_fixture)
    assert _ratio(cells, Nmax, 256) == Fraction(*g["ratio_256"])
    x = O.crossover(cells, Ms, Nmax)
    assert x.n_star == g["all_N_crossover"] and x.persistent_M == [0, 1]


@pytest.mark.parametrize("delta", [-1, 0, 1])
def test_K13_threshold_strict(delta):
    # SU^2 = 1.32; E_2N/E_N = 2/1.32 = 50/33 flips the crossover exactly (Eq. 6 strict)
    U = 10**9
    sc = dict(dataset_items=2**20, mini_batch=1, knot_G=[1, 2, 4, 8], grad_bytes=0, t1_ps=132 * U,
              knot_uepochs=[33 * 10**6, 33 * 10**6, 33 * 10**6, 50 * 10**6 + delta])
    S = O.Scenario.from_spec(sc)
    cells = S.project([1, 2], [132 * U, 100 * U], 8)
    x = O.crossover(cells, [1, 2], 8)
    assert (x.n_star == 8) == (delta > 0)
    if delta <= 0:
        assert x.n_star == 0


def test_K14_fig3_hypothetical():
    g = GOLD["K14_fig3"]
    u = 10**6
    T1 = 145 * 165 * u
    TM = [T1, T1 * g["su2"][1] // g["su2"][0], T1 * g["su4"][1] // g["su4"][0]]
    # DP scales perfectly to 32 workers, then epochs grow 1.5x per doubling
    G = [2**k for k in range(9)]
    E = [10**6] * 6 + [1_500_000, 2_250_000, 3_375_000]
    S = O.Scenario(dataset_items=2**20, mini_batch=1, knot_G=G, knot_uepochs=E, grad_bytes=0, t1_ps=T1)
    Ms = [1, 2, 4]
    cells = S.project(Ms, TM, 128)
    x = O.crossover(cells, Ms, 128)
    assert all(m == 1 for m in x.best_m[:32])           # DP up to 32 devices
    assert x.best_m[63] == 2                             # 32x2 at 64 devices
    C = lambda m, N: O.cell_C(cells, m, N, 128)
    assert C(1, 64) < C(0, 64)                           # 32x2 beats 64-way DP
    assert C(1, 64) < C(2, 64)                           # 16x4 worse than 32x2
    pow2 = [N for N in (2, 4, 8, 16, 32, 64, 128) if x.best_m[N - 1] != 1]
    assert pow2 == [64, 128] and x.best_m[127] == 2       # hybrid from 64 on; (·,2) best


def test_eq5_and_time_modes_coincide_without_ar():
    for fn in (synth.inception_fixture, synth.biglstm_fixture, synth.gnmt_fixture):
        sc, Ms, TM, Nmax = fn()
        a = O.Scenario.from_spec(dict(sc, ar_mode=0)).project(Ms, TM, Nmax)
        b = O.Scenario.from_spec(dict(sc, ar_mode=1)).project(Ms, TM, Nmax)
        assert [c.C for c in a] == [c.C for c in b]


def _rand_scenario(rng, ar_mode=0, ar_on=True):
    B = rng.choice([16, 32, 64, 128])
    n = rng.randint(3, 12)
    E = [rng.randint(10**5, 10**7)]
    for _ in range(n - 1):
        E.append(E[-1] * rng.randint(100, 300) // 100)
    t1 = rng.randint(10**8, 10**12)
    return dict(dataset_items=rng.randint(10**4, 10**8), mini_batch=B, knot_G=[B * 2**k for k in range(n)],
                knot_uepochs=E, grad_bytes=rng.randint(10**6, 10**10), t1_ps=t1,
                bw_intra_Bps=rng.randint(10**10, 10**12) if ar_on else 0, lat_intra_ps=rng.randint(0, 10**7),
                bw_inter_Bps=rng.randint(10**9, 10**11) if ar_on else 0, lat_inter_ps=rng.randint(0, 10**8),
                node_size=rng.choice([4, 8]), ar_mode=ar_mode)


@pytest.mark.parametrize("seed", range(30))
def test_R18_ar_never_lowers_hybrid_gain_in_eq5(seed):
    rng = random.Random(seed)
    sc = _rand_scenario(rng)
    t1 = sc["t1_ps"]
    Ms = [1, 2, 4, 8]
    TM = [t1] + [rng.randint(t1 // M, t1) for M in Ms[1:]]
    on = O.Scenario.from_spec(sc).project(Ms, TM, 256)
    off = O.Scenario.from_spec(dict(sc, bw_intra_Bps=0, bw_inter_Bps=0)).project(Ms, TM, 256)
    for m in range(1, 4):
        for N in range(1, 257):
            a_on, b_on = O.cell_C(on, 0, N, 256), O.cell_C(on, m, N, 256)
            a_off, b_off = O.cell_C(off, 0, N, 256), O.cell_C(off, m, N, 256)
            if b_on and b_off and a_on and a_off:
                assert a_on * b_off >= a_off * b_on


@pytest.mark.parametrize("seed", range(10))
def test_epoch_scale_invariance_of_decisions(seed):
    # scaling every epoch value by c changes no decision
    rng = random.Random(100 + seed)
    sc = _rand_scenario(rng, ar_on=rng.random() < 0.5)
    t1 = sc["t1_ps"]
    Ms = [1, 2, 4]
    TM = [t1] + [rng.randint(t1 // M, t1) for M in Ms[1:]]
    x1 = O.crossover(O.Scenario.from_spec(sc).project(Ms, TM, 200), Ms, 200)
    sc2 = dict(sc, knot_uepochs=[3 * e for e in sc["knot_uepochs"]])
    x2 = O.crossover(O.Scenario.from_spec(sc2).project(Ms, TM, 200), Ms, 200)
    assert (x1.n_star, x1.n_star_M, x1.persistent_M, x1.best_m) == \
           (x2.n_star, x2.n_star_M, x2.persistent_M, x2.best_m)


def test_cells_structure():
    sc, Ms, TM, Nmax = synth.inception_fixture()
    cells = O.Scenario.from_spec(sc).project(Ms, TM, Nmax)
    for N in range(1, Nmax + 1):
        assert cells[Nmax + N - 1].feasible == (N % 2 == 0)            # M ∤ N infeasible (R15)
        c = cells[N - 1]
        assert c.steps == -(-sc["dataset_items"] // (N * sc["mini_batch"]))   # ⌈D/G⌉
        assert c.C == c.step_ps * c.steps * c.uepochs
    # steps_per_epoch examples
    S = O.Scenario(dataset_items=1000, mini_batch=300, knot_G=[300, 600], knot_uepochs=[1, 1],
                   grad_bytes=0, t1_ps=1)
    assert S.project([1], [1], 1)[0].steps == 4
