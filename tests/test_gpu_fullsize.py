"""Parity at BASELINE.json's full size, in the launch configuration bench.py
times (Inception-V3-shaped, M = 2, PERTURB τ = 8/256, 10⁷ candidates per
round, EFT base): the oracle cannot evaluate 10⁸ placements, so the checks
are on outputs it CAN compute one by one (SURVEY.md §8(c) / task ③):

  * the round-0 argmin's makespan re-evaluated by the oracle;
  * 3,000 sampled candidates of the same round, each ≥ the argmin (and not
    smaller in index when equal);
  * a 4,096-candidate block at a random offset, element by element;
  * the 10-round search: the winner's placement re-evaluated by the oracle,
    and no worse than round 0.
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402

SEED, COUNT, ROUNDS, TAU, M = 13257, 10_000_000, 10, 8, 2


@pytest.fixture(scope="module")
def setup():
    spec = synth.inception_v3()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    base = g.eft_place(M)
    assert np.array_equal(base, od.eft(M))
    return spec, g, od, base


def test_round0_argmin_and_samples(setup):
    spec, g, od, base = setup
    base_pi = np.ascontiguousarray(base[od.pi])
    best = pp.u64(g.search_range(M, pp.GEN_PERTURB, SEED, TAU, base_pi, 0, COUNT))
    mk, idx = int(best[0]), int(best[1])
    assert od.makespan_pi(M, O.gen(od.K, M, O.GEN_PERTURB, SEED, TAU, base_pi, idx)) == mk
    rng = np.random.default_rng(1)
    for i in rng.integers(0, COUNT, 3000):
        v = od.makespan_pi(M, O.gen(od.K, M, O.GEN_PERTURB, SEED, TAU, base_pi, int(i)))
        assert v > mk or (v == mk and int(i) >= idx)
    assert mk <= od.makespan(M, base)          # candidate 0 is the base


def test_block_element_by_element(setup):
    spec, g, od, base = setup
    base_pi = np.ascontiguousarray(base[od.pi])
    lo = int(np.random.default_rng(2).integers(0, COUNT - 4096))
    got = pp.u64(g.eval_generated(M, pp.GEN_PERTURB, SEED, TAU, base_pi, lo, 4096))
    want = np.array([od.makespan_pi(M, O.gen(od.K, M, O.GEN_PERTURB, SEED, TAU, base_pi, i))
                     for i in range(lo, lo + 4096)], dtype=np.uint64)
    assert np.array_equal(got, want)


def test_full_search_winner(setup):
    spec, g, od, base = setup
    r = g.search_best(M, pp.GEN_PERTURB, SEED, COUNT, rounds=ROUNDS, tau=TAU, base=base)
    assert r.evaluated == COUNT * ROUNDS
    assert od.makespan(M, r.placement) == r.best_makespan_ps
    base_pi = np.ascontiguousarray(base[od.pi])
    r0 = int(pp.u64(g.search_range(M, pp.GEN_PERTURB, SEED, TAU, base_pi, 0, COUNT))[0])
    assert r.best_makespan_ps <= r0
    assert r.t1_ps == od.t1 and r.best_makespan_ps < r.t1_ps
