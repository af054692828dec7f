"""GPU parity of the exact schedule: the warp-per-
placement Giffler–Thompson branch and bound (exact_kernel.cuh) against the
oracle's enumeration of linear extensions (or_exact), bit for bit."""
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


def _check_explicit(spec, M, pl):
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    mk, ex = g.eval_exact(M, torch.as_tensor(pl, device="cuda"))
    got, ex = pp.u64(mk), ex.cpu().numpy()
    want = np.array([od.makespan_exact(M, row) for row in pl], dtype=np.uint64)
    assert ex.all()
    assert np.array_equal(got, want)
    lo = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
    assert (got <= lo).all()                      # never worse than in-order issue
    return got


def test_toy12_random_placements():
    spec = synth.toy12()
    rng = np.random.default_rng(0)
    for M in (2, 3, 4):
        pl = rng.integers(0, M, size=(300 + 17, 12), dtype=np.uint8)
        got = _check_explicit(spec, M, pl)
        assert (got < pp.u64(pp.Dfg(spec).eval_placements(M, torch.as_tensor(pl, device="cuda")))).any()


@pytest.mark.parametrize("seed", range(10))
def test_random_dags(seed):
    rng = random.Random(seed)
    K = rng.randint(1, 11)
    M = rng.randint(1, 5)
    spec = synth.random_dag(1000 + seed, K, max_cost=200, max_bytes=300, bw=10**12, lat_max=20, window=5)
    if seed % 3 == 0:
        spec["mem_bytes"] = [rng.randint(0, 100) for _ in range(K)]
        spec["dev_mem_cap_bytes"] = 150
    pl = np.random.default_rng(seed).integers(0, M, size=(257, K), dtype=np.uint8)
    _check_explicit(spec, M, pl)


@pytest.mark.parametrize("seed", range(4))
def test_hardware_graph(seed):
    nd = 3 + seed
    spec = synth.random_dag(1100 + seed, 9, max_cost=10**6, max_bytes=10**6, window=4)
    spec["hw"] = [H.ring(nd), H.switch(nd), H.random_hw(seed, nd, nr=1, extra_links=2), H.ring(nd)][seed]
    pl = np.random.default_rng(seed).integers(0, nd, size=(200, 9), dtype=np.uint8)
    _check_explicit(spec, nd, pl)


@pytest.mark.parametrize("gen", [O.GEN_GRAY, O.GEN_RANDOM, O.GEN_PERTURB])
@pytest.mark.parametrize("M", [2, 3])
def test_generated_and_search(gen, M):
    K = 7 if M == 2 else 5
    spec = synth.random_dag(1200 + M + gen, K, max_cost=100, max_bytes=150, bw=10**12, lat_max=10)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    base = np.random.default_rng(gen).integers(0, M, size=K, dtype=np.uint8)
    n = M**K if gen == O.GEN_GRAY else 1500
    mk, ex = g.eval_exact_generated(M, gen, 77, 64, base, 0, n)
    want = np.array([od.exact_pi(M, O.gen(K, M, gen, 77, 64, base, i)) for i in range(n)], dtype=np.uint64)
    assert ex.cpu().numpy().all()
    assert np.array_equal(pp.u64(mk), want)
    best, idx, unresolved = g.search_exact(M, gen, 77, 64, base, 0, n)
    assert unresolved == 0
    assert (best, idx) == od.round_exact(M, gen, 77, 64, base, 0, n)
    # a sub-range with a ragged start
    assert g.search_exact(M, gen, 77, 64, base, 13, n - 5)[:2] == od.round_exact(M, gen, 77, 64, base, 13, n - 5)


def test_toy12_exhaustive_exact_search():
    spec = synth.toy12()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    best, idx, unresolved = g.search_exact(2, pp.GEN_GRAY, 0, 0, None, 0, 4096)
    assert unresolved == 0
    assert (best, idx) == od.round_exact(2, O.GEN_GRAY, 0, 0, None, 0, 4096)
    assert best <= 920_000_000                     # the in-order optimum (K8)


def test_node_limit_reports_bound():
    spec = synth.toy12()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    pl = np.random.default_rng(3).integers(0, 3, size=(64, 12), dtype=np.uint8)
    mk, ex = g.eval_exact(3, torch.as_tensor(pl, device="cuda"), node_limit=3)
    mk, ex = pp.u64(mk), ex.cpu().numpy()
    want = np.array([od.makespan_exact(3, row) for row in pl], dtype=np.uint64)
    assert (mk >= want).all()
    assert (mk[ex == 1] == want[ex == 1]).all()
    assert (ex == 0).any()


def test_too_large_and_invalid():
    g = pp.Dfg(synth.inception_v3())                 # K = 324 > 32
    with pytest.raises(pp.PPError):
        g.search_exact(2, pp.GEN_RANDOM, 0, 0, None, 0, 10)
    g = pp.Dfg(synth.toy12())
    with pytest.raises(pp.PPError):
        g.search_exact(9, pp.GEN_RANDOM, 0, 0, None, 0, 10)
