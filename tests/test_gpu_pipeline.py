"""GPU parity of the pipeline-parallel MP evaluation:
pipeline_kernel against the oracle's or_pipeline, bit for bit."""
import itertools
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

MICRO = [1, 2, 4, 8, 16, 32]


@pytest.mark.parametrize("seed", range(8))
def test_every_candidate_small_dags(seed):
    rng = random.Random(seed)
    K = rng.randint(2, 16)
    M = rng.randint(1, min(8, K))
    spec = synth.random_dag(1700 + seed, K, max_cost=10**4, max_bytes=10**5, bw=10**11, lat_max=100, window=5)
    if seed % 3 == 1:
        spec["mem_bytes"] = [rng.randint(0, 10) for _ in range(K)]
        spec["dev_mem_cap_bytes"] = 30
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    micro = [1, 3, 4, 7]
    n = g.pipeline_space(M, len(micro))
    (bm, bi), vals = g.pipeline_range(M, micro, 0, n, all_values=True)
    combos = list(itertools.combinations(range(1, K), M - 1))
    assert n == len(combos) * len(micro)
    want = np.array([od.pipeline(M, list(combos[i // 4]), micro[i % 4]) for i in range(n)], dtype=np.uint64)
    assert np.array_equal(pp.u64(vals), want)
    assert (bm, bi) == od.pipeline_search(M, micro)


@pytest.mark.parametrize("name", ["gnmt", "biglstm", "inception_v3"])
def test_paper_dfgs_full_search(name):
    spec = getattr(synth, name)()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    for M in (2, 3):
        r = g.pipeline_search(M, MICRO)
        assert (r["makespan_ps"], r["index"]) == od.pipeline_search(M, MICRO)
        assert od.pipeline(M, r["cuts"], r["micro_batches"]) == r["makespan_ps"]
        assert r["makespan_ps"] < od.t1


@pytest.mark.parametrize("M", [4, 6, 8])
def test_paper_dfg_ranges(M):
    spec = synth.gnmt()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    n = g.pipeline_space(M, len(MICRO))
    rng = random.Random(M)
    for _ in range(3):
        lo = rng.randrange(0, n - 3000)
        (bm, bi), vals = g.pipeline_range(M, MICRO, lo, lo + 2999, all_values=True)
        assert (bm, bi) == od.pipeline_search(M, MICRO, lo, lo + 2999)
    # the last candidates of the space (ragged end)
    (bm, bi), _ = g.pipeline_range(M, MICRO, n - 777, n)
    assert (bm, bi) == od.pipeline_search(M, MICRO, n - 777, n)


def test_errors():
    g = pp.Dfg(dict(synth.toy12(), hw=H.ring(4)))
    with pytest.raises(pp.PPError):
        g.pipeline_search(2, MICRO)
    g = pp.Dfg(synth.toy12())
    with pytest.raises(pp.PPError):
        g.pipeline_search(13, MICRO)            # more stages than ops
    with pytest.raises(pp.PPError):
        g.pipeline_search(2, [0])
    # the u64 pipeline arithmetic is range-checked: a per-op
    # overhead that would wrap is PP_E_RANGE, not a silent overflow
    with pytest.raises(pp.PPError) as e:
        g.pipeline_search(2, [65536], overhead=2**50)
    assert e.value.code == -3


@pytest.mark.parametrize("overhead", [1, 5_000_000])
def test_op_overhead(overhead):
    spec = synth.gnmt()
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    for M in (2, 3):
        r = g.pipeline_search(M, MICRO, overhead=overhead)
        assert (r["makespan_ps"], r["index"]) == od.pipeline_search(M, MICRO, overhead=overhead)
    small = synth.random_dag(1900, 9, max_cost=10**4, max_bytes=10**5, bw=10**11, lat_max=100, window=4)
    g, od = pp.Dfg(small), O.Dfg.from_spec(small)
    n = g.pipeline_space(3, 4)
    _, vals = g.pipeline_range(3, [1, 2, 3, 5], 0, n, all_values=True, overhead=overhead)
    combos = list(itertools.combinations(range(1, 9), 2))
    want = np.array([od.pipeline(3, list(combos[i // 4]), [1, 2, 3, 5][i % 4], overhead=overhead) for i in range(n)],
                    dtype=np.uint64)
    assert np.array_equal(pp.u64(vals), want)
