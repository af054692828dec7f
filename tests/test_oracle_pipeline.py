"""Pins of the oracle's pipeline-parallel MP evaluation (
PAPER.md:100, :297; reading R26 in DESIGN.md §14)."""
import itertools
import random

import pytest

import oracle as O
import synth
from tests import brute


@pytest.mark.parametrize("M,m", [(2, 1), (2, 4), (4, 4), (4, 8), (8, 16), (3, 6)])
def test_gpipe_bubble_closed_form(M, m):
    # a uniform chain split into M equal stages with free transfers:
    # makespan = (m + M − 1)·(tf + tb), i.e. SU = M·m / (m + M − 1) (GPipe's bubble)
    q, d = 3, 48                                   # ops per stage, Δ per op (m | q·d)
    K = M * q
    spec = synth.chain(K, d, 2 * d, 0, lat=0)
    od = O.Dfg.from_spec(spec)
    cuts = [q * s for s in range(1, M)]
    tf, tb = q * d // m, q * 2 * d // m
    assert od.pipeline(M, cuts, m) == (m + M - 1) * (tf + tb)
    assert od.pipeline(M, cuts, m) * M * m == od.t1 * (m + M - 1)


def test_single_stage_is_serial():
    spec = synth.random_dag(3, 20, max_cost=64, window=5)
    spec["fwd_ps"] = [64 * x for x in spec["fwd_ps"]]
    spec["bwd_ps"] = [64 * x for x in spec["bwd_ps"]]
    od = O.Dfg.from_spec(spec)
    for m in (1, 2, 4, 8, 16, 32, 64):
        assert od.pipeline(1, [], m) == od.t1


def test_one_micro_batch_chain_pays_each_transfer_twice():
    # m = 1 on a chain: no overlap; one activation and one gradient transfer per cut
    spec = synth.chain(6, 10, 20, 1000, bw=10**12, lat=7)
    od = O.Dfg.from_spec(spec)
    assert od.pipeline(3, [2, 4], 1) == od.t1 + 2 * 2 * (1000 + 7)


@pytest.mark.parametrize("seed", range(10))
def test_matches_task_graph_brute_force(seed):
    rng = random.Random(seed)
    K = rng.randint(3, 14)
    M = rng.randint(1, min(4, K))
    spec = synth.random_dag(1500 + seed, K, max_cost=500, max_bytes=5000, bw=10**12 // 3, lat_max=50, window=4)
    if seed % 3 == 0:
        spec["mem_bytes"] = [rng.randint(0, 10) for _ in range(K)]
        spec["dev_mem_cap_bytes"] = 25
    od = O.Dfg.from_spec(spec)
    for cuts in itertools.islice(itertools.combinations(range(1, K), M - 1), 40):
        for m in (1, 2, 3, 5):
            assert od.pipeline(M, list(cuts), m) == brute.pipeline_makespan(spec, M, list(cuts), m), (cuts, m)


@pytest.mark.parametrize("seed", range(4))
def test_exhaustive_search(seed):
    K, M = 9, 2 + seed % 3
    spec = synth.random_dag(1600 + seed, K, max_cost=300, max_bytes=3000, bw=10**12, lat_max=30, window=4)
    od = O.Dfg.from_spec(spec)
    micro = [1, 2, 4, 8]
    best = None
    for r, cuts in enumerate(itertools.combinations(range(1, K), M - 1)):
        for j, m in enumerate(micro):
            v = (brute.pipeline_makespan(spec, M, list(cuts), m), r * len(micro) + j)
            best = v if best is None or v < best else best
    assert od.pipeline_search(M, micro) == best
    # a sub-range
    n = len(list(itertools.combinations(range(1, K), M - 1))) * len(micro)
    lo, hi = n // 3, 2 * n // 3
    sub = min((brute.pipeline_makespan(spec, M, list(c), micro[i % 4]), i)
              for i, c in ((i, list(itertools.combinations(range(1, K), M - 1))[i // 4]) for i in range(lo, hi)))
    assert od.pipeline_search(M, micro, lo, hi) == sub


def test_pipelining_helps_the_rnn_shaped_dfgs():
    for name in ("gnmt", "biglstm"):
        od = O.Dfg.from_spec(getattr(synth, name)())
        mk, idx = od.pipeline_search(2, [1, 2, 4, 8])
        assert mk < od.t1


@pytest.mark.parametrize("K,M", [(7, 1), (7, 2), (8, 3), (9, 4), (10, 5)])
def test_range_start_unranking(K, M):
    # every single-candidate range [i, i+1) must evaluate the i-th candidate of
    # the lexicographic order of itertools.combinations (the index layout)
    spec = synth.random_dag(1800 + K, K, max_cost=300, max_bytes=3000, bw=10**12, lat_max=30, window=4)
    od = O.Dfg.from_spec(spec)
    micro = [1, 3]
    for i, cuts in enumerate(itertools.combinations(range(1, K), M - 1)):
        for j, m in enumerate(micro):
            idx = 2 * i + j
            assert od.pipeline_search(M, micro, idx, idx + 1) == (od.pipeline(M, list(cuts), m), idx)


@pytest.mark.parametrize("M,m,o", [(2, 4, 5), (4, 8, 1), (3, 6, 100)])
def test_bubble_closed_form_with_op_overhead(M, m, o):
    # reading R27: every op pays o per micro-batch; on the uniform chain the
    # stage times grow by q·o and the bubble formula still holds
    q, d = 3, 48
    spec = synth.chain(M * q, d, 2 * d, 0, lat=0)
    od = O.Dfg.from_spec(spec)
    cuts = [q * s for s in range(1, M)]
    tf, tb = q * d // m + q * o, q * 2 * d // m + q * o
    assert od.pipeline(M, cuts, m, overhead=o) == (m + M - 1) * (tf + tb)
    assert od.pipeline(M, cuts, m, overhead=0) == od.pipeline(M, cuts, m)


def test_overhead_makes_many_micro_batches_lose():
    # with a per-op overhead the best micro-batch count is finite
    od = O.Dfg.from_spec(synth.gnmt())
    micro = [1, 2, 4, 8, 16, 32]
    _, idx0 = od.pipeline_search(2, micro)
    _, idx1 = od.pipeline_search(2, micro, overhead=20_000_000)     # 20 µs per op per micro-batch
    assert micro[idx0 % 6] == 32 and micro[idx1 % 6] < 32
