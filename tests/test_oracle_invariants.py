"""K15 invariants of the oracle schedule."""
import random

import pytest

import oracle as O
import synth
from tests import brute


def _spec(seed, K):
    return synth.random_dag(seed, K, avg_deg=1.8, max_cost=500, max_bytes=300, lat_max=20)


@pytest.mark.parametrize("seed", range(10))
def test_device_permutation_symmetry(seed):
    rng = random.Random(seed)
    spec = _spec(seed, 40)
    d = O.Dfg.from_spec(spec)
    for M in (2, 3, 5, 8):
        pl = [rng.randrange(M) for _ in range(d.K)]
        perm = list(range(M)); rng.shuffle(perm)
        assert d.makespan(M, pl) == d.makespan(M, [perm[x] for x in pl])


@pytest.mark.parametrize("seed", range(10))
def test_homogeneity(seed):
    # with BW = 1e12 B/s one byte is exactly one ps, so scaling bytes and L by c
    # scales every per-edge ps cost by c
    rng = random.Random(seed)
    spec = _spec(seed, 30)
    c = rng.randint(2, 9)
    s2 = dict(spec, fwd_ps=[c * x for x in spec["fwd_ps"]], bwd_ps=[c * x for x in spec["bwd_ps"]],
              edge_fwd_bytes=[c * x for x in spec["edge_fwd_bytes"]],
              edge_bwd_bytes=[c * x for x in spec["edge_bwd_bytes"]] if spec["edge_bwd_bytes"] else None,
              link_lat_ps=c * spec["link_lat_ps"])
    d1, d2 = O.Dfg.from_spec(spec), O.Dfg.from_spec(s2)
    for M in (2, 4):
        pl = [rng.randrange(M) for _ in range(d1.K)]
        assert d2.makespan(M, pl) == c * d1.makespan(M, pl)


@pytest.mark.parametrize("seed", range(10))
def test_monotone_in_costs(seed):
    rng = random.Random(seed)
    spec = _spec(seed, 30)
    d = O.Dfg.from_spec(spec)
    M = 3
    pl = [rng.randrange(M) for _ in range(d.K)]
    base = d.makespan(M, pl)
    for _ in range(5):
        s2 = dict(spec)
        k = rng.randrange(d.K)
        s2["fwd_ps"] = list(spec["fwd_ps"]); s2["fwd_ps"][k] += rng.randint(1, 100)
        if d.E:
            e = rng.randrange(d.E)
            s2["edge_fwd_bytes"] = list(spec["edge_fwd_bytes"]); s2["edge_fwd_bytes"][e] += rng.randint(1, 100)
        assert O.Dfg.from_spec(s2).makespan(M, pl) >= base


def _critical_path(spec):
    K = len(spec["fwd_ps"])
    order = brute.kahn_by_id(K, spec["op_id"], spec["edge_src"], spec["edge_dst"])
    f = [0] * K
    for k in order:
        f[k] = spec["fwd_ps"][k] + max([f[u] for u, v in zip(spec["edge_src"], spec["edge_dst"]) if v == k], default=0)
    b = [0] * K
    for k in reversed(order):
        b[k] = spec["bwd_ps"][k] + max([b[v] for u, v in zip(spec["edge_src"], spec["edge_dst"]) if u == k] + [f[k]])
    return max(b)


@pytest.mark.parametrize("seed", range(12))
def test_bounds_and_device_monotonicity(seed):
    rng = random.Random(seed)
    K = rng.randint(3, 7)
    spec = _spec(200 + seed, K)
    d = O.Dfg.from_spec(spec)
    t1 = d.t1
    cp = _critical_path(spec)
    prev = None
    for M in (1, 2, 3):
        best = d.search(M, O.GEN_GRAY, 0, M**K).best_makespan_ps
        assert -(-t1 // M) <= best <= t1                   # ⌈T_1/M⌉ ≤ best ≤ T_1, so SU ∈ [1, M]
        assert best >= cp                                  # zero-comm critical path is a lower bound
        if prev is not None:
            assert best <= prev                            # adding a device never hurts (superset)
        prev = best
    for _ in range(20):
        M = rng.randint(2, 4)
        pl = [rng.randrange(M) for _ in range(K)]
        cut = sum(O.edge_cost(spec["edge_fwd_bytes"][e], spec["link_bw_Bps"], spec["link_lat_ps"]) +
                  O.edge_cost((spec["edge_bwd_bytes"] or spec["edge_fwd_bytes"])[e], spec["link_bw_Bps"],
                              spec["link_lat_ps"])
                  for e in range(d.E) if pl[spec["edge_src"][e]] != pl[spec["edge_dst"][e]])
        assert cp <= d.makespan(M, pl) <= t1 + cut
