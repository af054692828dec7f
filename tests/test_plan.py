"""Host logic of pp_load_dfg without a device (pp_plan_dfg, pp.plan): the
validation errors equal the oracle's, T_1 and Σ param_bytes equal the
oracle's, the live-slot count W equals the peak number of simultaneously live
values computed independently (interval overlap over the forward+backward
step order built from the oracle's π), and the tier rule of DESIGN.md §6b."""
import numpy as np
import pytest

import oracle as O
import synth

pp = pytest.importorskip("paper_1907_13257_b200")


def _peak_live(spec):
    """max over steps s of |{v ≤ s : v read from a slot at a step > s}| for the
    loader's step order (forward in π, backward in reverse π, K padded to 8),
    an input produced by the previous step being forwarded in a register."""
    od = O.Dfg.from_spec(spec)
    pi = list(od.pi)
    K = len(pi)
    K8 = (K + 7) // 8 * 8
    S = 2 * K8
    pos = {d: i for i, d in enumerate(pi)}     # descriptor index → π position
    ins = [[] for _ in range(K)]
    outs = [[] for _ in range(K)]
    for a, b in zip(spec["edge_src"], spec["edge_dst"]):   # descriptor indices
        ins[pos[b]].append(pos[a])
        outs[pos[a]].append(pos[b])
    last = [-1] * S
    for s in range(S):
        fwd = s < K8
        p = s if fwd else S - 1 - s
        if p >= K:
            continue
        vals = list(ins[p]) if fwd else ([S - 1 - w for w in outs[p]] or [p])
        forwarded = False
        for v in vals:
            if v == s - 1 and not forwarded:
                forwarded = True
                continue
            last[v] = max(last[v], s)
    return max(sum(1 for v in range(s + 1) if last[v] > s) for s in range(S))


PAPER = ["toy12", "inception_v3", "gnmt", "biglstm"]


@pytest.mark.parametrize("name", PAPER)
def test_plan_of_paper_dfgs(name):
    spec = getattr(synth, name)()
    p, od = pp.plan(spec), O.Dfg.from_spec(spec)
    assert (p["K"], p["E"]) == (len(spec["fwd_ps"]), len(spec["edge_src"]))
    assert p["t1"] == od.t1 and p["grad_bytes"] == od.grad_bytes
    assert p["W"] == _peak_live(spec)
    assert p["tier"] == pp.TIER_SHARED
    # the shapes DESIGN.md §4 / §5 state
    assert {"toy12": 3, "inception_v3": 6, "gnmt": 22, "biglstm": 3}[name] == p["W"]


@pytest.mark.parametrize("seed", range(8))
def test_slot_count_is_the_peak_live_set(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.choice([5, 17, 64, 200]))
    spec = synth.random_dag(300 + seed, K, avg_deg=float(rng.choice([0.7, 1.5, 2.5])),
                            window=None if seed % 2 else 20)
    assert pp.plan(spec)["W"] == _peak_live(spec)


def test_tier_rule():
    assert pp.plan(synth.random_dag(5, 900, avg_deg=1.5))["tier"] == pp.TIER_GLOBAL          # W = 394
    long_ = pp.plan(synth.random_dag(11, 3200, avg_deg=1.2, max_in=3, window=40))
    assert long_["image_bytes"] > 96 * 1024 and long_["tier"] == pp.TIER_GLOBAL
    big_t = synth.random_dag(4901, 120, avg_deg=1.5, max_cost=10**15, max_bytes=10**9, bw=10**9)
    assert pp.plan(big_t)["tier"] == pp.TIER_GLOBAL                                            # T_1 ≥ 2^49 ps


def test_plan_errors_equal_the_oracle():
    base = synth.diamond()
    for bad, code in [(dict(base, edge_src=[0, 0, 1, 3], edge_dst=[1, 2, 3, 1]), -2),
                      (dict(base, edge_dst=[1, 2, 3, 9]), -1),
                      (dict(base, op_id=[1, 2, 2, 3]), -1),
                      (dict(base, fwd_ps=[2**60, 2**60, 8, 2]), -3)]:
        with pytest.raises(pp.PPError) as e:
            pp.plan(bad)
        assert e.value.code == code
        with pytest.raises(O.OracleError) as e2:
            O.Dfg.from_spec(bad)
        assert e2.value.code == code
