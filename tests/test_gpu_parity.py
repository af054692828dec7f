"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
bit for bit (integer ps; every compared value is an exact
integer, so the tolerance is zero)."""
import random

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1907_13257_b200 as pp  # noqa: E402

PAPER = ["toy12", "gnmt", "biglstm", "inception_v3"]


def _oracle_candidates(od, M, gen, seed_r, tau, base_pi, idx):
    return np.array([od.makespan_pi(M, O.gen(od.K, M, gen, seed_r, tau, base_pi, int(i))) for i in idx],
                    dtype=np.uint64)


@pytest.fixture(scope="module")
def dfgs():
    out = {}
    for name in PAPER:
        spec = getattr(synth, name)()
        out[name] = (spec, pp.Dfg(spec), O.Dfg.from_spec(spec))
    return out


def test_pi_and_t1_match(dfgs):
    for name, (spec, g, od) in dfgs.items():
        assert list(g.pi) == list(od.pi)
        assert g.t1 == od.t1
        assert g.grad_bytes == od.grad_bytes


def test_toy12_exhaustive_gray(dfgs):
    spec, g, od = dfgs["toy12"]
    r = g.search_best(2, pp.GEN_GRAY, 0, 4096)
    o = od.search(2, O.GEN_GRAY, 0, 4096)
    assert (r.best_makespan_ps, r.best_index, r.best_round, r.evaluated) == \
           (o.best_makespan_ps, o.best_index, o.best_round, o.evaluated)
    assert np.array_equal(r.placement, o.placement)
    assert (r.best_makespan_ps, r.best_index) == (920_000_000, 288)
    # every one of the 4096 makespans
    got = pp.u64(g.eval_generated(2, pp.GEN_GRAY, 0, 0, None, 0, 4096))
    want = _oracle_candidates(od, 2, O.GEN_GRAY, 0, 0, None, range(4096))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 8])
def test_eval_placements_paper_dfgs(dfgs, M):
    rng = np.random.default_rng(M)
    for name, (spec, g, od) in dfgs.items():
        count = 1000 + 37   # several CTAs and a ragged tail
        pl = rng.integers(0, M, size=(count, g.K), dtype=np.uint8)
        pl[0] = 0
        got = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
        want = np.array([od.makespan(M, row) for row in pl], dtype=np.uint64)
        assert np.array_equal(got, want), name
        assert got[0] == od.t1


@pytest.mark.parametrize("M", [2, 3, 4, 8])
def test_eval_placements_out_of_range_rows(dfgs, M):
    """A row holding a value ≥ M is reported infeasible and touches nothing
    else: the valid rows around it (same warps) keep their exact makespans
    (free[] indexed past the lane's M slots)."""
    rng = np.random.default_rng(100 + M)
    spec, g, od = dfgs["inception_v3"]
    count = 515
    pl = rng.integers(0, M, size=(count, g.K), dtype=np.uint8)
    bad = rng.choice(count, 40, replace=False)
    for i in bad:
        pl[i, rng.integers(0, g.K)] = rng.integers(M, 256)
    got = pp.u64(g.eval_placements(M, torch.as_tensor(pl, device="cuda")))
    for i in range(count):
        want = pp.INFEASIBLE if i in set(bad.tolist()) else od.makespan(M, pl[i])
        assert int(got[i]) == want, i
    ex = pp.u64(pp.Dfg(synth.toy12()).eval_exact(M, torch.as_tensor(
        np.array([[0] * 11 + [M], [0] * 12], dtype=np.uint8), device="cuda"))[0])
    assert int(ex[0]) == pp.INFEASIBLE and int(ex[1]) == O.Dfg.from_spec(synth.toy12()).t1


@pytest.mark.parametrize("gen", [O.GEN_RANDOM, O.GEN_PERTURB])
@pytest.mark.parametrize("M", [2, 3, 4, 8])
def test_eval_generated_paper_dfgs(dfgs, gen, M):
    rng = np.random.default_rng(10 * M + gen)
    for name, (spec, g, od) in dfgs.items():
        base = rng.integers(0, M, size=g.K, dtype=np.uint8)
        seed = int(rng.integers(0, 2**63))
        tau = 24
        begin, count = (0, 700) if name != "toy12" else (0, 4096)
        got = pp.u64(g.eval_generated(M, gen, seed, tau, base, begin, count))
        want = _oracle_candidates(od, M, gen, seed, tau, base, range(begin, begin + count))
        assert np.array_equal(got, want), name
        # far into the index space (ragged tail at an odd offset)
        begin = 10**9 + 13
        got = pp.u64(g.eval_generated(M, gen, seed, tau, base, begin, 77))
        want = _oracle_candidates(od, M, gen, seed, tau, base, range(begin, begin + 77))
        assert np.array_equal(got, want), name


@pytest.mark.parametrize("M", [2, 3, 4, 5, 6, 7, 8])
def test_gray_small_exhaustive_all_M(M):
    K = {2: 10, 3: 6, 4: 5, 5: 4, 6: 4, 7: 4, 8: 3}[M]
    spec = synth.random_dag(300 + M, K, avg_deg=1.7, max_cost=100, max_bytes=100)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    n = M**K
    got = pp.u64(g.eval_generated(M, pp.GEN_GRAY, 0, 0, None, 0, n))
    want = _oracle_candidates(od, M, O.GEN_GRAY, 0, 0, None, range(n))
    assert np.array_equal(got, want)
    r = g.search_best(M, pp.GEN_GRAY, 0, n)
    o = od.search(M, O.GEN_GRAY, 0, n)
    assert (r.best_makespan_ps, r.best_index) == (o.best_makespan_ps, o.best_index)
    assert np.array_equal(r.placement, o.placement)


def test_search_random_inception_prefix(dfgs):
    spec, g, od = dfgs["inception_v3"]
    for M in (2, 4):
        r = g.search_best(M, pp.GEN_RANDOM, 13257, 200_003)
        o = od.search(M, O.GEN_RANDOM, 13257, 200_003)
        assert (r.best_makespan_ps, r.best_index, r.best_round) == (o.best_makespan_ps, o.best_index, o.best_round)
        assert np.array_equal(r.placement, o.placement)


@pytest.mark.parametrize("name,M", [("gnmt", 2), ("gnmt", 4), ("biglstm", 2), ("inception_v3", 4), ("toy12", 3)])
def test_search_perturb_rounds(dfgs, name, M):
    spec, g, od = dfgs[name]
    count, rounds = (20_000, 4) if name != "toy12" else (500, 6)
    rng = np.random.default_rng(5)
    base = rng.integers(0, M, size=g.K, dtype=np.uint8)
    r = g.search_best(M, pp.GEN_PERTURB, 99, count, rounds=rounds, tau=8, base=base)
    o = od.search(M, O.GEN_PERTURB, 99, count, rounds=rounds, tau=8, base=base)
    assert (r.best_makespan_ps, r.best_index, r.best_round, r.evaluated) == \
           (o.best_makespan_ps, o.best_index, o.best_round, o.evaluated)
    assert np.array_equal(r.placement, o.placement)
    assert od.makespan(M, r.placement) == r.best_makespan_ps


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_random_dags(seed):
    rng = random.Random(seed)
    K = rng.choice([1, 2, 7, 33, 100, 257, 600, 1024])
    deg = rng.choice([0.5, 1.5, 3.0]) if K < 600 else 1.0
    spec = synth.random_dag(seed, K, avg_deg=deg, max_in=rng.choice([2, 4, 9]), window=None if K < 200 else 48,
                            max_cost=rng.choice([10, 10**6]), max_bytes=rng.choice([0, 100, 10**7]),
                            lat_max=rng.choice([0, 1000]))
    if rng.random() < 0.3:
        spec["mem_bytes"] = [rng.randint(0, 100) for _ in range(K)]
        spec["dev_mem_cap_bytes"] = rng.randint(1, 60 * K)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    M = rng.choice([1, 2, 3, 4, 5, 8])
    for gen in (O.GEN_RANDOM, O.GEN_PERTURB):
        base = np.array([rng.randrange(M) for _ in range(K)], dtype=np.uint8)
        s = rng.getrandbits(64)
        begin = rng.choice([0, 5, 10**12])
        got = pp.u64(g.eval_generated(M, gen, s, 40, base, begin, 333))
        want = _oracle_candidates(od, M, gen, s, 40, base, range(begin, begin + 333))
        assert np.array_equal(got, want)


def test_memory_cap_infeasible():
    spec = synth.random_dag(7, 20)
    spec["mem_bytes"] = [10] * 20
    spec["dev_mem_cap_bytes"] = 150          # needs ≥ 2 devices (200 B total)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    got = pp.u64(g.eval_generated(2, pp.GEN_RANDOM, 1, 0, None, 0, 500))
    want = _oracle_candidates(od, 2, O.GEN_RANDOM, 1, 0, None, range(500))
    assert np.array_equal(got, want)
    assert got[0] == pp.INFEASIBLE            # index 0 = all on device 0
    r = g.search_best(2, pp.GEN_RANDOM, 1, 500)
    assert r.best_makespan_ps == od.search(2, O.GEN_RANDOM, 1, 500).best_makespan_ps
    spec["dev_mem_cap_bytes"] = 5            # nothing fits
    g2 = pp.Dfg(spec)
    with pytest.raises(pp.PPError) as e:
        g2.search_best(2, pp.GEN_RANDOM, 1, 100)
    assert e.value.code == -5


def test_rank_slices_equal_full_search(dfgs):
    """Fake multi-rank on one GPU: slice the candidates exactly as the NCCL
    path does, reduce the packed keys on the host; GPU-count invariance."""
    spec, g, od = dfgs["gnmt"]
    count = 50_001
    full = g.search_best(2, pp.GEN_RANDOM, 3, count)
    for world in (1, 2, 3, 4, 8):
        keys, idx = [], []
        for r in range(world):
            b, e = pp.rank_slice(count, r, world)
            out = pp.u64(g.search_range(2, pp.GEN_RANDOM, 3, 0, None, b, e))
            keys.append(pp.pack_key(int(out[0]), r))
            idx.append(int(out[1]))
        k = min(keys)
        assert pp.key_makespan(k) == full.best_makespan_ps
        assert idx[pp.key_rank(k)] == full.best_index


def test_edge_cases():
    # single op, no edges; M = 1; empty eval
    spec = synth.independent(1, 5, 7)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.search_best(1, pp.GEN_GRAY, 0, 1).best_makespan_ps == 12
    r = g.search_best(4, pp.GEN_GRAY, 0, 4)
    assert r.best_makespan_ps == 12 and r.best_index == 0
    out = g.eval_placements(2, torch.zeros((0, 1), dtype=torch.uint8, device="cuda"))
    assert out.numel() == 0
    # independent ops: SU = M exactly (closed form, K7)
    spec = synth.independent(8, 4, 5)
    g = pp.Dfg(spec)
    assert g.search_best(4, pp.GEN_GRAY, 0, 4**8).best_makespan_ps == 2 * 9
    # chain: SU = 1 (K6)
    spec = synth.chain(9, 3, 6, 50)
    g = pp.Dfg(spec)
    assert g.search_best(3, pp.GEN_GRAY, 0, 3**9).best_makespan_ps == g.t1


def test_large_image_reduces_cta():
    # K + E near the 96 KB image cap, large W
    spec = synth.random_dag(77, 1050, avg_deg=0.9, max_in=3, window=40)
    g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
    assert g.image_bytes > 60_000
    for M in (2, 8):
        got = pp.u64(g.eval_generated(M, pp.GEN_RANDOM, 4, 0, None, 0, 100))
        want = _oracle_candidates(od, M, O.GEN_RANDOM, 4, 0, None, range(100))
        assert np.array_equal(got, want)


def test_error_codes_match_oracle():
    base = synth.diamond()
    for bad, code in [(dict(base, edge_src=[0, 0, 1, 3], edge_dst=[1, 2, 3, 1]), -2),
                      (dict(base, edge_dst=[1, 2, 3, 9]), -1),
                      (dict(base, op_id=[1, 2, 2, 3]), -1),
                      (dict(base, fwd_ps=[2**60, 2**60, 8, 2]), -3)]:
        with pytest.raises(pp.PPError) as e:
            pp.Dfg(bad)
        assert e.value.code == code
        with pytest.raises(O.OracleError) as e2:
            O.Dfg.from_spec(bad)
        assert e2.value.code == code
    g = pp.Dfg(synth.toy12())
    with pytest.raises(pp.PPError) as e:
        g.search_best(2, pp.GEN_GRAY, 0, 4097)
    assert e.value.code == -1
    g = pp.Dfg(synth.inception_v3())
    with pytest.raises(pp.PPError) as e:
        g.search_best(2, pp.GEN_GRAY, 0, 10)
    assert e.value.code == -4


def test_nccl_communicator_single_rank(dfgs):
    """The NCCL path of pp_search_best (key and index min all-reduces every
    round, winner decoded from the reduced key) at world size 1 equals the
    communicator-free path."""
    import os
    import socket
    import torch.distributed as dist
    spec, g, od = dfgs["gnmt"]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = pp.Comm(0, 1, 0)
        a = g.search_best(2, pp.GEN_PERTURB, 7, 30_001, rounds=3, tau=8, comm=comm)
        b = g.search_best(2, pp.GEN_PERTURB, 7, 30_001, rounds=3, tau=8)
        comm.close()
    finally:
        dist.destroy_process_group()
    assert (a.best_makespan_ps, a.best_index, a.best_round) == (b.best_makespan_ps, b.best_index, b.best_round)
    assert np.array_equal(a.placement, b.placement)
    o = od.search(2, O.GEN_PERTURB, 7, 30_001, rounds=3, tau=8)
    assert a.best_makespan_ps == o.best_makespan_ps and a.best_index == o.best_index


@pytest.mark.parametrize("np_", ["1", "2", "4"])
def test_every_placements_per_lane_variant(dfgs, np_, monkeypatch):
    """The search kernel is instantiated for NP = 1, 2, 4 placements per lane
    (chosen per launch); pin each and compare the argmin with the oracle."""
    monkeypatch.setenv("PP_NP", np_)
    for name, M, gen in [("gnmt", 2, O.GEN_PERTURB), ("inception_v3", 4, O.GEN_RANDOM), ("toy12", 3, O.GEN_GRAY),
                         ("biglstm", 8, O.GEN_PERTURB)]:
        spec, g, od = dfgs[name]
        count = 729 if name == "toy12" else 9_001
        base = np.zeros(g.K, dtype=np.uint8)
        got = pp.u64(g.search_range(M, gen, 77, 24, base, 3, 3 + count))
        want = od.round(M, gen, 77, 24, base, 3, 3 + count)
        assert (int(got[0]), int(got[1])) == want, (name, np_)


def test_sharded_exact_and_pipeline_searches():
    """The exact-schedule (§8(f) f1) and pipeline (f3) searches shard like the
    main search: per-rank slices + the packed-key argmin equal the full range
    (3 emulated ranks on one GPU), and pp_argmin_allreduce at world size 1
    leaves a rank's argmin unchanged."""
    import os
    import socket
    import torch.distributed as dist
    spec = synth.toy12()
    g = pp.Dfg(spec)
    full_x = g.search_exact(2, pp.GEN_GRAY, 0, 0, None, 0, 4096)
    micro = [1, 2, 4, 8]
    n_pipe = g.pipeline_space(3, len(micro))
    (full_p, full_pi), _ = g.pipeline_range(3, micro, 0, n_pipe)
    for world in (2, 3):
        keys_x, idx_x, keys_p, idx_p = [], {}, [], {}
        for r in range(world):
            b, e = pp.rank_slice(4096, r, world)
            mk, ix, _ = g.search_exact(2, pp.GEN_GRAY, 0, 0, None, b, e)
            keys_x.append(pp.pack_key(mk, r))
            idx_x[r] = ix
            b, e = pp.rank_slice(n_pipe, r, world)
            (mk, ix), _ = g.pipeline_range(3, micro, b, e)
            keys_p.append(pp.pack_key(mk, r))
            idx_p[r] = ix
        kx, kp = min(keys_x), min(keys_p)
        assert (pp.key_makespan(kx), idx_x[pp.key_rank(kx)]) == full_x[:2]
        assert (pp.key_makespan(kp), idx_p[pp.key_rank(kp)]) == (full_p, full_pi)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = pp.Comm(0, 1, 0)
        best = torch.tensor([full_x[0], full_x[1]], dtype=torch.int64, device="cuda")
        comm.argmin_allreduce(g, best)
        assert tuple(int(x) for x in pp.u64(best)) == full_x[:2]
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [2, 4, 8])
@pytest.mark.parametrize("np_", ["1", "2", "4"])
def test_perturb_m2_cut_words(dfgs, np_, M, monkeypatch):
    """M = 2 PERTURB runs the cut-word schedule (search_kernel.cuh
    schedule_m2p): 4 byte compares u < τ per SIMD word, whose two formulas
    meet at τ = 128, a packed base word per half-group, and pads in the last
    half-groups when K mod 8 ≠ 0.  Every τ boundary, a random base, begin = 0
    (candidate 0 = the base itself) and both the per-candidate (write-all,
    NP = 2 only) and the argmin kernels (NP pinned), against the oracle.
    M = 4 and 8 run the device-word schedule (schedule_mpw: revision-3
    re-draws base ⊕ (y mod M) as SIMD words) through the same cases."""
    rng = np.random.default_rng(128 + M)
    cases = [dfgs["toy12"][1:], dfgs["inception_v3"][1:]]
    for K in (13, 30):   # K mod 8 = 5 and 6: pad positions in the last half-groups
        spec = synth.random_dag(4000 + K, K, avg_deg=1.6, max_cost=10**6, max_bytes=10**6)
        cases.append((pp.Dfg(spec), O.Dfg.from_spec(spec)))
    for g, od in cases:
        base = rng.integers(0, M, size=g.K, dtype=np.uint8)
        for tau in (0, 1, 7, 8, 127, 128, 129, 200, 255, 256):
            seed = int(rng.integers(0, 2**63))
            monkeypatch.delenv("PP_NP", raising=False)
            got = pp.u64(g.eval_generated(M, pp.GEN_PERTURB, seed, tau, base, 0, 300))
            want = _oracle_candidates(od, M, O.GEN_PERTURB, seed, tau, base, range(300))
            assert np.array_equal(got, want), (g.K, tau)
            assert got[0] == od.makespan_pi(M, base)   # candidate 0 is the base
            monkeypatch.setenv("PP_NP", np_)
            r = pp.u64(g.search_range(M, pp.GEN_PERTURB, seed, tau, base, 0, 1_000))
            assert (int(r[0]), int(r[1])) == od.round(M, O.GEN_PERTURB, seed, tau, base, 0, 1_000), (g.K, tau)


@pytest.mark.parametrize("M", [2, 4, 8])
@pytest.mark.parametrize("np_", ["1", "2", "4"])
def test_perturb_m2_cut_words_memory_cap(np_, M, monkeypatch):
    """The cut-word schedule with a per-device memory cap:
    the memory use per device is summed from the same device words, and an
    over-cap candidate is infeasible.  Caps chosen so that some candidates
    fit and some do not."""
    rng = np.random.default_rng(487)
    for K in (29, 64, 131):
        spec = synth.random_dag(9000 + K, K, avg_deg=1.5, max_cost=10**6, max_bytes=10**6)
        spec["mem_bytes"] = [int(x) for x in rng.integers(0, 100, size=K)]
        spec["dev_mem_cap_bytes"] = int(sum(spec["mem_bytes"]) * {2: 0.55, 4: 0.3, 8: 0.16}[M])
        g, od = pp.Dfg(spec), O.Dfg.from_spec(spec)
        base = (np.arange(K) % M).astype(np.uint8)
        seed = int(rng.integers(0, 2**63))
        monkeypatch.delenv("PP_NP", raising=False)
        got = pp.u64(g.eval_generated(M, pp.GEN_PERTURB, seed, 64, base, 0, 500))
        want = _oracle_candidates(od, M, O.GEN_PERTURB, seed, 64, base, range(500))
        assert np.array_equal(got, want), K
        inf = int(np.sum(got == np.uint64(2**64 - 1)))
        assert 0 < inf < 500, (K, inf)   # both feasible and infeasible candidates occur
        monkeypatch.setenv("PP_NP", np_)
        r = pp.u64(g.search_range(M, pp.GEN_PERTURB, seed, 64, base, 0, 2_000))
        assert (int(r[0]), int(r[1])) == od.round(M, O.GEN_PERTURB, seed, 64, base, 0, 2_000), K
