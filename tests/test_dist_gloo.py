"""Multi-process (gloo, CPU) tests of the N > 1 protocol of pp_search_best
(SURVEY.md §8(e)): contiguous rank slices, the packed (makespan << 3 | rank)
min key, the winner-index exchange, and the NCCL unique-id hand-off.

The per-slice argmin here is the oracle's (no GPU on this box); slicing, the
exchange (key packing, both min all-reduces, decoding) and the base-move rule
are the product's own code: pp_round_exchange_host runs the protocol.h
template that pp_search_best instantiates with NCCL, here with a gloo
collective.  The result must not depend on the number
of ranks (GPU-count invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
I64_MAX = (1 << 63) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _u64_min_gloo(x):
    """min over ranks of a u64 through a signed int64 gloo all-reduce
    (x ^ 2^63 preserves the order)."""
    v = x ^ (1 << 63)
    t = torch.tensor([v - (1 << 64) if v >= 1 << 63 else v], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return (int(t.item()) % (1 << 64)) ^ (1 << 63)


def _sharded_search(rank, world, spec_name, M, gen, seed, count, rounds, tau):
    """pp_search_best's round loop with the oracle's per-slice argmin (no GPU
    here): the slice, the exchange and the base-move rule are the library's
    own code (pp_rank_slice, pp_round_exchange_host → csrc/protocol.h, the
    same template the NCCL path instantiates; pp_round_moves_base)."""
    import oracle as O
    import synth
    import paper_1907_13257_b200 as pp
    spec = getattr(synth, spec_name)() if spec_name != "random" else synth.random_dag(3, 40, window=8)
    od = O.Dfg.from_spec(spec)
    base = np.zeros(od.K, dtype=np.uint8)
    best = None
    for r in range(rounds):
        b, e = pp.rank_slice(count, rank, world)
        if e > b:
            mk, idx = od.round(M, gen, seed + r, tau, base, b, e)
        else:
            mk, idx = pp.INFEASIBLE, pp.INFEASIBLE          # empty slice
        wmk, widx = pp.round_exchange_host(mk, idx, rank, _u64_min_gloo)
        if best is None or wmk < best[0]:
            best = (wmk, widx, r)
        if gen == O.GEN_PERTURB and pp.round_moves_base(widx):
            base = O.gen(od.K, M, gen, seed + r, tau, base, widx)   # every rank moves to the winner
    return best


def _worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1907_13257_b200 as pp
        uid = pp.exchange_unique_id(rank)
        res = {"uid": uid.hex(), "best": [_sharded_search(rank, world, *c) for c in cases]}
        out[rank] = res
    finally:
        dist.destroy_process_group()


CASES = [("toy12", 2, 0, 0, 4096, 1, 0),          # GRAY exhaustive
         ("toy12", 3, 2, 17, 301, 4, 40),         # PERTURB rounds, ragged slices
         ("random", 4, 1, 99, 1001, 1, 0),        # RANDOM
         ("biglstm", 2, 2, 5, 203, 3, 16),
         ("toy12", 4, 2, 3, 2, 3, 128)]            # count < world at 3 ranks: rank 0's slice is empty


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_is_rank_count_invariant(world):
    import oracle as O
    import synth
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    results = [out[r] for r in range(world)]
    assert len({r["uid"] for r in results}) == 1 and len(results[0]["uid"]) == 256
    for ci, (name, M, gen, seed, count, rounds, tau) in enumerate(CASES):
        spec = getattr(synth, name)() if name != "random" else synth.random_dag(3, 40, window=8)
        ref = O.Dfg.from_spec(spec).search(M, gen, seed, count, rounds=rounds, tau=tau)
        for r in range(world):
            assert tuple(results[r]["best"][ci]) == (ref.best_makespan_ps, ref.best_index, ref.best_round)
