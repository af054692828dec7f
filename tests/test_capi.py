"""The C-ABI library loads and exports every symbol include/pp.h declares;
host-only protocol helpers; loader validation runs on the host before any CUDA
call, so its error codes are checked here against the oracle (no GPU)."""
import os
import re

import pytest

import oracle as O
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pp():
    from paper_1907_13257_b200 import _build
    _build.build()
    import paper_1907_13257_b200 as pp
    pp.lib()
    return pp


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "pp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(pp_[a-z0-9_]+)\s*\(", src))


def test_every_declared_symbol_is_exported(pp):
    declared = _declared_functions()
    assert len(declared) >= 19
    L = pp.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(pp.pp.SIGNATURES), declared ^ set(pp.pp.SIGNATURES)


def test_struct_sizes(pp):
    import ctypes as C
    assert C.sizeof(pp.pp.Cell) == 48
    assert C.sizeof(pp.pp.SearchDesc) == 40
    assert C.sizeof(pp.pp.CrossoverC) == 76


# every C-ABI struct the binding mirrors: (C typedef, ctypes class name)
STRUCTS = [("pp_dfg_desc", "DfgDesc"), ("pp_link_desc", "LinkDesc"), ("pp_hw_desc", "HwDesc"),
           ("pp_dfg_info", "DfgInfo"), ("pp_search_desc", "SearchDesc"), ("pp_search_result", "SearchResultC"),
           ("pp_pipeline_result", "PipelineResultC"), ("pp_scenario", "Scenario"), ("pp_cell", "Cell"),
           ("pp_crossover_result", "CrossoverC")]


def test_struct_layout_matches_header(pp, tmp_path):
    """gcc compiles include/pp.h and prints sizeof / offsetof of every field of
    every struct; the ctypes mirrors in pp.py must agree byte for byte."""
    import ctypes as C
    import subprocess
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "pp.h"', "int main(void) {"]
    for cname, pyname in STRUCTS:
        cls = getattr(pp.pp, pyname)
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'  printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {}
    for line in out:
        if line:
            a, b, v = line.split()
            got[(a, b)] = int(v)
    for cname, pyname in STRUCTS:
        cls = getattr(pp.pp, pyname)
        assert got[(cname, "size")] == C.sizeof(cls), cname
        for f in cls._fields_:
            assert got[(cname, f[0])] == getattr(cls, f[0]).offset, (cname, f[0])


def test_rank_slices_partition(pp):
    for count in (1, 7, 8, 1000, 10**8, 2**63 + 5):
        for world in range(1, 9):
            prev = 0
            for r in range(world):
                b, e = pp.rank_slice(count, r, world)
                assert b == prev and e >= b
                prev = e
            assert prev == count


def test_key_order_is_lexicographic(pp):
    # min key picks the smaller makespan, ties to the lower rank (lower global index)
    assert pp.pack_key(5, 7) < pp.pack_key(6, 0)
    assert pp.pack_key(5, 1) < pp.pack_key(5, 2)
    assert pp.key_makespan(pp.pack_key(123456789, 3)) == 123456789
    assert pp.key_rank(pp.pack_key(123456789, 3)) == 3
    assert pp.key_makespan(pp.pack_key(pp.INFEASIBLE, 4)) == pp.INFEASIBLE
    assert pp.pack_key(2**61 - 2, 0) < pp.pack_key(pp.INFEASIBLE, 0)


@pytest.mark.parametrize("bad,code", [
    (dict(edge_src=[0, 0, 1, 3], edge_dst=[1, 2, 3, 1]), -2),
    (dict(edge_dst=[1, 2, 3, 9]), -1),
    (dict(edge_src=[0, 0, 1, 2], edge_dst=[1, 2, 3, 2]), -1),
    (dict(op_id=[1, 2, 2, 3]), -1),
    (dict(op_id=[1, -2, 4, 3]), -1),
    (dict(fwd_ps=[2**60, 2**60, 8, 2]), -3),
    (dict(link_bw_Bps=0), -1),
])
def test_loader_validation_matches_oracle(pp, bad, code):
    spec = dict(synth.diamond(), **bad)
    with pytest.raises(pp.PPError) as e:
        pp.Dfg(spec)
    assert e.value.code == code
    with pytest.raises(O.OracleError) as e2:
        O.Dfg.from_spec(spec)
    assert e2.value.code == code
    if code == -2:
        # both name the same cycle's ids
        ids = lambda s: sorted(int(x) for x in s.split("cycle:")[1].split())
        assert ids(str(e.value)) == ids(str(e2.value)) == [1, 3]


def test_no_cpu_fallback(pp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pp.PPError) as e:
        pp.Dfg(synth.toy12())
    assert e.value.code == -6


def _threaded_exchange(pp, locals_):
    """Every rank's pp_round_exchange_host at once (one thread per rank), with
    an in-process min all-reduce built on a barrier."""
    import threading
    world = len(locals_)
    bar = threading.Barrier(world)
    vals = [None] * world
    out = [None] * world

    def worker(r):
        def allreduce_min(x):
            vals[r] = x
            bar.wait()
            m = min(vals)
            bar.wait()
            return m
        out[r] = pp.round_exchange_host(locals_[r][0], locals_[r][1], r, allreduce_min)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def test_round_exchange_protocol(pp):
    INF = pp.INFEASIBLE
    # the lexicographic (makespan, global index) winner, for any rank layout
    assert _threaded_exchange(pp, [(7, 3), (5, 40), (5, 90)]) == [(5, 40)] * 3
    assert _threaded_exchange(pp, [(9, 0), (9, 50)]) == [(9, 0)] * 2
    # empty slice on rank 0 and every real candidate infeasible: the empty
    # slice must not win (index 2^64-1 would move the base)
    assert _threaded_exchange(pp, [(INF, INF), (INF, 0), (INF, 1)]) == [(INF, 0)] * 3
    assert _threaded_exchange(pp, [(INF, INF), (12, 1)]) == [(12, 1)] * 2
    assert pp.round_key(5, INF, 3) == INF and pp.round_key(5, 0, 3) == pp.pack_key(5, 3)
    kg = pp.round_key(5, 9, 2)
    assert pp.round_contrib(kg, kg, 9) == 9                               # the winning rank
    assert pp.round_contrib(kg, pp.round_key(5, 4, 3), 4) == 4            # a tie on the makespan contributes too
    assert pp.round_contrib(kg, pp.round_key(6, 4, 1), 4) == INF          # a worse rank does not
    assert pp.round_contrib(INF, INF, 4) == INF and pp.round_contrib(kg, INF, 4) == INF
    # ties are resolved by the index, not the rank order (Gray indices of the
    # symmetry-reduced search are not ordered by rank)
    assert _threaded_exchange(pp, [(5, 70), (5, 30), (8, 1)]) == [(5, 30)] * 3
    # the base moves iff the winner is not candidate 0 (= the base)
    assert not pp.round_moves_base(0) and not pp.round_moves_base(INF) and pp.round_moves_base(17)


def test_round_exchange_callback_failure(pp):
    def bad(_x):
        raise RuntimeError("peer died")
    with pytest.raises(pp.PPError) as e:
        pp.round_exchange_host(5, 1, 0, bad)
    assert e.value.code == -7
