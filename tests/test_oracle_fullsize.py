"""The full-size golden's driver (tools/oracle_fullsize.py) replays O7 over
sliced oracle rounds; here it must equal the oracle's own or_search (and the
unsliced pipeline search) on counts small enough to run both.  This is what
lets tests/golden/fullsize_r02.json stand for `or_search` at full size."""
import concurrent.futures as cf
import importlib.util
import os

import numpy as np
import pytest

import oracle as O
import synth

_spec = importlib.util.spec_from_file_location(
    "oracle_fullsize", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "oracle_fullsize.py"))
F = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(F)


@pytest.fixture(scope="module")
def pool():
    with cf.ThreadPoolExecutor(max_workers=4) as p:
        yield p


@pytest.mark.parametrize("model,M,gen,count,rounds,tau", [
    ("toy12", 2, O.GEN_GRAY, 4096, 1, 0),
    ("toy12", 3, O.GEN_PERTURB, 700, 6, 64),
    ("gnmt", 2, O.GEN_PERTURB, 3000, 4, 8),
    ("biglstm", 4, O.GEN_PERTURB, 2000, 5, 40),
    ("inception_v3", 8, O.GEN_PERTURB, 1500, 3, 8),
    ("inception_v3", 2, O.GEN_RANDOM, 5000, 1, 0),
])
def test_sliced_search_equals_or_search(pool, model, M, gen, count, rounds, tau):
    od = O.Dfg.from_spec(getattr(synth, model)())
    base = od.eft(M) if gen == O.GEN_PERTURB else None
    want = od.search(M, gen, 99, count, rounds=rounds, tau=tau, base=base)
    for S in (1, 7, 64):
        got = F.sliced_search(pool, od, M, gen, 99, count, rounds, tau, base, S)
        assert (got["T_M"], got["best_index"], got["best_round"]) == \
               (want.best_makespan_ps, want.best_index, want.best_round), S
        assert got["placement"] == "".join(map(str, want.placement))


def test_perturb_base_moves_in_replay(pool):
    # a case where a later round improves (so the base-move rule is exercised)
    od = O.Dfg.from_spec(synth.toy12())
    want = od.search(2, O.GEN_PERTURB, 0, 30, rounds=8, tau=32)
    assert want.best_round > 0
    got = F.sliced_search(pool, od, 2, O.GEN_PERTURB, 0, 30, 8, 32, None, 5)
    assert (got["T_M"], got["best_index"], got["best_round"]) == \
           (want.best_makespan_ps, want.best_index, want.best_round)


def test_sliced_pipeline_equals_full(pool):
    od = O.Dfg.from_spec(synth.random_dag(77, 40, avg_deg=1.6, max_cost=10**6, max_bytes=10**6))
    for M in (2, 3):
        got = F.sliced_pipeline(pool, od, M, [1, 2, 4], 9)
        assert (got["makespan"], got["index"]) == od.pipeline_search(M, [1, 2, 4])
