"""B200-native placement evaluation and hybrid-parallelism projection
(the data-parallel hot path of arXiv 1907.13257).  See include/pp.h and
DESIGN.md.  The compute runs in libpp.so (hand-written sm_100a CUDA)."""
from .pp import (Dfg, Comm, plan, PPError, SearchResult, Crossover, project_e2e, crossover, cells_to_numpy,
                 rank_slice, exchange_unique_id, pack_key, key_makespan, key_rank, round_key, round_contrib,
                 round_moves_base, round_exchange_host, kernel_launch_count, lib, u64,
                 set_kernel_timing, get_kernel_timing,
                 GEN_GRAY, GEN_RANDOM, GEN_PERTURB, INFEASIBLE, LIB_PATH, TIER_SHARED, TIER_GLOBAL)

__all__ = ["Dfg", "Comm", "plan", "PPError", "SearchResult", "Crossover", "project_e2e", "crossover",
           "cells_to_numpy", "rank_slice", "exchange_unique_id", "pack_key", "key_makespan", "key_rank",
           "round_key", "round_contrib", "round_moves_base", "round_exchange_host",
           "kernel_launch_count", "set_kernel_timing", "get_kernel_timing", "lib", "u64", "GEN_GRAY", "GEN_RANDOM", "GEN_PERTURB", "INFEASIBLE", "TIER_SHARED", "TIER_GLOBAL",
           "LIB_PATH"]
