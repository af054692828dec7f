"""BASELINE.json's configs as search and projection parameters.

Plain data, no arithmetic of the method: which DFG, how many devices M, which
generator, how many candidates and rounds, the flip
threshold τ, the seed, and which projections (M set, N_max, scenario mode)
each config asks for.  `bench.py`, `tools/sweep.py`, `tools/oracle_fullsize.py`
(which writes the full-size golden `tests/golden/fullsize_r02.json` from the
oracle alone) and `tests/test_gpu_fullsize.py` all read it, so the GPU path
and the oracle run the same workloads.

Sizes are the ones BASELINE.json / SURVEY.md §8(d) state:

  1  toy-12, M = 2, GRAY exhaustive 2^12; projection N = 1..64
  2  GNMT-shaped, M = 2 and 4, PERTURB τ = 8, 10 rounds × 10^6 (10^7 sampled)
  3  BigLSTM-shaped, M = 2, PERTURB 10 × 10^6; crossover sweep N = 1..256
  4  Inception-V3-shaped, M = 2 and 4: PERTURB 10 × 10^7 (search) and
     RANDOM 1 × 10^8 (throughput) — 10^8 placements each
  5  the three DFGs × M ∈ {2, 4, 8}, PERTURB 10 × 10^6 each (+ the GPipe
     search for GNMT/BigLSTM at M = 2, 4); projection M ∈ {1,2,4,8} ×
     N = 1..1024 × 16 knots, EQ5 and TIME, crossover per model
  5x config 5 at the bench's size, 10 × 10^7 per search (tools/sweep.py)

Every PERTURB search starts from the EFT-greedy placement.
"""
from __future__ import annotations

SEED = 13257
TAU = 8                          # PERTURB τ = 8 (of 256)
MODELS = ["inception_v3", "gnmt", "biglstm"]
SWEEP_MS = [1, 2, 4, 8]
MICRO = [1, 2, 4, 8, 16, 32]     # GPipe micro-batch counts (§8(f) f3)
PIPELINED = {"gnmt": [2, 4], "biglstm": [2, 4]}   # the paper pipelined these


def search_key(model, M, gen, count, rounds, tau=TAU, seed=SEED, base="eft"):
    if gen != "perturb":
        tau, base = 0, "zero"
    return f"{model}|M{M}|{gen}|{rounds}x{count}|tau{tau}|seed{seed}|{base}"


def _s(model, M, gen, count, rounds):
    tau = TAU if gen == "perturb" else 0
    base = "eft" if gen == "perturb" else "zero"
    return dict(key=search_key(model, M, gen, count, rounds), model=model, M=M, gen=gen, count=count,
                rounds=rounds, tau=tau, seed=SEED, base=base)


def searches():
    """Every distinct search of configs 2–5x (configs 2 and 3 are subsets of 5)."""
    out = {}
    for s in ([_s("toy12", 2, "gray", 4096, 1)]                                               # config 1
              + [_s("gnmt", M, "perturb", 10**6, 10) for M in (2, 4)]                          # config 2
              + [_s("biglstm", 2, "perturb", 10**6, 10)]                                      # config 3
              + [_s("inception_v3", M, g, c, r) for M in (2, 4)                               # config 4
                 for g, c, r in (("perturb", 10**7, 10), ("random", 10**8, 1))]
              + [_s(m, M, "perturb", 10**6, 10) for m in MODELS for M in (2, 4, 8)]           # config 5
              + [_s(m, M, "perturb", 10**7, 10) for m in MODELS for M in (2, 4, 8)]):         # config 5x
        out.setdefault(s["key"], s)
    return list(out.values())


def pipelines():
    return [dict(key=f"{m}|M{M}|pipeline", model=m, M=M, micro=MICRO) for m, Ms in PIPELINED.items() for M in Ms]


def projections():
    """Each projection: the model, the M set, N_max, the scenario mode, and for
    each M ≥ 2 the search keys whose best makespan is T_M (the minimum over
    the listed searches/pipelines)."""
    out = []
    out.append(dict(name="c1_toy12", model="toy12", Ms=[1, 2], nmax=64, mode=0,
                    T={2: [search_key("toy12", 2, "gray", 4096, 1)]}))
    out.append(dict(name="c3_biglstm_M2_N256", model="biglstm", Ms=[1, 2], nmax=256, mode=0,
                    T={2: [search_key("biglstm", 2, "perturb", 10**6, 10)]}))
    out.append(dict(name="c4_bench_inception_M2", model="inception_v3", Ms=[1, 2], nmax=1024, mode=0,
                    T={2: [search_key("inception_v3", 2, "perturb", 10**7, 10)]}))
    for tag, count in (("c5", 10**6), ("c5x", 10**7)):
        for m in MODELS:
            for mode, mname in ((0, "EQ5"), (1, "TIME")):
                T = {}
                for M in SWEEP_MS[1:]:
                    keys = [search_key(m, M, "perturb", count, 10)]
                    if M in PIPELINED.get(m, []):
                        keys.append(f"{m}|M{M}|pipeline")
                    T[M] = keys
                out.append(dict(name=f"{tag}_{m}_{mname}", model=m, Ms=list(SWEEP_MS), nmax=1024, mode=mode, T=T))
    return out
