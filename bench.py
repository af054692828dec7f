"""Benchmark of the hot path (BASELINE.json metric: placements evaluated/sec).

One step = one pass of the whole path over one batch: a
placement search of the Inception-V3-shaped DFG on M devices (BASELINE
config 4: PERTURB, `--rounds` × `--count` candidates; on-device generation +
forward/backward list schedule + argmin, sharded over the ranks with an NCCL
min all-reduce of the packed key per round, the round/base update), then the
end-to-end projection over N = 1..N_max and the crossover.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pp|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL).  Rank 0 prints one JSON
line.  `--impl reference` times the CPU oracle (the reference arm of this
tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "placements evaluated/sec at 1/2/4/8 B200; crossover N bit-exact vs CPU oracle"
UNIT = "placements/s"
SEED = 13257


WORKLOADS = {"inception_v3": "Inception-V3-shaped (synth.inception_v3, batch 64)",
             "gnmt": "GNMT-shaped (synth.gnmt, 4+4 LSTM x 1024, 18 chunks)",
             "biglstm": "BigLSTM-shaped (synth.biglstm, 2 x LSTM 8192, 30 chunks)",
             "toy12": "toy-12 (SURVEY 8(d) config 1)"}


HW_GRAPHS = {"cube_mesh": "8 devices, DGX-1-style hybrid cube-mesh (synth.hw.hybrid_cube_mesh)",
             "switch": "8 devices on one switch (synth.hw.switch)",
             "ring": "8-device ring (synth.hw.ring)",
             "two_nodes": "2 nodes x 4 devices, switch per node, one network link (synth.hw.two_nodes)"}


def workload(args):
    spec = getattr(synth, args.workload)()
    if args.hw != "none":   # general hardware graph
        from synth import hw as H
        spec["hw"] = {"cube_mesh": H.hybrid_cube_mesh, "switch": lambda: H.switch(8), "ring": lambda: H.ring(8),
                      "two_nodes": lambda: H.two_nodes(4)}[args.hw]()
    return spec


def scenario(args, t1, grad):
    if args.workload == "toy12":
        return synth.toy12_scenario(t1)
    return synth.sweep_scenario(args.workload, t1, grad)


def alg_counts(spec):
    """Algorithmic work per placement:
    6 int32 ops per scheduled op (64-bit max with free + 64-bit add), 7 per
    edge visit (device compare, conditional 64-bit add, 64-bit max); shared
    memory: 8 B read per edge visit + 8 B written per scheduled op."""
    K, E = len(spec["fwd_ps"]), len(spec["edge_src"])
    ops = 6 * (2 * K) + 7 * (2 * E)
    smem = 8 * (2 * E) + 8 * (2 * K)
    return ops, smem


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index):
        self.idx = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks(sm_count, clock_mhz):
    """Roofline denominators for this ALU/shared-memory-bound path (DESIGN.md
    §Roofline): INT32 issue = 4 SMSPs × 32 lanes = 128 thread-ops/clk/SM;
    shared memory = 128 B/clk/SM; at the max SM clock from MEASURED_PEAKS.json."""
    return {"int32_ops_per_s": sm_count * 128 * clock_mhz * 1e6,
            "smem_bytes_per_s": sm_count * 128 * clock_mhz * 1e6}


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the search
    kernel from the committed ncu --set full capture (profiles/r*_traffic.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None
    d = json.load(open(files[-1]))
    return d["dram_bytes_read_per_launch"] + d["dram_bytes_write_per_launch"]


def measured_clock():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"]), "measured"
    except Exception:
        return 1965.0, "fallback (B200_PROFILING.md clocks.max.sm)"


# ------------------------------------------------------------ oracle arm
def cpu_oracle_sample(spec, M, gen_name, tau, base_kind, n_target_s=12.0):
    """The CPU oracle (oracle/) as it stands, single thread, on a bounded
    prefix of round 0 of the same candidate stream (placements/s, n, s)."""
    import oracle as O
    gen = O.GEN_PERTURB if gen_name == "perturb" else O.GEN_RANDOM
    od = O.Dfg.from_spec(spec)
    base_pi = od.eft(M)[od.pi] if (gen == O.GEN_PERTURB and base_kind == "eft") else None
    t = time.perf_counter()
    od.round(M, gen, SEED, tau, base_pi, 0, 20_000)
    rate = 20_000 / (time.perf_counter() - t)
    count = max(20_000, int(rate * n_target_s))
    t = time.perf_counter()
    od.round(M, gen, SEED, tau, base_pi, 0, count)
    dt = time.perf_counter() - t
    return count / dt, count, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    spec = workload(args)
    ops, _ = alg_counts(spec)
    gen = O.GEN_PERTURB if args.gen == "perturb" else O.GEN_RANDOM
    rounds = args.rounds if args.gen == "perturb" else 1
    per_round = max(1, args.ref_sample // rounds)
    n_step = per_round * rounds
    times = []
    for s in range(args.warmup + args.steps):
        t = time.perf_counter()
        od = O.Dfg.from_spec(spec)
        base = od.eft(args.M) if (gen == O.GEN_PERTURB and args.base == "eft") else None
        r = od.search(args.M, gen, SEED, per_round, rounds=rounds, tau=args.tau, base=base)
        sc = scenario(args, od.t1, od.grad_bytes)
        cells = O.Scenario.from_spec(sc).project([1, args.M], [od.t1, r.best_makespan_ps], args.nmax)
        x = O.crossover(cells, [1, args.M], args.nmax)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = n_step * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "gpu_launches": 0,
            "config": config_dict(args, spec, per_step=n_step),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{rounds} rounds x {per_round} {args.gen.upper()} candidates of the "
                                       f"{args.workload}-shaped DFG per step (the GPU step runs {rounds} x {args.count}) "
                                       f"+ projection N=1..{args.nmax} + crossover"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sample_result": {"T_M_ps": r.best_makespan_ps, "crossover_n_star": x.n_star,
                              "note": f"from the {n_step}-candidate sample above, not the full "
                                      f"{rounds} x {args.count} search: it differs from the GPU arm's full-size "
                                      f"result, which the GPU line's 'parity' key checks against the oracle"}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, spec, per_step=None):
    gen = (f"PERTURB tau={args.tau}/256, {args.rounds} rounds x {args.count:.0e}" if args.gen == "perturb"
           else f"RANDOM {args.count:.0e}").replace("+0", "")
    hw = f"_hw-{args.hw}" if args.hw != "none" else ""
    return {"workload": f"{args.workload}_shaped_M{args.M}_{args.gen}_{args.count * args.rounds:.0e}{hw}".replace("+0", ""),
            "dfg": WORKLOADS[args.workload], "K": len(spec["fwd_ps"]),
            "E": len(spec["edge_src"]), "M": args.M, "generator": gen + " (SplitMix64)", "seed": SEED,
            "candidates_per_step": per_step or args.count * args.rounds,
            "base": ("EFT greedy placement (pp_eft_place, SURVEY 8(f) f4)" if args.base == "eft" and args.gen == "perturb"
                     else "all ops on device 0"),
            "projection": f"M in {{1,{args.M}}}, N=1..{args.nmax}, EQ5, ring AR on",
            "l2": "flushed between timed steps (256 MiB write); inputs live on-chip",
            **({"hardware_graph": HW_GRAPHS[args.hw]} if args.hw != "none" else {})}


# ------------------------------------------------------------ parity leg
def parity_check(args, spec, r, x, cells_np, mode):
    """The GPU step's result against the CPU oracle (oracle/), outside the
    timed region: T_M, the winning index, round and placement, every
    projection cell, N* and N* vs the best DP.  mode "live" re-runs the full
    search with the oracle, its rounds sliced over the host's threads
    (tools/oracle_fullsize.py, the same driver that wrote the golden file);
    mode "golden" compares with tests/golden/fullsize_r02.json (written by
    that driver from oracle/ alone) when it holds this exact search."""
    import importlib.util
    import oracle as O
    from synth import configs
    out = {"mode": mode}
    t = time.perf_counter()
    od = O.Dfg.from_spec(spec)
    gen_name = args.gen
    if mode == "live":
        import concurrent.futures as cf
        sp = importlib.util.spec_from_file_location("oracle_fullsize", os.path.join(ROOT, "tools", "oracle_fullsize.py"))
        F = importlib.util.module_from_spec(sp)
        sp.loader.exec_module(F)
        threads = os.cpu_count() or 1
        base = od.eft(args.M) if (gen_name == "perturb" and args.base == "eft") else None
        gens = {"perturb": O.GEN_PERTURB, "random": O.GEN_RANDOM}
        with cf.ThreadPoolExecutor(max_workers=threads) as pool:
            want = F.sliced_search(pool, od, args.M, gens[gen_name], SEED, args.count, args.rounds,
                                   args.tau if gen_name == "perturb" else 0, base, 4 * threads)
        out["reference"] = f"oracle/ live, rounds sliced over {threads} host threads"
    else:
        key = configs.search_key(args.workload, args.M, gen_name, args.count, args.rounds, tau=args.tau, seed=SEED,
                                 base=args.base)
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_r02.json")))["searches"]
        if key not in gold:
            return {"mode": mode, "reference": f"no golden entry for {key}"}
        want = gold[key]
        out["reference"] = f"tests/golden/fullsize_r02.json[{key}] (written from oracle/ by tools/oracle_fullsize.py)"
    out["T_M"] = r.best_makespan_ps == want["T_M"]
    out["best_index"] = r.best_index == want["best_index"]
    out["best_round"] = r.best_round == want["best_round"]
    out["placement"] = "".join(map(str, r.placement)) == want["placement"]
    sc = scenario(args, od.t1, od.grad_bytes)
    oc = O.Scenario.from_spec(sc).project([1, args.M], [od.t1, want["T_M"]], args.nmax)
    ox = O.crossover(oc, [1, args.M], args.nmax)
    got = cells_np.reshape(-1)
    out["cells"] = all(((int(c["C_hi"]) << 64 | int(c["C_lo"])), int(c["feasible"])) == (o.C, o.feasible)
                       if o.feasible else int(c["feasible"]) == 0 for c, o in zip(got, oc))
    out["n_star"] = x.n_star == ox.n_star
    out["n_star_vs_best_dp"] = x.n_star_vs_best_dp == ox.n_star_vs_best_dp
    out["all"] = all(v for k, v in out.items() if isinstance(v, bool))
    out["oracle_s"] = round(time.perf_counter() - t, 1)
    return out


# ---------------------------------------------------------------- GPU arm
def run_pp(args):
    import torch
    import torch.distributed as dist
    import paper_1907_13257_b200 as pp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = pp.Comm(rank, world, local)
    stream = torch.cuda.current_stream()
    GEN = pp.GEN_PERTURB if args.gen == "perturb" else pp.GEN_RANDOM
    per_step = args.count * args.rounds
    spec = workload(args)
    g = pp.Dfg(spec, device=local)
    M = args.M
    sc = scenario(args, g.t1, g.grad_bytes)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    use_eft = GEN == pp.GEN_PERTURB and args.base == "eft"

    def step():
        base = g.eft_place(M, stream=stream) if use_eft else None      # SURVEY §8(f) f4 base seed
        r = g.search_best(M, GEN, SEED, args.count, rounds=args.rounds, tau=args.tau, base=base, comm=comm,
                          stream=stream)
        cells = pp.project_e2e(sc, [1, M], [g.t1, r.best_makespan_ps], args.nmax, device=local, stream=stream)
        x = pp.crossover(cells, [1, M], args.nmax, best_m=False, stream=stream)
        return r, x, cells

    for _ in range(args.warmup):
        step()
    barrier()
    # ---- device-timed steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = pp.kernel_launch_count()
    pp.set_kernel_timing(True)
    results = []
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.fill_(s & 0xFF)          # L2 flush outside the timed window
            barrier()
            ev[s][0].record(stream)
            results.append(step())
            ev[s][1].record(stream)
            torch.cuda.synchronize()
    launches = pp.kernel_launch_count() - launches0
    kern_ms, kern_n = pp.get_kernel_timing()
    pp.set_kernel_timing(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = torch.tensor([sum(step_ms), kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_ms, op=dist.ReduceOp.MAX)
    tot_ms, kern_ms_max = float(tot_ms[0]), float(tot_ms[1])
    value = per_step * args.steps / (tot_ms / 1e3)

    # ---- e2e through the C ABI with host buffers (load + search + projection + results)
    barrier()
    e2e_ms = []
    h2d = d2h = 0
    for s in range(max(1, args.steps)):
        flush.fill_(s & 0xFF)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        g2 = pp.Dfg(spec, device=local)                        # H2D of the DFG image
        base2 = g2.eft_place(M, stream=stream) if use_eft else None
        r2 = g2.search_best(M, GEN, SEED, args.count, rounds=args.rounds, tau=args.tau, base=base2, comm=comm,
                            stream=stream)
        cells2 = pp.project_e2e(sc, [1, M], [g2.t1, r2.best_makespan_ps], args.nmax, device=local, stream=stream)
        x2 = pp.crossover(cells2, [1, M], args.nmax, best_m=False, stream=stream)
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(t0.elapsed_time(t1))
        h2d = g2.image_bytes + ((g2.K + 15) // 16) * 16           # image + base upload
        d2h = 24 + ((g2.K + 15) // 16) * 16 + 4 + 76             # result, placement, range flag, crossover
        if use_eft:
            d2h += g2.K + 4                                      # EFT placement + status
        g2.close()
    e2 = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2, op=dist.ReduceOp.MAX)
    e2e_value = per_step * len(e2e_ms) / (float(e2[0]) / 1e3)

    if rank == 0:
        ops, smem_b = alg_counts(spec)
        clock, clock_src = measured_clock()
        pk = peaks(torch.cuda.get_device_properties(dev).multi_processor_count, clock)
        per_launch = args.count / world
        kern_avg_s = (kern_ms_max / max(1, kern_n)) / 1e3
        achieved_ops = ops * per_launch / kern_avg_s
        achieved_smem = smem_b * per_launch / kern_avg_s
        r, x, cells = results[-1]
        cells_np = pp.cells_to_numpy(cells)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {**config_dict(args, spec), "image_bytes": g.image_bytes, "live_slots": g.W},
            "gpu_launches": int(launches),
            "roofline": {"bound": "alu", "achieved": achieved_ops / 1e12, "peak": pk["int32_ops_per_s"] / 1e12,
                         "unit": "Tops/s (int32)", "frac": achieved_ops / pk["int32_ops_per_s"],
                         "traffic": ncu_traffic(), "traffic_unit": "DRAM bytes per launch (ncu)",
                         "kernel": f"pp::search_kernel<{M},{args.gen.upper()}>",
                         "kernel_ms_avg": kern_avg_s * 1e3, "kernel_share_of_step": kern_ms_max / tot_ms,
                         "alg_ops_per_placement": ops, "alg_smem_bytes_per_placement": smem_b,
                         "smem_frac": achieved_smem / pk["smem_bytes_per_s"],
                         "peak_note": f"148 SMs x 128 int32 lanes/clk x {clock:.0f} MHz ({clock_src} max SM clock)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "clocks": clk.summary(),
            "result": {"T1_ps": g.t1, "TM_ps": r.best_makespan_ps, "best_index": r.best_index,
                       "su_mp": g.t1 / r.best_makespan_ps, "crossover_n_star": x.n_star,
                       "n_star_vs_best_dp": x.n_star_vs_best_dp},
        }
        if world == 1 and not args.no_cpu_baseline:
            rate, n, dt = cpu_oracle_sample(spec, M, args.gen, args.tau, args.base)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                                    "sample": f"first {n} {args.gen.upper()} candidates of round 0 of the same "
                                              f"stream, {dt:.1f} s, single thread (nproc={os.cpu_count()})"}
        if args.parity != "off":
            mode = args.parity if args.parity != "auto" else ("live" if world == 1 else "golden")
            line["parity"] = parity_check(args, spec, r, x, cells_np, mode)
        print(json.dumps(line), flush=True)
    g.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pp", choices=["pp", "reference"])
    ap.add_argument("--M", type=int, default=2)
    ap.add_argument("--workload", default="inception_v3", choices=sorted(WORKLOADS))
    ap.add_argument("--count", type=int, default=10_000_000, help="candidates per round")
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--gen", default="perturb", choices=["perturb", "random"])
    ap.add_argument("--tau", type=int, default=8)
    ap.add_argument("--nmax", type=int, default=1024)
    ap.add_argument("--base", default="eft", choices=["eft", "zero"], help="PERTURB starting placement")
    ap.add_argument("--hw", default="none", choices=["none", *HW_GRAPHS],
                    help="evaluate on a general hardware graph instead of the uniform link")
    ap.add_argument("--ref-sample", type=int, default=200_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parity", default="auto", choices=["auto", "live", "golden", "off"],
                    help="check the step's result against the oracle: live (full oracle run over the host's "
                         "threads), golden (the committed oracle golden), auto = live at N=1, golden at N>1")
    args = ap.parse_args()
    if args.gen == "random":
        args.rounds = 1
    if args.impl == "reference":
        return run_reference(args)
    return run_pp(args)


if __name__ == "__main__":
    sys.exit(main())
