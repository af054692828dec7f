"""Summarise an ncu report (pipe utilisation, issue, smem) for profiles/."""
import csv, subprocess, sys

def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {k: (v, u) for k, u, v in zip(r[0], r[1], r[2])}

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]

if __name__ == "__main__":
    d = raw(sys.argv[1])
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k][0]} {d[k][1]}")
    # stall reasons per issued instruction, then the executed-opcode mix (SASS page)
    print("\nstall reasons per issued instruction (smsp__average_warps_issue_stalled_*_per_issue_active):")
    for k, (v, u) in sorted(d.items()):
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(v) >= 0.05:
                    print(f"  {k.split('stalled_')[1].replace('_per_issue_active.ratio', ''):28s} {float(v):.3f}")
            except ValueError:
                pass
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))[2:]
    import collections
    ops, tot = collections.Counter(), 0
    for r in rows:
        try:
            n = int(r[5])
        except (ValueError, IndexError):
            continue
        t = r[1].split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += n
        tot += n
    if tot:
        print("\nexecuted warp-instructions by opcode:")
        print("  " + ", ".join(f"{o} {100 * n / tot:.1f}%" for o, n in ops.most_common(16)))
