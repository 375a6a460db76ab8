"""Summarise an ncu report: key metrics + SASS opcode mix (run here, no GPU)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            res.append((d["Kernel Name"][:40], d["Metric Name"], d["Metric Unit"], d["Metric Value"]))
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        for n in names:
            if n in h:
                res[n] = (r[h.index(n)], u[h.index(n)])
    return res


def opmix(rep, top=22):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, ie, ist = h.index("Source"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    byop, stall = collections.Counter(), collections.Counter()
    tot = tots = 0
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        f = r[ia].split()
        if not f:
            continue
        op = f[1] if f[0].startswith("@") else f[0]
        op = op.split(".")[0]
        n, s = int(r[ie] or 0), int(r[ist] or 0)
        byop[op] += n
        stall[op] += s
        tot += n
        tots += s
    lines = [f"total warp-instructions {tot}, stall samples {tots}"]
    for op, n in byop.most_common(top):
        lines.append(f"  {op:10s} {100 * n / max(tot, 1):5.1f}% inst   {100 * stall[op] / max(tots, 1):5.1f}% stall")
    return lines


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, m, u, v in details(rep):
        print(f"{k:40s} {m:40s} {v} {u}")
    for n, (v, u) in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                               "sm__inst_executed.sum", "smsp__inst_executed.avg.per_cycle_active",
                               "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                               "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                               "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                               "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
                               "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                               "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
                               "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]).items():
        print(f"  {n:80s} {v} {u}")
    if "--ops" in sys.argv:
        print("\n".join(opmix(rep)))
