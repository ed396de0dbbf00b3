"""Summarise an .ncu-rep (raw page + source page) into text: key metrics, opcode mix, hot SASS."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, vals = rows[0], rows[2:]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_warps", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active"]
for v in vals:
    for k in KEYS:
        if k in h:
            print(f"{k} = {v[h.index(k)]} {rows[1][h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
isrc, ie, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(r[isrc].strip(), int(r[ie]), int(r[ist])) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot = sum(d[1] for d in data); tots = sum(d[2] for d in data)
print("total warp-inst", tot, "sass lines", len(data), "stall samples", tots)
ops = collections.Counter(); st = collections.Counter()
for s, e, w in data:
    f = s.split()
    op = (f[1] if f[0].startswith("@") else f[0]).split(".")[0]
    ops[op] += e; st[op] += w
for op, c in ops.most_common(24):
    print(f"  {op:8s} {100*c/tot:5.1f}% inst   {100*st[op]/max(tots,1):5.1f}% stall samples")
if len(sys.argv) > 2:
    thr = float(sys.argv[2]) * tot
    print("---- SASS with >= %.2f%% of instructions or stalls" % (100 * float(sys.argv[2])))
    for i, (s, e, w) in enumerate(data):
        if e >= thr or w >= float(sys.argv[2]) * tots:
            print(f"{i:5d} {100*e/tot:5.2f}% {100*w/max(tots,1):5.2f}%  {s[:100]}")
