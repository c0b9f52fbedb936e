"""Summarise an ncu report (details page) and the hottest SASS lines: python tools/ncu_summary.py rep [--sass N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
keys = {"Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Theoretical Active Warps per SM", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Limit Shared Mem",
        "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Compute (SM) Throughput",
        "No Eligible", "Eligible Warps Per Scheduler", "Avg. Active Threads Per Warp", "Branch Efficiency"}
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
iN, iV, iU, iK = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
for row in r[1:]:
    if row[iN] in keys:
        print(f"{row[iK][:30]:30s} {row[iN]:40s} {row[iV]} {row[iU]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_lsu.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "gpu__time_duration.sum"]
for i, name in enumerate(rr[0]):
    if name in want and len(rr) > 2:
        print(f"raw {name:60s} {rr[2][i]} {rr[1][i]}")
if "--sass" in sys.argv:
    n = int(sys.argv[sys.argv.index("--sass") + 1])
    s = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(s.splitlines()))
    hh = rows[1]
    iA, iS, iE, iW = hh.index("Address"), hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    tot = sum(int(x[iE] or 0) for x in data)
    totw = sum(int(x[iW] or 0) for x in data)
    print("total executed", tot, "stall samples", totw)
    mx = max(int(x[iE] or 0) for x in data)
    for x in data:
        e, w = int(x[iE] or 0), int(x[iW] or 0)
        if e > mx / n or w > totw * 0.004:
            print(f"{x[iA][-5:]:>6} {e:12d} {w:6d}  {x[iS][:100]}")
