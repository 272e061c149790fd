"""Summarise an ncu report: key SOL / memory / scheduler metrics per kernel.
usage: python tools/ncu_summary.py report.ncu-rep [name-filter]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name",
                                           "Metric Value", "Metric Unit"))
keep = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Theoretical Occupancy", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"}
seen = set()
for r in rows[1:]:
    if filt and filt not in r[ki]:
        continue
    key = (r[ki], r[mi])
    if r[mi] in keep and key not in seen:
        seen.add(key)
        print(f"{r[ki][:40]:40s} {r[mi]:38s} {r[vi]:>14s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rr = list(csv.reader(raw))
if len(rr) > 2:
    hh = rr[0]
    want = [i for i, n in enumerate(hh) if n in (
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "gpu__time_duration.sum")]
    for row in rr[2:]:
        if filt and filt not in row[hh.index("Kernel Name")]:
            continue
        print(row[hh.index("Kernel Name")][:40], {hh[i]: row[i] for i in want})
