"""Print the key ncu sections + pipe utilisation + stall reasons of a report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]
keep = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
        "Occupancy", "Warp State Statistics", "Launch Statistics")
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Section Name") in keep and d.get("Metric Name") in (
            "Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
            "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Grid Size",
            "Block Size", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Static Shared Memory Per Block", "Max Bandwidth"):
        print(f"{d['Section Name'][:24]:24} | {d['Metric Name'][:40]:40} | {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
for k, un, val in zip(h, u, v):
    if (("sm__inst_executed_pipe" in k and k.endswith(".avg.pct_of_peak_sustained_active"))
            or (k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"))
            or k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                     "sm__warps_active.avg.pct_of_peak_sustained_active")):
        try:
            if float(val.replace(",", "")) < 0.05:
                continue
        except ValueError:
            pass
        print(f"{k} = {val} {un}")
