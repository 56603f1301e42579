"""Summarise an .ncu-rep (details page metrics, dynamic instruction mix, stall reasons,
DRAM bytes) into a text file for profiles/.  Usage: ncu_summary.py REP OUT [elements]"""
import collections
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
elements = float(sys.argv[3]) if len(sys.argv) > 3 else None


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


lines = []
rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
hdr = {h: i for i, h in enumerate(rows[0])}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]
for r in rows[1:]:
    if r[hdr["Metric Name"]] in want:
        lines.append(f"{r[hdr['Kernel Name']][:60]:60s} {r[hdr['Metric Name']]:36s} {r[hdr['Metric Value']]} {r[hdr['Metric Unit']]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
names, vals = raw[0], raw[2]
lines.append("")
for h, v in zip(names, vals):
    if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active") or "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
        lines.append(f"  {h:70s} {v}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr2, data, kname = None, [], None
for r in src:
    if r and r[0] == "Kernel Name":
        if kname:
            break
        kname = r[1]
        continue
    if r and r[0] == "Address":
        hdr2 = r
        continue
    if hdr2 and r:
        data.append(r)
if hdr2:
    h2 = {k: i for i, k in enumerate(hdr2)}
    ops = collections.Counter()
    for r in data:
        toks = r[h2["Source"]].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += int(r[h2["Instructions Executed"]] or 0)
    tot = sum(ops.values())
    lines.append("")
    lines.append(f"dynamic SASS mix of {kname[:80]}: {tot} warp-instructions"
                 + (f" = {tot * 32 / elements:.1f} thread-instr per edge-codeword" if elements else ""))
    for op, n in ops.most_common(24):
        lines.append(f"  {op:10s} {n:12d} {100 * n / tot:5.1f}%" + (f"  {n * 32 / elements:6.2f}/elem" if elements else ""))
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:12]))
