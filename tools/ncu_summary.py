"""Summarise an ncu --set full report (details page) into the lines we track."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
iK, iS, iM, iU, iV = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
keys = sys.argv[2:] or ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread", "Achieved Occupancy",
                        "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
                        "Compute (SM) Throughput", "Executed Instructions", "Local Memory Spilling Requests", "Warp Cycles Per Issued Instruction",
                        "No Eligible", "Theoretical Occupancy", "Shared Memory Configuration Size"]
seen = set()
for r in rows[1:]:
    if len(r) <= iV or not r[iM]:
        continue
    if any(k in r[iM] for k in keys) and (r[iK], r[iM]) not in seen:
        seen.add((r[iK], r[iM]))
        print(f"{r[iK][:60]:60s} | {r[iM]:45s} | {r[iV]} {r[iU]}")
