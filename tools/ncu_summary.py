"""Key metrics per launch from an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions",
        "Grid Size", "Block Size", "Warp Cycles Per Issued Instruction"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
r = csv.reader(io.StringIO(out))
h = next(r)
cur = None
seen = set()
for row in r:
    d = dict(zip(h, row))
    k = (d["ID"], d["Kernel Name"][:60])
    m = d["Metric Name"]
    if m in WANT and (k, m) not in seen:
        seen.add((k, m))
        if k != cur:
            print("---", *k)
            cur = k
        print(f"    {m:36s} {d['Metric Value']:>14s} {d['Metric Unit']}")
