"""Print ncu --csv metric rows compactly: python tools/ncu_metrics.py <csv> [name-filter]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if flt in d["Kernel Name"]:
            print(d["ID"], d["Kernel Name"][:34], d["Metric Name"], d["Metric Value"])
