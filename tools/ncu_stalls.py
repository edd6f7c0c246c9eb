"""Stall summary of an ncu --page source --csv --print-source sass export.
python tools/ncu_stalls.py <sass.csv> [kernel-index] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(dict(zip(cur["hdr"], r)))
b = blocks[want]
print(b["name"][:90])
cols = [h for h in b["hdr"] if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(int(d[c] or 0) for d in b["rows"]) for c in cols}
allS = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in b["rows"])
print("samples", allS, {k: v for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
for d in sorted(b["rows"], key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    why = {c[6:]: int(d[c]) for c in cols if int(d[c] or 0) > 0}
    print(d["Address"][-5:], d["Warp Stall Sampling (All Samples)"], d["Instructions Executed"],
          d["Source"].strip()[:60], why)
