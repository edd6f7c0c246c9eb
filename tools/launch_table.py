"""Per-kernel totals of one ADMM sweep from an ncu launch list (gpu__time_duration.sum).

python tools/launch_table.py launches.csv [sweep_index]
A sweep cycle starts at each k_lrta_input launch (one per sweep); ncu serialises launches, so the
sum is the uncontended device time of the sweep.
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iK, iV, iID = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
seq = [(int(r[iID]), r[iK], float(r[iV].replace(",", ""))) for r in rows[1:]]
starts = [i for i, (_, k, _) in enumerate(seq) if "k_lrta_input" in k]
w = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sw = seq[starts[w]:starts[w + 1]]
print(f"sweep {w}: {len(sw)} launches, {sum(x[2] for x in sw) / 1e3:.1f} us serialised")
agg = collections.defaultdict(lambda: [0, 0.0])
for _, k, v in sw:
    name = re.sub(r"\(.*", "", k).replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += v / 1e3
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us  {n:4d}  {k[:90]}")
