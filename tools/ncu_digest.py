"""Digest an ncu --set full capture of one ADMM sweep into per-kernel and
per-category summaries (profiles/rNN/ncu_full_*.json, traffic.json).

python tools/ncu_digest.py report.ncu-rep out_prefix
Kernel -> bench category mapping follows the tr::launch categories.
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

CAT = [  # (kernel-name regex, category); first match wins
    (r"k_panel_mma<\d+, 1>|k_panel<.*, 1>", "panel_gram"),
    (r"k_panel_mma<\d+, 0>|k_panel<.*, 0>", "panel_sketch"),
    (r"k_proj_ws", "proj_tc"),
    (r"k_gemm_expand|k_expand_tc", "gemm_expand"),
    (r"k_expand_mode1", "expand_mode1"),
    (r"k_fft", "fft"),
    (r"k_sweep_tail", "sweep_tail"),
    (r"k_lrta_input", "lrta_input"),
    (r"k_orth_cluster|k_tsqr", "orth"),
    (r"k_ritz", "ritz"),
    (r"k_face_svt", "face_svt"),
]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

rep, prefix = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
kern = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("tr::", "")
    e = {"id": int(d["ID"]), "kernel": name}
    U = dict(zip(hdr, units))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
             "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "B": 1.0,
             "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for m in M:
        v = d.get(m, "")
        try:
            v = float(v.replace(",", "")) * scale.get(U.get(m, ""), 1.0)
        except ValueError:
            v = None
        e[m] = v
    e["duration_us"] = e.pop("gpu__time_duration.sum")
    rb, wb = e["dram__bytes_read.sum"] or 0, e["dram__bytes_write.sum"] or 0
    e["dram_GBps"] = (rb + wb) / (e["duration_us"] * 1e-6) / 1e9 if e["duration_us"] else None
    e["category"] = next((c for rx, c in CAT if re.search(rx, d["Kernel Name"].replace("tr::", ""))), None)
    kern.append(e)
json.dump({"how": "ncu --set full --clock-control none (one launch per row)", "launches": kern},
          open(prefix + "_full.json", "w"), indent=1)
cat = collections.defaultdict(lambda: {"bytes": 0.0, "launches": 0, "us": 0.0})
for e in kern:
    if e["category"]:
        c = cat[e["category"]]
        c["bytes"] += (e["dram__bytes_read.sum"] or 0) + (e["dram__bytes_write.sum"] or 0)
        c["launches"] += 1
        c["us"] += e["duration_us"] or 0
json.dump(dict(cat), open(prefix + "_categories.json", "w"), indent=1)
# per-step traffic by category (bench.py roofline "traffic": newest profiles/r*/traffic.json)
json.dump({"how": "ncu --set full of one uncontended ADMM sweep (TR_SERIAL_MODES=1 "
                  "tools/sweep_profile.py); DRAM read + write bytes summed per category",
           "categories": {k: {"bytes_per_step": v["bytes"], "launches": v["launches"],
                              "us_serialised": v["us"]} for k, v in cat.items()}},
          open(prefix + "_traffic.json", "w"), indent=1)
for k, v in sorted(cat.items(), key=lambda x: -x[1]["us"]):
    print(f"{k:14s} launches {v['launches']:3d}  {v['us']:9.1f} us  {v['bytes'] / 1e9:7.3f} GB  "
          f"{v['bytes'] / (v['us'] * 1e-6) / 1e9 if v['us'] else 0:7.1f} GB/s")
