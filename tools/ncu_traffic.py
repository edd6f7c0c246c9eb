"""profiles/rNN/traffic.json (DRAM bytes per ADMM sweep by kernel category) from
the targeted captures of tools/profile_kernels.sh.

python tools/ncu_traffic.py <dir with ncu_<tag>_{panel,fft,tail,proj}_raw.csv> <tag> <out.json>
Captured launches are the big (whole-tensor) ones of the 4th sweep; the per-sweep
figure multiplies each by its launches per sweep (3 t-SVTs) and adds the small
mode-1 launches where they were captured (proj) or estimates them from the core
size (panel passes over the 13 MB core unfolding)."""
import csv
import json
import sys

d, tag, out = sys.argv[1], sys.argv[2], sys.argv[3]


def launches(name):
    rows = list(csv.reader(open(f"{d}/ncu_{tag}_{name}_raw.csv")))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ms": 1e3, "ns": 1e-3}
    res = []
    for r in rows[2:]:
        e = dict(zip(hdr, r))

        def val(m):
            return float(e[m].replace(",", "")) * scale[units[hdr.index(m)]]

        res.append({"kernel": e["Kernel Name"].split("(")[0].replace("void ", ""),
                    "us": val("gpu__time_duration.sum"),
                    "bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum")})
    return res


cat = {}


def add(name, ls, per_step, extra_bytes=0.0, extra_launches=0):
    b = sum(x["bytes"] for x in ls) / len(ls) * per_step + extra_bytes
    cat[name] = {"bytes_per_step": b, "launches_per_step": per_step + extra_launches,
                 "captured_launches": len(ls), "us_per_captured_launch": sum(x["us"] for x in ls) / len(ls)}


pan = launches("panel")
core_mb = 13.4e6  # mode-1 unfolding of the bench core: 1024 x 3200 fp32
add("panel_sketch", [x for x in pan if "<2, 0" in x["kernel"]], 3, 3 * core_mb, 3)
add("panel_gram", [x for x in pan if "<2, 1" in x["kernel"]], 9, 9 * core_mb, 9)
fft = launches("fft")
cat["fft"] = {"bytes_per_step": sum(x["bytes"] for x in fft), "launches_per_step": len(fft),
              "captured_launches": len(fft), "us_per_step": sum(x["us"] for x in fft)}
tail = launches("tail")
add("lrta_input", [x for x in tail if "k_lrta_input" in x["kernel"]], 1)
add("sweep_tail", [x for x in tail if "k_sweep_tail" in x["kernel"]], 1)
prj = launches("proj")
pw = [x for x in prj if "k_proj_ws" in x["kernel"]]
cat["proj_tc"] = {"bytes_per_step": 3 * sum(x["bytes"] for x in pw), "launches_per_step": 6,
                  "captured_launches": len(pw), "us_per_tsvt": sum(x["us"] for x in pw)}
add("gemm_expand", [x for x in prj if "k_expand_tc" in x["kernel"]], 3)
json.dump({"how": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                  "--clock-control none on the 4th uncontended sweep of the bench workload "
                  "(TR_SERIAL_MODES=1 tools/sweep_profile.py 1; tools/profile_kernels.sh); "
                  "per-sweep = captured launch x launches per sweep (see tools/ncu_traffic.py)",
           "categories": cat}, open(out, "w"), indent=1)
for k, v in cat.items():
    print(f"{k:14s} {v['bytes_per_step'] / 1e9:8.3f} GB/sweep  {v['launches_per_step']} launches")
