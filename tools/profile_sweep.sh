#!/bin/bash
# ncu evidence of one ADMM sweep of the bench workload (run on the GPU box):
#   1. launch list of bench.py (--steps 2 --warmup 1): per-launch durations
#   2. --set full of the 4th uncontended sweep (TR_SERIAL_MODES=1 tools/sweep_profile.py 1)
#      digested into <out>_full.json / _categories.json / _traffic.json
# usage: tools/profile_sweep.sh OUTDIR TAG
set -e
out=${1:-gpurun_out}; tag=${2:-r2}
mkdir -p "$out"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$out/ncu_launches_admm_sweep_${tag}.csv" \
    python bench.py --steps 2 --warmup 1 --no-legs --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py "$out/ncu_launches_admm_sweep_${tag}.csv" 2 > "$out/launch_table_${tag}.txt" || true
# count the launches before the 4th sweep of sweep_profile (3 warm-up sweeps)
TR_SERIAL_MODES=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
    --log-file /tmp/sp_launches.csv python tools/sweep_profile.py 1 > /dev/null 2>&1
read skip count < <(python - <<'PY'
import csv
rows=[r for r in csv.reader(open('/tmp/sp_launches.csv')) if len(r) > 5]
h=rows[0]; iK=h.index("Kernel Name"); iID=h.index("ID")
ids=[]; seen=set()
for r in rows[1:]:
    if r[iID] in seen: continue
    seen.add(r[iID]); ids.append(r[iK])
st=[i for i,k in enumerate(ids) if "k_lrta_input" in k]
# the sweep starts with its FFT passes: 5 launches before k_lrta_input
a=st[3]-5; b=len(ids)
print(a, b-a)
PY
)
TR_SERIAL_MODES=1 ncu --set full --clock-control none --launch-skip $skip --launch-count $count \
    -o /tmp/sweep_full python tools/sweep_profile.py 1 > /dev/null 2>&1
python tools/ncu_digest.py /tmp/sweep_full.ncu-rep "$out/ncu_${tag}" > "$out/ncu_${tag}_digest.txt"
echo "skip $skip count $count"
