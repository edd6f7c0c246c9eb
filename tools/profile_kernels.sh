#!/bin/bash
# Targeted ncu --set full captures (with SASS source counters) of the hot
# kernels of the 4th uncontended sweep of the bench workload
# (TR_SERIAL_MODES=1 tools/sweep_profile.py 1: 3 warm-up sweeps, then 1).
# usage: tools/profile_kernels.sh OUTDIR TAG     (run on the GPU box); writes <name>_raw.csv (all metrics)
#   and <name>_sass.csv (per-instruction stall samples: tools/ncu_stalls.py)
out=${1:-gpurun_out}; tag=${2:-r2}
mkdir -p "$out"
cap() {  # name regex skip count
  TR_SERIAL_MODES=1 timeout 300 ncu --set full --clock-control none \
    -k "regex:$2" --launch-skip "$3" --launch-count "$4" -f -o "/tmp/ncu_${tag}_$1" \
    python tools/sweep_profile.py 1 > /dev/null 2>&1
  # the reports embed the library's cubin (~120 MB each): only the exports travel back
  ncu -i "/tmp/ncu_${tag}_$1.ncu-rep" --page raw --csv > "$out/ncu_${tag}_$1_raw.csv" 2>/dev/null
  ncu -i "/tmp/ncu_${tag}_$1.ncu-rep" --page source --csv --print-source sass \
    > "$out/ncu_${tag}_$1_sass.csv" 2>/dev/null
  rm -f "/tmp/ncu_${tag}_$1.ncu-rep"
}
# per sweep: 24 k_panel_mma (per t-SVT: sketch, 3 gram on mode 0, the same on mode 1),
# 3 k_fft4, 2 k_fft4_real, 1 tail, 6 k_proj_ws, 1 k_lrta_input, 3 k_expand_tc
cap panel 'k_panel_mma' 72 4
cap fft 'k_fft4' 15 5
cap tail 'k_sweep_tail|k_lrta_input' 6 2
cap proj 'k_proj_ws|k_expand_tc' 27 3
