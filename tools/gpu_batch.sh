set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_fullsize_gpu.py tests/test_lrta_gpu.py tests/test_baseline_configs_gpu.py -x -q -m gpu 2>&1 | tail -15
for c in 3 2; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>&1 | tail -1
TR_NO_PANEL_CLUSTER=1 timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>&1 | tail -1
done
timeout 300 python bench.py --step admm-sharded --steps 5 --warmup 3 2>&1 | tail -1
TR_NO_PANEL_CLUSTER=1 timeout 300 python bench.py --step admm-sharded --steps 5 --warmup 3 2>&1 | tail -1
