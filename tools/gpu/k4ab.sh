#!/bin/bash
# K4 A/B: work-unit form vs per-tile CTAs; parity subset first
mkdir -p gpurun_out
export TSR_PARITY_LOG=gpurun_out/parity_stats.jsonl; rm -f $TSR_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_raster.py tests/test_gpu_scene.py tests/test_gpu_capacity.py tests/test_gpu_trainer.py -q -x --timeout=600 > gpurun_out/pytest_k4.log 2>&1; echo pytest=$? >> gpurun_out/status_k4.txt
for f in units tiles units; do
  TSR_K4=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k4_$f.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
