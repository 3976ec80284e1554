#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_scene.py tests/test_gpu_raster.py -q -x --timeout=600 > gpurun_out/pytest_order.log 2>&1; echo pytest=$? > gpurun_out/status_order.txt
for cfg in c2 c3 c3lo; do for o in heavy raster; do
  TSR_TILE_ORDER=$o timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_order_${cfg}_$o.log 2>&1
done; done
