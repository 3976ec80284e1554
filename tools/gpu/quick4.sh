#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_loss.py tests/test_gpu_loss_contract.py -q -x --timeout=600 > gpurun_out/pytest_q4.log 2>&1; echo pytest=$? > gpurun_out/status_q4.txt
for c in c2 c1; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_q4_$c.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q4.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
