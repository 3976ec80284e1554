#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/k3hw_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py -q -x > gpurun_out/k3hw_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/k3hw_status.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_hw_on_$rep.log 2>&1
  TSR_K3_HW=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_hw_off_$rep.log 2>&1
done
