#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/px8b_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
TSR_K4R_PX=8 timeout 900 python -m pytest tests/test_gpu_regions.py -q -x > gpurun_out/px8b_pytest.log 2>&1; echo "pytest_px8=$?" >> gpurun_out/px8b_status.txt
for rep in 1 2; do
  TSR_K4R_REGION=8 TSR_K4R_PX=8 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r8p8_$rep.log 2>&1
  TSR_K4R_REGION=4 TSR_K4R_PX=8 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r4p8_$rep.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r4p4_$rep.log 2>&1
done
for c in c3 c3lo; do
  TSR_K4R_REGION=8 TSR_K4R_PX=8 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r8p8_$c.log 2>&1
  TSR_K4R_REGION=4 TSR_K4R_PX=8 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r4p8_$c.log 2>&1
done
