#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/k4lpt_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py tests/test_gpu_scene.py tests/test_gpu_capacity.py -q -x > gpurun_out/k4lpt_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/k4lpt_status.txt
for rep in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_lpt_$rep.log 2>&1; done
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_lpt_c3.log 2>&1
timeout 300 python bench.py --config c3lo --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_lpt_c3lo.log 2>&1

timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lpt_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
