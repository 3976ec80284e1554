#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_scene.py tests/test_gpu_trainer.py tests/test_gpu_capacity.py -q -x > gpurun_out/e2e_pytest.log 2>&1; echo pytest=$? > gpurun_out/e2e_status.txt
for rep in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e_$rep.log 2>&1; done
