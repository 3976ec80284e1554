#!/bin/bash
# one full ncu capture of K1b (source-level) + binning tests
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_binning.py -q -x > gpurun_out/k1_pytest.log 2>&1; echo "pytest=$?" > gpurun_out/k1_status.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:preprocess_kernel -s 3 -c 1 -o gpurun_out/k1_full -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/k1_ncu.log 2>&1
