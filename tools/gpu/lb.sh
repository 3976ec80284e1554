#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_binning.py tests/test_gpu_loss_contract.py tests/test_gpu_trainer.py tests/test_gpu_acceptance.py -q -x --timeout=600 > gpurun_out/pytest_lb.log 2>&1; echo pytest=$? > gpurun_out/status_lb.txt
for a in 1 8; do python -m paper_2601_19489_b200.benchtiling --n-splats 1000000 --anisotropy $a --width 1920 --height 1080 > gpurun_out/bt_1m_a$a.txt 2>&1; done
python -m paper_2601_19489_b200.benchtiling --n-splats 100000 --anisotropy 8 > gpurun_out/bt_100k.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_lbcheck.log 2>&1
