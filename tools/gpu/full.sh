#!/bin/bash
# full measurement session: tests, smoke, bench (+cpu baseline), reference arm, ncu evidence
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.draw --format=csv > gpurun_out/nvsmi.csv 2>&1
timeout 600 python -m pytest tests -m gpu -q -rf --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo benchref=$? >> gpurun_out/status.txt
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"render_bwd|render_fwd|vjp_adam|ssim_fwd" -s 4 -c 4 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/status.txt
