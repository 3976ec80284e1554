#!/bin/bash
make -j8 all > /dev/null 2>&1
# round-2 evidence session: tests, smoke, bench (+cpu baseline, e2e), reference arm,
# other configs, launch list, ncu full capture of the step's kernels
mkdir -p gpurun_out/r2n
O=gpurun_out/r2n
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.draw --format=csv > $O/nvsmi.csv 2>&1
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
export TSR_PARITY_LOG=$O/parity_stats.jsonl; rm -f $TSR_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=900 > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status.txt
timeout 900 python bench.py > $O/bench_c2.log 2>&1; echo bench=$? >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo benchref=$? >> $O/status.txt
for cfg in c1 c3 c3lo; do timeout 600 python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
timeout 600 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.log 2>&1
timeout 600 python bench.py --deterministic --no-cpu-baseline > $O/bench_c2_det.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu1=$? >> $O/status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"render_bwd|render_fwd|vjp_adam|ssim_|build_index|preprocess_kernel|cull_compact|tile_order" -s 9 -c 9 -o $O/prof_r2n python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1; echo ncu2=$? >> $O/status.txt
timeout 400 python bench.py --config c5 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo c5=$? >> $O/status.txt
timeout 600 python bench.py --vp --no-cpu-baseline > $O/bench_c2_vp.log 2>&1
