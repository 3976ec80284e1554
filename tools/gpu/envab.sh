#!/bin/bash
# env A/B on the default lib: bash tools/gpu/envab.sh "NAME=VAL" ...  ("base" = no env)
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for e in "$@"; do
  tag=$(echo "$e" | tr '=' '_')
  for rep in 1 2; do
    if [ "$e" = "base" ]; then timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_env_${tag}_$rep.log 2>&1
    else env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_env_${tag}_$rep.log 2>&1; fi
  done
done
