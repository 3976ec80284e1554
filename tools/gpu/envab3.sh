#!/bin/bash
# env A/B at C3 / C3-lo / C1: bash tools/gpu/envab3.sh "NAME=VAL" ... ("base" = no env)
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for e in "$@"; do
  tag=$(echo "$e" | tr '=' '_')
  for c in c3 c3lo c1; do
    if [ "$e" = "base" ]; then timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_env3_${tag}_$c.log 2>&1
    else env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_env3_${tag}_$c.log 2>&1; fi
  done
done
