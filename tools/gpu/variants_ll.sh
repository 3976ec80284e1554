#!/bin/bash
# per-variant C2 bench + launch list: bash tools/gpu/variants_ll.sh name1 name2 ...
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2601_19489_b200/libtilesplat_b200.so; else lib=build/libtilesplat_b200_$v.so; fi
  TSR_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.log 2>&1
  TSR_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$v.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
