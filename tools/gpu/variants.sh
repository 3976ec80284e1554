#!/bin/bash
# A/B of experiment variant libraries: bash tools/gpu/variants.sh name1 name2 ... (build/libtilesplat_b200_<name>.so; "base" = the default lib)
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2601_19489_b200/libtilesplat_b200.so; else lib=build/libtilesplat_b200_$v.so; fi
  TSR_LIB=$lib timeout 600 python -m pytest tests/test_gpu_regions.py -q -x --timeout=600 > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest=$?" >> gpurun_out/variants_status.txt
  for rep in 1 2; do
    TSR_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
done
