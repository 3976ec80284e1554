#!/bin/bash
# run selected GPU tests: bash tools/gpu/one.sh <pytest args...>
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest "$@" -q -x > gpurun_out/one_pytest.log 2>&1; echo pytest=$? > gpurun_out/one_status.txt
