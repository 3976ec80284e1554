#!/bin/bash
# full GPU parity suite (+ scale parity stats) and smoke
mkdir -p gpurun_out
export TSR_PARITY_LOG=gpurun_out/parity_stats.jsonl
rm -f $TSR_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=900 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
