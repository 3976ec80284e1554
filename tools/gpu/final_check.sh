#!/bin/bash
# round-end re-check of the committed tree: GPU tests, smoke, three C2 bench runs
make -j8 all > /dev/null 2>&1
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=900 > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status.txt
for i in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > $O/bench_c2_$i.log 2>&1; echo bench$i=$? >> $O/status.txt; done
