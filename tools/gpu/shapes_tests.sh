#!/bin/bash
# the non-default K4r shapes through the region / scale-parity / scene tests
mkdir -p gpurun_out; rm -f gpurun_out/shapes_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
TSR_K4R_REGION=4 timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py tests/test_gpu_scene.py -q -x > gpurun_out/shapes_r4.log 2>&1; echo "r4=$?" >> gpurun_out/shapes_status.txt
TSR_K4R_PX=4 timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py tests/test_gpu_scene.py -q -x > gpurun_out/shapes_p4.log 2>&1; echo "p4=$?" >> gpurun_out/shapes_status.txt
TSR_K4R_REGION=4 TSR_K4R_PX=4 timeout 900 python -m pytest tests/test_gpu_regions.py -q -x > gpurun_out/shapes_r4p4.log 2>&1; echo "r4p4=$?" >> gpurun_out/shapes_status.txt
