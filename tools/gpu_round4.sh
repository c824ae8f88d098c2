#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:srad_sweep -c 4 -o gpurun_out/prof_srad python tools/profile_driver.py srad > gpurun_out/ncu_srad.log 2>&1
ls -la gpurun_out
