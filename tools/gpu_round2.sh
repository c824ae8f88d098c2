#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bitonic_sort_kernel -c 2 -o gpurun_out/prof_bitonic python tools/profile_driver.py bitonic > gpurun_out/ncu_bitonic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nqueens_kernel -c 2 -o gpurun_out/prof_nqueens python tools/profile_driver.py nqueens > gpurun_out/ncu_nqueens.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out
