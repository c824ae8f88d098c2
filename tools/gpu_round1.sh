#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list, ncu captures.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bitonic_sort_kernel -c 2 -o gpurun_out/prof_bitonic python tools/profile_driver.py bitonic > gpurun_out/ncu_bitonic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:corpus_lanes -c 2 -o gpurun_out/prof_sb1 python tools/profile_driver.py sb1 > gpurun_out/ncu_sb1.log 2>&1
ls -la gpurun_out
