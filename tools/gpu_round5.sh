#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bitonic_sort_kernel -c 2 -o gpurun_out/prof_bitonic python tools/profile_driver.py bitonic > gpurun_out/ncu_bitonic.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_panel -s 100 -c 1 -o gpurun_out/prof_lud_unmelded python tools/profile_driver.py lud > gpurun_out/ncu_lud_u.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_panel -s 612 -c 1 -o gpurun_out/prof_lud_melded python tools/profile_driver.py lud > gpurun_out/ncu_lud_m.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lud2048.csv python tools/profile_driver.py lud 2048 > gpurun_out/ncu_lud_list.log 2>&1
ls -la gpurun_out
