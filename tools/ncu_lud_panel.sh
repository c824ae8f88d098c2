#!/bin/bash
# ncu --set full (with source) of one panel launch of LUD 8192^2 (the panel of
# step SKIP, default a P=3 panel late in the factorisation); kept as a report
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_panel_kernel -s ${SKIP:-403} -c 1 -o gpurun_out/prof_lud_panel${TAG:-} python tools/profile_driver.py lud > gpurun_out/ncu_lud_panel.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_lud_panel${TAG:-}.ncu-rep > gpurun_out/ncusum_lud_panel${TAG:-}.json
ncu -i gpurun_out/prof_lud_panel${TAG:-}.ncu-rep --page source --csv --print-source sass > gpurun_out/lud_panel_source${TAG:-}.csv 2>/dev/null
cat gpurun_out/ncusum_lud_panel${TAG:-}.json
