#!/bin/bash
# ncu --set full of one mid-size far-update launch of LUD 8192^2 (the 22nd), summarised on the box
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-lud_far} -s ${SKIP:-21} -c 1 -o gpurun_out/prof_lud_far${TAG:-} python tools/profile_driver.py lud > gpurun_out/ncu_lud_far.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_lud_far${TAG:-}.ncu-rep > gpurun_out/ncusum_lud_far${TAG:-}.json
cat gpurun_out/ncusum_lud_far${TAG:-}.json
