mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ms.csv python tools/profile_driver.py merge > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_sort -c 24 -o gpurun_out/prof_ms python tools/profile_driver.py merge > gpurun_out/ncu_ms.log 2>&1
