mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lud8192.csv python tools/profile_driver.py lud 8192 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_update -s 4 -c 1 -o gpurun_out/prof_lud_far python tools/profile_driver.py lud > gpurun_out/ncu_lud_far.log 2>&1
