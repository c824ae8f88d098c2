mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "lud" > gpurun_out/pytest_lud.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lud.log
timeout 300 python tools/time_lud.py 4096 8192 > gpurun_out/time_lud.log 2>&1
DARM_LUD_FAR=tiles timeout 300 python tools/time_lud.py 4096 8192 >> gpurun_out/time_lud.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_far_pipe -s 0 -c 1 -o gpurun_out/prof_lud_far python tools/profile_driver.py lud > gpurun_out/ncu_lud_far.log 2>&1
