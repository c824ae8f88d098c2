mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "lud" > gpurun_out/pytest_lud.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lud.log
timeout 300 python tools/time_lud.py 2048 4096 8192 > gpurun_out/time_lud.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lud8192.csv python tools/profile_driver.py lud 8192 > /dev/null 2>&1
