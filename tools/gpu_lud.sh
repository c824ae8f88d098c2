set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "lud" > gpurun_out/pytest_lud.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lud.log
timeout 300 python tools/time_lud.py 2048 4096 8192 > gpurun_out/time_lud.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lud2048.csv python tools/profile_driver.py lud 2048 > gpurun_out/ncu_lud_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_panel -s 100 -c 1 -o gpurun_out/prof_lud_unmelded python tools/profile_driver.py lud > gpurun_out/ncu_lud_u.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_panel -s 612 -c 1 -o gpurun_out/prof_lud_melded python tools/profile_driver.py lud > gpurun_out/ncu_lud_m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lud_update -s 40 -c 1 -o gpurun_out/prof_lud_update python tools/profile_driver.py lud > gpurun_out/ncu_lud_upd.log 2>&1
