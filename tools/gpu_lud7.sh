mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "lud" > gpurun_out/pytest_lud.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lud.log
for r in 0 4 8 16 24 32; do echo "panel_sms=$r"; DARM_LUD_PANEL_SMS=$r timeout 300 python tools/time_lud.py 8192; done > gpurun_out/time_lud.log 2>&1
