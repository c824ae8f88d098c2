mkdir -p gpurun_out
for r in 0 4 8 12 16 24; do echo "panel_sms=$r"; DARM_LUD_PANEL_SMS=$r timeout 300 python tools/time_lud.py 8192; done > gpurun_out/time_lud.log 2>&1
