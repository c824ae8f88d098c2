# time the bitonic register kernels built for 4 / 5 / 6 resident CTAs per SM
for m in 4 5 6; do cp paper_2107_05681_b200/_lib/var/minb$m.so paper_2107_05681_b200/_lib/libdarm_gpu.so; echo "MIN_CTAS=$m"; timeout 300 python tools/time_bitonic.py 64 256 1024 2>&1 | grep -v "kpt= 1"; done > gpurun_out/minb_sweep.txt 2>&1
cat gpurun_out/minb_sweep.txt
