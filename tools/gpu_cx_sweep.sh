set -x
for m in 0 2 3 4; do cp paper_2107_05681_b200/_lib/var/mod$m.so paper_2107_05681_b200/_lib/libdarm_gpu.so; echo "MOD=$m"; timeout 300 python tools/time_bitonic.py 64 256 1024 2>&1 | grep -v "^+"; done > gpurun_out/cx_sweep.txt 2>&1
cat gpurun_out/cx_sweep.txt
