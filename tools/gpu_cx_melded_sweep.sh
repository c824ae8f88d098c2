# time the bitonic register kernels with the melded form's FMA-pipe maxima every 2nd / 3rd / 4th / 8th pair
for m in 2 3 4 8; do cp paper_2107_05681_b200/_lib/var/mm$m.so paper_2107_05681_b200/_lib/libdarm_gpu.so; echo "MELDED_MOD=$m"; for r in 1 2; do timeout 300 python tools/time_bitonic.py 64 256 1024 2>&1 | grep "kpt=16"; done; done > gpurun_out/cx_melded_sweep.txt 2>&1
cat gpurun_out/cx_melded_sweep.txt
