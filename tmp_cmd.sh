nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,power.draw --format=csv
for v in default ahead minb16 default; do
  if [ $v = default ]; then L=""; else L="DARM_GPU_LIB=variants/$v/libdarm_gpu.so"; fi
  env $L timeout 300 python tools/time_srad.py $v 2>&1 | tail -2
done
