python -m pytest tests/test_srad.py -q -x -m gpu > gpurun_out/pytest_srad.log 2>&1; echo "srad tests rc=$?"; tail -5 gpurun_out/pytest_srad.log
for v in default srad_minb16 srad_minb20 srad_st4 srad_st16; do
  if [ $v = default ]; then L=""; else L="DARM_GPU_LIB=variants/$v/libdarm_gpu.so"; fi
  env $L timeout 300 python tools/time_srad.py $v 2>&1 | tail -2
done
