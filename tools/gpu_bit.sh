set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "bitonic" > gpurun_out/pytest_bit.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bit.log
timeout 300 python tools/time_bitonic.py 32 64 128 256 > gpurun_out/time_bit.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bitonic_sort_reg_kernel -c 2 -o gpurun_out/prof_bitonic_reg python tools/profile_driver.py bitonic > gpurun_out/ncu_bitonic_reg.log 2>&1
