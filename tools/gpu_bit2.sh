set -x
mkdir -p gpurun_out
timeout 300 python tools/time_bitonic.py 64 128 > gpurun_out/time_bit_nopf.log 2>&1
DARM_BITONIC_PF=1 timeout 300 python tools/time_bitonic.py 64 128 > gpurun_out/time_bit_pf.log 2>&1
DARM_BITONIC_PF=1 timeout 900 python -m pytest tests -q -m gpu -x -k "bitonic" > gpurun_out/pytest_bit_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bit_pf.log
