mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "bitonic or keys_per_thread" > gpurun_out/pytest_bit.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bit.log
timeout 600 python tools/time_bitonic.py ${BUCKETS:-64 256 1024 4096} > gpurun_out/time_bitonic.log 2>&1
