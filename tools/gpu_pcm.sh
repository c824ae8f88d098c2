set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "oddeven or pcm or abi" > gpurun_out/pytest_pcm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pcm.log
timeout 300 python tools/time_bitonic.py --oddeven 32 64 128 256 > gpurun_out/time_pcm.log 2>&1
