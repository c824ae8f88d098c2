set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "nqueens" > gpurun_out/pytest_nq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nq.log
timeout 300 python tools/time_nqueens.py 16 > gpurun_out/time_nq.log 2>&1
timeout 300 python tools/time_nqueens.py 17 >> gpurun_out/time_nq.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nqueens_kernel -c 2 -o gpurun_out/prof_nqueens python tools/profile_driver.py nqueens > gpurun_out/ncu_nqueens.log 2>&1
