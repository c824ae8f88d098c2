# One GPU session: the GPU test suite, then the timing tools given as arguments
# (each `name:command`), logs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1800 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
for spec in "$@"; do
  name="${spec%%:*}"; cmd="${spec#*:}"
  timeout 900 bash -c "$cmd" > "gpurun_out/$name.log" 2>&1
  echo "$name rc=$?"; tail -40 "gpurun_out/$name.log"
done
