#!/bin/bash
# One gpurun call (round 2): GPU tests, smoke, bench (+ reference arm), launch
# list, ncu captures (summarised on the box: gpurun copies back <= 64 MiB), the
# lane-efficiency sweep and the per-kernel timing tools.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
export DARM_PEER_TIMEOUT_S=60
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-kernel > gpurun_out/bench_under_ncu.log 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:bitonic_sort -c 8 -o gpurun_out/prof_bitonic python tools/profile_driver.py bitonic > gpurun_out/ncu_bitonic.log 2>&1
for b in 256 1024 4096; do
  timeout 900 $N -k regex:bitonic_sort -c 8 -o gpurun_out/prof_bitonic_b$b python tools/profile_driver.py bitonic $b > gpurun_out/ncu_bitonic_b$b.log 2>&1
done
timeout 600 $N -k regex:corpus_lanes -c 3 -o gpurun_out/prof_sb1 python tools/profile_driver.py sb1 > gpurun_out/ncu_sb1.log 2>&1
timeout 600 $N -k regex:srad_sweep -c 4 -o gpurun_out/prof_srad python tools/profile_driver.py srad > gpurun_out/ncu_srad.log 2>&1
timeout 600 $N -k regex:oddeven_sort -c 4 -o gpurun_out/prof_oddeven python tools/profile_driver.py oddeven > gpurun_out/ncu_oddeven.log 2>&1
timeout 600 $N -k regex:merge_sort -c 4 -o gpurun_out/prof_merge python tools/profile_driver.py merge 1048576 > gpurun_out/ncu_merge.log 2>&1
timeout 600 $N -k regex:"nqueens_kernel" -c 2 -o gpurun_out/prof_nqueens python tools/profile_driver.py nqueens > gpurun_out/ncu_nqueens.log 2>&1
timeout 600 $N -k regex:nqueens_step -c 2 -o gpurun_out/prof_nqueens_step python tools/profile_driver.py nqueens_step > gpurun_out/ncu_nqueens_step.log 2>&1
timeout 600 $N -k regex:ir_interp -c 1 -o gpurun_out/prof_interp python tools/profile_driver.py interp > gpurun_out/ncu_interp.log 2>&1
timeout 600 $N -k regex:lud_far -s 21 -c 1 -o gpurun_out/prof_lud_far python tools/profile_driver.py lud > gpurun_out/ncu_lud_far.log 2>&1
timeout 600 $N -k regex:lud_panel -s 100 -c 1 -o gpurun_out/prof_lud_unmelded python tools/profile_driver.py lud > gpurun_out/ncu_lud_u.log 2>&1
timeout 600 $N -k regex:lud_panel -s 612 -c 1 -o gpurun_out/prof_lud_melded python tools/profile_driver.py lud > gpurun_out/ncu_lud_m.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lud8192.csv python tools/profile_driver.py lud > gpurun_out/ncu_lud_list.log 2>&1
bash tools/lane_eff.sh
timeout 300 python tools/time_srad.py > gpurun_out/time_srad.log 2>&1
timeout 600 python tools/time_bitonic.py 64 256 1024 4096 > gpurun_out/time_bitonic.log 2>&1
timeout 600 python tools/time_bitonic.py --oddeven 64 256 > gpurun_out/time_oddeven.log 2>&1
timeout 300 python tools/time_corpus.py > gpurun_out/time_corpus.log 2>&1
timeout 300 python tools/time_lud.py 2048 4096 8192 > gpurun_out/time_lud.log 2>&1
timeout 300 python tools/trace_lud.py > gpurun_out/trace_lud.log 2>&1; python tools/trace_lud.py steps >> gpurun_out/trace_lud.log 2>&1
for k in bitonic bitonic_b256 bitonic_b1024 bitonic_b4096 sb1 srad srad_fast lud_far lud_melded lud_unmelded oddeven merge nqueens nqueens_step interp; do
  python tools/ncu_summary.py gpurun_out/prof_$k.ncu-rep > gpurun_out/ncusum_$k.json
  case " ${KEEP_REPS:-lud_far srad_fast} " in *" $k "*) ;; *) rm -f gpurun_out/prof_$k.ncu-rep ;; esac
done
ls -la gpurun_out
