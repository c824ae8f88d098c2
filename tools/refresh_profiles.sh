#!/bin/bash
# Copy one tools/gpu_round_r02.sh run (gpurun_out/) into the committed
# profiles/ under round tag $1 (default r02); files the run did not produce
# are skipped.
R=${1:-r02}
O=gpurun_out
P=profiles
cp_if() { [ -f "$1" ] && cp "$1" "$2"; }
[ -f $O/bench.json ] && tail -1 $O/bench.json > $P/${R}_bench.json
[ -f $O/bench_ref.json ] && tail -1 $O/bench_ref.json > $P/${R}_bench_reference.json
if [ -f $O/launches.csv ]; then
  cp $O/launches.csv $P/${R}_launches_bench.csv
  python tools/launch_share.py $O/launches.csv > $P/${R}_launches_bench_summary.txt
fi
if [ -f $O/launches_lud8192.csv ]; then
  cp $O/launches_lud8192.csv $P/${R}_launches_lud8192.csv
  python tools/launch_share.py $O/launches_lud8192.csv > $P/${R}_launches_lud8192_summary.txt
fi
for k in bitonic bitonic_b256 bitonic_b1024 bitonic_b4096 sb1 srad srad_fast lud_far lud_melded lud_unmelded oddeven merge nqueens nqueens_step interp; do
  if [ -s $O/ncusum_$k.json ]; then cp $O/ncusum_$k.json $P/${R}_ncu_$k.json
  elif [ -f $O/prof_$k.ncu-rep ]; then python tools/ncu_summary.py $O/prof_$k.ncu-rep > $P/${R}_ncu_$k.json; fi
done
if [ -f $O/lane_eff.csv ]; then
  cp $O/lane_eff.csv $P/${R}_lane_efficiency_ncu.csv
  python - "$R" <<'PY'
import json, subprocess, sys
r = sys.argv[1]
out = subprocess.run(["python", "tools/lane_eff.py", "gpurun_out/lane_eff.csv"], capture_output=True, text=True,
                     check=True).stdout
d = json.loads(out)
d["source"] = f"profiles/{r}_lane_efficiency_ncu.csv (tools/lane_eff.sh)"
json.dump(d, open(f"profiles/{r}_lane_efficiency.json", "w"), indent=1)
PY
fi
for t in lud srad bitonic oddeven corpus; do cp_if $O/time_$t.log $P/${R}_time_$t.txt; done
cp_if $O/trace_lud.log $P/${R}_trace_lud.txt
cp_if $O/pytest_gpu.log $P/${R}_pytest_gpu.log
cp_if $O/smoke.log $P/${R}_smoke.log
exit 0
