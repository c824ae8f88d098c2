#!/bin/bash
# Copy one tools/gpu_round7.sh run (gpurun_out/) into the committed profiles/
# (round tag $1, default r01) and summarise the ncu reports.
set -e
R=${1:-r01}
O=gpurun_out
P=profiles
tail -1 $O/bench.json > $P/${R}_bench.json
tail -1 $O/bench_ref.json > $P/${R}_bench_reference.json
cp $O/launches.csv $P/${R}_launches_bench.csv
python tools/launch_share.py $O/launches.csv > $P/${R}_launches_bench_summary.txt
cp $O/launches_lud8192.csv $P/${R}_launches_lud8192.csv
python tools/launch_share.py $O/launches_lud8192.csv > $P/${R}_launches_lud8192_summary.txt
for k in bitonic srad srad_fast lud_far lud_melded lud_unmelded oddeven merge nqueens; do
  if [ -f $O/ncusum_$k.json ]; then cp $O/ncusum_$k.json $P/${R}_ncu_$k.json
  else python tools/ncu_summary.py $O/prof_$k.ncu-rep > $P/${R}_ncu_$k.json; fi
done
cp $O/lane_eff.csv $P/${R}_lane_efficiency_ncu.csv
python tools/lane_eff.py $O/lane_eff.csv > /dev/null
python - "$R" <<'PY'
import json, subprocess, sys
r = sys.argv[1]
out = subprocess.run(["python", "tools/lane_eff.py", "gpurun_out/lane_eff.csv"], capture_output=True, text=True,
                     check=True).stdout
d = json.loads(out)
d["source"] = f"profiles/{r}_lane_efficiency_ncu.csv (tools/lane_eff.sh)"
json.dump(d, open(f"profiles/{r}_lane_efficiency.json", "w"), indent=1)
PY
cp $O/time_lud.log $P/${R}_time_lud.txt
cp $O/time_srad.log $P/${R}_time_srad.txt
cp $O/time_bitonic.log $P/${R}_time_bitonic_buckets.txt
cp $O/time_oddeven.log $P/${R}_time_oddeven.txt
cp $O/time_corpus.log $P/${R}_time_corpus.txt
cp $O/trace_lud.log $P/${R}_trace_lud.txt
cp $O/pytest_gpu.log $P/${R}_pytest_gpu.log
