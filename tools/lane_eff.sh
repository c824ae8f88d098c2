mkdir -p gpurun_out
timeout 1500 ncu --metrics smsp__thread_inst_executed_per_inst_executed.ratio,smsp__thread_inst_executed_pred_on_per_inst_executed.ratio,smsp__sass_average_branch_targets_threads_uniform.pct,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lane_eff.csv python tools/lane_eff_driver.py > gpurun_out/lane_eff.log 2>&1
