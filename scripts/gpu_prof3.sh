set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_r02g_verify_c4a3 -f python scripts/trace_search.py C4a@3 > gpurun_out/prof3a.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_root --launch-skip 150 --launch-count 1 -o gpurun_out/ncu_r02g_root_c5_5 -f python scripts/trace_search.py C5@5 > gpurun_out/prof3b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02g_metrics_c5_5.csv python scripts/trace_search.py C5@5 > gpurun_out/prof3c.log 2>&1
