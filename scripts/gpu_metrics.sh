set -x
python -c "import __graft_entry__ as g; g.build()"
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_lsu.sum
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/metrics_c2_4.csv python scripts/trace_search.py C2@4 > gpurun_out/metrics_run.log 2>&1
tail -3 gpurun_out/metrics_run.log
for wl in C4b C5@3 C3@12 C4a@3; do timeout 900 python scripts/trace_search.py $wl 2>&1 | head -1; done
