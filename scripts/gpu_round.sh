# full GPU round: parity tests, smoke, bench line, ncu launch lists of the bench workload
set -x
export TESSEL_BUDGET_SECS=1e9
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_lsu.sum
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/metrics_c2_8.csv python scripts/trace_search.py C2@8 > gpurun_out/metrics_run.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
for w in C1 C2@3 C2@4 C2@8 C4b C5@2 C5@3 C3@9 C3@12 C4a@3 C4a@4; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done
