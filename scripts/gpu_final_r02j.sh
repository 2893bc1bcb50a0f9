# round-2 final evidence: full GPU suite, smoke, ncu instruction counts of the
# bench workload (-> inst_counts.json for the roofline), the bench line, the
# ncu launch list of the bench command, full ncu captures of the dominant
# kernels (the heaviest k_resolve_warp level, the donation k_sp_tasks launch),
# per-config traces, the C5@5 bench line
set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02j_gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -40 > gpurun_out/r02j_pytest_gpu.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_lsu.sum
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02j_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02j_launches_bench.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sp_tasks -s 1 -c 1 -o gpurun_out/r02j_ncu_sptasks_c2_8 -f python scripts/trace_search.py C2@8 > gpurun_out/r02j_ncu_sptasks.log 2>&1
: > gpurun_out/r02j_traces.log
for w in C1 C2@3 C2@4 C2@8 C4b C5@2 C5@3 C5@4 C5@5 C3@9 C3@12 C4a@3 C4a@4; do timeout 900 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/r02j_traces.log; done
timeout 900 python bench.py --steps 3 --warmup 3 --workload C5@5 --no-cpu-baseline > gpurun_out/r02j_bench_c5_5.log 2>&1
