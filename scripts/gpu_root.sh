set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out/tl3
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py tests/test_to_search.py -q -x -m gpu 2>&1 | tail -3 > gpurun_out/root_tests.log
TSL_ROOT_DEVS=serial timeout 900 python -m pytest tests/test_gpu.py -q -x -m gpu -k "search" 2>&1 | tail -3 >> gpurun_out/root_tests.log
out=gpurun_out/root_traces.log
: > $out
for v in "TSL_LIB_VARIANT=" "TSL_LIB_VARIANT=base" "TSL_ROOT_DEVS=serial"; do
  for w in C5@5 C2@8 C5@4 C3@9 C4a@3 C2@4 C4b; do
    env $v TRACE_OUT=gpurun_out/tl3/$w.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_root --csv --log-file gpurun_out/r02h_root_c5_5.csv python scripts/trace_search.py C5@5 > gpurun_out/prof_root.log 2>&1
TSL_LIB_VARIANT=base timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_root --csv --log-file gpurun_out/r02h_root_c5_5_base.csv python scripts/trace_search.py C5@5 > gpurun_out/prof_root_base.log 2>&1
