set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dj_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_seam.py -q -x -k "search or seam" --durations=5 2>&1 | tail -8 > gpurun_out/dj_tests.log
out=gpurun_out/dj_traces.log
: > $out
for v in "" "TSL_DJ_SPLIT=1" "TSL_DJ_MODE=lane"; do
  for w in C2@8 C2@4 C5@4; do
    env $v TRACE_OUT=gpurun_out/trace_dj_${w}_${v}.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none --csv -k regex:k_resolve_warp --log-file gpurun_out/dj_resolve_launches.csv python scripts/trace_search.py C2@8 > gpurun_out/dj_ncu.log 2>&1
