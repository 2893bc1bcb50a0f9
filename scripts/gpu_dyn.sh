set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py -q -x -k "search or variants or sharded or probe" --durations=5 2>&1 | tail -6 > gpurun_out/dyn_tests.log
out=gpurun_out/dyn_traces.log
: > $out
for v in "TSL_RESOLVE_DYN=1" "TSL_RESOLVE_DYN=0"; do
  for w in C2@8 C2@4 C5@4 C5@5 C4a@3 C3@12 C4b; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
