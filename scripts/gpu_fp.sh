set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py tests/test_to_search.py -q -x -m gpu 2>&1 | tail -3 > gpurun_out/fp2_tests.log
out=gpurun_out/fp2_traces.log
: > $out
for v in "TSL_LIB_VARIANT=" "TSL_LIB_VARIANT=base" "TSL_LIB_VARIANT=fp2"; do
  for w in C4a@3 C4a@4 C3@9 C3@12 C5@4 C5@5; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
