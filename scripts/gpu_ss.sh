set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py -q -x -k "search or variants or sharded" 2>&1 | tail -3 > gpurun_out/ss_tests.log
out=gpurun_out/ss_traces.log
: > $out
for v in "TESSEL_SPEC_SMALL_NDEF=4096" "TESSEL_SPEC_SMALL_NDEF=512" "TESSEL_SPEC_SMALL_NDEF=32768" "TESSEL_SPEC_SMALL=4096" "TESSEL_SPEC_SMALL=256"; do
  for w in C2@8 C2@4 C4a@3 C4a@4 C3@9 C3@12 C5@4 C5@5 C4b C5@3; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
