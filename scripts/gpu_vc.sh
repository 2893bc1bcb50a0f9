set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py -q -x -k "search or variants or sharded or probe or verify" 2>&1 | tail -3 > gpurun_out/vc_tests.log
out=gpurun_out/vc_traces.log
: > $out
for v in "TSL_VERIFY_CANCEL=auto" "TSL_VERIFY_CANCEL=1" "TESSEL_SPEC_STAGE=4096" "TESSEL_SPEC_STAGE=1024" "TESSEL_SPEC_STAGE=65536"; do
  for w in C4a@3 C4a@4 C3@9 C3@12 C5@4 C5@5 C2@8; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
