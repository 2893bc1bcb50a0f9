set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/exs_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py -q -x -k "search or variants or sharded" --durations=5 2>&1 | tail -6 > gpurun_out/exs_tests.log
out=gpurun_out/exs_traces.log
: > $out
for v in "TSL_EXACT_STAGE=2048" "TSL_EXACT_STAGE=256" "TSL_EXACT_STAGE=100000000"; do
  for w in C3@9 C3@12 C4a@3 C4a@4 C5@4 C5@5 C2@8 C2@4; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
