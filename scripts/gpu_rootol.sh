set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rol_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py -q -x -k "search" --durations=5 2>&1 | tail -6 > gpurun_out/rol_tests.log
out=gpurun_out/rol_traces.log
: > $out
for v in "TSL_ROOT_DISJ=1" "TSL_ROOT_DISJ=0"; do
  for w in C2@8 C2@4 C5@4 C5@5 C3@9 C4a@4 C3@12; do
    env $v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "[$v] $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
