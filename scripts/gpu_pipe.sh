set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pipe_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu.py -q -x -k "search_matches_reference or variants" --durations=5 2>&1 | tail -8 > gpurun_out/pipe_tests.log
out=gpurun_out/pipe_traces.log
: > $out
for d in 3 6; do
  for w in C3@9 C3@12 C4a@3 C4a@4 C5@4 C2@8; do
    TESSEL_PIPELINE_DEPTH=$d timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "depth=$d $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
