set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/djinc_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py -q -x -k "disjunctive or search or variants" --durations=5 2>&1 | tail -6 > gpurun_out/djinc_tests.log
: > gpurun_out/djinc_traces.log
for w in C2@8 C2@4 C5@4 C5@5 C3@9 C4a@4 C3@12; do
  timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/djinc_traces.log
done
