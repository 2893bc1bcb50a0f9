set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wst_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -q -k "repetend_probe_kernel" 2>&1 | tail -12 > gpurun_out/wst_tests.log
timeout 1200 python -m pytest tests/test_gpu.py -q -x -k "search_matches_reference or search_random or variants" --durations=6 2>&1 | tail -12 >> gpurun_out/wst_tests.log
: > gpurun_out/wst_traces.log
for w in C2@4 C3@9 C5@4 C4a@3 C4a@4 C3@12 C2@8; do
  TRACE_OUT=gpurun_out/trace_wst_$w.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/wst_traces.log
done
