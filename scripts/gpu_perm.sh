set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/perm_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -q -k "repetend_probe_kernel" 2>&1 | tail -6 > gpurun_out/perm_tests.log
timeout 1500 python -m pytest tests/test_gpu.py tests/test_seam.py -q -x -k "search or seam" --durations=6 2>&1 | tail -10 >> gpurun_out/perm_tests.log
: > gpurun_out/perm_traces.log
for w in C2@4 C3@9 C5@4 C4a@3 C4a@4 C3@12 C2@8; do
  timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/perm_traces.log
done
