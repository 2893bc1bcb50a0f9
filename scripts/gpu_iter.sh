set -x
export TESSEL_BUDGET_SECS=1e9
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "disjunctive" 2>&1 | tail -15 > gpurun_out/pytest_dj.log
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for m in warp lane; do
TSL_DJ_MODE=$m TRACE_OUT=gpurun_out/trace_c2_4_$m.json timeout 600 python scripts/trace_search.py C2@4 > gpurun_out/trace_c2_4_$m.log 2>&1
done
for w in C2@3 C4b C5@2 C5@3 C3@9 C4a@3; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done
