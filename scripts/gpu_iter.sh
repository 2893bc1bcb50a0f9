set -x
export TESSEL_BUDGET_SECS=1e9
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "decide_batch_matches" --durations=20 2>&1 | tail -30 > gpurun_out/pytest_sp.log
for w in C3@9 C3@12 C4a@3; do timeout 300 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done
