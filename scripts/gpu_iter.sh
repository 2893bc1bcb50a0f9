set -x
export TESSEL_BUDGET_SECS=1e9
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "search_matches_reference or decide_batch" 2>&1 | tail -3 > gpurun_out/pytest_iter.log
for w in C2@8 C2@4 C5@3 C3@12 C4a@3; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done
