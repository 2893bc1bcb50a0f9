set -x
export TESSEL_BUDGET_SECS=1e9
timeout 1500 python -m pytest tests -m gpu -x -q -k "search" --durations=6 2>&1 | tail -12 > gpurun_out/pytest_iter.log
for pl in 1 0; do for w in C3@12 C4a@3 C4a@4 C5@4 C2@8 C3@9; do TESSEL_PIPELINE_WINDOWS=$pl timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "pipe=$pl" >> gpurun_out/traces.log; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done; done
