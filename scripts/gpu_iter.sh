set -x
export TESSEL_BUDGET_SECS=1e9
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q --durations=8 2>&1 | tail -15 > gpurun_out/pytest_iter.log
: > gpurun_out/traces.log
for w in C3@12 C4a@3 C4a@4 C5@4 C2@8 C3@9; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/traces.log; done
: > gpurun_out/sp_probe.log
for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0"; do timeout 120 python scripts/sp_probe.py $pr >> gpurun_out/sp_probe.log 2>&1; done
