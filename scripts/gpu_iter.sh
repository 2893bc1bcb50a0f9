set -x
export TESSEL_BUDGET_SECS=1e9
for w in C2@5 C2@6 C2@8; do timeout 900 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -3 gpurun_out/tr.tmp >> gpurun_out/traces_big.log; done
