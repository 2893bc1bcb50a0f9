set -x
export TESSEL_BUDGET_SECS=1e9
for sp in 1 0; do for w in C2@8 C2@4; do TSL_DJ_SPLIT=$sp TRACE_OUT=gpurun_out/trace_$w_$sp.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "split=$sp" >> gpurun_out/traces.log; head -4 gpurun_out/tr.tmp >> gpurun_out/traces.log; done; done
