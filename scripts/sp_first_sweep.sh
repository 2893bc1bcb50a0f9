# SP-DFS first-pass sweep on the long completion probes (timings only)
export TESSEL_BUDGET_SECS=1e9
out=gpurun_out/sp_first.log
: > $out
for first in 16384 1024; do
  echo "batch_first=$first" >> $out
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0"; do
    TSL_SP_BATCH_FIRST=$first timeout 120 python scripts/sp_probe.py $pr >> $out 2>&1
  done
  for w in C2@8 C3@12; do TSL_SP_BATCH_FIRST=$first timeout 300 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> $out; done
done
