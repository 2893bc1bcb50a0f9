set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sptb_build.log 2>&1
out=gpurun_out/sptb.log
: > $out
for tb in 4 3 2; do
  echo "tb=$tb" >> $out
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0"; do TSL_SP_TASK_BLOCKS=$tb timeout 120 python scripts/sp_probe.py $pr >> $out 2>&1; done
  for w in C2@8 C3@12 C5@4; do TSL_SP_TASK_BLOCKS=$tb timeout 300 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> $out; done
done
timeout 900 python -m pytest tests/test_gpu.py tests/test_to_search.py -q -x -k "subtree or decide_batch or to_" 2>&1 | tail -3 >> $out
