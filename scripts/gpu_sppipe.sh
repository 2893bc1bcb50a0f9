set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/spp_build.log 2>&1
out=gpurun_out/sppipe.log
: > $out
for v in "TSL_SP_PIPELINE=1" "TSL_SP_PIPELINE=0" "TSL_SP_TASK_BLOCKS=1" "TSL_SP_TASK_BLOCKS=8"; do
  echo "$v" >> $out
  for pr in "C2_8 0" "C3_12 0" "C4a_4 0"; do env $v timeout 120 python scripts/sp_probe.py $pr >> $out 2>&1; done
done
