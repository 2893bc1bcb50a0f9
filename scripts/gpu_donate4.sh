# donation at split depth 1: explored-node waste, sample size, check interval
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/don4_build.log 2>&1
: > gpurun_out/don4.log
for cfg in "TSL_SP_FIRST=2048 TSL_SP_DS_SHIFT=99" "TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99" "TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99 TSL_SP_DONATE_EVERY=16" "TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99 TSL_SP_DONATE_EVERY=256" "TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99 TSL_SP_TASK_BLOCKS=2" "TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99 TSL_SP_TASK_BLOCKS=3"; do
  echo "== $cfg" >> gpurun_out/don4.log
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0 a" "to_x4_n4 1 a" "to_m4_n3_cap6 0" "to_nn4_n2 0 a"; do
    env $cfg timeout 300 python scripts/sp_probe.py $pr >> gpurun_out/don4.log 2>&1
  done
done
for w in C2@8 C3@12 C4a@3 C4a@4 C5@4; do TSL_SP_FIRST=256 TSL_SP_DS_SHIFT=99 timeout 600 python scripts/trace_search.py $w 2>&1 | head -1 | cut -c1-300 >> gpurun_out/don4.log; done
