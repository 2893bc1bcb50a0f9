# donation window x check interval
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/win3_build.log 2>&1
: > gpurun_out/win3.log
for cfg in "TSL_SP_DONATE_WINDOW=4" "TSL_SP_DONATE_WINDOW=2" "TSL_SP_DONATE_WINDOW=8" "TSL_SP_DONATE_WINDOW=4 TSL_SP_DONATE_EVERY=16" "TSL_SP_DONATE_WINDOW=4 TSL_SP_DONATE_EVERY=256" "TSL_SP_DONATE_WINDOW=4 TSL_SP_FIRST=1024"; do
  echo "== $cfg" >> gpurun_out/win3.log
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0" "to_m4_n3_cap6 0"; do
    env $cfg timeout 300 python scripts/sp_probe.py $pr >> gpurun_out/win3.log 2>&1
  done
done
