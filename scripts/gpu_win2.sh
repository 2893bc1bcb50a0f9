# donation window sweep (leftmost open tasks only) + e2e breakdown
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/win_build.log 2>&1
: > gpurun_out/win.log
for wv in -1 0 1 4 16; do
  echo "== window $wv" >> gpurun_out/win.log
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0" "to_m4_n3_cap6 0"; do
    TSL_SP_DONATE_WINDOW=$wv timeout 300 python scripts/sp_probe.py $pr >> gpurun_out/win.log 2>&1
  done
done
timeout 600 python scripts/e2e_probe.py C2@8 3 > gpurun_out/e2e_probe.log 2>&1
