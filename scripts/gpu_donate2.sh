# donation tuning: split depth / sample size sweep on the long golden probes
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/don2_build.log 2>&1
: > gpurun_out/don2.log
TSL_SP_DEBUG=1 python scripts/sp_probe.py C2_8 0 >> gpurun_out/don2.log 2>&1
TSL_SP_DEBUG=1 python scripts/sp_probe.py to_x4_n4 0 >> gpurun_out/don2.log 2>&1
for cfg in "X=0" "TSL_SP_DS_SHIFT=2" "TSL_SP_DS_SHIFT=4" "TSL_SP_FIRST=2048" "TSL_SP_FIRST=2048 TSL_SP_DS_SHIFT=3" "TSL_SP_PAUSE=262144" "TSL_SP_DONATE_EVERY=16"; do
  echo "== $cfg" >> gpurun_out/don2.log
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0"; do
    env $cfg timeout 300 python scripts/sp_probe.py $pr >> gpurun_out/don2.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "donation or nested_runs or probes" > gpurun_out/don2_pytest.log 2>&1
