# donation with the sibling-aware DFS-prefix cut: split depth sweep
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/don3_build.log 2>&1
: > gpurun_out/don3.log
for cfg in "X=0" "TSL_SP_DS_SHIFT=4" "TSL_SP_DS_SHIFT=8" "TSL_SP_DS_SHIFT=16" "TSL_SP_DS_SHIFT=99" "TSL_SP_FIRST=2048 TSL_SP_DS_SHIFT=99"; do
  echo "== $cfg" >> gpurun_out/don3.log
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0" "to_x4_n4 0 a" "to_x4_n4 1 a" "to_m4_n3_cap6 0" "to_nn4_n2 0 a" "nn4_k3 0 a"; do
    env $cfg timeout 300 python scripts/sp_probe.py $pr >> gpurun_out/don3.log 2>&1
  done
done
TSL_SP_DEBUG=1 TSL_SP_DS_SHIFT=99 python scripts/sp_probe.py C2_8 0 >> gpurun_out/don3.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "donation or nested_runs or probes" > gpurun_out/don3_pytest.log 2>&1
TSL_SP_DS_SHIFT=99 timeout 900 python -m pytest tests/test_gpu.py -x -q -k "donation or nested_runs or probes" > gpurun_out/don3_pytest99.log 2>&1
