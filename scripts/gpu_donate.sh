# dynamic donation in SP task launches: exactness on every long golden probe,
# then per-probe timings with donation on / off and the C2@8 / C3@12 traces
set -x
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/don_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "donation or nested_runs" 2>&1 | tail -15
for mode in 1 0; do
  for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0" "to_x4_n4 1"; do
    TSL_SP_DONATE=$mode timeout 300 python scripts/sp_probe.py $pr
  done
done
for w in C2@8 C3@12 C4a@3; do timeout 600 python scripts/trace_search.py $w 2>&1 | head -1 | cut -c1-400; done
