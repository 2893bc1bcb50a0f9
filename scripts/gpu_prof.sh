set -x
export TESSEL_BUDGET_SECS=1e9
TRACE_OUT=gpurun_out/trace_c2_4.json timeout 600 python scripts/trace_search.py C2@4 > gpurun_out/trace_c2_4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_probe --launch-skip 30 --launch-count 1 -o gpurun_out/ncu_probe -f python scripts/trace_search.py C2@3 > gpurun_out/ncu_probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resolve_warp --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_resolve -f python scripts/trace_search.py C2@3 > gpurun_out/ncu_resolve.log 2>&1
