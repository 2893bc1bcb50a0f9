set -x
export TESSEL_BUDGET_SECS=1e9
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_verify_c39 -f python scripts/trace_search.py C3@9 > gpurun_out/ncu_verify.log 2>&1
