# ncu --set full captures of the latency-bound DFS kernels (source-correlated)
set -x
export TESSEL_BUDGET_SECS=1e9
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_resolve_warp --launch-skip 87 --launch-count 1 -o gpurun_out/ncu_resolve_big -f python scripts/trace_search.py C2@4 > gpurun_out/ncu_resolve_big.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_root --launch-skip 60 --launch-count 1 -o gpurun_out/ncu_root -f python scripts/trace_search.py C2@4 > gpurun_out/ncu_root.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_verify_c39 -f python scripts/trace_search.py C3@9 > gpurun_out/ncu_verify.log 2>&1
