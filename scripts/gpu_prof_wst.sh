set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wst_build.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_wst_verify_c4a3 -f python scripts/trace_search.py C4a@3 > gpurun_out/ncu_wst1.log 2>&1
