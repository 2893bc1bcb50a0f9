set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wrr_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -q -k "repetend_probe_kernel" 2>&1 | tail -15 > gpurun_out/wrr_probe.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int_peak scripts/int_peak.cu && /tmp/int_peak > gpurun_out/int_peak.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_wrr_verify_c4a3 -f python scripts/trace_search.py C4a@3 > gpurun_out/ncu_wrr1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_verify_warp --launch-count 1 -o gpurun_out/ncu_wrr_verify_c39 -f python scripts/trace_search.py C3@9 > gpurun_out/ncu_wrr2.log 2>&1
