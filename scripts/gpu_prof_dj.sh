# the heavy k_resolve_warp launches of C2@8 (deferred probes at N_R = 5): trace tops + one full ncu capture
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pdj_build.log 2>&1
timeout 600 python scripts/trace_search.py C2@8 > gpurun_out/pdj_trace.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_resolve_warp -s 110 -c 1 -o gpurun_out/pdj_resolve110 -f python scripts/trace_search.py C2@8 > gpurun_out/pdj_ncu.log 2>&1
