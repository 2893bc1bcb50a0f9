export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p_build.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_resolve_warp -s 110 -c 1 -o gpurun_out/r02p_ncu_resolve_c2_8 -f python scripts/trace_search.py C2@8 > gpurun_out/r02p_ncu_resolve.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_root -s 150 -c 1 -o gpurun_out/r02p_ncu_root_c2_8 -f python scripts/trace_search.py C2@8 > gpurun_out/r02p_ncu_root.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sp_tasks -s 1 -c 1 -o gpurun_out/r02p_ncu_sptasks_c2_8 -f python scripts/trace_search.py C2@8 > gpurun_out/r02p_ncu_sptasks.log 2>&1
