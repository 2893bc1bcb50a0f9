set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/psp_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sp_master -s 2 -c 1 -o gpurun_out/ncu_sp_master_c28 -f python scripts/sp_probe.py C2_8 0 > gpurun_out/ncu_psp1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sp_tasks -s 1 -c 1 -o gpurun_out/ncu_sp_tasks_c28 -f python scripts/sp_probe.py C2_8 0 > gpurun_out/ncu_psp2.log 2>&1
