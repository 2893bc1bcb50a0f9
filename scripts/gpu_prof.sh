set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sp_tasks --launch-count 1 -o gpurun_out/ncu_sptasks -f python scripts/sp_probe.py to_x4_n4 0 > gpurun_out/ncu_sptasks.log 2>&1
