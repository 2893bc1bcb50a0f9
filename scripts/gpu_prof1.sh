set -x
python -c "import __graft_entry__ as g; g.build()"
python scripts/profile_probe.py C4a_3 capped 100000 1
python scripts/profile_probe.py C4a_3 capped 100000 64
python scripts/profile_probe.py C3_12 completion 100000 1
TSL_DFS_MODE=thread python scripts/profile_probe.py C4a_3 capped 20000 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decide_warp -s 1 -c 1 -o gpurun_out/prof_wrx_c4a python scripts/profile_probe.py C4a_3 capped 20000 1 > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decide_warp -s 1 -c 1 -o gpurun_out/prof_wrx_c312 python scripts/profile_probe.py C3_12 completion 20000 1 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_4.csv python scripts/trace_search.py C2@4 > gpurun_out/ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_probe -s 40 -c 2 -o gpurun_out/prof_probe_c24 python scripts/trace_search.py C2@4 > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
