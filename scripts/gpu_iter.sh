set -x
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "decide_batch or nested_runs" 2>&1 | tail -3 > gpurun_out/pytest_iter.log
for f in "C3_12 0" "C3_12 1" "to_v4_n6_cap4 0" "to_x4_n4 0" "C4a_4 0"; do timeout 300 python scripts/sp_probe.py $f >> gpurun_out/sp_probe.log 2>&1; done
timeout 600 python scripts/phase_probe.py C2@8 2>&1 | head -1 >> gpurun_out/phase.log
