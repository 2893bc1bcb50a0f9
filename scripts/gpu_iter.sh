set -x
timeout 600 python scripts/phase_probe.py C2@8 > gpurun_out/phase_c2_8.log 2>&1
timeout 600 python scripts/phase_probe.py C3@12 > gpurun_out/phase_c3_12.log 2>&1
