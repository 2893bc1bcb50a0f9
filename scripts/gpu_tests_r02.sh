# round-2 parity session: the new GPU tests first, then the whole GPU suite
set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seam.py tests/test_extension_validate.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02b_new.log
timeout 1200 python -m pytest tests/test_gpu.py -m gpu -x -q -k "C5_4 or eager or gate" --durations=10 2>&1 | tail -25 >> gpurun_out/r02b_new.log
timeout 1800 python -m pytest tests -m "gpu and not slow" -q --durations=10 2>&1 | tail -25 > gpurun_out/r02b_pytest_gpu.log
