set -x
timeout 900 python -m pytest tests/test_extension_validate.py -x -q --durations=5 2>&1 | tail -25 > gpurun_out/pytest_iter.log
