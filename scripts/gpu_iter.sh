set -x
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "nested_runs" --durations=4 2>&1 | tail -8 > gpurun_out/pytest_iter.log
