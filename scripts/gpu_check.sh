# One GPU session: build, smoke, GPU tests, then short bench runs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests/test_gpu.py -x -q ${PYTEST_ARGS:-} 2>&1 | tail -30
for wl in ${BENCH_WORKLOADS:-C2@3 C2@4}; do
  timeout 900 python bench.py --steps 1 --warmup 1 --workload $wl --no-cpu-baseline 2>&1 | tail -3
done
