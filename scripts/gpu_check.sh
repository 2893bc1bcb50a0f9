set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 1 --warmup 1 --workload C2@3 --no-cpu-baseline 2>&1 | tail -5
