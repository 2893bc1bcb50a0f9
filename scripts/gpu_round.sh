set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
for w in C1 C2@3 C4b C5@2 C5@3 C3@9; do timeout 600 python scripts/trace_search.py $w 2>&1 | head -3 >> gpurun_out/traces.log; done
