# round-2 baseline GPU session: parity tests, smoke, bench line, per-config traces
set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt
nproc >> gpurun_out/r02a_gpu.txt; lscpu | grep "Model name" >> gpurun_out/r02a_gpu.txt
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q --durations=15 2>&1 | tail -40 > gpurun_out/r02a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a_bench.log 2>&1
: > gpurun_out/r02a_traces.log
for w in C2@4 C2@8 C4b C5@3 C5@4 C3@9 C3@12 C4a@3 C4a@4; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/r02a_traces.log; done
