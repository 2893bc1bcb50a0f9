export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -15 > gpurun_out/r02l_pytest_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02l_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02l_launches_bench.log 2>&1
: > gpurun_out/r02l_traces.log
for w in C2@8 C3@9 C3@12 C4a@3 C4a@4 C5@4 C5@5; do timeout 900 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/r02l_traces.log; done
