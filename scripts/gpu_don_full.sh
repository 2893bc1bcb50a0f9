# donation defaults: full GPU suite, smoke, bench, traces
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dg_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dg_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/dg_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/dg_bench.log 2>&1
: > gpurun_out/dg_traces.log
for w in C2@8 C3@9 C3@12 C4a@3 C4a@4 C5@4 C5@5; do timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/dg_traces.log; done
