export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/last_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/last_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/last_bench.log 2>&1
