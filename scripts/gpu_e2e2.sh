export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e2_build.log 2>&1
timeout 900 python scripts/e2e_var.py C2@8 6 > gpurun_out/e2e_var2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py -x -q -k "donation or epochs or nested_runs or decide_batch or search_matches" > gpurun_out/e2e2_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e2_bench.log 2>&1
