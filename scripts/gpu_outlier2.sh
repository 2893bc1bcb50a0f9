export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ol3_build.log 2>&1
timeout 900 python scripts/e2e_outlier.py C2@8 14 > gpurun_out/ol3.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ol3_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ol3_pytest.log
