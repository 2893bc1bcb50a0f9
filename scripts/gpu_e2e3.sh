export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e3_build.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e3_bench.log 2>&1
timeout 900 python scripts/e2e_var.py C2@8 3 > gpurun_out/e2e3_var.log 2>&1
