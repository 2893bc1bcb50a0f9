export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e_build.log 2>&1
timeout 900 python scripts/e2e_var.py C2@8 6 > gpurun_out/e2e_var.log 2>&1
