export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ol_build.log 2>&1
timeout 900 python scripts/e2e_outlier.py C2@8 14 > gpurun_out/ol.log 2>&1
