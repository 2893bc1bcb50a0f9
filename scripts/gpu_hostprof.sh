export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hp_build.log 2>&1
timeout 600 python scripts/host_profile.py C2@8 > gpurun_out/hp.log 2>&1
