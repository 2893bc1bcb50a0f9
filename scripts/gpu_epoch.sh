export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ep_build.log 2>&1
: > gpurun_out/ep.log
for f in C3_9 C4a_3 C3_12; do timeout 600 python scripts/sp_capped.py $f 6 >> gpurun_out/ep.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "donation or epochs or nested_runs" > gpurun_out/ep_pytest.log 2>&1
