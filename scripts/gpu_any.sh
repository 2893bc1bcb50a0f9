export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/any_build.log 2>&1
: > gpurun_out/any.log
for f in C3_9 C4a_3; do timeout 900 python scripts/sp_capped.py $f 6 >> gpurun_out/any.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu.py -x -q -k "donation or epochs or nested_runs or decide_batch" > gpurun_out/any_pytest.log 2>&1
