# DJ filter with per-item chunk masks and precomputed dependency lags
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dj2_build.log 2>&1
: > gpurun_out/dj2.log
for w in C2@8 C2@4 C5@5 C3@9 C4a@3; do timeout 600 python scripts/trace_search.py $w 2>&1 | head -2 | cut -c1-500 >> gpurun_out/dj2.log; done
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "disjunctive or search" > gpurun_out/dj2_pytest.log 2>&1
