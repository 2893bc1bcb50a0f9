set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wrg_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu.py tests/test_to_search.py -q -x -k "decide or subtree or to_ or C3_12 or C2_8 or C4a or k16" --durations=8 2>&1 | tail -15 > gpurun_out/wrg_tests.log
: > gpurun_out/wrg_sp.log
for pr in "C2_8 0" "C3_12 0" "C3_12 1" "C4a_4 0" "to_x4_n4 0"; do timeout 120 python scripts/sp_probe.py $pr >> gpurun_out/wrg_sp.log 2>&1; done
: > gpurun_out/wrg_traces.log
for w in C2@8 C3@12 C5@4 C4a@4; do
  timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/wrg_traces.log
done
