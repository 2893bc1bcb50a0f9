export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build2.log 2>&1
: > gpurun_out/r02o_traces.log
for w in C1 C2@3 C2@4 C2@8 C4b C5@2 C5@3 C5@4 C5@5 C3@9 C3@12 C4a@3 C4a@4; do timeout 900 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; head -1 gpurun_out/tr.tmp >> gpurun_out/r02o_traces.log; done
