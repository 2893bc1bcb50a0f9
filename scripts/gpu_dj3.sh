export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dj3_build.log 2>&1
: > gpurun_out/dj3.log
for o in 0 1 2 3 0; do for w in C2@8 C5@5; do echo "opt=$o" >> gpurun_out/dj3.log; TSL_DJ_OPT=$o timeout 600 python scripts/trace_search.py $w 2>&1 | head -2 | cut -c1-420 >> gpurun_out/dj3.log; done; done
