export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/spc_build.log 2>&1
: > gpurun_out/spc.log
for f in C3_9 C3_12 C4a_3 C4a_4 C5_4; do timeout 600 python scripts/sp_capped.py $f 6 >> gpurun_out/spc.log 2>&1; done
