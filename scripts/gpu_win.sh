set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/win_build.log 2>&1
out=gpurun_out/win_traces.log
: > $out
for wf in 512 128 32; do
  for w in C3@9 C3@12 C4a@3 C4a@4 C5@4 C2@8 C2@4; do
    TESSEL_PIPELINE_DEPTH=6 TESSEL_WINDOW_FIRST=$wf timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "wf=$wf $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
