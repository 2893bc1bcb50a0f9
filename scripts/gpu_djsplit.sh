# split disjunctive filter (k_dj_filter, 32 warps/SM, dynamic handout) vs the fused resolve
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/djs_build.log 2>&1
: > gpurun_out/djs.log
for m in 0 1; do for w in C2@8 C2@4 C5@5 C4a@3 C3@9; do
  echo "split=$m" >> gpurun_out/djs.log
  TSL_DJ_SPLIT=$m timeout 600 python scripts/trace_search.py $w 2>&1 | head -4 | cut -c1-600 >> gpurun_out/djs.log
done; done
