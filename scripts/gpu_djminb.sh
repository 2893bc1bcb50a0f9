# k_dj_filter occupancy variants (split filter launch) vs the fused resolve
export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/minb_build.log 2>&1
: > gpurun_out/minb.log
for v in base 3 2; do
  if [ "$v" != base ]; then cp paper_2311_15269_b200/libtessel_b200_minb$v.so paper_2311_15269_b200/libtessel_b200.so; touch paper_2311_15269_b200/libtessel_b200.so; fi
  for sp in 0 1; do
    echo "minb=$v split=$sp" >> gpurun_out/minb.log
    TSL_DJ_SPLIT=$sp timeout 600 python scripts/trace_search.py C2@8 2>&1 | head -3 | cut -c1-330 >> gpurun_out/minb.log
  done
done
