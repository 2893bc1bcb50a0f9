set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out/tl
for w in C4a@3 C4a@4 C3@9 C3@12 C5@4; do
  TRACE_OUT=gpurun_out/tl/$w.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tl/$w.log 2>&1
done
