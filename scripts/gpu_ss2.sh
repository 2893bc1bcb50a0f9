set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out/tl2
timeout 1500 python -m pytest tests/test_gpu.py tests/test_parallel.py tests/test_seam.py tests/test_to_search.py tests/test_extension_validate.py -q -x -m gpu 2>&1 | tail -3 > gpurun_out/ss2_tests.log
out=gpurun_out/ss2_traces.log
: > $out
for w in C2@8 C2@4 C4a@3 C4a@4 C3@9 C3@12 C5@4 C5@5 C4b C5@3 C1; do
  TRACE_OUT=gpurun_out/tl2/$w.json timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "$(head -1 gpurun_out/tr.tmp)" >> $out
done
