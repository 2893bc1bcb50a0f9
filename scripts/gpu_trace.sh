set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
for wl in ${TRACE_WORKLOADS:-C2@3 C2@4 C5@2 C3@9}; do
  timeout 600 python scripts/trace_search.py $wl 2>&1 | tail -18
done
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests/test_gpu.py -x -q --durations=25 ${PYTEST_ARGS:-} 2>&1 | tail -40
