# generic GPU session: smoke, selected pytest, traces, benches (env-configurable)
set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
if [ -n "${PYTEST_K:-}" ]; then
  timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests/test_gpu.py -q --durations=15 -k "$PYTEST_K" ${PYTEST_ARGS:-} 2>&1 | tail -40
fi
for wl in ${TRACE_WORKLOADS:-}; do
  timeout 600 python scripts/trace_search.py $wl 2>&1 | tail -${TRACE_LINES:-8}
done
for wl in ${BENCH_WORKLOADS:-}; do
  timeout 900 python bench.py --steps ${BENCH_STEPS:-1} --warmup ${BENCH_WARMUP:-1} --workload $wl ${BENCH_ARGS:---no-cpu-baseline} 2>&1 | tail -2
done
