export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02o_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02o_launches_bench.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --workload C5@5 --no-cpu-baseline > gpurun_out/r02o_bench_c5_5.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02o_bench_ref.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1
