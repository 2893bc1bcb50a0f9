export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/clk_build.log 2>&1
for per in 0 1.0 0.2; do BENCH_CLOCK_PERIOD=$per timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/clk_$per.log 2>&1; done
