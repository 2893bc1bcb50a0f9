export TESSEL_BUDGET_SECS=1e9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r02m_bench.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02m_bench2.log 2>&1
