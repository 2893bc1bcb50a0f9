# time-to-optimal on the box, both arms (reference CPU jobs=1 / jobs=nproc, B200)
set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tto_build.log 2>&1
nproc > gpurun_out/r02_ref_tto_host.txt; lscpu | grep "Model name" >> gpurun_out/r02_ref_tto_host.txt
timeout 3000 python scripts/ref_tto.py C1 C2@3 C5@2 C3@9 C4b C3@12 C4a@3 C4a@4 C2@4 C5@3 > gpurun_out/r02_ref_tto.jsonl 2> gpurun_out/r02_ref_tto.err
