# compile-time variants of the register-resident DFS, timed on the same box
set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/var_build.log 2>&1
cd paper_2311_15269_b200
for v in "r0d0 -DWRR_RELAX=0 -DWRR_DEVLIST=0" "r0d1 -DWRR_RELAX=0 -DWRR_DEVLIST=1" "r1d0 -DWRR_RELAX=1 -DWRR_DEVLIST=0"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared $2 $3 -o libtessel_b200_$1.so csrc/tessel_b200.cu >> ../gpurun_out/var_build.log 2>&1 &
done
wait
cd ..
out=gpurun_out/variants.log
: > $out
for v in r0d0 r0d1 r1d0; do
  for w in C3@9 C4a@3 C5@4 C2@8; do
    TSL_LIB_VARIANT=$v timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1; echo "$v $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
TSL_LIB_VARIANT=r0d1 timeout 900 python -m pytest tests/test_gpu.py -q -x -k "repetend_probe_kernel" 2>&1 | tail -3 >> $out
TSL_LIB_VARIANT=r1d0 timeout 900 python -m pytest tests/test_gpu.py -q -x -k "repetend_probe_kernel" 2>&1 | tail -3 >> $out
