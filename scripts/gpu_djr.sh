export TESSEL_BUDGET_SECS=1e9
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -DWDJ_COUNT_ROUNDS -o paper_2311_15269_b200/libtessel_b200.so paper_2311_15269_b200/csrc/tessel_b200.cu > gpurun_out/djr_build.log 2>&1
for w in C2@8 C2@4 C5@5; do timeout 600 python scripts/dj_rounds.py $w >> gpurun_out/djr.log 2>&1; done
