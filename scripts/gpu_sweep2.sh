set -x
export TESSEL_BUDGET_SECS=1e9
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sw2_build.log 2>&1
out=gpurun_out/sweep2.log
: > $out
for cfg in "200000 default" "0 default" "200000 4096" "0 4096" "0 1024"; do
  set -- $cfg
  for w in C3@9 C3@12 C4a@3 C4a@4 C5@4 C2@8 C2@4; do
    if [ "$2" = "default" ]; then
      TESSEL_DJ_BUDGET=$1 timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1
    else
      TESSEL_DJ_BUDGET=$1 TESSEL_SPEC_STAGE=$2 timeout 600 python scripts/trace_search.py $w > gpurun_out/tr.tmp 2>&1
    fi
    echo "dj=$1 stage=$2 $(head -1 gpurun_out/tr.tmp)" >> $out
  done
done
