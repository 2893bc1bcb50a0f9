# SP-DFS knob sweep on long completion probes (one GPU; timings only)
export TESSEL_BUDGET_SECS=1e9
out=gpurun_out/sp_sweep.log
: > $out
for pr in "C2_8 0" "C3_12 0" "to_x4_n4 0"; do
  for pause in 16384 65536 262144; do
    for tn in 65536 262144; do
      echo "pause=$pause task_nodes=$tn" >> $out
      TSL_SP_PAUSE=$pause TSL_SP_TASK_NODES=$tn timeout 120 python scripts/sp_probe.py $pr >> $out 2>&1
    done
  done
done
