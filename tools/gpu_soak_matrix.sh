#!/bin/bash
# GPU box: the serving-step soak (tools/soak_step.py) over the step-ring modes x geometries
# (G 2 / 4 / 8, page size 16 / 32, KEYS_ONLY, BF16 pool, learned R) -> gpurun_out/soak_matrix.txt
cd "${GRAFT_REPO_ROOT:-.}"
out=gpurun_out/soak_matrix.txt
: > $out
N=${SOAK_N:-4000}
for mode in 2 1 0; do
  for cfg in "" "SOAK_G=8" "SOAK_G=2" "SOAK_P=32" "SOAK_KEYS_ONLY=1" "SOAK_BF16=1" "SOAK_LEARNED=1" "SOAK_G=8 SOAK_P=32 SOAK_KEYS_ONLY=1"; do
    line=$(env KVR_STEP_DIRECT=$mode SOAK_EVERY=50 $cfg timeout 300 python tools/soak_step.py $N 2>&1 | tail -1)
    echo "mode $mode [${cfg:-default}] $line" >> $out
  done
done
cat $out
