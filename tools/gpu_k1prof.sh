#!/bin/bash
# GPU box: ncu captures of the tcgen05 K1 at 65536 tokens (rotated and plain launches)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
C1_TOKENS=65536 timeout 600 ncu --set full --clock-control none --import-source on -k regex:store_tc -s 2 -c 1 \
  -o gpurun_out/prof_k1_rot64k python tools/c1_store.py --ncu > /dev/null 2>&1; echo "rot rc=$?"
C1_TOKENS=65536 timeout 600 ncu --set full --clock-control none --import-source on -k regex:store_tc -s 6 -c 1 \
  -o gpurun_out/prof_k1_plain64k python tools/c1_store.py --ncu > /dev/null 2>&1; echo "plain rc=$?"
