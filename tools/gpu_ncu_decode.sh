#!/bin/bash
# GPU box: one full ncu capture of the C2 decode kernel (fused step) + launch list.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tma -s 30 -c 1 \
  -o gpurun_out/prof_decode python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_dec.out 2>&1
echo "ncu rc=$?"
