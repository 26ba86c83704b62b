#!/bin/bash
# GPU box: full bench (no CPU leg) under env-knob variants: VARIANTS="A=1,B=0 ..."
cd "${GRAFT_REPO_ROOT:-.}"
for v in ${VARIANTS:-default}; do
  echo "#### $v"
  env $(echo "$v" | tr ',' ' ' | sed 's/default//') timeout 900 python bench.py --steps 500 --no-cpu > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  grep "^\[bench\]" gpurun_out/bench_$v.err | head -40
done
