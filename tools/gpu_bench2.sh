#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:store_fast -s 0 -c 1 \
  -o gpurun_out/prof_store_big python bench.py --steps 20 --warmup 3 --no-cpu --sets 1 > gpurun_out/ncu_store.out 2>&1
