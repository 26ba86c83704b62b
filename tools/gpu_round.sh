#!/bin/bash
# GPU box: full GPU test suite, bench, ncu launch list + full captures of the hot kernels.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
MODE=${1:-all}
if [[ $MODE == all || $MODE == tests ]]; then
  timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
if [[ $MODE == all || $MODE == bench ]]; then
  timeout 600 python bench.py --steps 2000 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
  tail -3 gpurun_out/bench.err
fi
if [[ $MODE == all || $MODE == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"decode_tma|store_fast" -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_list.out 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tma -s 30 -c 1 \
    -o gpurun_out/prof_decode python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_dec.out 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:store_fast -s 0 -c 1 \
    -o gpurun_out/prof_store_big python bench.py --steps 20 --warmup 3 --no-cpu --sets 1 > gpurun_out/ncu_store.out 2>&1
fi
