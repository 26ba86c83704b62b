#!/bin/bash
# GPU box: decode tests, bench, ncu launch list + full captures of the two hot kernels.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
timeout 600 python -m pytest tests/test_gpu_decode.py -q -s -p no:cacheprovider > gpurun_out/pytest_decode.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_decode.log
timeout 600 python bench.py --steps 2000 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_mma|store_fast" -c 300 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_list.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 20 -c 1 \
  -o gpurun_out/prof_decode python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_dec.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:store_fast -s 60 -c 1 \
  -o gpurun_out/prof_store python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_store.out 2>&1
ls -la gpurun_out
