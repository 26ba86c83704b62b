#!/bin/bash
# GPU box: ncu launch list of a short bench run + full captures of the hot kernels.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"decode_tma|decode_merge|store_mma|store_tc|dequant_cells|stage_copy|rows_matmul|decode_bf16" -c 800 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 --quick > gpurun_out/ncu_list.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tma -s 30 -c 1 \
  -o gpurun_out/prof_decode python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 --quick > gpurun_out/ncu_dec.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:store_mma -s 2 -c 1 \
  -o gpurun_out/prof_store python tools/c1_store.py --ncu > gpurun_out/ncu_store.out 2>&1
C1_TOKENS=65536 timeout 900 ncu --set full --clock-control none --import-source on -k regex:store_tc -s 2 -c 1 \
  -o gpurun_out/prof_store_tc64k python tools/c1_store.py --ncu > gpurun_out/ncu_store_tc.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dequant_cells -s 2 -c 1 \
  -o gpurun_out/prof_k4 python bench.py --steps 40 --warmup 3 --no-cpu --sets 2 --quick > gpurun_out/ncu_k4.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:store_tc -s 1 -c 1 \
  -o gpurun_out/prof_learned python tools/k1_learned.py --ncu > gpurun_out/ncu_learned.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_bf16 -s 3 -c 1 \
  -o gpurun_out/prof_bf16 python bench.py --steps 20 --warmup 3 --no-cpu --sets 2 > gpurun_out/ncu_bf16.out 2>&1
ls -la gpurun_out
