#!/bin/bash
# GPU box: tcgen05 K1 -- timing vs the mma.sync kernel, parity tests, ncu capture
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for n in 4096 65536; do
  echo "== C1_TOKENS=$n tc";  C1_TOKENS=$n timeout 120 python tools/c1_store.py 2>&1 | tail -3
  echo "== C1_TOKENS=$n mma"; KVR_K1_IMPL=mma C1_TOKENS=$n timeout 120 python tools/c1_store.py 2>&1 | tail -3
done
timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_ops.py tests/test_gpu_learned.py tests/test_bf16_pool.py -q -x -p no:cacheprovider -s > gpurun_out/pytest_store.log 2>&1
echo "store tests rc=$?"; grep -E "nibble|passed|failed|Error|error" gpurun_out/pytest_store.log | tail -30
timeout 600 ncu --set full --clock-control none --import-source on -k regex:store_tc -s 2 -c 1 \
  -o gpurun_out/prof_store_tc python tools/c1_store.py --ncu > gpurun_out/ncu_store_tc.out 2>&1; echo "ncu rc=$?"
