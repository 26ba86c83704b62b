#!/bin/bash
# quick GPU iteration: decode/store tests + trace + bench
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_store.py -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -3 gpurun_out/pytest_quick.log
timeout 300 python tools/trace_decode.py 32768 0 > gpurun_out/trace.log 2>&1; tail -12 gpurun_out/trace.log
timeout 600 python bench.py --steps 2000 --warmup 10 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
