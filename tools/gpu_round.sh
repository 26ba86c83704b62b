#!/bin/bash
# GPU box: round evidence -- GPU tests, smoke, full bench (+ CPU leg), decode timelines, ncu.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
grep "^\[bench\]" gpurun_out/bench_full.err | tail -8
rm -f gpurun_out/trace.txt
for a in "32768 0 --step --steady" "32768 0 --step" "32768 0 --steady" "512 0 --step --steady" "512 0 --steady"; do
  timeout 300 python tools/trace_decode.py $a > /dev/null 2>> gpurun_out/trace.err
done
bash tools/gpu_profile.sh > /dev/null 2>&1; echo "profile rc=$?"
