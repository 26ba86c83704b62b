#!/bin/bash
# GPU box: full GPU suite + smoke + quick bench (headline + C1) + C2 trace
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 400 --warmup 10 --quick --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
grep "^\[bench\]" gpurun_out/bench_q.err
rm -f gpurun_out/trace.txt
timeout 300 python tools/trace_decode.py 32768 0 --step > /dev/null 2>> gpurun_out/trace.err
grep -E "==|loop|stored|merged|graph" gpurun_out/trace.txt
