#!/bin/bash
# GPU box: new parity tests + the existing GPU suite + a quick bench line
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_full.py -q -p no:cacheprovider -s > gpurun_out/pytest_parity.log 2>&1
echo "parity rc=$?"; grep -E "rel err|passed|failed|Error" gpurun_out/pytest_parity.log | tail -30
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/bench_q20.json 2> gpurun_out/bench_q20.err; echo "bench20 rc=$?"
timeout 600 python bench.py --steps 2000 --warmup 10 --quick --no-cpu > gpurun_out/bench_q2000.json 2> gpurun_out/bench_q2000.err; echo "bench2000 rc=$?"
grep "^\[bench\]" gpurun_out/bench_q20.err gpurun_out/bench_q2000.err
