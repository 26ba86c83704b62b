#!/bin/bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "SUMMARY|done" gpurun_out/sanitize_$tool.log
done
timeout 1500 compute-sanitizer --tool synccheck --num-cuda-barriers 65536 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "SUMMARY|done|Warning" gpurun_out/sanitize_synccheck.log
SAN_SKIP_TC=1 timeout 1500 compute-sanitizer --tool synccheck --num-cuda-barriers 65536 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck_notc.log 2>&1
echo "synccheck (no tcgen05 K1) rc=$?"; grep -E "SUMMARY|done|Warning" gpurun_out/sanitize_synccheck_notc.log
