#!/bin/bash
# decode timeline traces (tools/trace_decode.py) over the PDL / cache-policy knobs
cd "${GRAFT_REPO_ROOT:-.}"
rm -f gpurun_out/trace.txt
for pre in ${PRE_LIST:-0 2}; do for ef in ${EF_LIST:-0 1}; do
  echo "#### KVR_PREWAIT=$pre KVR_EVICT_FIRST=$ef" >> gpurun_out/trace.txt
  KVR_PREWAIT=$pre KVR_EVICT_FIRST=$ef timeout 300 python tools/trace_decode.py 32768 ${SPLITS:-0} --step --steady > /dev/null 2>gpurun_out/trace.err || tail -5 gpurun_out/trace.err
done; done
cat gpurun_out/trace.txt | grep -v "^=="
