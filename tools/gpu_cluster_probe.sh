#!/bin/bash
# GPU box: C2 with 16-CTA cluster merges vs the inline merge (split counts 12/16/18)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out; rm -f gpurun_out/trace.txt
for v in base cl16; do
  for sp in 16 18 12; do
    echo "#### $v splits $sp" >> gpurun_out/trace.txt
    KVR_LIB_PATH=paper_2604_19157_b200/_lib/variants/libkvrot_$v.so timeout 300 python tools/trace_decode.py 32768 $sp --step --steady > /dev/null 2>> gpurun_out/trace.err
    KVR_LIB_PATH=paper_2604_19157_b200/_lib/variants/libkvrot_$v.so timeout 300 python tools/trace_decode.py 32768 $sp --step > /dev/null 2>> gpurun_out/trace.err
  done
done
grep -E "####|==|graph|start|loop end|partial stored|merged|exit" gpurun_out/trace.txt
