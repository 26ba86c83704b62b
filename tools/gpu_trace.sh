#!/bin/bash
# GPU box: C2 decode timelines (tools/trace_decode.py) for the in-tree library and
# every A/B variant under _lib/variants/ (tools/build_variants.py NAME=-DKVR_...=..).
cd "${GRAFT_REPO_ROOT:-.}"
shopt -s nullglob
rm -f gpurun_out/trace.txt
for so in "" paper_2604_19157_b200/_lib/variants/libkvrot_*.so; do
  echo "#### ${so:-in-tree library}" >> gpurun_out/trace.txt
  KVR_LIB_PATH=$so timeout 300 python tools/trace_decode.py 32768 ${SPLITS:-0} --step --steady > /dev/null 2>gpurun_out/trace.err \
    || tail -5 gpurun_out/trace.err
done
grep -v "^==" gpurun_out/trace.txt
