#!/bin/bash
# GPU box: trace + back-to-back graph time of every variant library under _lib/variants/.
cd "${GRAFT_REPO_ROOT:-.}"
for so in paper_2604_19157_b200/_lib/variants/libkvrot_*.so; do
  echo "#### $(basename $so)"
  KVR_LIB_PATH=$so timeout 300 python tools/trace_decode.py ${CTX:-32768} ${SPLITS:-0} 2>&1 | grep -E "counter back|split weights|merged|exit|graph"
done
