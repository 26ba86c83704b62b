#!/bin/bash
# A/B of decode knobs: graph time per fused C2 step (tools/trace_decode.py)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_decode.py -q -x -p no:cacheprovider 2>&1 | tail -2
for mi in 0 1; do for ef in 0 1; do
 echo "#### MERGE_INLINE=$mi EF=$ef"; KVR_MERGE_INLINE=$mi KVR_EVICT_FIRST=$ef timeout 300 python tools/trace_decode.py 32768 0 12 24 32 --step --steady 2>&1 | grep "graph time\|^=="
done; done
