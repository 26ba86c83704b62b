#!/bin/bash
# GPU box: bench detail configs for every variant library under _lib/variants/.
cd "${GRAFT_REPO_ROOT:-.}"
for so in paper_2604_19157_b200/_lib/variants/libkvrot_*.so; do
  echo "#### $(basename $so)"
  KVR_LIB_PATH=$so timeout 600 python bench.py --steps 500 --no-cpu ${BENCH_ARGS} 2>&1 | grep "^\[bench\]"
done
