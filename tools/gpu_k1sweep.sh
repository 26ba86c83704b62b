cd "${GRAFT_REPO_ROOT:-.}"
for n in 1024 8192 16384 32768; do
  echo "== $n tc $(C1_TOKENS=$n timeout 120 python tools/c1_store.py 2>&1 | tr '\n' ' ')"
  echo "== $n mma $(KVR_K1_IMPL=mma C1_TOKENS=$n timeout 120 python tools/c1_store.py 2>&1 | tr '\n' ' ')"
done
