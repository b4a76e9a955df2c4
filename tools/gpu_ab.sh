#!/bin/bash
# A/B extraction timing: the baseline worktree _base (prebuilt here) vs the working tree, twice
# interleaved.  gpurun -- bash tools/gpu_ab.sh TAG [ext_time args]
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-ab}; shift
mkdir -p $O
for rep in 1 2; do
  echo "== base"; (cd _base && timeout 300 python ../tools/ext_time.py "$@") 2>&1 | tee -a $O/ab.txt
  echo "== new"; timeout 300 python tools/ext_time.py "$@" 2>&1 | tee -a $O/ab.txt
done
