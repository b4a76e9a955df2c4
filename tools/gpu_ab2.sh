#!/bin/bash
# ext_time.py in several argument sets for the base worktree and the working tree.
#   gpurun -- bash tools/gpu_ab2.sh TAG "args1" "args2" ...
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-ab2}; shift
mkdir -p $O
for a in "$@"; do
  echo "== base [$a]"; (cd _base && timeout 300 python ../tools/ext_time.py $a) 2>&1 | tee -a $O/ab.txt
  echo "== new [$a]"; timeout 300 python tools/ext_time.py $a 2>&1 | tee -a $O/ab.txt
done
