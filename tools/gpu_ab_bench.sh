#!/bin/bash
# bench.py step time, base worktree (_base) vs working tree (and _dbg with SIDES="base new dbg"),
# alternated, per argument set.  REPS (default 2) rounds.
#   gpurun -- bash tools/gpu_ab_bench.sh TAG "args1" "args2" ...
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-abb}; shift
mkdir -p $O
for rep in $(seq ${REPS:-2}); do
  for a in "$@"; do
    for side in ${SIDES:-base new}; do
      d=.; [ $side = base ] && d=_base; [ $side = dbg ] && d=_dbg
      r=$( (cd $d && timeout 300 python bench.py --skip-cpu --e2e-steps 1 $a 2>>$GRAFT_REPO_ROOT/$O/err.txt | tail -1) )
      echo "$side [$a] $(echo "$r" | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["value"], j["ms_per_step"], j["roofline"]["achieved"], j.get("gpu_launches"))')" | tee -a $O/ab.txt
    done
  done
done
