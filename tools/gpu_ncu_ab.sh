#!/bin/bash
# ncu --set full of one extraction launch (ext_time.py variant $2), base worktree and new tree.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-ncuab}; V=${2:-u8}
mkdir -p $O
(cd _base && timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist -s 3 -c 1 -o ../$O/base_$V python ../tools/ext_time.py 16384 5 $V > ../$O/base.log 2>&1); echo "base rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist -s 3 -c 1 -o $O/new_$V python tools/ext_time.py 16384 5 $V > $O/new.log 2>&1; echo "new rc=$?"
