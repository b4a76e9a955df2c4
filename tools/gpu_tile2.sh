#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-tile2}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
timeout 300 python tools/ext_time.py 16384 10 u16 hbm 200 > $O/ext200.txt 2>&1; echo "rc=$?"; tail -5 $O/ext200.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist_tile -s 3 -c 1 -o $O/tile64 python tools/ext_time.py 16384 5 u16 hbm 64 > $O/ncu64.log 2>&1; echo "ncu64 rc=$?"
