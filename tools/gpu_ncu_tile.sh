#!/bin/bash
# ncu --set full of the tile kernel at crop size $2 (ext_time u16, 16384 crops)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-ncutile}; T=${2:-200}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist_tile -s 3 -c 1 -o $O/tile$T python tools/ext_time.py 16384 5 u16 hbm $T > $O/ncu$T.log 2>&1; echo "ncu$T rc=$?"
