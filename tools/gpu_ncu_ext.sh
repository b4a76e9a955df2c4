#!/bin/bash
# ncu --set full of one lane59 launch per ext_time.py variant (args: TAG variant...)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; shift
mkdir -p $O
python __graft_entry__.py build > /dev/null 2>&1
for v in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist -s 3 -c 1 -o $O/$v python tools/ext_time.py 16384 5 $v > $O/$v.log 2>&1; echo "$v rc=$?"
done
