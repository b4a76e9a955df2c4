#!/bin/bash
# ext_time.py with alternative builds of the library (experiment variants under _dbg/vN).
cd "$GRAFT_REPO_ROOT" || exit 1
python __graft_entry__.py build > /dev/null 2>&1
for rep in 1 2; do
  echo "== main"; timeout 200 python tools/ext_time.py "$@"
  for v in _dbg/v*; do
    echo "== $v"; cp $v/liblbpfused.so _dbg/paper_1504_01883_b200/liblbpfused.so
    (cd _dbg && timeout 200 python ../tools/ext_time.py "$@")
  done
done
