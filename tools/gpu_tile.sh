#!/bin/bash
# Tile-kernel iteration: build, its GPU tests, extraction timing at 64 / 200 / 128.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-tile}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_tile_gpu.py -q -x > $O/test.log 2>&1; echo "tile tests rc=$? $(tail -1 $O/test.log)"
grep -E "^E |FAILED|Error" $O/test.log | head -20
timeout 300 python tools/ext_time.py 16384 20 u16 hbm 64 2>&1 | tee $O/ext.txt
timeout 120 python tools/ext_time.py 16384 10 u16 hbm 200 2>&1 | tee -a $O/ext.txt
timeout 300 python tools/ext_time.py 16384 20 u16 hbm 128 2>&1 | tee -a $O/ext.txt
