#!/bin/bash
# The fused database build on one GPU: its tests and the config-5 line with and without it.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-gather}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gather_gpu.py -q -x > $O/test.log 2>&1; echo "test rc=$? $(tail -1 $O/test.log)"
grep -E "FAILED|Error|assert" $O/test.log | head -20
for a in "" "--fused" "--chunks=1"; do
  timeout 300 python bench.py --workload config5 --steps 10 --warmup 3 $a > $O/c5$a.json 2> $O/c5$a.err; echo "c5 $a rc=$?"; tail -c 1200 "$O/c5$a.json"; echo
done
