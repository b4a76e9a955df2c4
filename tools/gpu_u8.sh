#!/bin/bash
# The compact (u8) recognition path: its GPU tests, then (args) bench lines.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-u8}
shift
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_u8_path_gpu.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/test.log 2>&1; echo "test rc=$? $(tail -1 $O/test.log)"
grep -E "^E |FAILED|Error" $O/test.log | head -30
for a in "$@"; do
  f=$O/bench_$(echo "$a" | tr ' =-' '___').json
  timeout 300 python bench.py $a > $f 2> $f.err; echo "bench [$a] rc=$?"; tail -c 1500 $f; echo; tail -3 $f.err
done
