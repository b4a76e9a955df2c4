#!/bin/bash
# Extraction iteration: build, ext_time (args), then the -m gpu tests (SKIP_TESTS=1 skips).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-ext}; shift
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
timeout 300 python tools/ext_time.py "$@" 2>&1 | tee $O/ext_time.txt
timeout 300 python tools/ext_time.py 131072 10 u8,u16 2>&1 | tee -a $O/ext_time.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/gputest.log 2>&1; echo "gputest rc=$? $(tail -1 $O/gputest.log)"
  grep -E "^E |FAILED|Error" $O/gputest.log | head -20
fi
