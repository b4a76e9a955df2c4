#!/bin/bash
# Quick GPU iteration: build, all -m gpu tests (or $PYTEST_K subset), then bench lines (args).
#   gpurun --timeout 900 -- bash tools/gpu_quick.sh TAG "bench args 1" "bench args 2" ...
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-quick}
shift
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/gputest.log 2>&1; echo "gputest rc=$? $(tail -1 $O/gputest.log)"
  grep -E "^E |FAILED|Error" $O/gputest.log | head -20
fi
for a in "$@"; do
  f=$O/bench_$(echo "$a" | tr ' =-' '___').json
  timeout 300 python bench.py $a > $f 2> $f.err; echo "bench [$a] rc=$?"
  python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline') or {}
    print(' value %.2f M/s step %.4f ms kern %s frac %s nom %s scorer %s' % (d['value']/1e6, d['ms_per_step'], r.get('kernel_ms'), r.get('frac'), r.get('frac_of_nominal_8000'), (r.get('scorer') or {}).get('kernel_ms')))
except Exception as e: print(' parse error', e)
PY
  tail -2 $f.err
done
