#!/bin/bash
# Full GPU test suite, smoke() and the tile bench lines in one gpurun call.
#   gpurun -- bash tools/gpu_final_check.sh TAG
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
for w in tile64 tile100 tile200; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > $O/$w.json 2> $O/$w.err
done
