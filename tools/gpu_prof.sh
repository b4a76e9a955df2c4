#!/bin/bash
# ncu captures: a launch list and one --set full capture per kernel regex of a bench command.
#   gpurun -- bash tools/gpu_prof.sh TAG "BENCH ARGS" "kregex1 kregex2 ..."
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-prof}
mkdir -p $O
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
CMD="python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 1 $2"
timeout 300 $CMD > $O/plain.json 2>&1; echo "plain rc=$?"; tail -c 600 $O/plain.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for K in $3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${NCU_SKIP:-3} -c 1 -o $O/prof_$K $CMD > $O/ncu_full_$K.log 2>&1; echo "ncu full $K rc=$?"; tail -2 $O/ncu_full_$K.log
done
