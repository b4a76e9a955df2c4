#!/bin/bash
# one gpurun call: every bench line of DESIGN.md §6 (measurement table) into gpurun_out/lines/
#   /usr/local/graft/bin/gpurun --timeout 1500 -- bash tools/gpu_all_lines.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/lines
python __graft_entry__.py build > gpurun_out/lines/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py "$@" > gpurun_out/lines/$name.json 2> gpurun_out/lines/$name.err
  echo "$name rc=$? $(tail -1 gpurun_out/lines/$name.json | cut -c1-160)"
}
run config3
run config3_depth --source depth --skip-cpu --e2e-steps 1
run config3_fused --source fused --skip-cpu --e2e-steps 1
run config3_bins256 --bins 256 --skip-cpu --e2e-steps 1
run config4 --workload config4 --skip-cpu --e2e-steps 1
run config1 --workload config1
run config2 --workload config2
run config2_split --workload config2 --api split --skip-cpu
run config2_resize200 --workload config2 --resize 200
run config5 --workload config5 --chunks 1
run train --workload train
run reference --impl reference --steps 3 --warmup 1
