#!/bin/bash
# Round-2 evidence in one gpurun call: every bench line into gpurun_out/$TAG/lines/, the ncu
# launch list of the headline step, and --set full captures of the kernels the lines report.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash tools/gpu_r02_lines.sh TAG
cd "$GRAFT_REPO_ROOT" || exit 1
T=${1:-r02_lines}
PART=${2:-lines}   # lines | ncu:NAME (see the case list below)  (one gpurun call each: gpurun_out/ comes back <= 64 MiB)
O=gpurun_out/$T
mkdir -p $O/lines $O/ncu
python __graft_entry__.py build > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
if [ "$PART" = lines ]; then
run() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py "$@" > $O/lines/$name.json 2> $O/lines/$name.err
  echo "$name rc=$? $(tail -1 $O/lines/$name.json | cut -c1-150)"
}
run config3 --steps 20 --warmup 5
run config3_u8 --steps 20 --warmup 5 --format u8 --skip-cpu
run config3_fused --source fused --skip-cpu --e2e-steps 1
run config3_depth --source depth --skip-cpu --e2e-steps 1
run config3_bins256 --bins 256 --skip-cpu --e2e-steps 1
run config4 --workload config4 --steps 10 --warmup 3 --skip-cpu --e2e-steps 1
run tile64 --workload tile64 --steps 20 --warmup 5
run tile100 --workload tile100 --steps 20 --warmup 5
run tile200 --workload tile200 --steps 10 --warmup 3
run config1 --workload config1
run config2 --workload config2
run config5 --workload config5 --chunks 1
run config5_fused --workload config5 --fused --chunks 1
run train --workload train
run reference --impl reference --steps 3 --warmup 1
# launch list (cold, serialised) of the headline step
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu/launches_config3.csv \
  python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 1 > $O/ncu/launches_config3.log 2>&1; echo "launches rc=$?"
fi
full() {  # name, kernel regex, bench args...
  local name=$1 k=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/ncu/$name \
    python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 1 "$@" > $O/ncu/$name.log 2>&1; echo "ncu $name rc=$?"
}
# one capture per call keeps gpurun_out/ under gpurun's 64 MiB copy-back limit: PART=ncu:NAME
case "$PART" in
  ncu:lane59_config3) full lane59_config3 lbp_hist_lane59 ;;
  ncu:svm_gemm_config3) full svm_gemm_config3 svm_gemm_kernel ;;
  ncu:lane59_fused) full lane59_fused lbp_hist_lane59 --source fused ;;
  ncu:tile64) full tile64 lbp_hist_tile --workload tile64 ;;
  ncu:tile100) full tile100 lbp_hist_tile --workload tile100 ;;
  ncu:tile200) full tile200 lbp_hist_tile --workload tile200 ;;
  ncu:svm_u8_config4) full svm_u8_config4 svm_gemm_u8 --workload config4 --crops 16384 ;;
  ncu:lane59_config3_u8) full lane59_config3_u8 lbp_hist_lane59 --format u8 ;;
esac
