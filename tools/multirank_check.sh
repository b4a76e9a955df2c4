#!/bin/bash
# Functional check of bench.py's multi-rank code paths on a ONE-GPU box: 2 ranks share the
# device over gloo (--dist-backend gloo).  Not a measurement (both ranks time-share one GPU).
#   /usr/local/graft/bin/gpurun --timeout 900 -- bash tools/multirank_check.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/multirank
python __graft_entry__.py build > gpurun_out/multirank/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() {  # name, args...
  local name=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 \
    --dist-backend gloo "$@" > gpurun_out/multirank/$name.json 2> gpurun_out/multirank/$name.err
  echo "$name rc=$? $(tail -1 gpurun_out/multirank/$name.json | cut -c1-200)"
}
run config3 --crops 4096 --steps 3 --warmup 3 --skip-cpu --e2e-steps 1
run config4 --workload config4 --crops 4096 --steps 3 --warmup 3 --skip-cpu --e2e-steps 1
run config5_serial --workload config5 --crops 8192 --chunks 1 --steps 3 --warmup 3
run config5_chunked --workload config5 --crops 8192 --chunks 4 --steps 3 --warmup 3
run config5_compact --workload config5 --crops 8192 --compact --steps 3 --warmup 3
run reference --impl reference --steps 2 --warmup 1
