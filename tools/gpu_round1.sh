#!/bin/bash
# one gpurun call: build, GPU tests, smoke, microbench, bench, ncu launch list + full capture
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_smem_hist tools/micro_smem_hist.cu
timeout 120 ./tools/micro_smem_hist > gpurun_out/micro.log 2>&1; echo "micro rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log
CMD="python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lbp_hist -s 3 -c 1 -o gpurun_out/prof_lbp_hist $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
