#!/bin/bash
# gpurun payload: build, GPU tests, smoke, bench; optional ncu (NCU=1) of the bench command.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
  timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
fi
BENCH_ARGS=${BENCH_ARGS:-""}
timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --skip-cpu --e2e-steps 1 $BENCH_ARGS"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  for K in ${NCU_KERNELS:-lbp_hist_lane59 svm_gemm_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${NCU_SKIP:-3} -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu full $K rc=$?"; tail -2 gpurun_out/ncu_full_$K.log
  done
fi
