#!/bin/bash
# Round-2 baseline session: gpu tests + smoke + bench lines (gpu_r02.sh), then the ncu launch
# list and --set full captures of the extraction and scorer kernels (gpu_prof.sh).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/gpu_r02b.sh TAG
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-r02b}
bash tools/gpu_r02.sh $TAG
bash tools/gpu_prof.sh ${TAG}_prof "" "lbp_hist svm_gemm_u8"
