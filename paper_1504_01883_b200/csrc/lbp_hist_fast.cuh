// lbp_hist_fast.cuh -- fast path for uniform crops (placeholder until the
// staged kernel lands; the generic kernel handles everything meanwhile).
#pragma once
#include "common.cuh"

namespace lbpf {

inline bool fast_path_applicable(const lbp_images_t&, const uint16_t*, int32_t, int32_t, int32_t) {
    return false;
}

inline cudaError_t launch_lbp_hist_fast(const uint8_t*, const uint16_t*, const lbp_images_t&,
                                        const lbp_roi_t*, int32_t, const DepthWindow&, int32_t,
                                        uint16_t*, int32_t*, int, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace lbpf
