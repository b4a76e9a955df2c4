// tma_util.cuh -- host helpers of the TMA-staged extraction kernels (lbp_hist_lane59.cuh,
// lbp_hist_lane256.cuh): whether a launch can use the 128x128 fast path (8x8 cells, 16-B
// aligned rows, TMA stride limits) and the 3-D tensor maps over an image stack.
#pragma once
#include <cudaTypedefs.h>
#include "common.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"

namespace lbpf {

constexpr int kFastCells = 8;

inline bool fast_path_applicable(const lbp_images_t& g, const uint8_t* grey, const uint16_t* depth,
                                 int32_t cells_x, int32_t cells_y, int32_t bins,
                                 const uint16_t* desc) {
    if (cells_x != kFastCells || cells_y != kFastCells) return false;
    if (reinterpret_cast<uintptr_t>(desc) & 15) return false;
    if (bins != 59 && bins != 256) return false;
    if (g.width < kFastTile || g.height < kFastTile) return false;
    if (grey && ((reinterpret_cast<uintptr_t>(grey) & 15) || (g.grey_pitch & 15) ||
                 (g.grey_img_stride & 15)))
        return false;  // (grey == NULL: depth-source launch, grey unused)
    if (depth && ((reinterpret_cast<uintptr_t>(depth) & 15) || ((g.depth_pitch * 2) & 15) ||
                  ((g.depth_img_stride * 2) & 15)))
        return false;
    // TMA: strides < 2^40 bytes
    if ((grey && g.grey_img_stride >= (int64_t(1) << 39)) ||
        (depth && g.depth_img_stride >= (int64_t(1) << 38)))
        return false;
    return true;
}

// The tile kernels (lbp_hist_tile.cuh): TMA-legal image stacks of any size (16-B aligned
// bases, pitches and image strides, strides < 2^40 bytes).
inline bool tile_path_applicable(const lbp_images_t& g, const uint8_t* grey, const uint16_t* depth) {
    if (!grey || (reinterpret_cast<uintptr_t>(grey) & 15) || (g.grey_pitch & 15) ||
        (g.grey_img_stride & 15) || g.grey_img_stride >= (int64_t(1) << 39))
        return false;
    if (depth && ((reinterpret_cast<uintptr_t>(depth) & 15) || ((g.depth_pitch * 2) & 15) ||
                  ((g.depth_img_stride * 2) & 15) || g.depth_img_stride >= (int64_t(1) << 38)))
        return false;
    return true;
}

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    // resolved once (thread-safe static init); immutable afterwards
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

inline bool encode_stack_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem,
                             const lbp_images_t& g, int64_t pitch, int64_t img_stride,
                             int box_w = kFastTile) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * elem), (cuuint64_t)(img_stride * elem)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, kFastTile, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace lbpf
