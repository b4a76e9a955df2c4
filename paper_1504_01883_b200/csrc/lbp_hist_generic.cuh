// lbp_hist_generic.cuh -- generic fused-depth LBP histogram kernel.
//
// Handles every geometry the ABI accepts (any ROI size / position / clamping,
// any grid, bins 59 or 256).  One CTA per ROI (grid-stride over ROIs); the
// cell histograms of a chunk of cells live in shared memory as u32 counters
// and are updated with shared-memory atomics (integer adds: order-independent,
// so the result is bit-exact whatever the thread schedule).  Grids whose
// histograms exceed the shared-memory budget are processed in chunks of whole
// cells, re-scanning only the rows of the chunk.  The fast path for uniform
// 128x128-class crops lives in lbp_hist_fast.cuh.
#pragma once
#include "common.cuh"

namespace lbpf {

constexpr int kGenericThreads = 256;
constexpr int kGenericHistCap = 12032;  // u32 counters per chunk (47 KB, static smem)

// Eq. 2 with the Fig. 7 weights: TL 1, T 2, TR 4, R 8, BR 16, B 32, BL 64, L 128.
__device__ __forceinline__ uint32_t lbp_code_scalar(const uint8_t* __restrict__ c, int64_t pitch) {
    const uint32_t gc = c[0];
    uint32_t code = 0;
    code |= (uint32_t)(c[-pitch - 1] >= gc) << 0;
    code |= (uint32_t)(c[-pitch] >= gc) << 1;
    code |= (uint32_t)(c[-pitch + 1] >= gc) << 2;
    code |= (uint32_t)(c[1] >= gc) << 3;
    code |= (uint32_t)(c[pitch + 1] >= gc) << 4;
    code |= (uint32_t)(c[pitch] >= gc) << 5;
    code |= (uint32_t)(c[pitch - 1] >= gc) << 6;
    code |= (uint32_t)(c[-1] >= gc) << 7;
    return code;
}

template <int BINS>
__global__ void __launch_bounds__(kGenericThreads)
lbp_hist_generic_kernel(const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                        lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                        DepthWindow win, int32_t cells_x, int32_t cells_y,
                        uint16_t* __restrict__ desc, int32_t* __restrict__ roi_status,
                        int skip_fast) {
    __shared__ uint32_t hist[kGenericHistCap];
    __shared__ uint8_t lut[256];
    constexpr int kCellsPerChunk = kGenericHistCap / BINS;
    const int64_t dim = (int64_t)cells_x * cells_y * BINS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kWarps = kGenericThreads / 32;

    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        lut[i] = (BINS == 59) ? kUniformLutDev.v[i] : (uint8_t)i;

    for (int32_t n = blockIdx.x; n < n_rois; n += gridDim.x) {
        const lbp_roi_t roi = rois[n];
        if (skip_fast && roi_is_fast(roi, geom)) continue;  // done by lbp_hist_fast_kernel
        const RoiGeom r = clamp_roi(roi, geom, cells_x, cells_y);
        uint16_t* out = desc + (int64_t)n * dim;
        if (threadIdx.x == 0 && roi_status) roi_status[n] = r.status;
        if (r.status != LBP_OK) {
            for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) out[i] = 0;
            continue;
        }
        const uint8_t* G = grey + (int64_t)r.img * geom.grey_img_stride;
        const uint16_t* D = depth ? depth + (int64_t)r.img * geom.depth_img_stride : nullptr;
        const int32_t n_cells = cells_x * cells_y;

        for (int32_t c0 = 0; c0 < n_cells; c0 += kCellsPerChunk) {
            const int32_t c1 = min(n_cells, c0 + kCellsPerChunk);
            __syncthreads();  // previous chunk's read-out done; lut visible
            for (int i = threadIdx.x; i < (c1 - c0) * BINS; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            // interior rows covered by cell rows [c0/Kx, (c1-1)/Kx]
            const int32_t cy_a = c0 / cells_x, cy_b = (c1 - 1) / cells_x;
            const int32_t i_begin = (int32_t)(((int64_t)cy_a * r.hi) / cells_y);
            const int32_t i_end = (int32_t)(((int64_t)(cy_b + 1) * r.hi) / cells_y);
            for (int32_t i = i_begin + warp; i < i_end; i += kWarps) {
                const int32_t cy = (int32_t)(((int64_t)(i + 1) * cells_y - 1) / r.hi);
                const int64_t yy = (int64_t)r.y0 + 1 + i;
                const uint8_t* grow = G + yy * geom.grey_pitch + r.x0 + 1;
                const uint16_t* drow = D ? D + yy * geom.depth_pitch + r.x0 + 1 : nullptr;
                for (int32_t j = lane; j < r.wi; j += 32) {
                    const int32_t cx = (int32_t)(((int64_t)(j + 1) * cells_x - 1) / r.wi);
                    const int32_t cell = cy * cells_x + cx;
                    if (cell < c0 || cell >= c1) continue;
                    if (drow) {
                        const uint32_t d = drow[j];
                        if (win.none_valid || (d - win.lo) > win.span) continue;
                    }
                    const uint32_t code = lbp_code_scalar(grow + j, geom.grey_pitch);
                    atomicAdd(&hist[(cell - c0) * BINS + lut[code]], 1u);
                }
            }
            __syncthreads();
            uint16_t* o = out + (int64_t)c0 * BINS;
            for (int i = threadIdx.x; i < (c1 - c0) * BINS; i += blockDim.x) o[i] = (uint16_t)hist[i];
        }
        __syncthreads();
    }
}

}  // namespace lbpf
