// lbp_resize.cuh -- resized-ROI descriptors ("The detected face ... is
// resized to 200x200 pixels"): every ROI is clamped to its image, resized to
// size x size (grey: bilinear, half-pixel centres, rounded half up; depth: nearest neighbour,
// half-pixel centres, ties toward the smaller index) and described like a full
// size x size crop -- with the resize fused into the staging of the histogram kernel, so the
// resized crops never reach HBM.
//
// One CTA per (ROI, cell row) unit, as the band kernel.  A unit stages the resized rows its
// cell row needs (its interior rows plus the 1-px halo, in row chunks that fit the staging
// buffer) straight from the source frame into shared memory, then runs Eq. 2 / the depth
// window / the cell histograms on the staged tile.  Exact integer arithmetic (size <= 1024
// keeps every weighted sum below 2^31): the sample point of output column c is
// sx = Nx / Dx with Nx = (2c + 1) w - size, Dx = 2 size (clamped at 0), so the bilinear value
// is an integer over Dx * Dy and round-half-up is an integer floor; the nearest source
// column is floor(((2c + 1) w - 1) / (2 size)).
#pragma once
#include "common.cuh"

namespace lbpf {

constexpr int kResizeThreads = 512;
constexpr int kResizeMaxSize = 1024;
constexpr int kResizeStageBytes = 28 * 1024;  // grey u8 + depth u16 rows of one chunk
constexpr int kResizeHistCap = 4096;          // u32 counters per cell chunk (both planes)

// floor(q / m) for q < 2^32 and an estimate from a float reciprocal, corrected exactly
__device__ __forceinline__ uint32_t udiv_fix(uint32_t q, uint32_t m, float inv_m) {
    uint32_t r = (uint32_t)((float)q * inv_m);
    if ((uint64_t)r * m > q) --r;
    if ((uint64_t)(r + 1) * m <= q) ++r;
    return r;
}

// SRC: 0 = codes on grey, 1 = codes on depth, 2 = both (fused grey||depth descriptor)
template <int BINS, int SRC>
__global__ void __launch_bounds__(kResizeThreads)
lbp_hist_resize_kernel(const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                       lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                       int32_t size, DepthWindow win, int32_t cells_x, int32_t cells_y,
                       uint16_t* __restrict__ desc, int64_t desc_stride,
                       int32_t* __restrict__ roi_status) {
    constexpr int kPlanes = SRC == 2 ? 2 : 1;
    constexpr int NT = kResizeThreads, kWarps = NT / 32;
    __shared__ __align__(16) uint8_t stage[kResizeStageBytes];
    __shared__ uint32_t hist[kResizeHistCap];
    __shared__ uint8_t lut[256];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < 256; i += NT) lut[i] = (BINS == 59) ? kUniformLutDev.v[i] : (uint8_t)i;
    for (int i = t; i < kResizeHistCap; i += NT) hist[i] = 0;
    __syncthreads();

    const int32_t S = size, Wi = S - 2, Hi = S - 2;
    const int64_t dim = (int64_t)cells_x * cells_y * BINS;
    const uint32_t D = 2u * (uint32_t)S;            // Dx = Dy
    const uint32_t den = D * D;                     // bilinear denominator
    const float inv_2den = 1.0f / (2.0f * (float)den);
    const float inv_D = 1.0f / (float)D;
    const bool has_depth = depth != nullptr;
    const int32_t cells_per_chunk = kResizeHistCap / (BINS * kPlanes);
    const int64_t n_units = (int64_t)n_rois * cells_y;

    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int32_t n = (int32_t)(u / cells_y), cy = (int32_t)(u - (int64_t)n * cells_y);
        const lbp_roi_t roi = rois[n];
        // crop = clamp(roi, image)
        int64_t x0 = roi.x, y0 = roi.y, x1 = x0 + roi.w, y1 = y0 + roi.h;
        x0 = x0 < 0 ? 0 : x0;
        y0 = y0 < 0 ? 0 : y0;
        x1 = x1 > geom.width ? geom.width : x1;
        y1 = y1 > geom.height ? geom.height : y1;
        int32_t status = LBP_OK;
        if (roi.img < 0 || roi.img >= geom.n_images || x1 <= x0 || y1 <= y0) status = LBP_E_ROI;
        else if (cells_x > Wi || cells_y > Hi) status = LBP_E_GRID;
        else if ((int64_t)((Wi + cells_x - 1) / cells_x) * ((Hi + cells_y - 1) / cells_y) > 65535)
            status = LBP_E_OVERFLOW;
        uint16_t* out = desc + (int64_t)n * desc_stride;
        const int64_t seg0 = (int64_t)cy * cells_x * BINS, seg1 = seg0 + (int64_t)cells_x * BINS;
        if (cy == 0 && t == 0 && roi_status) roi_status[n] = status;
        if (status != LBP_OK) {
            for (int p = 0; p < kPlanes; ++p)
                for (int64_t i = seg0 + t; i < seg1; i += NT) out[p * dim + i] = 0;
            continue;
        }
        const uint32_t cw = (uint32_t)(x1 - x0), ch = (uint32_t)(y1 - y0);
        const uint8_t* G = (SRC != 1) ? grey + (int64_t)roi.img * geom.grey_img_stride +
                                            y0 * geom.grey_pitch + x0
                                      : nullptr;
        const uint16_t* Dp = has_depth ? depth + (int64_t)roi.img * geom.depth_img_stride +
                                             y0 * geom.depth_pitch + x0
                                       : nullptr;
        // interior rows of this cell row: [ib, ie)
        const int32_t ib = (int32_t)(((int64_t)cy * Hi) / cells_y);
        const int32_t ie = (int32_t)(((int64_t)(cy + 1) * Hi) / cells_y);

        for (int32_t c0 = 0; c0 < cells_x; c0 += cells_per_chunk) {
            const int32_t c1 = min(cells_x, c0 + cells_per_chunk);
            const int32_t jb = (int32_t)(((int64_t)c0 * Wi) / cells_x);
            const int32_t je = (int32_t)(((int64_t)c1 * Wi) / cells_x);
            const int32_t scols = je - jb + 2;              // staged resized columns [jb, je+2)
            const int32_t rows_max = (kResizeStageBytes - 2) / (3 * scols) - 2;  // >= 1 (S <= 1024)
            uint8_t* sg = stage;                            // [rows][scols] u8
            for (int32_t r0 = ib; r0 < ie; r0 += rows_max) {
                const int32_t r1 = min(ie, r0 + rows_max);
                const int32_t srows = r1 - r0 + 2;          // resized rows [r0, r1+2)
                uint16_t* sd = reinterpret_cast<uint16_t*>(stage + ((srows * scols + 1) & ~1));
                // ---- stage the resized rows (threads own columns; per column the x sample
                //      points are computed once)
                for (int32_t cc = t; cc < scols; cc += NT) {
                    const uint32_t c = (uint32_t)(jb + cc);
                    const uint32_t qx = (2 * c + 1) * cw;  // < 2^32: width <= 2^20, c < 1024
                    const uint32_t Nx = qx > (uint32_t)S ? qx - (uint32_t)S : 0u;  // sx >= 0
                    uint32_t gx0 = udiv_fix(Nx, D, inv_D);
                    uint32_t rx = Nx - gx0 * D;
                    if (gx0 > cw - 1) { gx0 = cw - 1; rx = 0; }
                    const uint32_t gx1 = gx0 + 1 < cw ? gx0 + 1 : cw - 1;
                    uint32_t dx = udiv_fix((2 * c + 1) * cw - 1, D, inv_D);
                    dx = dx > cw - 1 ? cw - 1 : dx;
                    for (int32_t rr = 0; rr < srows; ++rr) {
                        const uint32_t r = (uint32_t)(r0 + rr);
                        if (SRC != 1) {
                            const uint32_t qy = (2 * r + 1) * ch;
                            const uint32_t Ny = qy > (uint32_t)S ? qy - (uint32_t)S : 0u;
                            uint32_t gy0 = udiv_fix(Ny, D, inv_D);
                            uint32_t ry = Ny - gy0 * D;
                            if (gy0 > ch - 1) { gy0 = ch - 1; ry = 0; }
                            const uint32_t gy1 = gy0 + 1 < ch ? gy0 + 1 : ch - 1;
                            const uint8_t* a = G + (int64_t)gy0 * geom.grey_pitch;
                            const uint8_t* b = G + (int64_t)gy1 * geom.grey_pitch;
                            const uint32_t num = (D - rx) * (D - ry) * __ldg(a + gx0) +
                                                 rx * (D - ry) * __ldg(a + gx1) +
                                                 (D - rx) * ry * __ldg(b + gx0) +
                                                 rx * ry * __ldg(b + gx1);
                            sg[rr * scols + cc] = (uint8_t)udiv_fix(2 * num + den, 2 * den, inv_2den);
                        }
                        if (has_depth) {
                            uint32_t dy = udiv_fix((2 * r + 1) * ch - 1, D, inv_D);
                            dy = dy > ch - 1 ? ch - 1 : dy;
                            sd[rr * scols + cc] = __ldg(Dp + (int64_t)dy * geom.depth_pitch + dx);
                        }
                    }
                }
                __syncthreads();
                // ---- codes, depth window, cell histograms over interior rows [r0, r1)
                for (int32_t i = r0 + warp; i < r1; i += kWarps) {
                    const int32_t sr = i - r0 + 1;  // staged row of the centre
                    for (int32_t j = jb + lane; j < je; j += 32) {
                        const int32_t sc = j - jb + 1;
                        if (has_depth) {
                            const uint32_t dc = sd[sr * scols + sc];
                            if (win.none_valid || (dc - win.lo) > win.span) continue;
                        }
                        const int32_t cx =
                            (int32_t)(((uint32_t)(j + 1) * (uint32_t)cells_x - 1u) / (uint32_t)Wi) - c0;
#pragma unroll
                        for (int p = 0; p < kPlanes; ++p) {
                            const bool on_depth = (SRC == 1) || (SRC == 2 && p == 1);
                            uint32_t code = 0;
                            if (on_depth) {
                                const uint16_t* q = sd + sr * scols + sc;
                                const uint32_t gc = q[0];
                                code = ((uint32_t)(q[-scols - 1] >= gc) << 0) |
                                       ((uint32_t)(q[-scols] >= gc) << 1) |
                                       ((uint32_t)(q[-scols + 1] >= gc) << 2) |
                                       ((uint32_t)(q[1] >= gc) << 3) |
                                       ((uint32_t)(q[scols + 1] >= gc) << 4) |
                                       ((uint32_t)(q[scols] >= gc) << 5) |
                                       ((uint32_t)(q[scols - 1] >= gc) << 6) |
                                       ((uint32_t)(q[-1] >= gc) << 7);
                            } else {
                                const uint8_t* q = sg + sr * scols + sc;
                                const uint32_t gc = q[0];
                                code = ((uint32_t)(q[-scols - 1] >= gc) << 0) |
                                       ((uint32_t)(q[-scols] >= gc) << 1) |
                                       ((uint32_t)(q[-scols + 1] >= gc) << 2) |
                                       ((uint32_t)(q[1] >= gc) << 3) |
                                       ((uint32_t)(q[scols + 1] >= gc) << 4) |
                                       ((uint32_t)(q[scols] >= gc) << 5) |
                                       ((uint32_t)(q[scols - 1] >= gc) << 6) |
                                       ((uint32_t)(q[-1] >= gc) << 7);
                            }
                            atomicAdd(&hist[(p * (c1 - c0) + cx) * BINS + lut[code]], 1u);
                        }
                    }
                }
                __syncthreads();  // the stage is rewritten by the next row chunk
            }
            // ---- cells [cy*cells_x + c0, cy*cells_x + c1) of every plane -> descriptor
            const int32_t nb = (c1 - c0) * BINS;
            for (int p = 0; p < kPlanes; ++p) {
                uint16_t* o = out + p * dim + seg0 + (int64_t)c0 * BINS;
                for (int32_t k = t; k < nb; k += NT) {
                    o[k] = (uint16_t)hist[p * nb + k];
                    hist[p * nb + k] = 0;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace lbpf
