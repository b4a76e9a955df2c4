// lbp_hist_generic.cuh -- generic fused-depth LBP histogram code path.
//
// Handles every geometry the ABI accepts (any ROI size / position / clamping,
// any grid, bins 59 or 256).  `extract_roi_generic` processes ONE ROI with a
// group of NT threads; the cell histograms of a chunk of cells live in shared
// memory as u32 counters updated with shared-memory atomics (integer adds:
// order-independent, so the result is bit-exact whatever the schedule).  Grids
// whose histograms exceed the chunk capacity are processed in chunks of whole
// cells, re-scanning only the rows of the chunk.  It is used by the generic
// kernel (one CTA per ROI) and, for the odd ROI, inside the TMA fast kernel.
#pragma once
#include "common.cuh"

namespace lbpf {

constexpr int kGenericThreads = 256;
constexpr int kGenericHistCap = 4096;  // u32 counters per chunk (16 KB static smem)

// Eq. 2 with the Fig. 7 weights: TL 1, T 2, TR 4, R 8, BR 16, B 32, BL 64, L 128.
// T = uint8_t (grey source) or uint16_t (depth source); pitch in elements.
template <typename T>
__device__ __forceinline__ uint32_t lbp_code_scalar(const T* __restrict__ c, int64_t pitch) {
    const uint32_t gc = __ldg(c);
    uint32_t code = 0;
    code |= (uint32_t)(__ldg(c - pitch - 1) >= gc) << 0;
    code |= (uint32_t)(__ldg(c - pitch) >= gc) << 1;
    code |= (uint32_t)(__ldg(c - pitch + 1) >= gc) << 2;
    code |= (uint32_t)(__ldg(c + 1) >= gc) << 3;
    code |= (uint32_t)(__ldg(c + pitch + 1) >= gc) << 4;
    code |= (uint32_t)(__ldg(c + pitch) >= gc) << 5;
    code |= (uint32_t)(__ldg(c + pitch - 1) >= gc) << 6;
    code |= (uint32_t)(__ldg(c - 1) >= gc) << 7;
    return code;
}

// The image plane the codes are computed on: grey (u8) or depth (u16), pitches in elements.
template <typename T>
struct CodePlane {
    const T* base;
    int64_t pitch, img_stride;
};

// One ROI (index n) by a group of NT threads (t = 0..NT-1), hist = `cap` u32 of smem
// that is all-zero on entry and is all-zero again on return.  lut[code] >> lut_shift is
// the bin.  `sync()` synchronises the group.  The descriptor row of ROI n starts at
// desc + n * desc_stride (desc_stride >= dim; the fused grey||depth layout passes 2 * dim and
// a desc already offset to its block).
// Only the cells [cell_begin, cell_end) (row-major cell indices) are computed and written;
// the whole grid by default.  The unit holding cell 0 writes roi_status.  KEEP (one chunk
// only): the counts stay in hist (not re-zeroed, no trailing sync) for the caller to read.
template <int BINS, int NT, typename T, typename Sync, bool KEEP = false>
__device__ __forceinline__ void extract_roi_generic(
    const CodePlane<T> plane, const uint16_t* __restrict__ depth, const lbp_images_t& geom,
    const lbp_roi_t roi, int32_t n, const DepthWindow& win, int32_t cells_x, int32_t cells_y,
    uint16_t* __restrict__ desc, int64_t desc_stride, int32_t* __restrict__ roi_status,
    uint32_t* hist, int cap, const uint8_t* lut, int lut_shift, int t, Sync sync,
    int32_t cell_begin = 0, int32_t cell_end = -1) {
    if (cell_end < 0) cell_end = cells_x * cells_y;
    const int warp = t >> 5, lane = t & 31;
    constexpr int kWarps = NT / 32;
    const RoiGeom r = clamp_roi(roi, geom, cells_x, cells_y);
    uint16_t* out = desc + (int64_t)n * desc_stride;
    if (t == 0 && roi_status && cell_begin == 0) roi_status[n] = r.status;
    if (r.status != LBP_OK) {
        for (int64_t i = (int64_t)cell_begin * BINS + t; i < (int64_t)cell_end * BINS; i += NT)
            out[i] = 0;
        return;
    }
    const T* G = plane.base + (int64_t)r.img * plane.img_stride;
    const uint16_t* D = depth ? depth + (int64_t)r.img * geom.depth_img_stride : nullptr;
    const int32_t cells_per_chunk = cap / BINS;
    // cell of interior column j: ((j+1)*Kx - 1) / W' -- in 32 bits when it cannot overflow
    // (every realistic geometry), 64 bits otherwise
    const bool narrow = (uint64_t)(r.wi + 1) * (uint64_t)cells_x < (1ull << 32);
    auto cell_x = [&](int32_t j) -> int32_t {
        return narrow ? (int32_t)(((uint32_t)(j + 1) * (uint32_t)cells_x - 1u) / (uint32_t)r.wi)
                      : (int32_t)(((int64_t)(j + 1) * cells_x - 1) / r.wi);
    };

    for (int32_t c0 = cell_begin; c0 < cell_end; c0 += cells_per_chunk) {
        const int32_t c1 = min(cell_end, c0 + cells_per_chunk);
        // interior rows covered by cell rows [c0/Kx, (c1-1)/Kx]
        const int32_t cy_a = c0 / cells_x, cy_b = (c1 - 1) / cells_x;
        const int32_t i_begin = (int32_t)(((int64_t)cy_a * r.hi) / cells_y);
        const int32_t i_end = (int32_t)(((int64_t)(cy_b + 1) * r.hi) / cells_y);
        for (int32_t i = i_begin + warp; i < i_end; i += kWarps) {
            const int32_t cy = (int32_t)(((int64_t)(i + 1) * cells_y - 1) / r.hi);
            const int64_t yy = (int64_t)r.y0 + 1 + i;
            const T* grow = G + yy * plane.pitch + r.x0 + 1;
            const uint16_t* drow = D ? D + yy * geom.depth_pitch + r.x0 + 1 : nullptr;
            // 4 columns per lane per iteration: their 4 x 10 independent global loads are in
            // flight together (latency-bound otherwise: one ROI per CTA, L2/DRAM latency)
            for (int32_t j0 = lane; j0 < r.wi; j0 += 128) {
                uint32_t code[4], ok[4];
                int32_t cell[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t j = j0 + 32 * u;
                    const bool in = j < r.wi;
                    const int32_t jj = in ? j : j0;
                    cell[u] = cy * cells_x + cell_x(jj);
                    ok[u] = in && cell[u] >= c0 && cell[u] < c1;
                    if (drow) {
                        const uint32_t d = __ldg(drow + jj);
                        ok[u] = ok[u] && !win.none_valid && (d - win.lo) <= win.span;
                    }
                    code[u] = lbp_code_scalar(grow + jj, plane.pitch);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (ok[u]) atomicAdd(&hist[(cell[u] - c0) * BINS + (lut[code[u]] >> lut_shift)], 1u);
            }
        }
        sync();
        uint16_t* o = out + (int64_t)c0 * BINS;
        for (int i = t; i < (c1 - c0) * BINS; i += NT) {
            o[i] = (uint16_t)hist[i];
            if (!KEEP) hist[i] = 0;
        }
        if (!KEEP) sync();
    }
}

struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// One CTA per (ROI, cell row) unit: the rows of one cell row of one ROI, all its cells.
// Cell rows are disjoint in the descriptor, so units never share a counter and no global
// atomics are needed; a handful of ROIs (the frame-stream and single-crop configs) still
// spread over cells_y times as many SMs.
// NT = 512 for small batches of tall ROIs (one interior row per warp, one L2 round trip),
// 256 otherwise.
template <int BINS, typename T, int NT = kGenericThreads>
__global__ void __launch_bounds__(NT)
lbp_hist_generic_kernel(const CodePlane<T> plane, const uint16_t* __restrict__ depth,
                        lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                        DepthWindow win, int32_t cells_x, int32_t cells_y,
                        uint16_t* __restrict__ desc, int64_t desc_stride,
                        int32_t* __restrict__ roi_status) {
    __shared__ uint32_t hist[kGenericHistCap];
    __shared__ uint8_t lut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        lut[i] = (BINS == 59) ? kUniformLutDev.v[i] : (uint8_t)i;
    // only the counters of one chunk are ever used: (cap / BINS) cells, or one cell row
    const int used = min(kGenericHistCap / BINS, cells_x) * BINS;
    for (int i = threadIdx.x; i < used; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int64_t n_units = (int64_t)n_rois * cells_y;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int32_t n = (int32_t)(u / cells_y), cy = (int32_t)(u - (int64_t)n * cells_y);
        extract_roi_generic<BINS, NT>(plane, depth, geom, rois[n], n, win, cells_x,
                                                   cells_y, desc, desc_stride, roi_status, hist,
                                                   kGenericHistCap, lut, 0, (int)threadIdx.x,
                                                   CtaSync{}, cy * cells_x, (cy + 1) * cells_x);
    }
}

}  // namespace lbpf
