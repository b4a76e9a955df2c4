// common.cuh -- shared device helpers of the CUDA hot path (product code; never
// includes or links anything under oracle/).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "lbpfused.h"

namespace lbpf {

// ---------------------------------------------------------------------------
// Uniform-pattern bin map (bins = 59), built at compile time.  A code is
// uniform iff its circular 8-bit pattern (the Fig. 7 sampling points go round
// the centre) has at most two 0/1 transitions; uniform codes are
// numbered 0..57 in ascending code order, every other code maps to bin 58
// (reading R4).
// ---------------------------------------------------------------------------
struct BinLut {
    uint8_t v[256];
};

constexpr int popcount8(unsigned x) {
    int n = 0;
    for (int i = 0; i < 8; ++i) n += (x >> i) & 1u;
    return n;
}

constexpr BinLut make_uniform_lut() {
    BinLut t{};
    int next = 0;
    for (unsigned c = 0; c < 256; ++c) {
        unsigned rot = ((c >> 1) | (c << 7)) & 0xFFu;  // neighbour p+1 aligned onto p
        t.v[c] = popcount8(c ^ rot) <= 2 ? static_cast<uint8_t>(next++) : 0xFF;
    }
    for (unsigned c = 0; c < 256; ++c)
        if (t.v[c] == 0xFF) t.v[c] = static_cast<uint8_t>(next);
    return t;
}

constexpr BinLut kUniformLut = make_uniform_lut();
static_assert(kUniformLut.v[0] == 0 && kUniformLut.v[255] == 57 && kUniformLut.v[85] == 58,
              "uniform LUT");
// device copy (constant bank); kernels stage it into shared memory
static __constant__ BinLut kUniformLutDev = make_uniform_lut();

// Launch with programmatic stream serialization: the kernel's CTAs may be scheduled before
// the previous kernel on the stream completes (once that kernel has run launch_dependents),
// so the kernel must call grid_dependency_wait() before it touches memory the previous kernel
// writes or reads.  Without a triggering predecessor this is an ordinary launch.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, int smem,
                              cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

// Depth-window predicate parameters: valid(d) <=> d != 0 && dmin <= d <= dmax
//   <=> (uint32)(d - lo) <= span with lo = max(dmin, 1), span = dmax - lo,
// and nothing is valid when dmax < lo (i.e. dmax == 0): `none_valid`.
struct DepthWindow {
    uint32_t lo, span;
    int none_valid;
};

inline DepthWindow make_window(uint16_t dmin, uint16_t dmax) {
    DepthWindow w;
    w.lo = dmin < 1 ? 1u : dmin;
    w.none_valid = (dmax < w.lo);
    w.span = w.none_valid ? 0u : (uint32_t)dmax - w.lo;
    return w;
}

// Geometry of one clamped ROI, computed identically on every thread.
struct RoiGeom {
    int32_t status;
    int32_t img;
    int32_t x0, y0;  // top-left of the clamped ROI in the image
    int32_t wi, hi;  // interior size W' = w-2, H' = h-2
};

__device__ __forceinline__ RoiGeom clamp_roi(const lbp_roi_t r, const lbp_images_t& g,
                                             int cells_x, int cells_y) {
    RoiGeom o;
    int64_t x0 = r.x, y0 = r.y;
    int64_t x1 = x0 + r.w, y1 = y0 + r.h;
    x0 = x0 < 0 ? 0 : x0;
    y0 = y0 < 0 ? 0 : y0;
    x1 = x1 > g.width ? g.width : x1;
    y1 = y1 > g.height ? g.height : y1;
    int64_t w = x1 - x0, h = y1 - y0;
    o.img = r.img;
    o.x0 = (int32_t)x0;
    o.y0 = (int32_t)y0;
    o.wi = (int32_t)(w - 2);
    o.hi = (int32_t)(h - 2);
    o.status = LBP_OK;
    if (r.img < 0 || r.img >= g.n_images || w < 3 || h < 3) {
        o.status = LBP_E_ROI;
    } else if (cells_x > o.wi || cells_y > o.hi) {
        o.status = LBP_E_GRID;
    } else {
        // largest cell of the floor partition spans ceil(W'/K) pixels
        int64_t mw = (o.wi + cells_x - 1) / cells_x, mh = (o.hi + cells_y - 1) / cells_y;
        if (mw * mh > 65535) o.status = LBP_E_OVERFLOW;
    }
    return o;
}

// ROIs handled by the TMA fast kernel: fully inside the image, exactly kFastTile square, and
// x a multiple of 16 px (a TMA box must start 16-B aligned in its innermost dimension:
// tools/tma_probe.cu measured "illegal instruction" for unaligned starts on B200).
constexpr int kFastTile = 128;
__device__ __forceinline__ bool roi_is_fast(const lbp_roi_t& r, const lbp_images_t& g) {
    return r.w == kFastTile && r.h == kFastTile && r.img >= 0 && r.img < g.n_images && r.x >= 0 &&
           (r.x & 15) == 0 &&
           r.y >= 0 && (int64_t)r.x + kFastTile <= g.width && (int64_t)r.y + kFastTile <= g.height;
}
// Same for the frame variant of the lane-private kernel, which stages a wider box at the
// aligned-down column and takes any x.
__device__ __forceinline__ bool roi_is_fast_frame(const lbp_roi_t& r, const lbp_images_t& g) {
    return r.w == kFastTile && r.h == kFastTile && r.img >= 0 && r.img < g.n_images && r.x >= 0 &&
           r.y >= 0 && (int64_t)r.x + kFastTile <= g.width && (int64_t)r.y + kFastTile <= g.height;
}

}  // namespace lbpf
