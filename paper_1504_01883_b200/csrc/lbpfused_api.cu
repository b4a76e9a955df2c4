// lbpfused_api.cu -- the C ABI (include/lbpfused.h): argument validation,
// dispatch between kernel variants, launches on the caller's stream.
#include <cmath>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "desc_pack.cuh"
#include "gather.cuh"
#include "lbp_hist_generic.cuh"
#include "tma_util.cuh"
#include "lbp_hist_lane59.cuh"
#include "lbp_hist_lane256.cuh"
#include "lbp_hist_tile.cuh"
#include "lbp_resize.cuh"
#include "lbp_recognize.cuh"
#include "svm_fp64.cuh"
#include "svm_gemm.cuh"
#include "svm_gemm_i8.cuh"
#include "svm_gemm_u8.cuh"
#include "svm_train.cuh"

using namespace lbpf;

namespace {

int32_t launch_status(cudaError_t e) {
    if (e == cudaSuccess) return LBP_OK;
    if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorInvalidDeviceFunction)
        return LBP_E_UNSUPPORTED;
    return LBP_E_CUDA;
}

int32_t check_geometry(const lbp_images_t& g, bool has_grey, bool has_depth) {
    if (g.n_images < 1 || g.height < 1 || g.width < 1 || g.reserved != 0) return LBP_E_ARG;
    if (has_grey && (g.grey_pitch < g.width ||
                     g.grey_img_stride < g.grey_pitch * (g.height - 1) + g.width))
        return LBP_E_ARG;
    if (has_depth && (g.depth_pitch < g.width ||
                      g.depth_img_stride < g.depth_pitch * (g.height - 1) + g.width))
        return LBP_E_ARG;
    return LBP_OK;
}

// Workspace format of svm_prepare for a [C][dim] model: the INT8 digit planes for many classes
// (more than one fp16 TMEM pass), else the fp16 digit planes.
bool svm_choose_layout(int32_t C, int32_t dim, lbpf::SvmPrepHeader* h) {
    if (C > lbpf::kPassClasses && lbpf::svm_layout_i8(C, dim, h)) return true;
    return lbpf::svm_layout(C, dim, h);
}
size_t svm_layout_total(const lbpf::SvmPrepHeader& h) {
    const size_t elem = h.magic == lbpf::kPrep8Magic ? 1 : 2;
    return (size_t)h.q_off + (size_t)h.total_rows * h.dim_pad * elem;
}

int num_sms() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace

extern "C" {

int32_t lbp_descriptor_dim(int32_t cells_x, int32_t cells_y, int32_t bins) {
    if (cells_x < 1 || cells_y < 1 || (bins != 59 && bins != 256)) return LBP_E_ARG;
    int64_t d = (int64_t)cells_x * cells_y * bins;
    return d > 0x7FFFFFFF ? LBP_E_ARG : (int32_t)d;
}

const char* lbp_status_string(int32_t s) {
    switch (s) {
        case LBP_OK: return "LBP_OK";
        case LBP_E_ARG: return "LBP_E_ARG: invalid argument";
        case LBP_E_ROI: return "LBP_E_ROI: ROI empty, smaller than 3x3 after clamping, or bad image";
        case LBP_E_GRID: return "LBP_E_GRID: grid larger than the ROI interior";
        case LBP_E_OVERFLOW: return "LBP_E_OVERFLOW: a cell has more than 65535 pixels";
        case LBP_E_UNSUPPORTED: return "LBP_E_UNSUPPORTED: unsupported device or configuration";
        case LBP_E_CUDA: return "LBP_E_CUDA: CUDA error";
        default: return "unknown status";
    }
}

}  // extern "C"

namespace {

// One descriptor block: codes of `plane` (grey u8 or depth u16), depth-window mask from
// `depth`, rows of desc_stride elements starting at `desc`.
int32_t extract_block(const uint8_t* grey, const uint16_t* depth, bool depth_source,
                      const lbp_images_t& geom, const lbp_roi_t* rois, int32_t n_rois,
                      const DepthWindow& win, int32_t cells_x, int32_t cells_y, int32_t bins,
                      uint16_t* desc, int64_t desc_stride, int32_t* roi_status,
                      cudaStream_t stream) {
    // Small batches (the frame-stream and single-crop configs): the band kernel spreads every
    // ROI over cells_y CTAs; the persistent TMA kernel would give each ROI one 8-warp group.
    const bool small_batch = n_rois < num_sms();
    // Frames wider than a crop: the FRAME variant of the lane-private kernel stages a wider
    // box so that 128x128 ROIs at any column take the TMA path (crop stacks keep the
    // 128-wide boxes).
    const bool frame = geom.width >= l59::Layout<true>::kGreyW;
    // crop stacks of 64x64, 100x100 or 200x200 images (8x8 cells, 59 bins, grey codes): the
    // tile variant of the TMA kernel (two 64-px crops per warp row / one 100-px crop / four
    // 200-px quadrant tiles)
    if (!depth_source && !small_batch && bins == 59 && cells_x == 8 && cells_y == 8 &&
        geom.width == geom.height &&
        (geom.width == 64 || geom.width == 100 || geom.width == 200) &&
        tile_path_applicable(geom, grey, depth) &&
        // whole rows leave the 64-px tiles by bulk copies (16 B), the 200-px quadrants' runs
        // of 4 cells by 8-B stores
        (reinterpret_cast<uintptr_t>(desc) & 15) == 0 && ((desc_stride * 2) & 15) == 0) {
        const cudaError_t e =
            geom.width == 64
                ? launch_lbp_hist_tile<64>(grey, depth, geom, rois, n_rois, win, desc, desc_stride,
                                           roi_status, num_sms(), stream)
            : geom.width == 100
                ? launch_lbp_hist_tile<100>(grey, depth, geom, rois, n_rois, win, desc,
                                            desc_stride, roi_status, num_sms(), stream)
                : launch_lbp_hist_tile<200>(grey, depth, geom, rois, n_rois, win, desc,
                                            desc_stride, roi_status, num_sms(), stream);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    if (!depth_source && !small_batch) {
        // Fast path (8x8 cells, 16-B aligned rows): one TMA-staged persistent kernel; ROIs
        // that are not fully-inside 128x128 boxes take the generic code path inside it.
        if (fast_path_applicable(geom, grey, depth, cells_x, cells_y, bins, desc) &&
            ((desc_stride * 2) & 15) == 0) {
            // conflict-free lane-private kernels (59 bins: the headline configuration).
            // cudaErrorNotSupported = refused on the host before any launch (a tensor map
            // that cannot be encoded, a shared-memory layout that does not fit): the generic
            // kernel below takes the batch.
            const cudaError_t e =
                bins == 59 ? launch_lbp_hist_lane59(grey, depth, geom, rois, n_rois, win, desc,
                                                    desc_stride, roi_status, num_sms(), stream,
                                                    false, frame)
                           : launch_lbp_hist_lane256(grey, depth, geom, rois, n_rois, win, desc,
                                                     desc_stride, roi_status, num_sms(), stream);
            if (e != cudaErrorNotSupported) return launch_status(e);
        }
    }
    // depth source, headline geometry: the same TMA kernel with the codes on the depth tile
    // (exact while dmax <= 0x7BFE, see lbp_hist_lane59.cuh)
    if (depth_source && !small_batch && bins == 59 && win.span + win.lo <= 0x7BFEu &&
        !win.none_valid &&
        fast_path_applicable(geom, nullptr, depth, cells_x, cells_y, bins, desc) &&
        ((desc_stride * 2) & 15) == 0) {
        const cudaError_t e = launch_lbp_hist_lane59(grey, depth, geom, rois, n_rois, win, desc,
                                                     desc_stride, roi_status, num_sms(), stream,
                                                     true, frame);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    // one CTA per (ROI, cell row) unit, grid-strided; 512 threads when the batch is small and
    // the images tall (the frame-stream config: one interior row per warp)
    const int grid = (int)std::min<int64_t>((int64_t)n_rois * cells_y, (int64_t)num_sms() * 8);
    const bool wide = (int64_t)n_rois * cells_y < 2 * num_sms() && geom.height >= 128;
    auto band = [&](auto plane) {
        using T = typename std::remove_const<
            typename std::remove_pointer<decltype(plane.base)>::type>::type;
        auto k = bins == 59 ? (wide ? lbp_hist_generic_kernel<59, T, 512>
                                    : lbp_hist_generic_kernel<59, T, kGenericThreads>)
                            : (wide ? lbp_hist_generic_kernel<256, T, 512>
                                    : lbp_hist_generic_kernel<256, T, kGenericThreads>);
        k<<<grid, wide ? 512 : kGenericThreads, 0, stream>>>(plane, depth, geom, rois, n_rois, win,
                                                           cells_x, cells_y, desc, desc_stride,
                                                           roi_status);
    };
    if (depth_source)
        band(CodePlane<uint16_t>{depth, geom.depth_pitch, geom.depth_img_stride});
    else
        band(CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride});
    return launch_status(cudaGetLastError());
}

}  // namespace

extern "C" {

int32_t lbp_extract_source(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                           const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins, int32_t source,
                           uint16_t* desc, int32_t* roi_status, lbp_stream_t stream_) {
    if (n_rois < 0) return LBP_E_ARG;
    if (source != LBP_SRC_GREY && source != LBP_SRC_DEPTH && source != LBP_SRC_FUSED)
        return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (source == LBP_SRC_FUSED && dim > 0x3FFFFFFF) return LBP_E_ARG;
    if (dmin > dmax) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    const bool need_grey = source != LBP_SRC_DEPTH, need_depth = source != LBP_SRC_GREY;
    if (!rois || !desc || (need_grey && !grey) || (need_depth && !depth)) return LBP_E_ARG;
    int32_t st = check_geometry(geom, need_grey, depth != nullptr);
    if (st != LBP_OK) return st;
    cudaStream_t stream = (cudaStream_t)stream_;
    const DepthWindow win = make_window(dmin, dmax);
    const int64_t stride = source == LBP_SRC_FUSED ? 2 * (int64_t)dim : dim;
    // grey || depth in ONE pass of the TMA kernel (both code planes of one staged tile, depth
    // read from HBM once) for crop stacks of the headline geometry; else two blocks
    if (source == LBP_SRC_FUSED && n_rois >= num_sms() && bins == 59 &&
        geom.width < l59::Layout<true>::kGreyW &&
        fast_path_applicable(geom, grey, depth, cells_x, cells_y, bins, desc)) {
        const cudaError_t e = launch_lbp_hist_lane59(grey, depth, geom, rois, n_rois, win, desc,
                                                     stride, roi_status, num_sms(), stream, false,
                                                     false, nullptr, nullptr, nullptr, true);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    if (need_grey) {
        st = extract_block(grey, depth, false, geom, rois, n_rois, win, cells_x, cells_y, bins,
                           desc, stride, roi_status, stream);
        if (st != LBP_OK) return st;
    }
    if (need_depth)
        st = extract_block(grey, depth, true, geom, rois, n_rois, win, cells_x, cells_y, bins,
                           desc + (source == LBP_SRC_FUSED ? dim : 0), stride, roi_status, stream);
    return st;
}

int32_t lbp_extract_resized(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                            const lbp_roi_t* rois, int32_t n_rois, int32_t size, uint16_t dmin,
                            uint16_t dmax, int32_t cells_x, int32_t cells_y, int32_t bins,
                            int32_t source, uint16_t* desc, int32_t* roi_status,
                            lbp_stream_t stream_) {
    if (n_rois < 0 || size < 3 || size > kResizeMaxSize) return LBP_E_ARG;
    if (source != LBP_SRC_GREY && source != LBP_SRC_DEPTH && source != LBP_SRC_FUSED)
        return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (source == LBP_SRC_FUSED && dim > 0x3FFFFFFF) return LBP_E_ARG;
    if (dmin > dmax) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    const bool need_grey = source != LBP_SRC_DEPTH, need_depth = source != LBP_SRC_GREY;
    if (!rois || !desc || (need_grey && !grey) || (need_depth && !depth)) return LBP_E_ARG;
    int32_t st = check_geometry(geom, need_grey, depth != nullptr);
    if (st != LBP_OK) return st;
    if (geom.width > (1 << 20) || geom.height > (1 << 20)) return LBP_E_UNSUPPORTED;
    cudaStream_t stream = (cudaStream_t)stream_;
    const DepthWindow win = make_window(dmin, dmax);
    const int64_t stride = source == LBP_SRC_FUSED ? 2 * (int64_t)dim : dim;
    const int grid = (int)std::min<int64_t>((int64_t)n_rois * cells_y, (int64_t)num_sms() * 8);
    const uint8_t* g = need_grey ? grey : nullptr;
#define LBPF_RESIZE_LAUNCH(B, SRCV)                                                          \
    lbp_hist_resize_kernel<B, SRCV><<<grid, kResizeThreads, 0, stream>>>(                  \
        g, depth, geom, rois, n_rois, size, win, cells_x, cells_y, desc, stride, roi_status)
    if (bins == 59) {
        if (source == LBP_SRC_GREY) LBPF_RESIZE_LAUNCH(59, 0);
        else if (source == LBP_SRC_DEPTH) LBPF_RESIZE_LAUNCH(59, 1);
        else LBPF_RESIZE_LAUNCH(59, 2);
    } else {
        if (source == LBP_SRC_GREY) LBPF_RESIZE_LAUNCH(256, 0);
        else if (source == LBP_SRC_DEPTH) LBPF_RESIZE_LAUNCH(256, 1);
        else LBPF_RESIZE_LAUNCH(256, 2);
    }
#undef LBPF_RESIZE_LAUNCH
    return launch_status(cudaGetLastError());
}

int32_t lbp_recognize(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                      const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                      int32_t cells_x, int32_t cells_y, int32_t bins, const float* W,
                      const float* bias, int32_t n_classes, const void* prepared,
                      size_t prepared_bytes, float reject_threshold, uint16_t* desc,
                      int32_t* roi_status, float* scores, int32_t* labels, float* top_score,
                      lbp_stream_t stream_) {
    if (n_rois < 0 || n_classes < 1) return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (prepared && prepared_bytes < svm_workspace_bytes(n_classes, dim)) return LBP_E_ARG;
    if (dmin > dmax) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    if (!grey || !rois || !desc || !W || !bias) return LBP_E_ARG;
    int32_t st = check_geometry(geom, true, depth != nullptr);
    if (st != LBP_OK) return st;
    cudaStream_t stream = (cudaStream_t)stream_;
    // small batches: one launch, a cluster of cells_y CTAs per ROI (extract + score via DSMEM)
    if (n_rois < num_sms() && cells_y <= kRecMaxCluster && n_classes <= kRecMaxClasses &&
        (int64_t)n_rois * cells_y <= 0x7FFFFFFF) {
        const DepthWindow win = make_window(dmin, dmax);
        return launch_status(launch_lbp_recognize_cluster(
            grey, depth, geom, rois, n_rois, win, cells_x, cells_y, bins, desc, roi_status, W,
            bias, n_classes, scores, labels, top_score, reject_threshold, stream));
    }
    st = lbp_extract_source(grey, depth, geom, rois, n_rois, dmin, dmax, cells_x, cells_y, bins,
                            LBP_SRC_GREY, desc, roi_status, stream_);
    if (st != LBP_OK) return st;
    return svm_score(desc, n_rois, dim, W, bias, n_classes, prepared, prepared_bytes, scores,
                     labels, top_score, reject_threshold, stream_);
}

int32_t lbp_extract_gather(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                           const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins,
                           const int32_t* labels, lbp_gather_dst_t dst, uint16_t* scratch,
                           int32_t* roi_status, lbp_stream_t stream_) {
    if (n_rois < 0) return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (dmin > dmax) return LBP_E_ARG;
    if (dst.mode == LBP_GATHER_MULTIMEM) {
        if (dst.n_dst != 1) return LBP_E_ARG;
    } else if (dst.mode == LBP_GATHER_PEERS) {
        if (dst.n_dst < 1 || dst.n_dst > LBP_GATHER_MAX_DST) return LBP_E_ARG;
    } else {
        return LBP_E_ARG;
    }
    for (int r = 0; r < dst.n_dst; ++r)
        if (dst.base[r] == 0 || (dst.base[r] & 15)) return LBP_E_ARG;
    if (dst.desc_offset < 0 || (dst.desc_offset & 15) || dst.desc_pitch < dim ||
        (dst.desc_pitch & 7) || dst.row_base < 0)
        return LBP_E_ARG;
    if (dst.labels_offset >= 0 && (dst.labels_offset & 3)) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    if (!grey || !rois || !scratch) return LBP_E_ARG;
    int32_t st = check_geometry(geom, true, depth != nullptr);
    if (st != LBP_OK) return st;
    cudaStream_t stream = (cudaStream_t)stream_;
    const DepthWindow win = make_window(dmin, dmax);
    // fused: the headline TMA kernel writes every row from its epilogue (crop stacks; frames
    // wider than a crop, small batches and other geometries take extraction + forwarding)
    const bool frame = geom.width >= l59::Layout<true>::kGreyW;
    if (n_rois >= num_sms() && bins == 59 && !frame &&
        fast_path_applicable(geom, grey, depth, cells_x, cells_y, bins, scratch)) {
        const cudaError_t e = launch_lbp_hist_lane59(grey, depth, geom, rois, n_rois, win, scratch,
                                                     dim, roi_status, num_sms(), stream, false,
                                                     false, &dst, labels);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    st = lbp_extract_source(grey, depth, geom, rois, n_rois, dmin, dmax, cells_x, cells_y, bins,
                            LBP_SRC_GREY, scratch, roi_status, stream_);
    if (st != LBP_OK) return st;
    const int grid = (int)std::min<int64_t>(((int64_t)n_rois * 32 + 255) / 256,
                                            (int64_t)num_sms() * 8);
    lbp_gather_forward_kernel<<<grid, 256, 0, stream>>>(scratch, n_rois, dim, labels, dst);
    return launch_status(cudaGetLastError());
}

int32_t lbp_u8_exc_cap_min(lbp_images_t geom, int32_t dim) {
    if (dim < 1 || geom.width < 1 || geom.height < 1) return LBP_E_ARG;
    const int64_t inner = (int64_t)std::max(geom.width - 2, 0) * std::max(geom.height - 2, 0);
    return (int32_t)std::min<int64_t>(inner / 256, dim);
}

int32_t lbp_extract_u8(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                       const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                       int32_t cells_x, int32_t cells_y, int32_t bins, uint8_t* packed,
                       int64_t pitch, int32_t* exc_n, uint32_t* exc, int32_t exc_cap,
                       uint16_t* scratch, int32_t* roi_status, lbp_stream_t stream_) {
    if (n_rois < 0) return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (dim > 65535 || pitch < dim || dmin > dmax) return LBP_E_ARG;
    int32_t st = check_geometry(geom, true, depth != nullptr);
    if (st != LBP_OK) return st;
    if (exc_cap < lbp_u8_exc_cap_min(geom, dim)) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    if (!grey || !rois || !packed || !exc_n || (exc_cap > 0 && !exc)) return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    const DepthWindow win = make_window(dmin, dmax);
    const bool frame = geom.width >= l59::Layout<true>::kGreyW;
    if (n_rois >= num_sms() && bins == 59 && !frame && (pitch & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(packed) & 15) == 0 &&
        fast_path_applicable(geom, grey, depth, cells_x, cells_y, bins, nullptr)) {
        const U8Out uo{packed, exc_n, exc, exc_cap, pitch};
        const cudaError_t e = launch_lbp_hist_lane59(grey, depth, geom, rois, n_rois, win,
                                                     nullptr, 0, roi_status, num_sms(), stream,
                                                     false, false, nullptr, nullptr, &uo);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    if (!scratch) return LBP_E_ARG;
    st = lbp_extract_source(grey, depth, geom, rois, n_rois, dmin, dmax, cells_x, cells_y, bins,
                            LBP_SRC_GREY, scratch, roi_status, stream_);
    if (st != LBP_OK) return st;
    const int grid = (int)std::min<int64_t>(((int64_t)n_rois * 32 + 255) / 256,
                                            (int64_t)num_sms() * 8);
    desc_pack_rows_kernel<<<grid, 256, 0, stream>>>(scratch, n_rois, dim, packed, pitch, exc_n,
                                                     exc, exc_cap);
    return launch_status(cudaGetLastError());
}

int32_t lbp_fused_extract(const uint8_t* grey, const uint16_t* depth, lbp_images_t geom,
                          const lbp_roi_t* rois, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                          int32_t cells_x, int32_t cells_y, int32_t bins, uint16_t* desc,
                          int32_t* roi_status, lbp_stream_t stream) {
    return lbp_extract_source(grey, depth, geom, rois, n_rois, dmin, dmax, cells_x, cells_y, bins,
                              LBP_SRC_GREY, desc, roi_status, stream);
}

int32_t svm_score(const uint16_t* desc, int32_t n, int32_t dim, const float* W, const float* bias,
                  int32_t n_classes, const void* prepared, size_t prepared_bytes, float* scores,
                  int32_t* labels, float* top_score, float reject_threshold,
                  lbp_stream_t stream_) {
    if (n < 0 || dim < 1 || n_classes < 1) return LBP_E_ARG;
    if (prepared && prepared_bytes < svm_workspace_bytes(n_classes, dim)) return LBP_E_ARG;
    if (n == 0) return LBP_OK;
    if (!desc || !W || !bias) return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    // Tensor-core path: exact integer digit-plane GEMM (needs svm_prepare()'s workspace);
    // below one 128-crop tile the CUDA-core kernel has the lower latency.
    SvmPrepHeader h;
    if (prepared && n >= kGemmM && svm_choose_layout(n_classes, dim, &h) &&
        (reinterpret_cast<uintptr_t>(desc) & 15) == 0) {
        cudaError_t e = h.magic == kPrep8Magic
                            ? launch_svm_gemm_i8(desc, n, dim, W, bias, h, (const uint8_t*)prepared,
                                                 scores, labels, top_score, reject_threshold,
                                                 num_sms(), stream)
                            : launch_svm_gemm(desc, n, dim, W, bias, h, (const uint8_t*)prepared,
                                              scores, labels, top_score, reject_threshold,
                                              num_sms(), stream);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    // CUDA-core path: exact fp64 accumulation; 8 crops per CTA, 1 for tiny batches
    if (n < 8) {
        svm_score_fp64_kernel<false, 1, 1024><<<n, 1024, 0, stream>>>(
            desc, n, dim, W, bias, n_classes, scores, labels, top_score, reject_threshold);
        return launch_status(cudaGetLastError());
    }
    const int grid = (int)((n + kSvmRowsMax - 1) / kSvmRowsMax);
    const size_t smem = (size_t)kSvmRowsMax * dim * sizeof(float);
    if (smem <= 200 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(svm_score_fp64_kernel<true, kSvmRowsMax>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return launch_status(e);
        svm_score_fp64_kernel<true, kSvmRowsMax><<<grid, kSvmThreads, smem, stream>>>(
            desc, n, dim, W, bias, n_classes, scores, labels, top_score, reject_threshold);
    } else {
        svm_score_fp64_kernel<false, kSvmRowsMax><<<grid, kSvmThreads, 0, stream>>>(
            desc, n, dim, W, bias, n_classes, scores, labels, top_score, reject_threshold);
    }
    return launch_status(cudaGetLastError());
}

int32_t svm_score_l1(const uint16_t* desc, int32_t n, int32_t dim, int32_t block, const float* W,
                     const float* bias, int32_t n_classes, float* scores, int32_t* labels,
                     float* top_score, float reject_threshold, lbp_stream_t stream_) {
    if (n < 0 || dim < 1 || n_classes < 1 || block < 1 || dim % block != 0) return LBP_E_ARG;
    if (n == 0) return LBP_OK;
    if (!desc || !W || !bias) return LBP_E_ARG;
    const int nblk = dim / block;
    auto smem_for = [&](int rows) {
        return (size_t)rows * dim * sizeof(float) + 8 + (size_t)rows * nblk * sizeof(double);
    };
    cudaStream_t stream = (cudaStream_t)stream_;
    if (smem_for(kSvmRowsMax) <= 200 * 1024) {  // 8 crops per CTA
        const size_t smem = smem_for(kSvmRowsMax);
        cudaError_t e = cudaFuncSetAttribute(svm_score_l1_kernel<kSvmRowsMax>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return launch_status(e);
        const int grid = (int)((n + kSvmRowsMax - 1) / kSvmRowsMax);
        svm_score_l1_kernel<kSvmRowsMax><<<grid, kSvmThreads, smem, stream>>>(
            desc, n, dim, block, W, bias, n_classes, scores, labels, top_score, reject_threshold);
        return launch_status(cudaGetLastError());
    }
    if (smem_for(1) > 200 * 1024) return LBP_E_UNSUPPORTED;
    cudaError_t e = cudaFuncSetAttribute(svm_score_l1_kernel<1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_for(1));
    if (e != cudaSuccess) return launch_status(e);
    svm_score_l1_kernel<1><<<n, kSvmThreads, smem_for(1), stream>>>(
        desc, n, dim, block, W, bias, n_classes, scores, labels, top_score, reject_threshold);
    return launch_status(cudaGetLastError());
}

int32_t svm_train_ovr(const uint16_t* desc, int32_t n, int32_t dim, const int32_t* labels,
                      int32_t n_classes, const int32_t* order, int64_t T, int32_t inv_lambda,
                      float* W, float* bias, int64_t* z_out, lbp_stream_t stream_) {
    if (n < 1 || dim < 1 || n_classes < 1 || T < 1 || inv_lambda < 1) return LBP_E_ARG;
    if (T > (int64_t(1) << 31)) return LBP_E_ARG;
    if (!desc || !labels || !order || !W || !bias) return LBP_E_ARG;
    if (dim > kTrainMaxDim) return LBP_E_UNSUPPORTED;
    cudaStream_t stream = (cudaStream_t)stream_;
    // even dim, 4-B aligned rows: z in registers, one barrier per step (svm_train.cuh)
    if ((dim & 1) == 0 && (reinterpret_cast<uintptr_t>(desc) & 3) == 0) {
        const bool z32 = T * 65535 < (int64_t(1) << 31);  // |z_T[d]| <= T * 65535
        if (dim <= 2 * 256 * 8) {
            auto k = z32 ? svm_train_ovr_reg_kernel<256, 8, true>
                         : svm_train_ovr_reg_kernel<256, 8, false>;
            k<<<std::min(n_classes, 4 * num_sms()), 256, 0, stream>>>(
                desc, n, dim, labels, n_classes, order, T, inv_lambda, W, bias, z_out);
        } else {
            auto k = z32 ? svm_train_ovr_reg_kernel<1024, 8, true>
                         : svm_train_ovr_reg_kernel<1024, 8, false>;
            k<<<std::min(n_classes, 2 * num_sms()), 1024, 0, stream>>>(
                desc, n, dim, labels, n_classes, order, T, inv_lambda, W, bias, z_out);
        }
        return launch_status(cudaGetLastError());
    }
    const size_t smem = (size_t)(dim + 1) * sizeof(int64_t);
    if (dim <= 256 * 16) {  // 59-bin descriptors: 256 threads x 16 entries (cheaper barriers)
        auto k = svm_train_ovr_kernel<256, 16>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return launch_status(e);
        k<<<std::min(n_classes, 4 * num_sms()), 256, smem, stream>>>(
            desc, n, dim, labels, n_classes, order, T, inv_lambda, W, bias, z_out);
        return launch_status(cudaGetLastError());
    }
    auto k = svm_train_ovr_kernel<1024, 16>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return launch_status(e);
    k<<<std::min(n_classes, 2 * num_sms()), 1024, smem, stream>>>(
        desc, n, dim, labels, n_classes, order, T, inv_lambda, W, bias, z_out);
    return launch_status(cudaGetLastError());
}

int32_t lbp_desc_pack_u8(const uint16_t* desc, int64_t n, int32_t dim, int64_t row_base,
                         uint8_t* packed, lbp_desc_exc_t* exc, int32_t exc_cap,
                         int32_t* exc_count, lbp_stream_t stream_) {
    if (n < 0 || dim < 1 || exc_cap < 0 || !exc_count) return LBP_E_ARG;
    if (n > 0 && (!desc || !packed || (exc_cap > 0 && !exc))) return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    cudaError_t e = cudaMemsetAsync(exc_count, 0, sizeof(int32_t), stream);
    if (e != cudaSuccess) return launch_status(e);
    if (n == 0) return LBP_OK;
    const int64_t total = n * (int64_t)dim;
    const bool vec = ((reinterpret_cast<uintptr_t>(desc) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(packed) & 7) == 0);
    const int64_t work = vec ? (total >> 3) + 8 : total;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((work + kPackThreads - 1) / kPackThreads, (int64_t)num_sms() * 8));
    if (vec)
        desc_pack_u8_kernel<true><<<grid, kPackThreads, 0, stream>>>(
            desc, total, dim, row_base, packed, exc, exc_cap, exc_count);
    else
        desc_pack_u8_kernel<false><<<grid, kPackThreads, 0, stream>>>(
            desc, total, dim, row_base, packed, exc, exc_cap, exc_count);
    return launch_status(cudaGetLastError());
}

int32_t lbp_desc_unpack_u8(const uint8_t* packed, int64_t n, int32_t dim, int64_t row_base,
                           const lbp_desc_exc_t* exc, const int32_t* exc_counts, int32_t n_lists,
                           int32_t exc_cap, uint16_t* desc, lbp_stream_t stream_) {
    if (n < 0 || dim < 1 || n_lists < 0 || exc_cap < 0) return LBP_E_ARG;
    if (n == 0) return LBP_OK;
    if (!packed || !desc || (n_lists > 0 && exc_cap > 0 && (!exc || !exc_counts)))
        return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    const int64_t total = n * (int64_t)dim;
    const bool vec = ((reinterpret_cast<uintptr_t>(desc) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(packed) & 7) == 0);
    const int64_t work = vec ? (total >> 3) + 8 : total;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((work + kPackThreads - 1) / kPackThreads, (int64_t)num_sms() * 8));
    if (vec)
        desc_unpack_u8_kernel<true><<<grid, kPackThreads, 0, stream>>>(packed, total, desc);
    else
        desc_unpack_u8_kernel<false><<<grid, kPackThreads, 0, stream>>>(packed, total, desc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return launch_status(e);
    const int64_t recs = (int64_t)n_lists * exc_cap;
    if (recs == 0) return LBP_OK;
    const int sgrid = (int)std::min<int64_t>((recs + kPackThreads - 1) / kPackThreads,
                                             (int64_t)num_sms() * 4);
    desc_exc_scatter_kernel<<<sgrid, kPackThreads, 0, stream>>>(exc, exc_counts, n_lists, exc_cap,
                                                                row_base, n, dim, desc);
    return launch_status(cudaGetLastError());
}

#ifdef LBP_SVM_TRACE  // developer builds only (not declared in the public header)
int32_t lbp_debug_svm_trace(unsigned long long* out32) {
    return cudaMemcpyFromSymbol(out32, g_svm_trace, sizeof(g_svm_trace)) == cudaSuccess ? 0 : -1;
}
#endif

size_t svm_workspace_bytes(int32_t n_classes, int32_t dim) {
    SvmPrepHeader h;
    if (!svm_choose_layout(n_classes, dim, &h)) return 0;
    return svm_layout_total(h);
}

int32_t svm_prepare(const float* W, int32_t n_classes, int32_t dim, void* workspace,
                    size_t workspace_bytes, lbp_stream_t stream) {
    if (!W || !workspace || n_classes < 1 || dim < 1) return LBP_E_ARG;
    SvmPrepHeader h;
    if (!svm_choose_layout(n_classes, dim, &h)) return LBP_E_UNSUPPORTED;
    if (workspace_bytes < svm_layout_total(h)) return LBP_E_ARG;
    if (h.magic == kPrep8Magic)
        svm_prepare_i8_kernel<<<h.total_rows, 256, 0, (cudaStream_t)stream>>>(W, h,
                                                                             (uint8_t*)workspace);
    else
        svm_prepare_kernel<<<h.total_rows, 256, 0, (cudaStream_t)stream>>>(W, h,
                                                                          (uint8_t*)workspace);
    return launch_status(cudaGetLastError());
}

size_t svm_workspace_u8_bytes(int32_t n_classes, int32_t dim) {
    SvmPrepHeader h;
    if (!svm_layout_u8(n_classes, dim, &h)) return 0;
    return svm_layout_u8_total(h);
}

int32_t svm_prepare_u8(const float* W, int32_t n_classes, int32_t dim, void* workspace,
                       size_t workspace_bytes, lbp_stream_t stream) {
    if (!W || !workspace || n_classes < 1 || dim < 1) return LBP_E_ARG;
    SvmPrepHeader h;
    if (!svm_layout_u8(n_classes, dim, &h)) return LBP_E_UNSUPPORTED;
    if (workspace_bytes < svm_layout_u8_total(h)) return LBP_E_ARG;
    svm_prepare_u8_kernel<kU8Digits><<<h.total_rows, 256, 0, (cudaStream_t)stream>>>(
        W, h, (uint8_t*)workspace);
    const U8Layout L4 = u8_layout(n_classes, 4);
    svm_prepare_u8_kernel<4><<<L4.N * L4.n_pass, 256, 0, (cudaStream_t)stream>>>(
        W, h, (uint8_t*)workspace);
    return launch_status(cudaGetLastError());
}

int32_t svm_score_u8(const uint8_t* packed, int64_t pitch, const int32_t* exc_n,
                     const uint32_t* exc, int32_t exc_cap, int32_t n, int32_t dim,
                     const float* W, const float* bias, int32_t n_classes, const void* prepared,
                     size_t prepared_bytes, float* scores, int32_t* labels, float* top_score,
                     float reject_threshold, lbp_stream_t stream_) {
    if (n < 0 || dim < 1 || dim > 65535 || n_classes < 1 || pitch < dim || exc_cap < 0)
        return LBP_E_ARG;
    if (prepared && prepared_bytes < svm_workspace_u8_bytes(n_classes, dim)) return LBP_E_ARG;
    if (n == 0) return LBP_OK;
    if (!packed || !exc_n || (exc_cap > 0 && !exc) || !W || !bias) return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    SvmPrepHeader h;
    if (prepared && n >= kGemmM && svm_layout_u8(n_classes, dim, &h) && (pitch & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(packed) & 15) == 0) {
        const cudaError_t e = launch_svm_gemm_u8(packed, pitch, exc_n, exc, exc_cap, n, dim, W,
                                                 bias, h, (const uint8_t*)prepared, scores,
                                                 labels, top_score, reject_threshold, num_sms(),
                                                 stream);
        if (e != cudaErrorNotSupported) return launch_status(e);
    }
    const size_t smem = (size_t)dim * sizeof(float);
    if (smem > 200 * 1024) return LBP_E_UNSUPPORTED;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            svm_score_u8_fp64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return launch_status(e);
    }
    const int grid = (int)std::min<int64_t>(n, (int64_t)num_sms() * 8);
    svm_score_u8_fp64_kernel<<<grid, kU8F64Threads, smem, stream>>>(
        packed, pitch, exc_n, exc, exc_cap, n, dim, W, bias, n_classes, scores, labels,
        top_score, reject_threshold);
    return launch_status(cudaGetLastError());
}

// --------------------------------------------------------------------------
// end-to-end entry point from host buffers
// --------------------------------------------------------------------------
namespace {
struct RecognizeLayout {
    size_t grey_off, grey_bytes, depth_off, depth_bytes, rois_off, rois_bytes;
    size_t desc_off, desc_bytes, labels_off, top_off, total;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

RecognizeLayout recognize_layout(const lbp_images_t& g, bool has_depth, int32_t n_rois,
                                 int32_t dim) {
    RecognizeLayout L{};
    L.grey_bytes = (size_t)(g.grey_img_stride * (g.n_images - 1) + g.grey_pitch * (g.height - 1) +
                            g.width);
    L.depth_bytes = has_depth ? 2 * (size_t)(g.depth_img_stride * (g.n_images - 1) +
                                             g.depth_pitch * (g.height - 1) + g.width)
                              : 0;
    L.rois_bytes = (size_t)n_rois * sizeof(lbp_roi_t);
    L.desc_bytes = (size_t)n_rois * dim * sizeof(uint16_t);
    size_t o = 0;
    L.grey_off = o;
    o = align256(o + L.grey_bytes);
    L.depth_off = o;
    o = align256(o + L.depth_bytes);
    L.rois_off = o;
    o = align256(o + L.rois_bytes);
    L.desc_off = o;
    o = align256(o + L.desc_bytes);
    L.labels_off = o;
    o = align256(o + (size_t)n_rois * 4);
    L.top_off = o;
    o = align256(o + (size_t)n_rois * 4);
    L.total = o;
    return L;
}
}  // namespace

size_t lbp_recognize_workspace_bytes(lbp_images_t geom, int32_t has_depth, int32_t n_rois,
                                     int32_t cells_x, int32_t cells_y, int32_t bins) {
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0 || n_rois < 0 || check_geometry(geom, true, has_depth != 0) != LBP_OK) return 0;
    return recognize_layout(geom, has_depth != 0, n_rois, dim).total;
}

int32_t lbp_recognize_host(const uint8_t* grey_h, const uint16_t* depth_h, lbp_images_t geom,
                           const lbp_roi_t* rois_h, int32_t n_rois, uint16_t dmin, uint16_t dmax,
                           int32_t cells_x, int32_t cells_y, int32_t bins, const float* W,
                           const float* bias, int32_t n_classes, const void* prepared,
                           size_t prepared_bytes, float reject_threshold, void* workspace,
                           size_t workspace_bytes, int32_t* labels_h, float* top_h,
                           lbp_stream_t stream_) {
    if (n_rois < 0 || n_classes < 1) return LBP_E_ARG;
    const int32_t dim = lbp_descriptor_dim(cells_x, cells_y, bins);
    if (dim < 0) return dim;
    if (dmin > dmax) return LBP_E_ARG;
    if (n_rois == 0) return LBP_OK;
    if (!grey_h || !rois_h || !W || !bias || !workspace) return LBP_E_ARG;
    int32_t st = check_geometry(geom, true, depth_h != nullptr);
    if (st != LBP_OK) return st;
    const RecognizeLayout L = recognize_layout(geom, depth_h != nullptr, n_rois, dim);
    if (workspace_bytes < L.total) return LBP_E_ARG;
    cudaStream_t stream = (cudaStream_t)stream_;
    char* ws = (char*)workspace;
    uint8_t* grey = (uint8_t*)(ws + L.grey_off);
    uint16_t* depth = depth_h ? (uint16_t*)(ws + L.depth_off) : nullptr;
    lbp_roi_t* rois = (lbp_roi_t*)(ws + L.rois_off);
    uint16_t* desc = (uint16_t*)(ws + L.desc_off);
    int32_t* labels = (int32_t*)(ws + L.labels_off);
    float* top = (float*)(ws + L.top_off);
    cudaError_t e = cudaMemcpyAsync(grey, grey_h, L.grey_bytes, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && depth_h)
        e = cudaMemcpyAsync(depth, depth_h, L.depth_bytes, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(rois, rois_h, L.rois_bytes, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return LBP_E_CUDA;
    st = lbp_fused_extract(grey, depth, geom, rois, n_rois, dmin, dmax, cells_x, cells_y, bins,
                           desc, nullptr, stream_);
    if (st != LBP_OK) return st;
    st = svm_score(desc, n_rois, dim, W, bias, n_classes, prepared, prepared_bytes, nullptr,
                   labels, top, reject_threshold, stream_);
    if (st != LBP_OK) return st;
    if (labels_h) e = cudaMemcpyAsync(labels_h, labels, (size_t)n_rois * 4, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess && top_h)
        e = cudaMemcpyAsync(top_h, top, (size_t)n_rois * 4, cudaMemcpyDeviceToHost, stream);
    return e == cudaSuccess ? LBP_OK : LBP_E_CUDA;
}

}  // extern "C"

