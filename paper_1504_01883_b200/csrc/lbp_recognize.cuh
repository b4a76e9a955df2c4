// lbp_recognize.cuh -- extraction + linear-SVM scoring fused into ONE launch for small batches
// (the frame-stream and single-crop latency configs; SURVEY §8f-3 "fused extract -> score").
//
// A thread-block cluster of cells_y CTAs serves one ROI: CTA r (cluster rank r) computes the
// histograms of cell row r exactly as the band kernel (extract_roi_generic over the cells of
// that row) and writes them to the descriptor, then the partial decision values of every
// class over its own 472 (cells_x * bins) descriptor entries -- u16 x fp32 products exact in
// fp64, summed in a fixed order.  After a cluster barrier, rank 0 reads the cells_y partials
// of each class from the other CTAs' shared memory (DSMEM, ld.shared::cluster), adds them in
// rank order plus the bias, rounds once to fp32 and takes the argmax (ties -> lowest class):
// the descriptor never makes an HBM round trip between two launches, and the two dependent
// launches of the unfused path become one.
#pragma once
#include "common.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"

namespace lbpf {

constexpr int kRecMaxClasses = 2048;          // fp64 partials in smem (16 KB)
constexpr int kRecMaxCluster = 8;             // portable cluster size: cells_y <= 8
constexpr int kRecPrefetch = 16;              // W entries per lane requested before extraction

__device__ __forceinline__ double ld_dsmem_f64(const double* local_ptr, uint32_t rank) {
    const uint32_t a = mapa_shared(smem_u32(local_ptr), rank);
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}

// NT threads per CTA: 512 (one interior row per warp for 128-px crops, where 256 threads
// left two dependent L2 round trips per warp: config2 11.9 -> 9.0 us) for tall images, 256
// for small crops (64x64: 7-8 rows per cell row)
template <int BINS, int NT>
__global__ void __launch_bounds__(NT)
lbp_recognize_cluster_kernel(const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                             lbp_images_t geom, const lbp_roi_t* __restrict__ rois,
                             int32_t n_rois, DepthWindow win, int32_t cells_x, int32_t cells_y,
                             uint16_t* __restrict__ desc, int32_t* __restrict__ roi_status,
                             const float* __restrict__ W, const float* __restrict__ bias,
                             int32_t n_classes, float* __restrict__ scores,
                             int32_t* __restrict__ labels, float* __restrict__ top_score,
                             float reject_threshold) {
    __shared__ uint32_t hist[kGenericHistCap];
    __shared__ uint8_t lut[256];
    __shared__ double part[kRecMaxClasses];
    __shared__ float wbest[NT / 32];
    __shared__ int wbest_c[NT / 32];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    constexpr int kWarps = NT / 32;
    for (int i = t; i < 256; i += NT) lut[i] = (BINS == 59) ? kUniformLutDev.v[i] : (uint8_t)i;
    const int used = min(kGenericHistCap / BINS, cells_x) * BINS;
    for (int i = t; i < used; i += NT) hist[i] = 0;
    __syncthreads();

    const uint32_t rank = cluster_ctarank();         // = cell row
    const int32_t n = (int32_t)cluster_id_x();       // ROI of this cluster
    const int32_t dim = cells_x * cells_y * BINS;
    const int32_t seg = cells_x * BINS, seg0 = (int32_t)rank * seg;

    // W of this warp's first class over the segment, requested before the extraction so the
    // loads overlap it (segments up to kRecPrefetch * 32 entries)
    float wpre[kRecPrefetch];
    const bool prefetch = seg <= kRecPrefetch * 32 && warp < n_classes;
    if (prefetch) {
        const float* w = W + (int64_t)warp * dim + seg0;
#pragma unroll
        for (int u = 0; u < kRecPrefetch; ++u) {
            const int k = lane + 32 * u;
            wpre[u] = k < seg ? __ldg(w + k) : 0.0f;
        }
    }
    // ---- histograms of cell row `rank` (writes desc[n][seg0, seg0 + seg) and, rank 0, the
    // status); when the row's counters fit one chunk they stay in smem for the scoring
    const bool keep = seg <= kGenericHistCap;
    const CodePlane<uint8_t> plane{grey, geom.grey_pitch, geom.grey_img_stride};
    if (keep)
        extract_roi_generic<BINS, NT, uint8_t, CtaSync, true>(
            plane, depth, geom, rois[n], n, win, cells_x, cells_y, desc, dim, roi_status, hist,
            kGenericHistCap, lut, 0, t, CtaSync{}, (int32_t)rank * cells_x,
            ((int32_t)rank + 1) * cells_x);
    else
        extract_roi_generic<BINS, NT>(
            plane, depth, geom, rois[n], n, win, cells_x, cells_y, desc, dim, roi_status, hist,
            kGenericHistCap, lut, 0, t, CtaSync{}, (int32_t)rank * cells_x,
            ((int32_t)rank + 1) * cells_x);
    __syncthreads();  // this CTA's counts are complete (smem) / its segment written (global)

    // ---- partial decision values over this segment: warp per class, fp64 (exact products)
    const uint16_t* x = desc + (int64_t)n * dim + seg0;
    auto xat = [&](int k) -> double { return keep ? (double)hist[k] : (double)x[k]; };
    for (int c = warp; c < n_classes; c += kWarps) {
        double acc = 0.0;
        if (prefetch && c == warp) {
#pragma unroll
            for (int u = 0; u < kRecPrefetch; ++u) {
                const int k = lane + 32 * u;
                if (k < seg) acc = fma((double)wpre[u], xat(k), acc);
            }
        } else {
            const float* w = W + (int64_t)c * dim + seg0;
            for (int k = lane; k < seg; k += 32) acc = fma((double)__ldg(w + k), xat(k), acc);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
        if (lane == 0) part[c] = acc;
    }
    cluster_sync();  // every CTA's partials are in its shared memory

    if (rank == 0) {
        // s[c] = fp32(b[c] + sum_r part_r[c]), ranks in order; argmax, ties -> lowest class
        float best = -INFINITY;
        int best_c = 0x7FFFFFFF;
        for (int c = t; c < n_classes; c += NT) {
            double acc = (double)__ldg(bias + c);
            for (int r = 0; r < cells_y; ++r) acc += ld_dsmem_f64(&part[c], (uint32_t)r);
            const float s = (float)acc;
            if (scores) scores[(int64_t)n * n_classes + c] = s;
            if (best_c == 0x7FFFFFFF || s > best) {  // c ascending within the thread
                best = s;
                best_c = c;
            }
        }
        // block argmax, ties -> lowest class
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
            const int oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, off);
            if (oc != 0x7FFFFFFF && (best_c == 0x7FFFFFFF || ob > best || (ob == best && oc < best_c))) {
                best = ob;
                best_c = oc;
            }
        }
        if (lane == 0) {
            wbest[warp] = best;
            wbest_c[warp] = best_c;
        }
        __syncthreads();
        if (t == 0) {
            float b = wbest[0];
            int bc = wbest_c[0];
            for (int w2 = 1; w2 < kWarps; ++w2) {
                const float ob = wbest[w2];
                const int oc = wbest_c[w2];
                if (oc != 0x7FFFFFFF && (bc == 0x7FFFFFFF || ob > b || (ob == b && oc < bc))) {
                    b = ob;
                    bc = oc;
                }
            }
            if (top_score) top_score[n] = b;
            if (labels) labels[n] = (b < reject_threshold) ? -1 : bc;
        }
    }
    cluster_sync();  // the partials stay alive until rank 0 has read them
}

inline cudaError_t launch_lbp_recognize_cluster(const uint8_t* grey, const uint16_t* depth,
                                                const lbp_images_t& geom, const lbp_roi_t* rois,
                                                int32_t n_rois, const DepthWindow& win,
                                                int32_t cells_x, int32_t cells_y, int32_t bins,
                                                uint16_t* desc, int32_t* roi_status,
                                                const float* W, const float* bias, int32_t C,
                                                float* scores, int32_t* labels, float* top,
                                                float reject, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_rois * cells_y), 1, 1);
    const bool tall = geom.height >= 128;
    cfg.blockDim = dim3(tall ? 512 : 256, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cells_y;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = bins == 59 ? (tall ? lbp_recognize_cluster_kernel<59, 512>
                                   : lbp_recognize_cluster_kernel<59, 256>)
                           : (tall ? lbp_recognize_cluster_kernel<256, 512>
                                   : lbp_recognize_cluster_kernel<256, 256>);
    return cudaLaunchKernelEx(&cfg, kern, grey, depth, geom, rois, n_rois, win, cells_x, cells_y,
                              desc, roi_status, W, bias, C, scores, labels, top, reject);
}

}  // namespace lbpf
