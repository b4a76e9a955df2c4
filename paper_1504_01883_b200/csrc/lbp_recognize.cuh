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

constexpr int kRecThreads = kGenericThreads;  // 256
constexpr int kRecMaxClasses = 2048;          // fp64 partials in smem (16 KB)
constexpr int kRecMaxCluster = 8;             // portable cluster size: cells_y <= 8

__device__ __forceinline__ double ld_dsmem_f64(const double* local_ptr, uint32_t rank) {
    const uint32_t a = mapa_shared(smem_u32(local_ptr), rank);
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}

template <int BINS>
__global__ void __launch_bounds__(kRecThreads)
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
    __shared__ float wbest[kRecThreads / 32];
    __shared__ int wbest_c[kRecThreads / 32];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    constexpr int kWarps = kRecThreads / 32;
    for (int i = t; i < 256; i += kRecThreads) lut[i] = (BINS == 59) ? kUniformLutDev.v[i] : (uint8_t)i;
    const int used = min(kGenericHistCap / BINS, cells_x) * BINS;
    for (int i = t; i < used; i += kRecThreads) hist[i] = 0;
    __syncthreads();

    const uint32_t rank = cluster_ctarank();         // = cell row
    const int32_t n = (int32_t)cluster_id_x();       // ROI of this cluster
    const int32_t dim = cells_x * cells_y * BINS;
    const int32_t seg = cells_x * BINS, seg0 = (int32_t)rank * seg;

    // ---- histograms of cell row `rank` (writes desc[n][seg0, seg0 + seg) and, rank 0, the status)
    extract_roi_generic<BINS, kRecThreads>(CodePlane<uint8_t>{grey, geom.grey_pitch,
                                                              geom.grey_img_stride},
                                           depth, geom, rois[n], n, win, cells_x, cells_y, desc,
                                           dim, roi_status, hist, kGenericHistCap, lut, 0, t,
                                           CtaSync{}, (int32_t)rank * cells_x,
                                           ((int32_t)rank + 1) * cells_x);
    __syncthreads();  // this CTA's descriptor segment is written (and visible to the CTA)

    // ---- partial decision values over this segment: warp per class, fp64 (exact products)
    const uint16_t* x = desc + (int64_t)n * dim + seg0;
    for (int c = warp; c < n_classes; c += kWarps) {
        const float* w = W + (int64_t)c * dim + seg0;
        double acc = 0.0;
        for (int k = lane; k < seg; k += 32) acc = fma((double)__ldg(w + k), (double)x[k], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
        if (lane == 0) part[c] = acc;
    }
    cluster_sync();  // every CTA's partials are in its shared memory

    if (rank == 0) {
        // s[c] = fp32(b[c] + sum_r part_r[c]), ranks in order; argmax, ties -> lowest class
        float best = -INFINITY;
        int best_c = 0x7FFFFFFF;
        for (int c = t; c < n_classes; c += kRecThreads) {
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
    cfg.blockDim = dim3(kRecThreads, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cells_y;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (bins == 59)
        return cudaLaunchKernelEx(&cfg, lbp_recognize_cluster_kernel<59>, grey, depth, geom, rois,
                                  n_rois, win, cells_x, cells_y, desc, roi_status, W, bias, C,
                                  scores, labels, top, reject);
    return cudaLaunchKernelEx(&cfg, lbp_recognize_cluster_kernel<256>, grey, depth, geom, rois,
                              n_rois, win, cells_x, cells_y, desc, roi_status, W, bias, C,
                              scores, labels, top, reject);
}

}  // namespace lbpf
