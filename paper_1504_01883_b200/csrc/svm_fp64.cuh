// svm_fp64.cuh -- CUDA-core linear-SVM scorer with exact fp64 accumulation.
//
// s[n][c] = fp32(b[c] + sum_d W[c][d] * h[n][d]): every product of a u16 count
// and an fp32 weight is exact in fp64 (16 + 24 significant bits), so the only
// rounding is the fp64 summation (relative 2^-53 per add) and the final
// fp32 rounding -- the oracle's definition up to summation order (SURVEY §8c
// step 8, "Score precision" reading).
//
// CTA = kSvmRows crops; its warps take (class, dimension slice) items round-robin; each
// lane strides the slice and keeps kSvmRows fp64 partial sums, reduced with warp shuffles;
// with few classes every class is split into slices so that all warps have loads in flight
// (a latency-bound kernel for the frame-stream / single-crop configs).  The descriptors of
// the CTA's crops are staged in shared memory as fp32 (counts <= 65535 are exact in fp32).
// Tiny batches use 1 crop and 1,024 threads per CTA.
#pragma once
#include "common.cuh"

namespace lbpf {

constexpr int kSvmThreads = 256;
constexpr int kSvmRowsMax = 8;  // crops per CTA (1 for tiny batches: latency)

__device__ __forceinline__ bool better(float s, int c, float best, int best_c) {
    // argmax over fp32 scores, ties -> lowest class index
    return s > best || (s == best && c < best_c);
}

template <bool kStage, int kSvmRows, int NT = kSvmThreads>
__global__ void __launch_bounds__(NT)
svm_score_fp64_kernel(const uint16_t* __restrict__ desc, int32_t n, int32_t dim,
                      const float* __restrict__ W, const float* __restrict__ bias,
                      int32_t n_classes, float* __restrict__ scores, int32_t* __restrict__ labels,
                      float* __restrict__ top_score, float reject_threshold) {
    extern __shared__ float xs[];  // [kSvmRows][dim]
    constexpr int kWarps = NT / 32;
    constexpr int kItems = 2 * kWarps;  // (class, slice) items when classes are few
    __shared__ float wbest[kWarps][kSvmRows];
    __shared__ int wbest_c[kWarps][kSvmRows];
    __shared__ double part[kItems][kSvmRows];  // [slice * C + class][row], few classes
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * kSvmRows;
    const int rows = (int)((n - row0) < kSvmRows ? (n - row0) : kSvmRows);

    if (kStage) {
        const uint16_t* src = desc + row0 * dim;
#pragma unroll 4
        for (int i = threadIdx.x; i < kSvmRows * dim; i += blockDim.x)
            xs[i] = i < rows * dim ? (float)__ldg(src + i) : 0.0f;
        __syncthreads();
    }
    // unstaged: rows past the end re-read the last valid row (results discarded)
    auto x = [&](int k, int d) -> double {
        if (kStage) return (double)xs[k * dim + d];
        return (double)__ldg(desc + (row0 + min(k, rows - 1)) * dim + d);
    };

    // work items (class, slice of the dimension): with fewer classes than 2x the warps each
    // class is split into S slices so that every warp has loads in flight
    const int S = n_classes >= kWarps ? 1 : kItems / n_classes;
    const int items = n_classes * S;
    float best[kSvmRows];
    int best_c[kSvmRows];
#pragma unroll
    for (int k = 0; k < kSvmRows; ++k) {
        best[k] = -INFINITY;
        best_c[k] = 0x7FFFFFFF;
    }
    for (int item = warp; item < items; item += kWarps) {
        const int c = item / S, sl = item - c * S;
        const int d0 = (int)((int64_t)sl * dim / S), d1 = (int)((int64_t)(sl + 1) * dim / S);
        const float* w = W + (int64_t)c * dim;
        double acc[kSvmRows];
#pragma unroll
        for (int k = 0; k < kSvmRows; ++k) acc[k] = 0.0;
        for (int d = d0 + lane; d < d1; d += 128) {
            double wd[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) wd[u] = d + 32 * u < d1 ? (double)__ldg(w + d + 32 * u) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (d + 32 * u < d1) {
#pragma unroll
                    for (int k = 0; k < kSvmRows; ++k) acc[k] = fma(wd[u], x(k, d + 32 * u), acc[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kSvmRows; ++k) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xFFFFFFFFu, acc[k], off);
        }
        if (S > 1) {  // partial sums, combined below in slice order
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < kSvmRows; ++k) part[sl * n_classes + c][k] = acc[k];
            continue;
        }
        const double b = (double)__ldg(bias + c);
#pragma unroll
        for (int k = 0; k < kSvmRows; ++k) {
            const float s = (float)(acc[k] + b);
            if (lane == 0 && k < rows && scores) scores[(row0 + k) * n_classes + c] = s;
            if (better(s, c, best[k], best_c[k]) || best_c[k] == 0x7FFFFFFF) {
                best[k] = s;
                best_c[k] = c;
            }
        }
    }
    if (S > 1) {
        __syncthreads();
        if (threadIdx.x < rows) {
            const int k = threadIdx.x;
            float b = 0.0f;
            int bc = 0;
            for (int c = 0; c < n_classes; ++c) {
                double acc = 0.0;
                for (int sl = 0; sl < S; ++sl) acc += part[sl * n_classes + c][k];
                const float s = (float)(acc + (double)__ldg(bias + c));
                if (scores) scores[(row0 + k) * n_classes + c] = s;
                if (c == 0 || s > b) {
                    b = s;
                    bc = c;
                }
            }
            if (top_score) top_score[row0 + k] = b;
            if (labels) labels[row0 + k] = (b < reject_threshold) ? -1 : bc;
        }
        return;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kSvmRows; ++k) {
            wbest[warp][k] = best[k];
            wbest_c[warp][k] = best_c[k];
        }
    }
    __syncthreads();
    if (threadIdx.x < rows) {
        const int k = threadIdx.x;
        float b = wbest[0][k];
        int bc = wbest_c[0][k];
        for (int w = 1; w < kWarps; ++w) {
            if (wbest_c[w][k] == 0x7FFFFFFF) continue;
            if (bc == 0x7FFFFFFF || better(wbest[w][k], wbest_c[w][k], b, bc)) {
                b = wbest[w][k];
                bc = wbest_c[w][k];
            }
        }
        if (top_score) top_score[row0 + k] = b;
        if (labels) labels[row0 + k] = (b < reject_threshold) ? -1 : bc;
    }
}

}  // namespace lbpf
