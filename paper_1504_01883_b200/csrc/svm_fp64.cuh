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

namespace lbpf {

// ---------------------------------------------------------------------------- L1 variant
// s[n][c] = fp32(b[c] + sum_k (sum_{d in block k} W[c][d] h[n][d]) / N_k), N_k = the block's
// count sum (blocks with N_k = 0 contribute 0): the SVM on per-block L1-normalised
// descriptors, with the division applied to each block's exact-product fp64
// partial sum (the same real number as the oracle's sum of W * (h / N_k)).  CTA = R (8, or 1
// for long descriptors) crops staged in smem as fp32 (exact counts); a warp per class; lane l owns blocks
// l, l+32, ... and sums them in order, then one shuffle reduction per class.
template <int R>
__global__ void __launch_bounds__(kSvmThreads)
svm_score_l1_kernel(const uint16_t* __restrict__ desc, int32_t n, int32_t dim, int32_t block,
                    const float* __restrict__ W, const float* __restrict__ bias,
                    int32_t n_classes, float* __restrict__ scores, int32_t* __restrict__ labels,
                    float* __restrict__ top_score, float reject_threshold) {
    extern __shared__ float l1s[];  // [rows][dim] fp32 counts, then [rows][nblk] fp64 N_k
    constexpr int kWarps = kSvmThreads / 32;
    __shared__ float wbest[kWarps][R];
    __shared__ int wbest_c[kWarps][R];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = dim / block;
    const int64_t row0 = (int64_t)blockIdx.x * R;
    const int rows = (int)((n - row0) < R ? (n - row0) : R);
    float* xs = l1s;
    double* nk = reinterpret_cast<double*>(l1s + ((R * dim + 1) & ~1));
    for (int i = threadIdx.x; i < R * dim; i += blockDim.x)
        xs[i] = i < rows * dim ? (float)__ldg(desc + row0 * dim + i) : 0.0f;
    __syncthreads();
    for (int i = threadIdx.x; i < R * nblk; i += blockDim.x) {
        const int r = i / nblk, k = i - r * nblk;
        double sum = 0.0;  // exact: integer counts
        for (int d = k * block; d < (k + 1) * block; ++d) sum += (double)xs[r * dim + d];
        nk[i] = sum;
    }
    __syncthreads();
    float best[R];
    int best_c[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        best[r] = -INFINITY;
        best_c[r] = 0x7FFFFFFF;
    }
    for (int c = warp; c < n_classes; c += kWarps) {
        const float* w = W + (int64_t)c * dim;
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
        for (int k = lane; k < nblk; k += 32) {
            double p[R];
#pragma unroll
            for (int r = 0; r < R; ++r) p[r] = 0.0;
            for (int d = k * block; d < (k + 1) * block; ++d) {
                const double wd = (double)__ldg(w + d);
#pragma unroll
                for (int r = 0; r < R; ++r) p[r] = fma(wd, (double)xs[r * dim + d], p[r]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double N = nk[r * nblk + k];
                if (N > 0.0) acc[r] += p[r] / N;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xFFFFFFFFu, acc[r], off);
        }
        const double b = (double)__ldg(bias + c);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float sc = (float)(acc[r] + b);
            if (lane == 0 && r < rows && scores) scores[(row0 + r) * n_classes + c] = sc;
            if (better(sc, c, best[r], best_c[r]) || best_c[r] == 0x7FFFFFFF) {
                best[r] = sc;
                best_c[r] = c;
            }
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            wbest[warp][r] = best[r];
            wbest_c[warp][r] = best_c[r];
        }
    }
    __syncthreads();
    if (threadIdx.x < rows) {
        const int r = threadIdx.x;
        float b = wbest[0][r];
        int bc = wbest_c[0][r];
        for (int w2 = 1; w2 < kWarps; ++w2) {
            if (wbest_c[w2][r] == 0x7FFFFFFF) continue;
            if (bc == 0x7FFFFFFF || better(wbest[w2][r], wbest_c[w2][r], b, bc)) {
                b = wbest[w2][r];
                bc = wbest_c[w2][r];
            }
        }
        if (top_score) top_score[row0 + r] = b;
        if (labels) labels[row0 + r] = (b < reject_threshold) ? -1 : bc;
    }
}

}  // namespace lbpf
