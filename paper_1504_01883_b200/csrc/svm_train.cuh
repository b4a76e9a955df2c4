// svm_train.cuh -- one-vs-rest linear SVM training on the GPU (
// S:449-466; reading R20), computed exactly in integers so that the model is
// bit-identical to the oracle's whatever the reduction order:
//   z_0 = 0; for t = 1..T: i = order[t-1], y = +1 if label[i] == c else -1, x~ = (x_i, 1);
//   violated iff t == 1 or y (z_{t-1} . x~) < ceil((t - 1) / inv_lambda);
//   z_t = z_{t-1} + [violated] y x~;   model w = inv_lambda z_T / T (fp64, then fp32).
// (z_t = lambda t w_t of Pegasos' w_t = (1 - 1/t) w_{t-1} + [viol] y x~ / (lambda t).)
//
// One CTA (NT threads) per class; z (int64, dim + 1) lives in shared memory; each thread
// owns the descriptor entries d = tid + k * NT and keeps the current and the next sample's
// counts in registers (the next sample is prefetched while the current step reduces).  A
// step is an int64 dot product (warp shuffles + one smem pass), one uniform decision and, when
// violated, an integer update of the thread's z entries.  The step chain of a class is
// sequential by definition; classes run in parallel.
#pragma once
#include "common.cuh"

namespace lbpf {

constexpr int kTrainMaxDim = 16384;  // 8x8 cells x 256 bins

// NT threads, PER descriptor entries per thread (dim <= NT * PER)
template <int kTrainThreads, int kTrainPerThread>
__global__ void __launch_bounds__(kTrainThreads)
svm_train_ovr_kernel(const uint16_t* __restrict__ desc, int32_t n, int32_t dim,
                     const int32_t* __restrict__ labels, int32_t n_classes,
                     const int32_t* __restrict__ order, int64_t T, int32_t inv_lambda,
                     float* __restrict__ W, float* __restrict__ bias,
                     int64_t* __restrict__ z_out) {
    extern __shared__ int64_t z[];  // [dim + 1]
    __shared__ int64_t red[kTrainThreads / 32];
    __shared__ int viol_s;
    const int t0 = threadIdx.x, warp = t0 >> 5, lane = t0 & 31;
    constexpr int kWarps = kTrainThreads / 32;

    for (int32_t c = blockIdx.x; c < n_classes; c += gridDim.x) {
        for (int d = t0; d <= dim; d += kTrainThreads) z[d] = 0;
        uint32_t cur[kTrainPerThread], nxt[kTrainPerThread];
        int32_t i = __ldg(order);
        {
            const uint16_t* x = desc + (int64_t)i * dim;
#pragma unroll
            for (int k = 0; k < kTrainPerThread; ++k) {
                const int d = t0 + k * kTrainThreads;
                cur[k] = d < dim ? __ldg(x + d) : 0u;
            }
        }
        __syncthreads();
        for (int64_t t = 1; t <= T; ++t) {
            const int64_t y = (__ldg(labels + i) == c) ? 1 : -1;
            // prefetch the next sample's counts
            const int32_t i_next = t < T ? __ldg(order + t) : i;
            {
                const uint16_t* x = desc + (int64_t)i_next * dim;
#pragma unroll
                for (int k = 0; k < kTrainPerThread; ++k) {
                    const int d = t0 + k * kTrainThreads;
                    nxt[k] = d < dim ? __ldg(x + d) : 0u;
                }
            }
            bool viol = true;
            if (t > 1) {
                long long part = 0;
#pragma unroll
                for (int k = 0; k < kTrainPerThread; ++k) {
                    const int d = t0 + k * kTrainThreads;
                    if (d < dim) part += (long long)z[d] * (long long)cur[k];
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, off);
                if (lane == 0) red[warp] = part;
                __syncthreads();
                if (t0 == 0) {
                    long long dot = z[dim];  // the constant feature 1
                    for (int w2 = 0; w2 < kWarps; ++w2) dot += red[w2];
                    const long long thr = (long long)((t - 1 + inv_lambda - 1) / inv_lambda);
                    viol_s = (y * dot < thr) ? 1 : 0;
                }
                __syncthreads();
                viol = viol_s != 0;
            }
            if (viol) {
#pragma unroll
                for (int k = 0; k < kTrainPerThread; ++k) {
                    const int d = t0 + k * kTrainThreads;
                    if (d < dim) z[d] += y * (int64_t)cur[k];
                }
                if (t0 == 0) z[dim] += y;
            }
            __syncthreads();  // z complete before the next step's dot product
#pragma unroll
            for (int k = 0; k < kTrainPerThread; ++k) cur[k] = nxt[k];
            i = i_next;
        }
        // model: w = inv_lambda z_T / T, one fp64 division (correctly rounded) then fp32
        const double Td = (double)T;
        for (int d = t0; d < dim; d += kTrainThreads)
            W[(int64_t)c * dim + d] = (float)((double)((int64_t)inv_lambda * z[d]) / Td);
        if (t0 == 0) bias[c] = (float)((double)((int64_t)inv_lambda * z[dim]) / Td);
        if (z_out)
            for (int d = t0; d <= dim; d += kTrainThreads) z_out[(int64_t)c * (dim + 1) + d] = z[d];
        __syncthreads();  // z is reset for the next class
    }
}

}  // namespace lbpf
