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
#include <type_traits>

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

// Register-resident variant (even dim): each thread owns the descriptor entry PAIRS
// (2p, 2p+1), p = tid + k * NT, and keeps its z entries in registers (they are private to the
// thread: the update of entry d only needs z[d] and x[d]).  The dot product's warp partials go
// to a double-buffered smem array; after ONE barrier every thread sums the partials itself
// and takes the (identical, integer) decision, so no second barrier and no smem z.  The bias
// entry z[dim] is kept by every thread redundantly.  Z32: int32 z, exact while T * 65535 <
// 2^31 (|z_T[d]| <= T max x); the products accumulate in int64 (IMAD.WIDE).
template <int NT, int PAIRS, bool Z32>
__global__ void __launch_bounds__(NT)
svm_train_ovr_reg_kernel(const uint16_t* __restrict__ desc, int32_t n, int32_t dim,
                         const int32_t* __restrict__ labels, int32_t n_classes,
                         const int32_t* __restrict__ order, int64_t T, int32_t inv_lambda,
                         float* __restrict__ W, float* __restrict__ bias,
                         int64_t* __restrict__ z_out) {
    using ZT = typename std::conditional<Z32, int32_t, int64_t>::type;
    constexpr int kWarps = NT / 32;
    __shared__ long long red[2][kWarps];
    const int t0 = threadIdx.x, warp = t0 >> 5, lane = t0 & 31;
    const int half = dim >> 1;
    const uint32_t* __restrict__ d32 = reinterpret_cast<const uint32_t*>(desc);

    for (int32_t c = blockIdx.x; c < n_classes; c += gridDim.x) {
        ZT z[2 * PAIRS];
#pragma unroll
        for (int k = 0; k < 2 * PAIRS; ++k) z[k] = 0;
        ZT zb = 0;
        // software pipeline over a 3-slot register ring, the step loop unrolled by 3 so that
        // every slot is a fixed register set (a register copy of a just-requested load would
        // wait for it): step t (slot r = (t-1) % 3) uses the counts in buf[r] requested two
        // steps ago, requests the counts of step t+2 into buf[(r+2)%3] from the index ids[..]
        // loaded one step ago, and loads the index of step t+3 into ids[r].
        auto idx = [&](int64_t j) { return __ldg(order + (j < T ? j : T - 1)); };
        // (the visit-order index of step t+2 is loaded three steps earlier: slot (r+1) % 3 of
        // ids holds it at step t and is then reloaded with the index of step t+5)
        uint32_t buf[3][PAIRS];
        int32_t ids[3] = {idx(4), idx(2), idx(3)};
        int32_t labs[3];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int32_t i0 = idx(r);
#pragma unroll
            for (int k = 0; k < PAIRS; ++k) {
                const int p = t0 + k * NT;
                buf[r][k] = p < half ? __ldg(d32 + (int64_t)i0 * half + p) : 0u;
            }
            labs[r] = __ldg(labels + i0);
        }
        for (int64_t t0s = 1; t0s <= T; t0s += 3) {
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const int64_t t = t0s + r;
                if (t > T) break;  // uniform
                const int rn = (r + 2) % 3, ri = (r + 1) % 3;
                const int32_t i_n = ids[ri];  // sample of step t+2
#pragma unroll
                for (int k = 0; k < PAIRS; ++k) {
                    const int p = t0 + k * NT;
                    buf[rn][k] = p < half ? __ldg(d32 + (int64_t)i_n * half + p) : 0u;
                }
                labs[rn] = __ldg(labels + i_n);
                ids[ri] = idx(t + 4);          // sample of step t+5
                const ZT y = (labs[r] == c) ? 1 : -1;
                bool viol = true;
                if (t > 1) {
                    // two independent accumulators (even / odd entries): half the dependent
                    // chain of 64-bit multiply-adds
                    long long pe = 0, po = 0;
#pragma unroll
                    for (int k = 0; k < PAIRS; ++k) {
                        pe += (long long)z[2 * k] * (long long)(buf[r][k] & 0xFFFFu);
                        po += (long long)z[2 * k + 1] * (long long)(buf[r][k] >> 16);
                    }
                    long long part = pe + po;
                    if constexpr (Z32) {
                        // |part| < 16 * 2^31 * 2^16 = 2^51: three 17-bit pieces (the top one
                        // signed) each summed over the warp by one redux.sync -- exact (every
                        // sum < 2^22) and without the five dependent shuffle rounds
                        const unsigned long long u = (unsigned long long)part;
                        const int pc = (int)(u & 0x1FFFFu), pb = (int)((u >> 17) & 0x1FFFFu);
                        const int pa = (int)(part >> 34);
                        const int sc = __reduce_add_sync(0xFFFFFFFFu, pc);
                        const int sb = __reduce_add_sync(0xFFFFFFFFu, pb);
                        const int sa = __reduce_add_sync(0xFFFFFFFFu, pa);
                        part = (long long)sa * (1ll << 34) + (long long)sb * (1ll << 17) + sc;
                    } else {
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1)
                            part += __shfl_xor_sync(0xFFFFFFFFu, part, off);
                    }
                    const int rb = (int)(t & 1);
                    if (lane == 0) red[rb][warp] = part;
                    __syncthreads();
                    // the warp partials summed as a tree (exact in int64, any order)
                    long long rs[kWarps];
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) rs[w] = red[rb][w];
#pragma unroll
                    for (int h = kWarps / 2; h > 0; h >>= 1)
#pragma unroll
                        for (int w = 0; w < h; ++w) rs[w] += rs[w + h];
                    const long long dot = (long long)zb + rs[0];
                    // (an incremental loop-carried threshold and a 32-bit division both
                    // measured slower: this form depends only on t and overlaps the reduction)
                    const long long thr = (long long)((t - 1 + inv_lambda - 1) / inv_lambda);
                    viol = (long long)y * dot < thr;
                }
                if (viol) {
#pragma unroll
                    for (int k = 0; k < PAIRS; ++k) {
                        z[2 * k] += y * (ZT)(buf[r][k] & 0xFFFFu);
                        z[2 * k + 1] += y * (ZT)(buf[r][k] >> 16);
                    }
                    zb += y;
                }
            }
        }
        // model: w = inv_lambda z_T / T, one fp64 division (correctly rounded) then fp32
        const double Td = (double)T;
#pragma unroll
        for (int k = 0; k < PAIRS; ++k) {
            const int p = t0 + k * NT;
            if (p < half) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int d = 2 * p + e;
                    const int64_t zd = (int64_t)z[2 * k + e];
                    W[(int64_t)c * dim + d] = (float)((double)((int64_t)inv_lambda * zd) / Td);
                    if (z_out) z_out[(int64_t)c * (dim + 1) + d] = zd;
                }
            }
        }
        if (t0 == 0) {
            bias[c] = (float)((double)((int64_t)inv_lambda * (int64_t)zb) / Td);
            if (z_out) z_out[(int64_t)c * (dim + 1) + dim] = (int64_t)zb;
        }
        __syncthreads();  // the partial buffers are reused by the next class
    }
}

}  // namespace lbpf
