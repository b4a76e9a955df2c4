// svm_gemm_i8.cuh -- the exact linear-SVM scorer on the INT8 tensor cores (tcgen05.mma
// kind::i8, s32 accumulators), used for many classes (C > kPassClasses) where the fp16
// digit-plane kernel of svm_gemm.cuh needs many TMEM passes.
//
// Weights as unsigned base-256 digits of an offset fraction:  with m_c = 2^e > max|W[c]|,
//   u = (W[c][d] / m_c + 1) / 2 in (0, 1),  U = rint(u * 2^40) = sum_{k<5} d_k 2^(8(4-k)),
//   d_k in [0, 255]  (|u - U 2^-40| <= 2^-41),
// so  sum_d x_d W[c][d] = m_c (2 sum_d x_d u_d - X),  X = sum_d x_d, and the GEMM computes the
// five digit products S_k = sum_d x_d d_k[d] and X (an all-ones row) EXACTLY in s32 (counts
// <= 255 as u8 operands: 255 * 255 * dim < 2^31 for dim <= 32,768).  The epilogue forms
// Q = sum_k S_k 2^(8(4-k)) = sum_d (x_d & 255) U_d in int64 (exact: < 255 * dim * 2^40 < 2^63
// for dim <= 32,768) and s = b + m_c (Q 2^-39 - X) in fp64,
// rounded once to fp32 -- the oracle's definition up to the 2^-40 m_c quantisation of W and
// fp64 rounding.  A count above 255 enters the GEMM as its low byte; its
// high part (x - (x & 255)) W is added exactly in fp64 by the row's epilogue thread (rows with
// more than kI8BigMax such entries are recomputed in fp64).
//
// The descriptor tile is u16 in HBM: the producer loads K = 128 columns as two 64-column
// 128-B-swizzled boxes, and converter warps (one thread per row) pack the row in place into
// the u8 operand tile (the first box's space), flagging counts > 255; the leader of the CTA
// pair then issues tcgen05.mma.cta_group::2.kind::i8 (M = 256, K = 32 per instruction).
// TMEM columns of a pass: digit k of the pass's class j at column k * 96 + j, the X column at
// 480 (pass = at most 96 classes, 512 columns).
#pragma once
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "svm_gemm.cuh"

namespace lbpf {

constexpr int kI8Digits = 5;
constexpr int kI8PassClasses = 96;   // digit planes of 96 classes + X = 481 of 512 columns
constexpr int kI8OnesCol = kI8Digits * kI8PassClasses;  // 480
constexpr int kI8K = 128;            // K per stage: one 128-B u8 row
constexpr int kI8DimAlign = 128;
constexpr int kI8MaxDim = 32768;     // 255 * 255 * dim < 2^31 (digit products, s32) and
                                     // Q = sum_d (x_d & 255) U_d < 255 * dim * 2^40 < 2^63
constexpr int kI8Threads = 448;      // warp 0 producer, 1 MMA, 2-5 converters + epilogue,
                                     // 6-13 epilogue helpers (two per TMEM lane quarter)
constexpr int kI8EpiWays = 3;        // epilogue warps per lane quarter
constexpr int kI8Chunk = 8;          // classes per epilogue chunk (x8 TMEM loads)
constexpr uint32_t kPrep8Magic = 0x53564D38u;  // "SVM8"
constexpr int kI8BigMax = 4;         // recorded entries above 255 per descriptor row
constexpr int kI8Distinct = 40;      // distinct such columns per CTA tile with W staged in smem
constexpr int kI8DbitsWords = (kI8MaxDim + 31) / 32;

__host__ __device__ inline int i8_pass_classes(int C, int p) {
    const int lo = p * kI8PassClasses;
    return (C - lo) < kI8PassClasses ? (C - lo) : kI8PassClasses;
}
inline bool svm_layout_i8(int32_t C, int32_t D, SvmPrepHeader* h) {
    if (C < 1 || D < 1 || (D % 8) != 0 || D > kI8MaxDim) return false;
    h->magic = kPrep8Magic;
    h->n_classes = C;
    h->dim = D;
    h->dim_pad = (D + kI8DimAlign - 1) / kI8DimAlign * kI8DimAlign;
    h->n_pass = (C + kI8PassClasses - 1) / kI8PassClasses;
    h->rows_max = 512;
    h->total_rows = 512 * h->n_pass;
    h->scale_off = 1024;
    h->q_off = (1024 + 4 * C + 1023) / 1024 * 1024;
    return true;
}

// One block per stored B row (pass-major, pair-major inside a pass as in svm_gemm.cuh).
__global__ void svm_prepare_i8_kernel(const float* __restrict__ W, SvmPrepHeader h,
                                      uint8_t* __restrict__ ws) {
    __shared__ float red[32];
    const int row = blockIdx.x;
    if (row == 0 && threadIdx.x == 0) write_prep_header(ws, h, W);
    const int p = row / 512, sr = row % 512;
    const int nc = i8_pass_classes(h.n_classes, p);
    // pair-major storage: 512 rows = 2 MMA halves of 256; CTA r holds rows hh*256 + r*128 + j
    const int cr = sr / 256, within = sr % 256;
    const int lr = (within / 128) * 256 + cr * 128 + within % 128;  // natural row = TMEM column
    uint8_t* q = ws + h.q_off + (size_t)row * h.dim_pad;
    const int k = lr / kI8PassClasses, j = lr % kI8PassClasses;
    if (lr >= kI8OnesCol || j >= nc) {  // X row (all ones over the real dim) or padding
        const uint8_t v = (lr == kI8OnesCol) ? 1 : 0;
        for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x) q[d] = d < h.dim ? v : 0;
        return;
    }
    const int c = p * kI8PassClasses + j;
    const float* w = W + (size_t)c * h.dim;
    float mx = 0.0f;
    for (int d = threadIdx.x; d < h.dim; d += blockDim.x) mx = fmaxf(mx, fabsf(w[d]));
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
        if (threadIdx.x == 0) red[0] = mx;
    }
    __syncthreads();
    mx = red[0];
    int e = 0;
    if (mx > 0.0f) frexpf(mx, &e);  // mx = f 2^e, f in [0.5, 1): m = 2^e > mx strictly
    const double m = ldexp(1.0, e);
    if (k == 0 && threadIdx.x == 0) reinterpret_cast<float*>(ws + h.scale_off)[c] = (float)m;
    for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x) {
        uint8_t dig = 0;
        if (d < h.dim) {
            const double u = ((double)w[d] / m + 1.0) * 0.5;           // exact in fp64
            const long long U = llrint(u * 1099511627776.0);           // 2^40, < 2^40
            dig = (uint8_t)((U >> (8 * (kI8Digits - 1 - k))) & 0xFF);
        }
        q[d] = dig;
    }
}

__device__ __forceinline__ void mma_i8_ss_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// instruction descriptor, kind::i8: A, B unsigned 8-bit K-major, D s32, shape M x N
__host__ __device__ constexpr uint32_t idesc_u8_s32(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// stage: A u16 K=128 as two 16 KB boxes (the u8 operand is packed into the first), B u8
// (256 rows x 128 B = 32 KB)
constexpr int kI8StageA = 2 * kGemmM * 128;  // 32 KB
constexpr int kI8StageB = 256 * 128;         // 32 KB
constexpr int kI8StageBytes = kI8StageA + kI8StageB;

// What one accumulator row's epilogue needs for a pass (svm_gemm_i8_kernel)
struct I8Epi {
    uint32_t lane_addr;   // TMEM address of the row's lane quarter
    const double2* tab;   // (scale, bias) of the pass's classes
    int nc, class0, C;
    int32_t X;            // sum_d x_d (ones column)
    bool live, staged;
    int n_big, row;
    double hi_r[kI8BigMax];
    uint32_t woff[kI8BigMax];
    const int32_t* big_d;
    const int32_t* big_hi;
    const float* W;
    int dim;
    float* scores;
    int64_t crop;
};

// kI8Chunk classes [c0, c0 + kI8Chunk) of the pass: Q by Horner over the 5 digit planes,
// s = b + m (Q 2^-39 - X) [+ the exact high parts of entries above 255]; running argmax over
// ascending classes (ties -> lowest).  kBig: the warp has rows with entries above 255.
template <bool kBig>
__device__ __forceinline__ void i8_combine16(const I8Epi& e, int c0, float& best, int& best_c) {
    long long q[kI8Chunk];
    uint32_t v[kI8Chunk];
#pragma unroll
    for (int j = 0; j < kI8Chunk; ++j) q[j] = 0;
#pragma unroll
    for (int k = 0; k < kI8Digits; ++k) {
        tmem_ld8(e.lane_addr + (uint32_t)(k * kI8PassClasses + c0), v);
        tmem_ld_wait_regs(v);
#pragma unroll
        for (int j = 0; j < kI8Chunk; ++j) q[j] = (q[j] << 8) + (int32_t)v[j];
    }
#pragma unroll
    for (int j = 0; j < kI8Chunk; ++j) {
        const int lc = c0 + j;
        const double2 sb = e.tab[lc < kI8PassClasses ? lc : 0];
        const double sm = fma((double)q[j], 0x1p-39, -(double)e.X);
        double acc = fma(sb.x, sm, sb.y);
        if (kBig && lc < e.nc) {
            if (e.staged) {  // independent shared loads, no dependent chain
#pragma unroll
                for (int t = 0; t < kI8BigMax; ++t)
                    acc = fma(e.hi_r[t],
                              (double)__uint_as_float(ld_shared_u32(e.woff[t] + (uint32_t)lc * 4)),
                              acc);
            } else {
                const float* wc = e.W + (size_t)(e.class0 + lc) * e.dim;
                for (int t = 0; t < e.n_big; ++t)
                    acc = fma((double)e.big_hi[e.row * kI8BigMax + t],
                              (double)__ldg(wc + e.big_d[e.row * kI8BigMax + t]), acc);
            }
        }
        const float sc = (float)acc;
        if (lc < e.nc && e.live) {
            if (e.scores) e.scores[e.crop * e.C + e.class0 + lc] = sc;
            if (best_c < 0 || sc > best) {
                best = sc;
                best_c = e.class0 + lc;
            }
        }
    }
}

// the row's correction terms (smem addresses of its staged W columns; zero weights beyond
// n_big), hoisted out of the class loop
__device__ __forceinline__ void i8_epi_corrections(I8Epi& e, const float* wcol) {
    const uint32_t wcol0 = smem_u32(wcol);
#pragma unroll
    for (int t = 0; t < kI8BigMax; ++t) {
        const bool on = e.staged && t < e.n_big;
        e.hi_r[t] = on ? (double)e.big_hi[e.row * kI8BigMax + t] : 0.0;
        e.woff[t] = on ? wcol0 + (uint32_t)e.big_d[e.row * kI8BigMax + t] * (kI8PassClasses * 4)
                       : wcol0;
    }
}

// the chunks c0 = kI8Chunk (par + kI8EpiWays i) of the pass (par 0: converter warp, 1..:
// its helpers)
__device__ __forceinline__ void i8_epi_chunks(const I8Epi& e, int par, float& best, int& best_c) {
    const bool warp_big = __any_sync(0xFFFFFFFFu, e.n_big != 0);  // warp-uniform variant
    for (int c0 = kI8Chunk * par; c0 < e.nc; c0 += kI8Chunk * kI8EpiWays) {
        if (warp_big) i8_combine16<true>(e, c0, best, best_c);
        else i8_combine16<false>(e, c0, best, best_c);
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kI8Threads, 1)
svm_gemm_i8_kernel(const __grid_constant__ CUtensorMap a_map,
                   const __grid_constant__ CUtensorMap b_map, const uint16_t* __restrict__ desc,
                   int32_t n, const float* __restrict__ W, const float* __restrict__ bias,
                   const uint8_t* __restrict__ ws, SvmPrepHeader h, int stages,
                   float* __restrict__ scores, int32_t* __restrict__ labels,
                   float* __restrict__ top_score, float reject_threshold) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kI8StageBytes);
    uint64_t* conv = full + stages;
    uint64_t* empty = conv + stages;
    uint64_t* tmem_full = empty + stages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
    double2* epi_tab = reinterpret_cast<double2*>(smem + stages * kI8StageBytes + 512);
    // per-row lists of the descriptor entries above 255 (their high part x - (x & 255) is
    // added on CUDA cores: x W = (x & 255) W [GEMM] + (x - (x & 255)) W [exact fp64])
    int32_t* big_d = reinterpret_cast<int32_t*>(epi_tab + 2 * kI8PassClasses);
    int32_t* big_hi = big_d + kGemmM * kI8BigMax;
    // the tile's distinct columns holding an entry above 255 (a bitmap dedups them) and, per
    // pass, W of the pass's classes at those columns: the epilogue's high-part corrections
    // then read shared memory (a 16x16 cell whose 256 pixels share one bin is the usual case)
    uint32_t* dbits = reinterpret_cast<uint32_t*>(big_hi + kGemmM * kI8BigMax);
    int32_t* dlist = reinterpret_cast<int32_t*>(dbits + kI8DbitsWords);
    int32_t* dcount = dlist + kI8Distinct;
    float* wcol = reinterpret_cast<float*>(dcount + 4);  // [kI8Distinct][kI8PassClasses]
    // per row: its count of entries above 255 (for the helpers) and the helpers' argmax
    int32_t* nbig = reinterpret_cast<int32_t*>(wcol + kI8Distinct * kI8PassClasses);
    float* hbest = reinterpret_cast<float*>(nbig + kGemmM);           // [helper set][row]
    int32_t* hcls = reinterpret_cast<int32_t*>(hbest + (kI8EpiWays - 1) * kGemmM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = (int)cluster_id_x(), n_pairs_grid = (int)n_clusters_x();
    const int C = h.n_classes;
    const int KC = h.dim_pad / kI8K;
    const float* scales = reinterpret_cast<const float*>(ws + h.scale_off);

    if (threadIdx.x == 0) {
        tmem_slot[1] = prep_header_ok(ws, h, W) ? 0u : 1u;  // (read after __syncthreads)
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 8);  // 4 converter warps x 2 CTAs
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 8);
        fence_mbar_init();
        prefetch_tensormap(&a_map);
        prefetch_tensormap(&b_map);
    }
    if (warp == 1) {
        tmem_alloc_pair(tmem_slot, 512);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // a workspace that does not belong to this model: nothing past its header is read, every
    // row gets LBP_LABEL_BAD_MODEL below
    const bool bad_model = tmem_slot[1] != 0u;
    const int n_tiles = bad_model ? 0 : (n + 2 * kGemmM - 1) / (2 * kGemmM);
    // programmatic dependent launch: the prologue above may overlap the tail of the kernel
    // that wrote the descriptors; everything below reads them (no-op without PDL).  The next
    // kernel on the stream (the next batch's extraction) may be scheduled from now on: it waits
    // for this grid's completion before it touches the descriptors.
    launch_dependents();
    grid_dependency_wait();

    if (warp == 0) {
        // ===================== TMA producer: A = two 64-column u16 boxes, B = this CTA's half
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                const int arow = t * 2 * kGemmM + (int)rank * kGemmM;
                for (int p = 0; p < h.n_pass; ++p) {
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&empty[s], ph ^ 1);
                        mbar_arrive_expect_tx(&full[s], kI8StageBytes);
                        uint8_t* st = smem + s * kI8StageBytes;
                        tma_load_2d(st, &a_map, &full[s], kc * kI8K, arow);
                        tma_load_2d(st + kI8StageA / 2, &a_map, &full[s], kc * kI8K + 64, arow);
                        tma_load_2d(st + kI8StageA, &b_map, &full[s], kc * kI8K,
                                    p * 512 + (int)rank * 256);
                        if (++s == stages) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; whole warp, one elected lane issues)
        if (rank == 0) {
            int s = 0;
            uint32_t ph = 0, acc_ph = 0;
            const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
            const uint32_t d_hi = (uint32_t)(d0 >> 32), d_lo0 = (uint32_t)d0;
            const uint32_t idesc = idesc_u8_s32(2 * kGemmM, 256);
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                for (int p = 0; p < h.n_pass; ++p) {
                    mbar_wait(tmem_empty, acc_ph ^ 1);
                    acc_ph ^= 1;
                    tc_fence_after();
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&conv[s], ph);
                        tc_fence_after();
                        const uint32_t a_lo = d_lo0 + (uint32_t)(s * kI8StageBytes) / 16;
                        const uint32_t b_lo = a_lo + (uint32_t)kI8StageA / 16;
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < kI8K / 32; ++ks) {
                                const uint64_t ad = ((uint64_t)d_hi << 32) | (a_lo + 2 * ks);
                                const uint32_t acc = (kc | ks) != 0;
                                // two MMAs of N = 256: TMEM columns [0, 256) and [256, 512)
                                mma_i8_ss_pair(tmem_base, ad, ((uint64_t)d_hi << 32) | (b_lo + 2 * ks),
                                               idesc, acc);
                                mma_i8_ss_pair(tmem_base + 256, ad,
                                               ((uint64_t)d_hi << 32) | (b_lo + 128 * 128 / 16 + 2 * ks),
                                               idesc, acc);
                            }
                            mma_commit_pair(&empty[s], 0x3);
                        }
                        __syncwarp();
                        if (++s == stages) { s = 0; ph ^= 1; }
                    }
                    if (elect_one()) mma_commit_pair(tmem_full, 0x3);
                    __syncwarp();
                }
            }
        }
    } else if (warp >= 6) {
        const int par = 1 + (warp - 6) / 4;  // helper set 1 (warps 6..9) or 2 (10..13)
        // ===================== epilogue helpers (warps 6..9): the odd 16-class chunks of the
        // TMEM lane quarter of converter warp (warp & 3); their per-row argmax is merged by
        // the converter through shared memory
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        int pc = 0;
        uint32_t acc_ph = 0;
        for (int t = pair; t < n_tiles; t += n_pairs_grid) {
            const int64_t crop = (int64_t)t * 2 * kGemmM + (int64_t)rank * kGemmM + row;
            int class0 = 0;
            for (int p = 0; p < h.n_pass; ++p) {
                const int nc = i8_pass_classes(C, p);
                named_barrier_sync(2, 128 * kI8EpiWays);
                I8Epi e;
                e.tab = epi_tab + (pc & 1) * kI8PassClasses;
                e.nc = nc; e.class0 = class0; e.C = C;
                e.live = crop < n; e.staged = *dcount <= kI8Distinct; e.n_big = nbig[row];
                e.row = row; e.big_d = big_d; e.big_hi = big_hi; e.W = W; e.dim = h.dim;
                e.scores = scores; e.crop = crop;
                i8_epi_corrections(e, wcol);
                mbar_wait(tmem_full, acc_ph);
                acc_ph ^= 1;
                tc_fence_after();
                e.lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
                e.X = (int32_t)tmem_ld1(e.lane_addr + kI8OnesCol);
                tmem_ld_wait();
                float best = 0.0f;
                int best_c = -1;
#ifndef LBP_I8_NOEPI
                i8_epi_chunks(e, par, best, best_c);
#endif
                hbest[(par - 1) * kGemmM + row] = best;
                hcls[(par - 1) * kGemmM + row] = best_c;
                tc_fence_before();
                named_barrier_sync(3, 128 * kI8EpiWays);
                class0 += nc;
                ++pc;
            }
        }
    } else {
        // ===================== converters (one thread per A row) + epilogue
        const int et = threadIdx.x - 64;  // 0..127 = A row of this CTA = TMEM lane
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t conv_leader = mapa_shared(smem_u32(conv), 0);
        const uint32_t tmem_empty_leader = mapa_shared(smem_u32(tmem_empty), 0);
        int s = 0, pc = 0;
        uint32_t ph = 0, acc_ph = 0;
        for (int t = pair; t < n_tiles; t += n_pairs_grid) {
            const int64_t crop = (int64_t)t * 2 * kGemmM + (int64_t)rank * kGemmM + row;
            float best = 0.0f;
            int best_c = -1;
            int class0 = 0;
            int n_big = 0;          // entries of this row above 255 (recorded in pass 0)
            bool row_over = false;  // more than kI8BigMax of them: the row is scored in fp64
            for (int i = et; i < kI8DbitsWords; i += 128) dbits[i] = 0;
            if (et == 0) *dcount = 0;
            named_barrier_sync(1, 128);  // bitmap clear before the tile's first record
            for (int p = 0; p < h.n_pass; ++p) {
                const int nc = i8_pass_classes(C, p);
                for (int kc = 0; kc < KC; ++kc) {
                    mbar_wait(&full[s], ph);
                    // row et: u16 chunks of box 0 (cols 0-63) and box 1 (cols 64-127), 128-B
                    // swizzle (chunk c of row r at (c ^ (r & 7)) * 16) -> u8 row in box 0
                    // this thread converts A row `row` -- the TMEM lane its epilogue reads, so
                    // the row's entries above 255 are known to the thread that scores it
                    const uint32_t b0 = smem_u32(smem + s * kI8StageBytes) + row * 128;
                    const uint32_t b1 = b0 + kI8StageA / 2;
                    const uint32_t sw = (uint32_t)(row & 7);
                    uint4 v[16];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        v[c] = ld_shared_u32x4(b0 + ((c ^ sw) << 4));
                        v[8 + c] = ld_shared_u32x4(b1 + ((c ^ sw) << 4));
                    }
                    uint32_t big = 0;
#pragma unroll
                    for (int J = 0; J < 8; ++J) {  // u8 chunk J = u16 chunks 2J, 2J+1
                        const uint4 a = v[2 * J], b = v[2 * J + 1];
                        big |= (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) & 0xFF00FF00u;
                        const uint4 o = make_uint4(prmt(a.x, a.y, 0x6420), prmt(a.z, a.w, 0x6420),
                                                   prmt(b.x, b.y, 0x6420), prmt(b.z, b.w, 0x6420));
                        st_shared_u32x4(b0 + ((J ^ sw) << 4), o);
                    }
                    if (big && p == 0) {  // rare: record the entries above 255 of this row
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const uint32_t val = (w4[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                                if (val > 255u) {
                                    const int d = kc * kI8K + 8 * i + e;
                                    if (n_big < kI8BigMax) {
                                        big_d[row * kI8BigMax + n_big] = d;
                                        big_hi[row * kI8BigMax + n_big] = (int32_t)(val & 0xFF00u);
                                        ++n_big;
                                    } else {
                                        row_over = true;
                                    }
                                    const uint32_t bit = 1u << (d & 31);
                                    if (!(atomicOr(&dbits[d >> 5], bit) & bit)) {
                                        const int k = atomicAdd(dcount, 1);
                                        if (k < kI8Distinct) dlist[k] = d;
                                    }
                                }
                            }
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(conv_leader + s * 8);
                    if (++s == stages) { s = 0; ph ^= 1; }
                }
                // ---- epilogue of this pass
                double2* tab = epi_tab + (pc & 1) * kI8PassClasses;
                for (int i = et; i < kI8PassClasses; i += 128)
                    tab[i] = i < nc ? make_double2((double)__ldg(scales + class0 + i),
                                                   (double)__ldg(bias + class0 + i))
                                    : make_double2(0.0, 0.0);
                named_barrier_sync(1, 128);  // (scale, bias) table and the tile's column list
                const int nd = *dcount;
                const bool staged = nd <= kI8Distinct;  // else: corrections read W in global
                if (nd > 0 && staged) {
                    for (int i = et; i < nd * kI8PassClasses; i += 128) {
                        const int k = i / kI8PassClasses, lc = i - k * kI8PassClasses;
                        wcol[i] = lc < nc ? __ldg(W + (size_t)(class0 + lc) * h.dim + dlist[k])
                                          : 0.0f;
                    }
                    if (p == 0)  // the row's entries -> indices into the tile's column list
                        for (int e = 0; e < n_big; ++e) {
                            const int d = big_d[row * kI8BigMax + e];
                            int k = 0;
                            while (dlist[k] != d) ++k;
                            big_d[row * kI8BigMax + e] = k;
                        }
                    named_barrier_sync(1, 128);  // W columns staged
                }
                if (p == 0) nbig[row] = n_big;  // final after pass 0's conversion
                named_barrier_sync(2, 128 * kI8EpiWays);  // table, lists, counts for the helpers
                mbar_wait(tmem_full, acc_ph);
                acc_ph ^= 1;
                tc_fence_after();
                I8Epi e;
                e.lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
                e.X = (int32_t)tmem_ld1(e.lane_addr + kI8OnesCol);
                tmem_ld_wait();
                e.tab = tab; e.nc = nc; e.class0 = class0; e.C = C;
                e.live = crop < n; e.staged = staged; e.n_big = n_big; e.row = row;
                e.big_d = big_d; e.big_hi = big_hi; e.W = W; e.dim = h.dim;
                e.scores = scores; e.crop = crop;
                i8_epi_corrections(e, wcol);
                const bool live = e.live;
                const float best_prev = best;
                const int best_c_prev = best_c;
#ifndef LBP_I8_NOEPI  // (developer ablation: the class loops removed)
                i8_epi_chunks(e, 0, best, best_c);
#endif
                named_barrier_sync(3, 128 * kI8EpiWays);  // the helpers' partial argmaxes
#pragma unroll
                for (int hset = 0; hset < kI8EpiWays - 1; ++hset) {
                    const float hb = hbest[hset * kGemmM + row];
                    const int hc = hcls[hset * kGemmM + row];
                    if (hc >= 0 && (best_c < 0 || hb > best || (hb == best && hc < best_c))) {
                        best = hb;
                        best_c = hc;
                    }
                }
                if (row_over && live) {  // many entries above 255: the row in fp64
                    best = best_prev;
                    best_c = best_c_prev;
                    for (int lc = 0; lc < nc; ++lc) {
                        const int c = class0 + lc;
                        double acc = (double)__ldg(bias + c);
                        for (int d = 0; d < h.dim; ++d)
                            acc += (double)__ldg(W + (size_t)c * h.dim + d) *
                                   (double)desc[crop * h.dim + d];
                        const float sc = (float)acc;
                        if (scores) scores[crop * C + c] = sc;
                        if (best_c < 0 || sc > best) {
                            best = sc;
                            best_c = c;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tmem_empty_leader);
                class0 += nc;
                ++pc;
            }
            if (crop < n) {
                if (top_score) top_score[crop] = best;
                if (labels) labels[crop] = (best < reject_threshold) ? -1 : best_c;
            }
        }
    }
    if (bad_model) write_bad_model(n, C, scores, labels, top_score);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair(tmem_base, 512);
}

inline cudaError_t launch_svm_gemm_i8(const uint16_t* desc, int32_t n, int32_t dim,
                                      const float* W, const float* bias, const SvmPrepHeader& h,
                                      const uint8_t* ws, float* scores, int32_t* labels,
                                      float* top, float reject, int sms, cudaStream_t stream) {
    CUtensorMap am, bm;
    if (!encode_2d(&am, desc, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (uint64_t)dim, (uint64_t)n,
                   (uint64_t)dim * 2, 64, kGemmM))
        return cudaErrorNotSupported;
    if (!encode_2d(&bm, ws + h.q_off, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)h.dim_pad,
                   (uint64_t)h.total_rows, (uint64_t)h.dim_pad, kI8K, 256))
        return cudaErrorNotSupported;
    const int stages = 3;
    const int smem = stages * kI8StageBytes + 1024 + 512 + 2 * kI8PassClasses * 16 +
                     2 * kGemmM * kI8BigMax * 4 + kI8DbitsWords * 4 + (kI8Distinct + 4) * 4 +
                     kI8Distinct * kI8PassClasses * 4 + (1 + 2 * (kI8EpiWays - 1)) * kGemmM * 4;
    cudaError_t e = cudaFuncSetAttribute(svm_gemm_i8_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (n + 2 * kGemmM - 1) / (2 * kGemmM);
    const int pairs = tiles < sms / 2 ? tiles : sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(kI8Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (grid_dependency_wait)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, svm_gemm_i8_kernel, am, bm, desc, n, W, bias, ws, h, stages,
                              scores, labels, top, reject);
}

}  // namespace lbpf
