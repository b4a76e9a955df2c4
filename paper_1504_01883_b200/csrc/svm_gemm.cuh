// svm_gemm.cuh -- exact linear-SVM scoring on the 5th-gen tensor cores (tcgen05, TMEM, TMA).
//
// s[n][c] = b[c] + sum_d W[c][d] * x[n][d]  (P:142 hyperplane) as a GEMM
// X (crops x D, u16 counts) * Q^T where Q holds W split into fixed-point INTEGER digit planes:
//     W[c][d] ~= m_c * sum_{k<4} 2^-(8+9k) * q_k[c][d],  q_k in [-256, 256],  m_c = 2^e >= max|W[c]|
// (svm_prepare; |error| <= 2^-36 m_c).  The u16 descriptor tile is fed to the tensor core
// UNCONVERTED: the bits of a count x < 2048 read as fp16 are exactly x * 2^-24 (subnormal below
// 1024, exponent field 1 up to 2047).  Digits are exact in fp16, every product is an integer
// times 2^-24 and every partial sum stays below 2^24 * 2^-24 while sum_d x_d < 2^16, so the
// fp32 tensor-core accumulation is EXACT and order-independent.  The epilogue combines the
// four digit accumulators in fp64 (exact), adds the bias and rounds once to fp32 -- the
// oracle's definition up to the 2^-36 m_c quantisation of W.  Rows that break
// the exactness preconditions (sum_d x_d >= 2^16, detected with an all-ones B row, or a count
// >= 2048 in the CTA's tile, detected by the checker warps) are recomputed in fp64 on CUDA
// cores by the epilogue thread.
//
// Kernel: persistent CTA PAIRS (clusters of 2, one CTA per SM), 6 warps per CTA, 256 crops
// per pair tile:
//   warp 0  TMA producer: A = this CTA's 128 x 64 u16 descriptor tile, B = this CTA's half
//           (rows/2 x 64 fp16) of the pass's digit rows, both 128-B swizzled, into a ring of
//           `stages` smem stages (mbarrier full/empty)
//   warp 1  TMEM allocator (cta_group::2) + on the leader CTA the single-thread MMA issuer
//           (tcgen05.mma.cta_group::2 kind::f16, M=256: both CTAs' A and B halves)
//   warps 2-5  check the A tile for counts >= 2048 (off the MMA's critical path), then run
//           the epilogue: tcgen05.ld accumulators, fp64 digit combine, bias, argmax.
//   warp 6  relay: one lane forwards "stage s landed in this CTA" to the leader's ready[s].
// Classes are processed in TMEM passes of <= 124 classes (4 digits each + a ones block =
// 512 fp32 columns); the running argmax of a crop lives in its epilogue thread's registers.
#pragma once
#ifdef LBP_SVM_TRACE
__device__ unsigned long long g_svm_trace[32];
#endif
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ptx.cuh"

namespace lbpf {

constexpr int kPassClasses = 124;
constexpr int kGemmM = 128;
constexpr int kGemmK = 64;                  // K per pipeline stage (fp16 elements)
constexpr int kRowBytes = kGemmK * 2;       // one swizzled smem row: 128 B (SWIZZLE_128B)
constexpr int kDimAlign = 64;               // workspace dim padding
constexpr int kGemmThreads = 480;  // 15 warps (see svm_gemm_kernel)
constexpr int kEpiWays = 3;        // epilogue warps per TMEM lane quarter (checker + 2 helpers)
constexpr uint32_t kPrepMagic = 0x53564D31u;  // "SVM1"

constexpr int kPrepSamples = 8;
struct SvmPrepHeader {
    uint32_t magic;
    int32_t n_classes, dim, dim_pad, n_pass, rows_max, total_rows;
    int32_t scale_off, q_off;  // byte offsets inside the workspace
    // bits of W at kPrepSamples fixed positions (svm_prepare): the scorers compare them with
    // the W of the call, so a workspace prepared for another model is refused (labels
    // LBP_LABEL_BAD_MODEL) instead of silently scoring with the wrong digit planes
    uint32_t w_sample[kPrepSamples];
};

__host__ __device__ inline int64_t w_sample_pos(int i, int32_t C, int32_t dim) {
    return (int64_t)i * ((int64_t)C * dim - 1) / (kPrepSamples - 1);
}

// svm_prepare's header write (one thread): the layout plus the W fingerprint
__device__ inline void write_prep_header(uint8_t* ws, SvmPrepHeader h, const float* W) {
    for (int i = 0; i < kPrepSamples; ++i)
        h.w_sample[i] = __float_as_uint(W[w_sample_pos(i, h.n_classes, h.dim)]);
    *reinterpret_cast<SvmPrepHeader*>(ws) = h;
}

// The scorers' check (one thread, in the prologue, before any TMA of the workspace): the
// workspace header must describe this call's layout (same magic, classes, dim, padding, row
// count and offsets) and carry the bits of this call's W at the sample positions.
__device__ inline bool prep_header_ok(const uint8_t* ws, const SvmPrepHeader& h,
                                      const float* W) {
    const SvmPrepHeader* g = reinterpret_cast<const SvmPrepHeader*>(ws);
    if (g->magic != h.magic || g->n_classes != h.n_classes || g->dim != h.dim ||
        g->dim_pad != h.dim_pad || g->n_pass != h.n_pass || g->total_rows != h.total_rows ||
        g->scale_off != h.scale_off || g->q_off != h.q_off)
        return false;
    for (int i = 0; i < kPrepSamples; ++i)
        if (g->w_sample[i] != __float_as_uint(W[w_sample_pos(i, h.n_classes, h.dim)]))
            return false;
    return true;
}

// Outputs of a refused call: label LBP_LABEL_BAD_MODEL, NaN top score and scores.
__device__ inline void write_bad_model(int32_t n, int32_t C, float* scores, int32_t* labels,
                                       float* top_score) {
    const float nan = __uint_as_float(0x7FC00000u);
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i < n; i += nt) {
        if (labels) labels[i] = LBP_LABEL_BAD_MODEL;
        if (top_score) top_score[i] = nan;
    }
    if (scores)
        for (int64_t i = t0; i < (int64_t)n * C; i += nt) scores[i] = nan;
}

__host__ __device__ inline int pass_classes(int C, int p) {
    const int lo = p * kPassClasses;
    return (C - lo) < kPassClasses ? (C - lo) : kPassClasses;
}
__host__ __device__ inline int pass_rows(int nc) { return ((4 * nc + 16) + 31) / 32 * 32; }

inline bool svm_layout(int32_t C, int32_t D, SvmPrepHeader* h) {
    if (C < 1 || D < 1 || (D % 8) != 0) return false;  // TMA row stride must be 16-B aligned
    h->magic = kPrepMagic;
    h->n_classes = C;
    h->dim = D;
    h->dim_pad = (D + kDimAlign - 1) / kDimAlign * kDimAlign;
    h->n_pass = (C + kPassClasses - 1) / kPassClasses;
    h->rows_max = pass_rows(pass_classes(C, 0));
    int rows = 0;
    for (int p = 0; p < h->n_pass; ++p) rows += pass_rows(pass_classes(C, p));
    h->total_rows = rows;
    h->scale_off = 1024;
    h->q_off = (1024 + 4 * C + 1023) / 1024 * 1024;
    return true;
}

// ---------------------------------------------------------------------------- prepare

// One block per Q row.  Natural rows of a pass: 4 digit rows per class (row 4c+k = digit k
// of W[c][.]), the all-ones row, zero padding; stored in pair-major order (svm_gemm_kernel).
__global__ void svm_prepare_kernel(const float* __restrict__ W, SvmPrepHeader h,
                                   uint8_t* __restrict__ ws) {
    __shared__ float red[32];
    const int row = blockIdx.x;
    if (row == 0 && threadIdx.x == 0) write_prep_header(ws, h, W);
    // locate (pass, local row)
    int p = 0, base = 0;
    while (p < h.n_pass && row >= base + pass_rows(pass_classes(h.n_classes, p))) {
        base += pass_rows(pass_classes(h.n_classes, p));
        ++p;
    }
    const int nc = pass_classes(h.n_classes, p);
    // pair-major storage: storage row sr of a pass of R rows belongs to CTA r = sr / (R/2) of
    // the pair and to MMA half hh; its natural row (TMEM column) is hh*nn + r*nn/2 + j
    const int R = pass_rows(nc), nh = R > 256 ? 2 : 1, nn = R / nh;
    const int sr = row - base, cr = sr / (R / 2), within = sr % (R / 2);
    const int lr = (within / (nn / 2)) * nn + cr * (nn / 2) + within % (nn / 2);
    __half* q = reinterpret_cast<__half*>(ws + h.q_off) + (size_t)row * h.dim_pad;
    if (lr >= 4 * nc) {  // ones row (column sum check) or zero padding
        const float v = (lr == 4 * nc) ? 1.0f : 0.0f;
        for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x)
            q[d] = __float2half_rn(d < h.dim ? v : 0.0f);
        return;
    }
    const int c = p * kPassClasses + lr / 4, k = lr % 4;
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
    if (mx > 0.0f) frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1) -> m = 2^e >= mx
    const float m = ldexpf(1.0f, e);
    if (k == 0 && threadIdx.x == 0) reinterpret_cast<float*>(ws + h.scale_off)[c] = m;
    for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x) {
        float v = d < h.dim ? (w[d] / m) * 256.0f : 0.0f;  // exact: power-of-two scalings
        float qk = 0.0f;
        for (int j = 0; j <= k; ++j) {
            qk = rintf(v);            // in [-256, 256]
            v = (v - qk) * 512.0f;    // exact residual
        }
        q[d] = __float2half_rn(qk);
    }
}

// ---------------------------------------------------------------------------- GEMM kernel

struct GemmSmem {
    int stages, stage_bytes;
    __device__ __forceinline__ uint8_t* a(uint8_t* base, int s) const { return base + s * stage_bytes; }
    __device__ __forceinline__ uint8_t* b(uint8_t* base, int s) const {
        return base + s * stage_bytes + kGemmM * kGemmK * 2;
    }
};

// A CTA pair (cluster of 2) computes a 256-crop tile: CTA r stages crops [256t + 128r, +128)
// as A and HALF of each pass's B rows (the pair-major storage order of svm_prepare), the
// leader (rank 0) issues tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem and
// writing both CTAs' TMEM.  Per CTA, B traffic from L2 is half of a 1-CTA M=128 kernel's.
//
// Barriers (same smem offsets in both CTAs):
//   full[s]    local: this CTA's TMA bytes landed           (count 1, expect_tx)
//   ready[s]   leader: both CTAs' stage s landed              (count 2, one relay per CTA)
//   empty[s]   both: pair MMAs and this CTA's 4 checker warps done with stage s (count 5)
//   tmem_full  both: accumulators of the pass complete        (multicast commit)
//   tmem_empty leader: both CTAs' epilogues drained TMEM      (count 8)
// Epilogue of one pass for one accumulator row: the 4-class groups c4 = 4 (par + kEpiWays i)
// (par 0: the checker warp, 1..kEpiWays-1: its helpers), 16 TMEM columns per tcgen05.ld,
// double-buffered (the next own group is in flight while the current one is combined).
// Accumulators hold (integer sum) * 2^-24, so digit k weighs 2^(16-9k); the fp64 combination
// is exact and fma(scale, q, bias) rounds once.  Running argmax over ascending classes (ties
// -> lowest).
__device__ __forceinline__ void svm_epilogue_groups(uint32_t lane_addr, const double2* tab,
                                                    int nc, int par, bool live, float* scores,
                                                    int64_t crop, int C, int class0,
                                                    float& best, int& best_c) {
    auto combine4 = [&](const uint32_t (&v)[16], int c4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int lc = c4 + j;
            const double2 sb = tab[lc < kPassClasses ? lc : 0];
            double q = (double)__uint_as_float(v[4 * j + 0]) * 0x1p16;
            q = fma((double)__uint_as_float(v[4 * j + 1]), 0x1p7, q);
            q = fma((double)__uint_as_float(v[4 * j + 2]), 0x1p-2, q);
            q = fma((double)__uint_as_float(v[4 * j + 3]), 0x1p-11, q);
            const float sc = (float)fma(sb.x, q, sb.y);
            if (lc < nc && live) {
                if (scores) scores[crop * C + class0 + lc] = sc;
                if (best_c < 0 || sc > best) {
                    best = sc;
                    best_c = class0 + lc;
                }
            }
        }
    };
    constexpr int kStep = 4 * kEpiWays;
    uint32_t va[16], vb[16];
    int c4 = 4 * par;
    if (c4 < nc) {
        tmem_ld16(lane_addr + (uint32_t)(4 * c4), va);
        tmem_ld_wait_regs(va);
    }
    for (; c4 < nc; c4 += 2 * kStep) {
        const bool has_b = c4 + kStep < nc, has_a2 = c4 + 2 * kStep < nc;  // warp-uniform
        if (has_b) tmem_ld16(lane_addr + (uint32_t)(4 * (c4 + kStep)), vb);
        combine4(va, c4);
        if (has_b) {
            tmem_ld_wait_regs(vb);
            if (has_a2) tmem_ld16(lane_addr + (uint32_t)(4 * (c4 + 2 * kStep)), va);
            combine4(vb, c4 + kStep);
            if (has_a2) tmem_ld_wait_regs(va);
        }
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
svm_gemm_kernel(const __grid_constant__ CUtensorMap a_map, const __grid_constant__ CUtensorMap b_map,
                const __grid_constant__ CUtensorMap b_last_map,
                const uint16_t* __restrict__ desc, int32_t n, const float* __restrict__ W,
                const float* __restrict__ bias, const uint8_t* __restrict__ ws, SvmPrepHeader h,
                int stages, int stage_bytes, float* __restrict__ scores,
                int32_t* __restrict__ labels, float* __restrict__ top_score,
                float reject_threshold) {
    extern __shared__ uint8_t smem_raw[];
#ifdef LBP_SVM_TRACE  // developer phase timestamps (globaltimer) of cluster 0 and the last one:
                      // entry, prologue done, last MMA issued, MMAs done, epilogue done, exit
#define SVM_TRACE(slot)                                                                    \
    do {                                                                                   \
        const uint32_t cl_ = cluster_id_x();                                               \
        if (cl_ == 0 || cl_ == n_clusters_x() - 1) {                                       \
            unsigned long long gt;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                         \
            g_svm_trace[(cl_ == 0 ? 0 : 1) * 16 + cluster_ctarank() * 8 + (slot)] = gt;    \
        }                                                                                  \
    } while (0)
#else
#define SVM_TRACE(slot) do {} while (0)
#endif
    if (threadIdx.x == 0) SVM_TRACE(0);
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const GemmSmem L{stages, stage_bytes};
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* ready = full + stages;
    uint64_t* empty = ready + stages;
    uint64_t* tmem_full = empty + stages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = (int)cluster_id_x(), n_pairs_grid = (int)n_clusters_x();
    const int C = h.n_classes;
    const int KC = h.dim_pad / kGemmK;
    const float* scales = reinterpret_cast<const float*>(ws + h.scale_off);

    if (threadIdx.x == 0) {
        tmem_slot[1] = prep_header_ok(ws, h, W) ? 0u : 1u;  // (read after __syncthreads)
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 2);
            mbar_init(&empty[s], 5);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 8);
        fence_mbar_init();
        prefetch_tensormap(&a_map);
        prefetch_tensormap(&b_map);
        prefetch_tensormap(&b_last_map);
    }
    if (warp == 1) {
        tmem_alloc_pair(tmem_slot, 512);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // a workspace that does not belong to this model: no tile is scored (nothing of the
    // workspace is read past its header), every row gets LBP_LABEL_BAD_MODEL below
    const bool bad_model = tmem_slot[1] != 0u;
    const int n_tiles = bad_model ? 0 : (n + 2 * kGemmM - 1) / (2 * kGemmM);
    // programmatic dependent launch: the prologue above may overlap the tail of the kernel
    // that wrote the descriptors; everything below reads them (no-op without PDL).  The next
    // kernel on the stream (the next batch's extraction) may be scheduled from now on: it waits
    // for this grid's completion before it touches the descriptors.
    launch_dependents();
    grid_dependency_wait();
    if (threadIdx.x == 0) SVM_TRACE(1);

    if (warp == 0) {
        // ===================== TMA producer (each CTA: its A rows and its half of B)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                int row0 = 0;
                for (int p = 0; p < h.n_pass; ++p) {
                    const int rows = pass_rows(pass_classes(C, p));
                    const int half = rows / 2;
                    const CUtensorMap* bm = (p + 1 < h.n_pass || h.n_pass == 1) ? &b_map : &b_last_map;
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&empty[s], ph ^ 1);
                        mbar_arrive_expect_tx(&full[s], (kGemmM + half) * kRowBytes);
                        tma_load_2d(L.a(smem, s), &a_map, &full[s], kc * kGemmK,
                                    t * 2 * kGemmM + (int)rank * kGemmM);
                        tma_load_2d(L.b(smem, s), bm, &full[s], kc * kGemmK, row0 + (int)rank * half);
                        if (++s == stages) { s = 0; ph ^= 1; }
                    }
                    row0 += rows;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA, single thread)
        // The whole warp runs the loop (warp-uniform control flow keeps the descriptor
        // arithmetic in uniform registers); one elected lane issues the MMAs and commits.
        if (rank == 0) {
            int s = 0;
            uint32_t ph = 0, acc_ph = 0;
            // 128-B swizzle descriptors differ only in the 14-bit start-address field of the
            // low word: desc(base + off) = desc(base) + off / 16 while the address stays < 256 KB
            const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
            const uint32_t d_hi = (uint32_t)(d0 >> 32), d_lo0 = (uint32_t)d0;
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                for (int p = 0; p < h.n_pass; ++p) {
                    const int rows = pass_rows(pass_classes(C, p));
                    const bool two = rows > 256;
                    const int nn = two ? rows / 2 : rows;  // N per MMA (multiple of 16)
                    const uint32_t idesc = idesc_f16_f32(2 * kGemmM, nn);
                    const uint32_t b2_off = (uint32_t)(nn / 2) * kRowBytes / 16;  // 2nd half's B rows
                    mbar_wait(tmem_empty, acc_ph ^ 1);  // both epilogues drained TMEM
                    acc_ph ^= 1;
                    tc_fence_after();
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&ready[s], ph);
                        tc_fence_after();
                        const uint32_t a_lo = d_lo0 + (uint32_t)(s * stage_bytes) / 16;
                        const uint32_t b_lo = a_lo + (uint32_t)(kGemmM * kGemmK * 2) / 16;
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < kGemmK / 16; ++ks) {
                                const uint64_t ad = ((uint64_t)d_hi << 32) | (a_lo + 2 * ks);
                                const uint32_t acc = (kc | ks) != 0;
                                mma_f16_ss_pair(tmem_base, ad, ((uint64_t)d_hi << 32) | (b_lo + 2 * ks),
                                                idesc, acc);
                                if (two)
                                    mma_f16_ss_pair(tmem_base + nn, ad,
                                                    ((uint64_t)d_hi << 32) | (b_lo + b2_off + 2 * ks),
                                                    idesc, acc);
                            }
                            mma_commit_pair(&empty[s], 0x3);  // stage free in both CTAs
                        }
                        __syncwarp();
                        if (++s == stages) { s = 0; ph ^= 1; }
                    }
                    if (elect_one()) mma_commit_pair(tmem_full, 0x3);  // pass accumulators done
                    __syncwarp();
                    if (lane == 0) SVM_TRACE(2);
                }
            }
        }
    } else if (warp == 6) {
        // ===================== relay: "stage s landed in this CTA" -> leader's MMA issuer
        if (lane == 0) {
            const uint32_t ready_leader = mapa_shared(smem_u32(ready), 0);
            int s = 0;
            uint32_t ph = 0;
            const int chunks = ((n_tiles - pair + n_pairs_grid - 1) / n_pairs_grid) * h.n_pass * KC;
            for (int i = 0; i < chunks; ++i) {
                mbar_wait(&full[s], ph);
                mbar_arrive_cluster(ready_leader + s * 8);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= 7) {
        // ===================== epilogue helpers (warps 7..10): the odd 8-class groups of the
        // same TMEM lane quarter as checker warp (warp & 3); their per-row argmax is merged
        // by the checker through shared memory
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        double2* epi_tab = reinterpret_cast<double2*>(smem + stages * stage_bytes + 512);
        const int par = 1 + (warp - 7) / 4;  // helper set 1 (warps 7..10) or 2 (11..14)
        float* hbest = reinterpret_cast<float*>(epi_tab + 2 * kPassClasses) + (par - 1) * kGemmM;
        int* hcls = reinterpret_cast<int*>(reinterpret_cast<float*>(epi_tab + 2 * kPassClasses) +
                                           (kEpiWays - 1) * kGemmM) + (par - 1) * kGemmM;
        int pc = 0;
        uint32_t acc_ph = 0;
        for (int t = pair; t < n_tiles; t += n_pairs_grid) {
            const int64_t crop = (int64_t)t * 2 * kGemmM + (int64_t)rank * kGemmM + row;
            int class0 = 0;
            for (int p = 0; p < h.n_pass; ++p) {
                const int nc = pass_classes(C, p);
                const double2* tab = epi_tab + (pc & 1) * kPassClasses;
                named_barrier_sync(2, 128 * kEpiWays);  // the pass's (scale, bias) table
                mbar_wait(tmem_full, acc_ph);
                acc_ph ^= 1;
                tc_fence_after();
                const uint32_t lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
                const bool live = crop < n;
                float best = 0.0f;
                int best_c = -1;
                svm_epilogue_groups(lane_addr, tab, nc, par, live, scores, crop, C, class0, best,
                                    best_c);
                hbest[row] = best;
                hcls[row] = best_c;
                tc_fence_before();
                named_barrier_sync(3, 128 * kEpiWays);  // partial argmaxes for the checkers
                class0 += nc;
                ++pc;
            }
        }
    } else {
        // ===================== checkers + epilogue (warps 2..5, 128 threads per CTA)
        const int et = threadIdx.x - 64;           // 0..127
        const int quarter = warp & 3;              // TMEM lane quarter accessible by this warp
        const int row = quarter * 32 + lane;       // accumulator row = crop within the CTA's half
        const uint32_t tmem_empty_leader = mapa_shared(smem_u32(tmem_empty), 0);
        double2* epi_tab = reinterpret_cast<double2*>(smem + stages * stage_bytes + 512);
        int s = 0, pc = 0;
        uint32_t ph = 0, acc_ph = 0;
        for (int t = pair; t < n_tiles; t += n_pairs_grid) {
            const int64_t crop = (int64_t)t * 2 * kGemmM + (int64_t)rank * kGemmM + row;
            float best = 0.0f;
            int best_c = -1;
            int class0 = 0;
            uint32_t flag_or = 0;
            for (int p = 0; p < h.n_pass; ++p) {
                const int nc = pass_classes(C, p);
                for (int kc = 0; kc < KC; ++kc) {
                    mbar_wait(&full[s], ph);
                    // the A tile is used AS IS: a u16 count x < 2048 read as fp16 bits is
                    // exactly x * 2^-24 (subnormal for x < 1024, exponent field 1 below 2048);
                    // larger counts are flagged here and their tile takes the fp64 fallback
                    const uint32_t a_addr = smem_u32(L.a(smem, s));
                    uint32_t big = 0;
#pragma unroll
                    for (int j = 0; j < (kGemmM * kRowBytes) / (16 * 128); ++j) {
                        const uint4 v = ld_shared_u32x4(a_addr + (j * 128 + et) * 16);
                        big |= (v.x | v.y | v.z | v.w) & 0xF800F800u;
                    }
                    flag_or |= big;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done reading stage s
                    if (++s == stages) { s = 0; ph ^= 1; }
                }
                // ---- epilogue of this pass (this CTA's 128 rows; its own count flag: the
                // rows of the two CTAs are disjoint).  (scale, bias) of the pass's classes are
                // staged in smem, double-buffered by pass parity; the barrier below orders them.
                double2* tab = epi_tab + (pc & 1) * kPassClasses;
                for (int i = et; i < kPassClasses; i += 128)
                    tab[i] = i < nc ? make_double2((double)__ldg(scales + class0 + i),
                                                   (double)__ldg(bias + class0 + i))
                                    : make_double2(0.0, 0.0);
                const bool tile_big = named_barrier_or(1, 128, flag_or != 0);
                named_barrier_sync(2, 128 * kEpiWays);  // the table for the helper warps
                mbar_wait(tmem_full, acc_ph);
                if (et == 0) SVM_TRACE(3);
                acc_ph ^= 1;
                tc_fence_after();
                const uint32_t lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
                // column sum sum_d x_d from the all-ones row (exactness precondition)
                const uint32_t colsum_bits = tmem_ld1(lane_addr + (uint32_t)(4 * nc));
                tmem_ld_wait();
                const float colsum = __uint_as_float(colsum_bits);
                const bool exact = (colsum < 0x1p-8f) && !tile_big;
                const bool live = crop < n;
                const float best_prev = best;  // argmax over the earlier passes
                const int best_c_prev = best_c;
                // the 4-class groups 0, 3, 6, .. here, the others in the two helper warps
                svm_epilogue_groups(lane_addr, tab, nc, 0, live, scores, crop, C, class0, best,
                                    best_c);
                named_barrier_sync(3, 128 * kEpiWays);  // the helpers' partial argmaxes
                {
                    const float* hbest = reinterpret_cast<const float*>(epi_tab + 2 * kPassClasses);
                    const int* hcls = reinterpret_cast<const int*>(hbest + (kEpiWays - 1) * kGemmM);
#pragma unroll
                    for (int hset = 0; hset < kEpiWays - 1; ++hset) {
                        const float hb = hbest[hset * kGemmM + row];
                        const int hc = hcls[hset * kGemmM + row];
                        if (hc >= 0 && (best_c < 0 || hb > best || (hb == best && hc < best_c))) {
                            best = hb;
                            best_c = hc;
                        }
                    }
                }
                if (!exact && live) {
                    // exactness preconditions broken for this row: redo the pass in fp64 on
                    // CUDA cores (rare: huge cells or sums; the oracle's definition)
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
            if (et == 0) SVM_TRACE(4);
        }
    }
    if (bad_model) write_bad_model(n, C, scores, labels, top_score);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's TMEM / smem are no longer used by the leader's MMAs
    if (warp == 1) tmem_dealloc_pair(tmem_base, 512);
    if (threadIdx.x == 0) SVM_TRACE(5);
}

// ---------------------------------------------------------------------------- host side

inline bool encode_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize,
                      uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                      uint32_t box_outer) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    (void)esize;
    return fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline cudaError_t launch_svm_gemm(const uint16_t* desc, int32_t n, int32_t dim, const float* W,
                                   const float* bias, const SvmPrepHeader& h, const uint8_t* ws,
                                   float* scores, int32_t* labels, float* top, float reject,
                                   int sms, cudaStream_t stream) {
    CUtensorMap am, bm, blm;
    const int rows_last = pass_rows(pass_classes(h.n_classes, h.n_pass - 1));
    if (!encode_2d(&am, desc, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (uint64_t)dim, (uint64_t)n,
                   (uint64_t)dim * 2, kGemmK, kGemmM))
        return cudaErrorNotSupported;
    // one TMA box = one CTA's half of a pass (<= 256 rows)
    if (!encode_2d(&bm, ws + h.q_off, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)h.dim_pad,
                   (uint64_t)h.total_rows, (uint64_t)h.dim_pad * 2, kGemmK, h.rows_max / 2) ||
        !encode_2d(&blm, ws + h.q_off, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)h.dim_pad,
                   (uint64_t)h.total_rows, (uint64_t)h.dim_pad * 2, kGemmK, rows_last / 2))
        return cudaErrorNotSupported;
    const int stage_bytes = kGemmM * kGemmK * 2 + (h.rows_max / 2) * kGemmK * 2;
    const int budget = 216 * 1024;
    int stages = budget / stage_bytes;
    stages = stages > 12 ? 12 : stages;
    if (stages < 2) return cudaErrorNotSupported;
    // + 1024 alignment slack + 512 barriers + epilogue table
    const int smem = stages * stage_bytes + 1024 + 512 + 2 * kPassClasses * 16 +
                     2 * (kEpiWays - 1) * kGemmM * 4 + 16;  // + the helpers' per-row argmax
    cudaError_t e = cudaFuncSetAttribute(svm_gemm_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (n + 2 * kGemmM - 1) / (2 * kGemmM);
    const int pairs = tiles < sms / 2 ? tiles : sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (grid_dependency_wait)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, svm_gemm_kernel, am, bm, blm, desc, n, W, bias, ws, h, stages,
                              stage_bytes, scores, labels, top, reject);
}

}  // namespace lbpf
