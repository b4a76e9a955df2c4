// svm_gemm_u8.cuh -- the exact linear-SVM scorer (P:142 hyperplane, P:144
// one identity against the others) reading the COMPACT descriptor of lbp_extract_u8:
// packed[n][d] = count & 255 (u8, rows of `pitch` bytes) plus, per row, the entries whose
// count exceeds 255 as (d << 16 | count) records (include/lbpfused.h).  The u8 rows are the
// tcgen05 A operand as they are: TMA loads them straight into the 128-B-swizzled stage, no
// conversion (the u16 kernel of svm_gemm_i8.cuh packs every tile in shared memory first and
// reads twice the bytes).
//
// Weights as unsigned base-256 digits of an offset fraction (as in svm_gemm_i8.cuh): with
// m_c = 2^e > max|W[c]|,  u = (W[c][d] / m_c + 1) / 2 in (0, 1),  U = rint(u 2^(8 D)) =
// sum_{k<D} d_k 2^(8(D-1-k)),  d_k in [0, 255],  so
//   sum_d x_d W[c][d] = m_c (2 sum_d x_d u_d - X),  X = sum_d x_d,
// and the GEMM computes the D digit products S_k = sum_d p_d d_k[d] and X (an all-ones row)
// EXACTLY in s32 (p = packed, 255 * 255 * dim < 2^31 for dim <= 32,768).  The epilogue forms
// Q = sum_k S_k 2^(8(D-1-k)) in int64 and s = b + m_c (Q 2^-(8D-1) - X) in fp64; an entry
// above 255 adds (count & ~255) W[c][d] exactly in fp64 (its low byte went through the GEMM).
// The result is the oracle's definition up to the 2^-(8D) m_c quantisation of W and fp64
// rounding, rounded once to fp32.  D = 5 when scores are requested (|W error|
// <= 2^-40 m_c).  Labels and top scores only: D = 4 (|W error| <= 2^-32 m_c, a fifth fewer
// MMAs) with a PROOF per row -- every approximate score a_c is within
//   E = max_c m_c * X * 2^-32 (1 + 2^-20) + (max_c m_c * Xt + max_c |b_c|) * 2^-40
// (Xt = sum of the true counts) of the exact score, so the row's argmax is certain when the
// two largest a_c differ by more than 2E, and its top score is within R13 when E <= 2^-21 |a1|;
// a row that fails either test (or lies within E of the reject threshold) gets
// LBP_LABEL_RECHECK and the fix-up kernel (svm_u8_fixup_kernel) recomputes it exactly in fp64.
//
// TMEM / B layout of one pass of P classes: column j*D + k = digit k of the pass's class j
// (class-major: 8 classes are 8*D consecutive columns, one x32 + one x8 load for D = 5),
// column D*P = X, zero columns up to N = roundup(D*P + 1, 16) <= 256.  One MMA of N columns
// per K step (cta_group::2, M = 256: 128 crops per CTA); CTA r of the pair holds the B rows of
// columns r*N/2 + [0, N/2) (svm_prepare_u8 stores them in that order, so each CTA's half of a
// pass is one TMA box).  P = ceil(C / n_pass), n_pass = ceil(C / floor(255/D)): C = 100 is two
// passes of 50 classes, C = 1000 twenty.  TMEM holds TWO accumulators (columns 0 and 256), so
// the epilogue of pass p overlaps the MMAs of pass p + 1 (tmem_full / tmem_empty per buffer).
//
// Warps: 0 = TMA producer (A 128 x 128 B + B N/2 x 128 B per stage), 1 = TMEM allocator and,
// on the leader CTA, the MMA issuer, 2 = relay ("stage s landed here" -> the leader's
// ready[s]), 3..14 = epilogue, three warps per TMEM lane quarter (quarter = warp & 3); the
// first of each quarter's warps also loads its rows' exception records and stages the W
// columns they need.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ptx.cuh"
#include "svm_gemm.cuh"
#include "svm_gemm_i8.cuh"

namespace lbpf {

constexpr uint32_t kPrepU8Magic = 0x35554D53u;  // "SMU5": D = 5 planes, then D = 4 planes
constexpr int kU8Digits = 5;                    // (the scores layout; D = 4: label-only)
constexpr int32_t kLabelRecheck = -3;           // row left for svm_u8_fixup_kernel
constexpr int kU8K = 128;              // K per stage: one 128-B u8 row
constexpr int kU8Threads = 480;        // 15 warps (see above)
constexpr int kU8EpiWays = 3;          // epilogue warps per TMEM lane quarter
constexpr int kU8Chunk = 8;            // classes per epilogue chunk
constexpr int kU8BigMax = 8;           // entries above 255 per row kept in shared memory
constexpr int kU8Distinct = 32;        // distinct such columns per CTA tile with W staged
constexpr int kU8MaxDim = 32768;       // s32 digit products, int64 Q (as svm_gemm_i8.cuh)
constexpr int kU8DbitsWords = kU8MaxDim / 32;
constexpr int kU8Stages = 6;             // 32-KB stages (A 16 KB + B 128 x 128 B)

struct U8Layout {
    int P, N, n_pass;
};
__host__ __device__ inline U8Layout u8_layout(int C, int D = kU8Digits) {
    const int pmax = 255 / D;  // one 256-column TMEM buffer per pass
    const int np = (C + pmax - 1) / pmax;
    const int P = (C + np - 1) / np;
    return {P, (D * P + 1 + 15) / 16 * 16, np};
}
// the header describes the D = 5 planes; the D = 4 planes follow them
inline bool svm_layout_u8(int32_t C, int32_t D, SvmPrepHeader* h) {
    if (C < 1 || D < 1 || D > kU8MaxDim) return false;
    const U8Layout L = u8_layout(C);
    h->magic = kPrepU8Magic;
    h->n_classes = C;
    h->dim = D;
    h->dim_pad = (D + kU8K - 1) / kU8K * kU8K;
    h->n_pass = L.n_pass;
    h->rows_max = L.N;
    h->total_rows = L.N * L.n_pass;
    h->scale_off = 1024;
    h->q_off = (1024 + 4 * C + 1023) / 1024 * 1024;
    return true;
}
__host__ __device__ inline size_t u8_q4_off(const SvmPrepHeader& h) {
    return (size_t)h.q_off + (size_t)h.total_rows * h.dim_pad;
}
inline size_t svm_layout_u8_total(const SvmPrepHeader& h) {
    const U8Layout L4 = u8_layout(h.n_classes, 4);
    return u8_q4_off(h) + (size_t)L4.N * L4.n_pass * h.dim_pad;
}

// One block per stored B row of the D-digit planes.
template <int D>
__global__ void svm_prepare_u8_kernel(const float* __restrict__ W, SvmPrepHeader h,
                                      uint8_t* __restrict__ ws) {
    __shared__ float red[32];
    const int row = blockIdx.x;
    if (D == kU8Digits && row == 0 && threadIdx.x == 0) write_prep_header(ws, h, W);
    const U8Layout L = u8_layout(h.n_classes, D);
    const int p = row / L.N, col = row % L.N;  // storage row = natural column (CTA r: r*N/2..)
    uint8_t* q = ws + (D == kU8Digits ? (size_t)h.q_off : u8_q4_off(h)) + (size_t)row * h.dim_pad;
    const int j = col / D, k = col % D;
    const int c = p * L.P + j;
    if (col >= D * L.P || c >= h.n_classes) {  // X row (all ones) or padding
        const uint8_t v = (col == D * L.P) ? 1 : 0;
        for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x) q[d] = d < h.dim ? v : 0;
        return;
    }
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
    if (D == kU8Digits && k == 0 && threadIdx.x == 0)
        reinterpret_cast<float*>(ws + h.scale_off)[c] = (float)m;
    for (int d = threadIdx.x; d < h.dim_pad; d += blockDim.x) {
        uint8_t dig = 0;
        if (d < h.dim) {
            const double u = ((double)w[d] / m + 1.0) * 0.5;                 // exact in fp64
            const long long U = llrint(ldexp(u, 8 * D));                     // < 2^(8D)
            dig = (uint8_t)((U >> (8 * (D - 1 - k))) & 0xFF);
        }
        q[d] = dig;
    }
}

struct U8Epi {
    uint32_t lane_addr;   // TMEM address of the row's lane quarter in the pass's buffer
    const double2* tab;   // (scale, bias) of the pass's classes
    int nc, class0, C;
    int32_t X;            // sum_d packed[d] (ones column)
    bool live;
    int n_big, row;
    const uint32_t* big;  // smem [kGemmM][kU8BigMax]: (column-list index << 16) | (count & ~255)
    uint32_t wcol0;       // smem address of the staged W columns [kU8Distinct][P]
    int P;
    float* scores;
    int64_t crop;
};

// The running result of a row: argmax over fp32 scores (scores mode), or the two largest
// fp64 approximations (label-only mode: a1 of class c1, a2).
struct U8Best {
    double a1, a2;
    int c1;
};

// TMEM columns of the chunk of classes [c0, c0 + kU8Chunk) of a buffer: 8 D columns (x32 + x8
// loads for D = 5, one x32 for D = 4).  A chunk that would cross the buffer's end (the last
// chunk of a pass of more than 48 (D = 5) classes) holds at most 3 real classes = 15 columns:
// one x16 load (real columns lie below D P + 1 <= 256).
struct U8Chunk {
    uint32_t a[32], b[8];
};
template <int D>
__device__ __forceinline__ void u8_load_wait(const U8Epi& e, int c0, U8Chunk& v) {
    if (c0 * D + 8 * D <= 256) {  // warp-uniform
        tmem_ld32(e.lane_addr + (uint32_t)(c0 * D), v.a);
        if (D > 4) tmem_ld8(e.lane_addr + (uint32_t)(c0 * D + 32), v.b);
        tmem_ld_wait_regs(v.a);
        if (D > 4) tmem_ld_wait_regs(v.b);
    } else {
        uint32_t (&h)[16] = *reinterpret_cast<uint32_t (*)[16]>(v.a);
        tmem_ld16(e.lane_addr + (uint32_t)(c0 * D), h);
        tmem_ld_wait_regs(h);
    }
}

// classes [c0, c0 + kU8Chunk) of the pass from their loaded columns: Q by Horner over the D
// digits, s = b + m (Q 2^-(8D-1) - X) [+ the exact high parts of the entries above 255].
// Scores mode (LBL false): fp32 scores, running argmax over ascending classes (ties ->
// lowest).  LBL: the fp64 values feed the two-largest tracker.  kBig: the warp has rows with
// entries above 255.
template <int D, bool LBL, bool kBig>
__device__ __forceinline__ void u8_combine(const U8Epi& e, int c0, const U8Chunk& v, U8Best& r) {
#pragma unroll
    for (int j = 0; j < kU8Chunk; ++j) {
        long long q = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int i = j * D + k;
            q = (q << 8) + (int32_t)(i < 32 ? v.a[i] : v.b[i - 32]);
        }
        const int lc = c0 + j;
        const double2 sb = e.tab[lc < e.nc ? lc : 0];
        const double sm = fma((double)q, ldexp(1.0, 1 - 8 * D), -(double)e.X);
        double acc = fma(sb.x, sm, sb.y);
        if (kBig && lc < e.nc) {
            for (int t = 0; t < e.n_big; ++t) {
                const uint32_t rec = e.big[e.row * kU8BigMax + t];
                const float w = __uint_as_float(
                    ld_shared_u32(e.wcol0 + ((rec >> 16) * (uint32_t)e.P + (uint32_t)lc) * 4));
                acc = fma((double)(rec & 0xFFFFu), (double)w, acc);
            }
        }
        if (lc < e.nc && e.live) {
            if constexpr (LBL) {
                if (r.c1 < 0 || acc > r.a1) {
                    r.a2 = r.a1;
                    r.a1 = acc;
                    r.c1 = e.class0 + lc;
                } else if (acc > r.a2) {
                    r.a2 = acc;
                }
            } else {
                const float sc = (float)acc;
                if (e.scores) e.scores[e.crop * e.C + e.class0 + lc] = sc;
                if (r.c1 < 0 || sc > (float)r.a1) {
                    r.a1 = sc;
                    r.c1 = e.class0 + lc;
                }
            }
        }
    }
}

// this warp's chunks c0 = kU8Chunk (par + kU8EpiWays i) of the pass
template <int D, bool LBL, bool kBig>
__device__ __forceinline__ void u8_epi_chunks_t(const U8Epi& e, int par, U8Best& r) {
    for (int c0 = kU8Chunk * par; c0 < e.nc; c0 += kU8Chunk * kU8EpiWays) {
        U8Chunk v;
        u8_load_wait<D>(e, c0, v);
        u8_combine<D, LBL, kBig>(e, c0, v, r);
    }
}
template <int D, bool LBL>
__device__ __forceinline__ void u8_epi_chunks(const U8Epi& e, int par, U8Best& r) {
    if (__any_sync(0xFFFFFFFFu, e.n_big != 0)) u8_epi_chunks_t<D, LBL, true>(e, par, r);
    else u8_epi_chunks_t<D, LBL, false>(e, par, r);
}

// merge b into a (label-only mode: the two largest values; scores mode: the argmax with ties
// to the lower class)
template <bool LBL>
__device__ __forceinline__ void u8_merge(U8Best& a, const U8Best& b) {
    if (b.c1 < 0) return;
    if constexpr (LBL) {
        if (a.c1 < 0 || b.a1 > a.a1 || (b.a1 == a.a1 && b.c1 < a.c1)) {
            a.a2 = fmax(a.c1 < 0 ? -INFINITY : a.a1, fmax(a.a2, b.a2));
            a.a1 = b.a1;
            a.c1 = b.c1;
        } else {
            a.a2 = fmax(a.a2, fmax(b.a1, b.a2));
        }
    } else {
        if (a.c1 < 0 || b.a1 > a.a1 || (b.a1 == a.a1 && b.c1 < a.c1)) a = b;
    }
}

// Rows with more than kU8BigMax entries above 255 (or a tile with more than kU8Distinct
// distinct such columns): the pass's classes in fp64 on CUDA cores from the packed row and its
// exception records (exact products; rare -- a crop with many uniform 16 x 16 cells).
template <bool LBL>
__device__ __noinline__ void u8_row_fp64(const uint8_t* __restrict__ packed, int64_t pitch,
                                         const uint32_t* __restrict__ exc, int32_t exc_cap,
                                         int n_exc, int64_t crop, int dim, const float* W,
                                         const float* bias, int class0, int nc, int C,
                                         float* scores, U8Best& r) {
    const uint8_t* x = packed + crop * pitch;
    for (int lc = 0; lc < nc; ++lc) {
        const int c = class0 + lc;
        const float* w = W + (size_t)c * dim;
        double acc = (double)__ldg(bias + c);
        for (int d = 0; d < dim; ++d) acc = fma((double)__ldg(w + d), (double)x[d], acc);
        for (int t = 0; t < n_exc; ++t) {
            const uint32_t rc = exc[crop * exc_cap + t];
            acc = fma((double)(rc & 0xFF00u), (double)__ldg(w + (rc >> 16)), acc);
        }
        U8Best one{LBL ? acc : (double)(float)acc, -INFINITY, c};
        if (!LBL && scores) scores[crop * C + c] = (float)acc;
        u8_merge<LBL>(r, one);
    }
}

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kU8Threads, 1)
svm_gemm_u8_kernel(const __grid_constant__ CUtensorMap a_map,
                   const __grid_constant__ CUtensorMap b_map, const uint8_t* __restrict__ packed,
                   int64_t pitch, const int32_t* __restrict__ exc_n,
                   const uint32_t* __restrict__ exc, int32_t exc_cap, int32_t n,
                   const float* __restrict__ W, const float* __restrict__ bias,
                   const uint8_t* __restrict__ ws, SvmPrepHeader h, float* __restrict__ scores,
                   int32_t* __restrict__ labels, float* __restrict__ top_score,
                   float reject_threshold) {
    constexpr bool LBL = D < kU8Digits;  // label-only mode (scores == NULL)
    extern __shared__ uint8_t smem_raw[];
    // (developer builds with -DLBP_SVM_TRACE: phase timestamps, svm_gemm.cuh's SVM_TRACE;
    // slots: 0 entry, 1 dependency wait done, 6 first stage ready, 2 last MMA issued,
    // 3 accumulators complete, 4 epilogue done, 5 exit)
    if (threadIdx.x == 0) SVM_TRACE(0);
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const U8Layout LY = u8_layout(h.n_classes, D);
    const int stage_a = kGemmM * kU8K;          // 16 KB
    const int stage_bytes = stage_a + (LY.N / 2) * kU8K;
    uint8_t* tail = smem + kU8Stages * stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(tail);
    uint64_t* ready = full + kU8Stages;
    uint64_t* empty = ready + kU8Stages;
    uint64_t* tmem_full = empty + kU8Stages;   // [2]: accumulator buffer b complete
    uint64_t* tmem_empty = tmem_full + 2;      // [2]: both CTAs' epilogues drained buffer b
    uint64_t* hdr_bar = tmem_empty + 2;        // the workspace-header check has completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hdr_bar + 1);  // [0] TMEM, [1] bad model
    float* maxes = reinterpret_cast<float*>(tmem_slot + 2);           // [2] max m_c, max |b_c|
    double2* epi_tab = reinterpret_cast<double2*>(tail + 256);            // [2][P]
    uint32_t* big = reinterpret_cast<uint32_t*>(epi_tab + 2 * 128);      // [kGemmM][kU8BigMax]
    uint32_t* dbits = big + kGemmM * kU8BigMax;                          // [kU8DbitsWords]
    int32_t* dlist = reinterpret_cast<int32_t*>(dbits + kU8DbitsWords);  // [kU8Distinct]
    int32_t* dcount = dlist + kU8Distinct;                               // [4]
    float* wcol = reinterpret_cast<float*>(dcount + 4);                  // [kU8Distinct][P]
    int32_t* nbig = reinterpret_cast<int32_t*>(wcol + kU8Distinct * 128);  // [kGemmM]
    double* ha1 = reinterpret_cast<double*>(nbig + kGemmM);   // [kU8EpiWays - 1][kGemmM] x3
    double* ha2 = ha1 + (kU8EpiWays - 1) * kGemmM;
    int32_t* hc1 = reinterpret_cast<int32_t*>(ha2 + (kU8EpiWays - 1) * kGemmM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = (int)cluster_id_x(), n_pairs_grid = (int)n_clusters_x();
    const int C = h.n_classes;
    const int KC = h.dim_pad / kU8K;
    const float* scales = reinterpret_cast<const float*>(ws + h.scale_off);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kU8Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 2);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 8);  // the 4 first epilogue warps of each CTA
        }
        mbar_init(hdr_bar, 1);
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
    // The workspace was sized by the host (prepared_bytes >= svm_workspace_u8_bytes), so every
    // TMA of it stays inside the allocation; whether it belongs to this model (header + W
    // fingerprint, prep_header_ok) is checked by the relay warp concurrently with the MMAs and
    // only the epilogue waits for the verdict (hdr_bar) before it writes any output.
    const int n_tiles = (n + 2 * kGemmM - 1) / (2 * kGemmM);
    // Programmatic dependent launch: the prologue above may overlap the tail of the extraction
    // kernel.  Only the threads that read its output wait (griddepcontrol.wait is per thread):
    // the producer before its descriptor (A) loads -- the weight (B) loads of the first
    // stages go out before it -- and the epilogue before the exception records.  The fix-up
    // kernel of the label-only mode may be scheduled from now on.
    launch_dependents();

    if (warp == 0) {
        // ===================== TMA producer: A = 128 u8 rows x 128 B, B = this CTA's N/2 rows
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const int chunks = ((n_tiles - pair + n_pairs_grid - 1) / n_pairs_grid) * LY.n_pass * KC;
            const int pre = chunks < kU8Stages ? chunks : kU8Stages;
            // B of the first `pre` chunks (chunk i = pass i / KC, K block i % KC) before the wait
            for (int i = 0; i < pre; ++i) {
                mbar_arrive_expect_tx(&full[i], stage_bytes);
                tma_load_2d(smem + i * stage_bytes + stage_a, &b_map, &full[i], (i % KC) * kU8K,
                            ((i / KC) % LY.n_pass) * LY.N + (int)rank * (LY.N / 2));
            }
            grid_dependency_wait();
            SVM_TRACE(1);
            int i = 0;
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                const int arow = t * 2 * kGemmM + (int)rank * kGemmM;
                for (int p = 0; p < LY.n_pass; ++p) {
                    for (int kc = 0; kc < KC; ++kc, ++i) {
                        uint8_t* st = smem + s * stage_bytes;
                        if (i >= pre) {
                            mbar_wait(&empty[s], ph ^ 1);
                            mbar_arrive_expect_tx(&full[s], stage_bytes);
                            tma_load_2d(st + stage_a, &b_map, &full[s], kc * kU8K,
                                        p * LY.N + (int)rank * (LY.N / 2));
                        }
                        tma_load_2d(st, &a_map, &full[s], kc * kU8K, arow);
                        if (++s == kU8Stages) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; whole warp runs the loop, one lane issues)
        if (rank == 0) {
            int s = 0, gp = 0;  // gp: pass counter -> accumulator buffer gp & 1
            uint32_t ph = 0;
            const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
            const uint32_t d_hi = (uint32_t)(d0 >> 32), d_lo0 = (uint32_t)d0;
            const uint32_t idesc = idesc_u8_s32(2 * kGemmM, LY.N);
            for (int t = pair; t < n_tiles; t += n_pairs_grid) {
                for (int p = 0; p < LY.n_pass; ++p, ++gp) {
                    const int buf = gp & 1;
                    const uint32_t d_tmem = tmem_base + (uint32_t)(256 * buf);
                    // both CTAs' epilogues drained this buffer (its previous use, pass gp - 2)
                    mbar_wait(&tmem_empty[buf], (((uint32_t)gp >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                    for (int kc = 0; kc < KC; ++kc) {
                        mbar_wait(&ready[s], ph);
                        tc_fence_after();
                        if (kc == 0 && p == 0 && lane == 0) SVM_TRACE(6);
                        const uint32_t a_lo = d_lo0 + (uint32_t)(s * stage_bytes) / 16;
                        const uint32_t b_lo = a_lo + (uint32_t)stage_a / 16;
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < kU8K / 32; ++ks) {
                                const uint64_t ad = ((uint64_t)d_hi << 32) | (a_lo + 2 * ks);
                                const uint32_t acc = (kc | ks) != 0;
                                mma_i8_ss_pair(d_tmem, ad,
                                               ((uint64_t)d_hi << 32) | (b_lo + 2 * ks), idesc, acc);
                            }
                            mma_commit_pair(&empty[s], 0x3);  // stage free in both CTAs
                        }
                        __syncwarp();
                        if (++s == kU8Stages) { s = 0; ph ^= 1; }
                    }
                    if (elect_one()) mma_commit_pair(&tmem_full[buf], 0x3);
                    __syncwarp();
                    if (lane == 0) SVM_TRACE(2);
                }
            }
        }
    } else if (warp == 2) {
        // ===================== relay: "stage s landed in this CTA" -> the leader's ready[s]
        if (lane == 0) {
            // first, the workspace check (a few dependent global loads, off the MMA's path)
            tmem_slot[1] = prep_header_ok(ws, h, W) ? 0u : 1u;
            mbar_arrive(hdr_bar);  // (release: the flag is visible to the waiters)
            const uint32_t ready_leader = mapa_shared(smem_u32(ready), 0);
            int s = 0;
            uint32_t ph = 0;
            const int chunks = ((n_tiles - pair + n_pairs_grid - 1) / n_pairs_grid) * LY.n_pass * KC;
            for (int i = 0; i < chunks; ++i) {
                mbar_wait(&full[s], ph);
                mbar_arrive_cluster(ready_leader + s * 8);
                if (++s == kU8Stages) { s = 0; ph ^= 1; }
            }
        }
    } else {
        // ===================== epilogue: warps 3..14, three per TMEM lane quarter; par 0 (warps
        // 3..6) owns the row's exceptions, the (scale, bias) table and the final result
        const int quarter = warp & 3;
        const int par = (warp - 3) / 4;
        const int row = quarter * 32 + lane;
        const int et = par == 0 ? quarter * 32 + lane : -1;  // 0..127 for the par-0 warps
        const uint32_t tmem_empty_leader = mapa_shared(smem_u32(tmem_empty), 0);  // [2]
        const uint32_t lane_addr = tmem_base + ((uint32_t)(quarter * 32) << 16);
        if (LBL && par == 0) {  // max_c m_c and max_c |b_c| for the error bound E
            float ms = 0.0f, bs = 0.0f;
            for (int c = et; c < C; c += 128) {
                ms = fmaxf(ms, __ldg(scales + c));
                bs = fmaxf(bs, fabsf(__ldg(bias + c)));
            }
            if (et < 2) maxes[et] = 0.0f;
            named_barrier_sync(1, 128);
            atomicMax(reinterpret_cast<unsigned int*>(&maxes[0]), __float_as_uint(ms));
            atomicMax(reinterpret_cast<unsigned int*>(&maxes[1]), __float_as_uint(bs));
            named_barrier_sync(1, 128);
        }
        grid_dependency_wait();      // the exception records come from the extraction
        mbar_wait(hdr_bar, 0);       // the workspace verdict (long done when the MMAs finish)
        const bool bad = tmem_slot[1] != 0u;
        float* const out_scores = bad ? nullptr : scores;
        int pc = 0;  // pass counter -> accumulator buffer pc & 1 (as the MMA issuer's gp)
        for (int t = pair; t < n_tiles; t += n_pairs_grid) {
            const int64_t crop = (int64_t)t * 2 * kGemmM + (int64_t)rank * kGemmM + row;
            const bool live = crop < n;
            U8Best best{-INFINITY, -INFINITY, -1};
            int n_big = 0, n_exc = 0, X = 0;
            uint32_t xhi = 0;  // sum of the entries' high parts (count & ~255) of the row
            bool row_over = false;
            if (par == 0) {
                // ---- this tile's exception records: per row (<= kU8BigMax) and the tile's
                // distinct columns (bitmap dedup), indices into the column list
                for (int i = et; i < kU8DbitsWords; i += 128) dbits[i] = 0;
                if (et == 0) *dcount = 0;
                named_barrier_sync(1, 128);
                n_exc = live ? min(exc_n[crop], exc_cap) : 0;
                row_over = n_exc > kU8BigMax;
                for (int e = 0; e < n_exc; ++e) {
                    const uint32_t r = exc[crop * exc_cap + e];
                    xhi += r & 0xFF00u;
                    if (row_over) continue;
                    const uint32_t d = r >> 16;
                    const uint32_t bit = 1u << (d & 31);
                    if (!(atomicOr(&dbits[d >> 5], bit) & bit)) {
                        const int k = atomicAdd(dcount, 1);
                        if (k < kU8Distinct) dlist[k] = (int)d;
                    }
                }
                named_barrier_sync(1, 128);  // column list complete
                const int nd = *dcount;
                if (nd > kU8Distinct && n_exc > 0) row_over = true;  // W not staged: fp64 row
                if (!row_over) {
                    for (int e = 0; e < n_exc; ++e) {
                        const uint32_t r = exc[crop * exc_cap + e];
                        int k = 0;
                        while (dlist[k] != (int)(r >> 16)) ++k;
                        big[row * kU8BigMax + e] = ((uint32_t)k << 16) | (r & 0xFF00u);
                    }
                    n_big = n_exc;
                }
                nbig[row] = n_big;
            }
            int class0 = 0;
            for (int p = 0; p < LY.n_pass; ++p) {
                const int nc = min(LY.P, C - class0);
                double2* tab = epi_tab + (pc & 1) * 128;
                if (par == 0) {
                    for (int i = et; i < LY.P; i += 128)
                        tab[i] = i < nc ? make_double2((double)__ldg(scales + class0 + i),
                                                       (double)__ldg(bias + class0 + i))
                                        : make_double2(0.0, 0.0);
                    const int nd = min(*dcount, kU8Distinct);
                    for (int i = et; i < nd * LY.P; i += 128) {
                        const int k = i / LY.P, lc = i - k * LY.P;
                        wcol[i] = lc < nc ? __ldg(W + (size_t)(class0 + lc) * h.dim + dlist[k]) : 0.0f;
                    }
                }
                named_barrier_sync(2, 128 * kU8EpiWays);  // table, W columns, lists ready
                const int buf = pc & 1;
                mbar_wait(&tmem_full[buf], ((uint32_t)pc >> 1) & 1u);
                tc_fence_after();
                if (et == 0) SVM_TRACE(3);
                U8Epi e;
                e.lane_addr = lane_addr + (uint32_t)(256 * buf);
                e.X = (int32_t)tmem_ld1(e.lane_addr + (uint32_t)(D * LY.P));
                tmem_ld_wait();
                X = e.X;
                e.tab = tab; e.nc = nc; e.class0 = class0; e.C = C;
                e.live = live; e.n_big = nbig[row]; e.row = row; e.big = big;
                e.wcol0 = smem_u32(wcol); e.P = LY.P; e.scores = out_scores; e.crop = crop;
                U8Best pb{-INFINITY, -INFINITY, -1};
                u8_epi_chunks<D, LBL>(e, par, pb);
                if (par > 0) {
                    ha1[(par - 1) * kGemmM + row] = pb.a1;
                    ha2[(par - 1) * kGemmM + row] = pb.a2;
                    hc1[(par - 1) * kGemmM + row] = pb.c1;
                }
                tc_fence_before();
                named_barrier_sync(3, 128 * kU8EpiWays);  // TMEM read, helpers' results written
                if (par == 0) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tmem_empty_leader + 8 * buf);  // buffer free
#pragma unroll
                    for (int hs = 0; hs < kU8EpiWays - 1; ++hs)
                        u8_merge<LBL>(pb, U8Best{ha1[hs * kGemmM + row], ha2[hs * kGemmM + row],
                                                 hc1[hs * kGemmM + row]});
                    if (row_over && live) {  // the pass's classes in fp64 (rare)
                        pb = U8Best{-INFINITY, -INFINITY, -1};
                        u8_row_fp64<LBL>(packed, pitch, exc, exc_cap, n_exc, crop, h.dim, W, bias,
                                         class0, nc, C, out_scores, pb);
                    }
                    // passes ascend in class: on equal values the earlier pass's class stays
                    u8_merge<LBL>(best, pb);
                }
                class0 += nc;
                ++pc;
            }
            if (et == 0) SVM_TRACE(4);
            if (par == 0 && live && !bad) {
                float top = (float)best.a1;
                int32_t label = (top < reject_threshold) ? -1 : best.c1;
                if constexpr (LBL) {
                    // the proof of DESIGN.md §5 (label-only mode): every a_c is within E of the
                    // exact score; row_over rows were scored in fp64 (rounding term only)
                    const double mx = (double)maxes[0], bx = (double)maxes[1];
                    const double xt = (double)X + (double)xhi;
                    const double E = (row_over ? 0.0 : mx * (double)X * 0x1p-32 * (1.0 + 0x1p-20)) +
                                     (mx * xt + bx) * 0x1p-40;
                    const bool clear = (best.a2 == -INFINITY || best.a1 - best.a2 > 2.0 * E) &&
                                       E <= 0x1p-21 * fabs(best.a1) &&
                                       !(fabs(best.a1 - (double)reject_threshold) <= E);
                    if (!clear) {
                        label = kLabelRecheck;
                        top = __uint_as_float(0x7FC00000u);
                    }
                }
                if (top_score) top_score[crop] = top;
                if (labels) labels[crop] = label;
            }
            if (par == 0) named_barrier_sync(1, 128);  // nbig / lists consumed before reuse
        }
    }
    tc_fence_before();
    __syncthreads();  // (the relay's flag is visible to every thread after this)
    if (tmem_slot[1] != 0u) write_bad_model(n, C, scores, labels, top_score);
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair(tmem_base, 512);
    if (threadIdx.x == 0) SVM_TRACE(5);
}

// One row by one CTA on CUDA cores: the row staged in shared memory as fp32 (its entries
// above 255 restored from the records), one warp per class at a time, exact products
// accumulated in fp64, argmax over the fp32 scores (ties -> lowest class).
constexpr int kU8F64Threads = 256;
__device__ __forceinline__ void u8_score_row_cta(int64_t row, const uint8_t* __restrict__ packed,
                                                 int64_t pitch, const int32_t* __restrict__ exc_n,
                                                 const uint32_t* __restrict__ exc, int32_t exc_cap,
                                                 int32_t dim, const float* __restrict__ W,
                                                 const float* __restrict__ bias, int32_t C,
                                                 float* scores, int32_t* labels, float* top_score,
                                                 float reject_threshold, float* xs, float* wb,
                                                 int* wc) {
    constexpr int kWarps = kU8F64Threads / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* x = packed + row * pitch;
    for (int d = threadIdx.x; d < dim; d += blockDim.x) xs[d] = (float)x[d];
    __syncthreads();
    const int ne = min(exc_n[row], exc_cap);
    for (int t = threadIdx.x; t < ne; t += blockDim.x) {
        const uint32_t r = exc[row * exc_cap + t];
        xs[r >> 16] = (float)(r & 0xFFFFu);
    }
    __syncthreads();
    float best = 0.0f;
    int best_c = -1;
    for (int c = warp; c < C; c += kWarps) {
        const float* w = W + (size_t)c * dim;
        double acc = 0.0;
        for (int d = lane; d < dim; d += 32) acc = fma((double)__ldg(w + d), (double)xs[d], acc);
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
        const float sc = (float)(acc + (double)__ldg(bias + c));
        if (lane == 0 && scores) scores[row * C + c] = sc;
        if (best_c < 0 || sc > best) {  // classes ascend within the warp
            best = sc;
            best_c = c;
        }
    }
    if (lane == 0) {
        wb[warp] = best;
        wc[warp] = best_c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float b = 0.0f;
        int bc = -1;
        for (int i = 0; i < kWarps; ++i)
            if (wc[i] >= 0 && (bc < 0 || wb[i] > b || (wb[i] == b && wc[i] < bc))) {
                b = wb[i];
                bc = wc[i];
            }
        if (top_score) top_score[row] = b;
        if (labels) labels[row] = (b < reject_threshold) ? -1 : bc;
    }
    __syncthreads();
}

// CUDA-core scorer of the compact descriptor (batches under one 128-crop tile, rows not
// TMA-addressable, no prepared workspace): one CTA per crop.
__global__ void __launch_bounds__(kU8F64Threads)
svm_score_u8_fp64_kernel(const uint8_t* __restrict__ packed, int64_t pitch,
                         const int32_t* __restrict__ exc_n, const uint32_t* __restrict__ exc,
                         int32_t exc_cap, int32_t n, int32_t dim, const float* __restrict__ W,
                         const float* __restrict__ bias, int32_t C, float* __restrict__ scores,
                         int32_t* __restrict__ labels, float* __restrict__ top_score,
                         float reject_threshold) {
    extern __shared__ float xs[];  // [dim]
    __shared__ float wb[kU8F64Threads / 32];
    __shared__ int wc[kU8F64Threads / 32];
    for (int64_t row = blockIdx.x; row < n; row += gridDim.x)
        u8_score_row_cta(row, packed, pitch, exc_n, exc, exc_cap, dim, W, bias, C, scores,
                         labels, top_score, reject_threshold, xs, wb, wc);
}

// Label-only mode's fix-up (launched after svm_gemm_u8_kernel<4>, programmatic dependent
// launch): every row the tensor-core kernel could not prove (label kLabelRecheck) is scored
// exactly on CUDA cores.  Each CTA scans blocks of 256 labels (one coalesced load per thread)
// and scores the few flagged rows of its blocks.
__global__ void __launch_bounds__(kU8F64Threads)
svm_u8_fixup_kernel(const uint8_t* __restrict__ packed, int64_t pitch,
                    const int32_t* __restrict__ exc_n, const uint32_t* __restrict__ exc,
                    int32_t exc_cap, int32_t n, int32_t dim, const float* __restrict__ W,
                    const float* __restrict__ bias, int32_t C, int32_t* __restrict__ labels,
                    float* __restrict__ top_score, float reject_threshold) {
    extern __shared__ float xs[];  // [dim]
    __shared__ float wb[kU8F64Threads / 32];
    __shared__ int wc[kU8F64Threads / 32];
    __shared__ int list[kU8F64Threads];
    __shared__ int count;
    // (no launch_dependents here: scheduling the next batch's extraction this early measured
    // ~1 % slower per config4 step, tools/gpu_ab_bench.sh; it launches when this grid ends)
    grid_dependency_wait();  // the labels come from the tensor-core kernel
    for (int64_t base = (int64_t)blockIdx.x * kU8F64Threads; base < n;
         base += (int64_t)gridDim.x * kU8F64Threads) {
        if (threadIdx.x == 0) count = 0;
        __syncthreads();
        const int64_t row = base + threadIdx.x;
        if (row < n && labels[row] == kLabelRecheck) list[atomicAdd(&count, 1)] = (int)threadIdx.x;
        __syncthreads();
        const int m = count;
        for (int i = 0; i < m; ++i)
            u8_score_row_cta(base + list[i], packed, pitch, exc_n, exc, exc_cap, dim, W, bias, C,
                             nullptr, labels, top_score, reject_threshold, xs, wb, wc);
        __syncthreads();
    }
}

inline int u8_smem_bytes(int N) {
    return kU8Stages * (kGemmM * kU8K + (N / 2) * kU8K) + 1024 + 256 + 2 * 128 * 16 +
           kGemmM * kU8BigMax * 4 + kU8DbitsWords * 4 + (kU8Distinct + 4) * 4 +
           kU8Distinct * 128 * 4 + kGemmM * 4 + (kU8EpiWays - 1) * kGemmM * (8 + 8 + 4);
}

// D = 5 when scores are requested (or labels are not: the recheck marker lives in them) or
// the model fits two D = 5 passes (C <= 102: one tile's two passes, where the fix-up launch
// would cost more than the fifth of the MMAs it saves); else the label-only D = 4 kernel
// followed by its fix-up.
inline cudaError_t launch_svm_gemm_u8(const uint8_t* packed, int64_t pitch,
                                      const int32_t* exc_n, const uint32_t* exc, int32_t exc_cap,
                                      int32_t n, int32_t dim, const float* W, const float* bias,
                                      const SvmPrepHeader& h, const uint8_t* ws, float* scores,
                                      int32_t* labels, float* top, float reject, int sms,
                                      cudaStream_t stream) {
    const bool lbl = scores == nullptr && labels != nullptr && u8_layout(h.n_classes).n_pass > 2;
    const int D = lbl ? 4 : kU8Digits;
    const U8Layout LY = u8_layout(h.n_classes, D);
    if (LY.P > 128) return cudaErrorNotSupported;  // (the epilogue tables hold 128 classes)
    CUtensorMap am, bm;
    if (!encode_2d(&am, packed, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)dim, (uint64_t)n,
                   (uint64_t)pitch, kU8K, kGemmM))
        return cudaErrorNotSupported;
    const uint8_t* q = ws + (lbl ? u8_q4_off(h) : (size_t)h.q_off);
    if (!encode_2d(&bm, q, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)h.dim_pad,
                   (uint64_t)LY.N * LY.n_pass, (uint64_t)h.dim_pad, kU8K, LY.N / 2))
        return cudaErrorNotSupported;
    const int smem = u8_smem_bytes(LY.N);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    auto kern = lbl ? svm_gemm_u8_kernel<4> : svm_gemm_u8_kernel<kU8Digits>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (n + 2 * kGemmM - 1) / (2 * kGemmM);
    const int pairs = tiles < sms / 2 ? tiles : sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(kU8Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (grid_dependency_wait)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, am, bm, packed, pitch, exc_n, exc, exc_cap, n, W, bias, ws,
                           h, scores, labels, top, reject);
    if (e != cudaSuccess || !lbl) return e;
    // the fix-up: one 256-label block per CTA up to 4 CTAs per SM
    const size_t fsm = (size_t)dim * sizeof(float);
    if (fsm > 48 * 1024) {
        e = cudaFuncSetAttribute(svm_u8_fixup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)fsm);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t fc = {};
    const int64_t blocks = ((int64_t)n + kU8F64Threads - 1) / kU8F64Threads;
    fc.gridDim = dim3((unsigned)std::min<int64_t>(blocks, 4 * (int64_t)sms), 1, 1);
    fc.blockDim = dim3(kU8F64Threads, 1, 1);
    fc.dynamicSmemBytes = fsm;
    fc.stream = stream;
    fc.attrs = attr;
    fc.numAttrs = 1;
    return cudaLaunchKernelEx(&fc, svm_u8_fixup_kernel, packed, pitch, exc_n, exc, exc_cap, n, dim,
                              W, bias, h.n_classes, labels, top, reject);
}

}  // namespace lbpf
