// lbp_hist_fast.cuh -- TMA-staged fused-depth LBP histogram kernel for 128x128 ROIs,
// 8x8 cells, 59 or 256 bins (the workload of BASELINE configs[1..4]).
//
// Design:
//  * Persistent: one CTA per SM, 512 threads = two independent groups of 8 warps.  Each
//    group owns `kStages` smem stages (grey 16 KB + depth 32 KB per crop) filled by 3-D
//    TMA tensor loads (cp.async.bulk.tensor, mbarrier complete_tx) while it computes the
//    previous crop, plus its own histogram buffer.  Crops are dealt round-robin to the
//    2*#SM groups; a group synchronises only itself (named barriers).
//  * Warp w of a group computes cell row w: with Ky = 8 the floor partition of the 126
//    interior rows gives warp w exactly rows [floor(126w/8), floor(126(w+1)/8)).
//  * Lane l owns image columns 4l..4l+3 of every row.  Grey bytes are widened to fp16
//    halves 1024+g (exact; comparisons unchanged), so one HSET2 compares two pixels with
//    one neighbour; the eight masks are merged into the Eq. 2 code with one LOP3 each
//    (Fig. 7 weights: TL 1, T 2, TR 4, R 8, BR 16, B 32, BL 64, L 128).  Left/right
//    neighbours come from one shuffle each way per row; rows roll down in registers.
//  * Depth window at the centre pixel -> predicate; bins via a 256-B LUT in smem holding
//    4*bin (59 bins) or the code itself (256 bins); histogram update = fire-and-forget
//    shared-memory increment (ATOMS), integer and order-independent -> bit-exact.
//  * Epilogue: u32 counters -> u16, 16-B vector stores of the 7,552-B descriptor, counters
//    re-zeroed in the same pass.
// ROIs that are not fully-inside 128x128 boxes are processed by the same group with the
// generic code path (extract_roi_generic), so one launch covers every ROI.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"

namespace lbpf {

constexpr int kFastGroupThreads = 256;     // 8 warps = 8 cell rows
constexpr int kFastGroups = 2;
constexpr int kFastThreads = kFastGroupThreads * kFastGroups;
constexpr int kFastCells = 8;

template <int BINS>
struct FastCfg {
    static constexpr int kStages = (BINS == 59) ? 2 : 1;
    static constexpr int kGreyBytes = kFastTile * kFastTile;
    static constexpr int kDepthBytes = kFastTile * kFastTile * 2;
    static constexpr int kStageBytes = kGreyBytes + kDepthBytes;
    static constexpr int kDim = kFastCells * kFastCells * BINS;      // descriptor length
    // packed histogram: u32 word (cell % 32, bin) holds cell c in its low half and cell c+32
    // in its high half (counts <= 256 per cell for 128x128 crops, no carry between halves)
    static constexpr int kHistWords = (kFastCells * kFastCells / 2) * BINS;
    static constexpr int kHistBytes = kHistWords * 4;
    // per group: stages + two histogram buffers (double-buffered across crops)
    static constexpr int kGroupBytes = kStages * kStageBytes + 2 * kHistBytes;
    static constexpr int kLutOff = kFastGroups * kGroupBytes;          // 256-aligned
    static constexpr int kBarOff = kLutOff + 256;
    static constexpr int kSmemBytes = kBarOff + kFastGroups * kStages * 8 + 1024;  // +align slack
    static_assert(kLutOff % 256 == 0, "LUT must be 256-B aligned (PRMT address trick)");
    static_assert(kHistBytes % 16 == 0, "vector epilogue");
};

struct FastRow {
    uint32_t h0, h1;   // fp16x2 (1024+g) of columns 4l..4l+1, 4l+2..4l+3
    uint32_t lh0, mh, rh1;  // shifted pairs: (4l-1,4l), (4l+1,4l+2), (4l+3,4l+4)
};

// grey_word_addr: smem address of this lane's 4 pixels (columns 4l..4l+3) of the row
__device__ __forceinline__ FastRow make_row(uint32_t grey_word_addr, int lane) {
    (void)lane;
    const uint32_t w = ld_shared_u32(grey_word_addr);
    FastRow r;
    r.h0 = prmt(w, 0x64646464u, 0x5140);  // [g0, 0x64, g1, 0x64]
    r.h1 = prmt(w, 0x64646464u, 0x7362);  // [g2, 0x64, g3, 0x64]
    const uint32_t left = __shfl_up_sync(0xFFFFFFFFu, r.h1, 1);
    const uint32_t right = __shfl_down_sync(0xFFFFFFFFu, r.h0, 1);
    r.lh0 = prmt(left, r.h0, 0x5432);
    r.mh = prmt(r.h0, r.h1, 0x5432);
    r.rh1 = prmt(r.h1, right, 0x5432);
    return r;
}

__device__ __forceinline__ uint32_t hfma2_sat(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.sat.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// Eq. 2 for the two pixels of fp16x2 centre `c` (values 1024+g).  Returns per 16-bit half
// 0x64 | code (code = sum_p [g_p >= g_c] 2^p, Fig. 7 weights).  Half of the eight
// comparisons run on the FMA pipe as sat(g_p - g_c + 1) in {0,1} accumulated with the weight
// onto 1024.0 (exact small integers in fp16), half on the ALU pipe as HSET2 masks merged
// with LOP3, which balances the two pipes.
__device__ __forceinline__ uint32_t code2(uint32_t c, uint32_t tl, uint32_t t, uint32_t tr,
                                          uint32_t r, uint32_t br, uint32_t b, uint32_t bl,
                                          uint32_t l) {
    constexpr uint32_t kOne = 0x3C003C00u, kMinusOne = 0xBC00BC00u, k1024 = 0x64006400u;
    const uint32_t negc1 = hfma2(c, kMinusOne, kOne);  // 1 - g_c
    uint32_t acc = hfma2(hfma2_sat(tl, kOne, negc1), kOne, k1024);         // TL  1
    acc = hfma2(hfma2_sat(t, kOne, negc1), 0x40004000u, acc);              // T   2
    acc = hfma2(hfma2_sat(tr, kOne, negc1), 0x44004400u, acc);             // TR  4
    acc = hfma2(hfma2_sat(r, kOne, negc1), 0x48004800u, acc);              // R   8
    acc |= hge2_mask(br, c) & 0x00100010u;                                 // BR  16
    acc |= hge2_mask(b, c) & 0x00200020u;                                  // B   32
    acc |= hge2_mask(bl, c) & 0x00400040u;                                 // BL  64
    acc |= hge2_mask(l, c) & 0x00800080u;                                  // L   128
    return acc;
}

template <int BINS, bool HAS_DEPTH>
__global__ void __launch_bounds__(kFastThreads, 1)
lbp_hist_fast_kernel(const __grid_constant__ CUtensorMap grey_map,
                     const __grid_constant__ CUtensorMap depth_map,
                     const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                     lbp_images_t geom,
                     const lbp_roi_t* __restrict__ rois, int32_t n_rois, DepthWindow win,
                     uint16_t* __restrict__ desc, int64_t desc_stride,
                     int32_t* __restrict__ roi_status) {
    using Cfg = FastCfg<BINS>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

    const int tid = threadIdx.x;
    const int group = tid / kFastGroupThreads;
    const int gtid = tid % kFastGroupThreads;
    const int warp = gtid >> 5, lane = gtid & 31;
    uint8_t* gbase = smem + group * Cfg::kGroupBytes;
    uint32_t* hist = reinterpret_cast<uint32_t*>(gbase + S * Cfg::kStageBytes);  // 2 buffers
    uint8_t* lut = smem + Cfg::kLutOff;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff) + group * S;

    // ---- one-time setup
    if (tid < 256) lut[tid] = (BINS == 59) ? (uint8_t)(kUniformLutDev.v[tid] * 4) : (uint8_t)tid;
    for (int i = gtid; i < 2 * Cfg::kHistWords; i += kFastGroupThreads) hist[i] = 0;
    if (gtid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
        if (HAS_DEPTH) prefetch_tensormap(&depth_map);
    }
    __syncthreads();

    const int n_groups = gridDim.x * kFastGroups;
    const int gid = blockIdx.x * kFastGroups + group;
    const uint32_t bar_id = 1 + group;

    // producer: thread 0 of the group issues the TMA loads of crop `n` into stage s
    auto issue = [&](int32_t n, int s) {
        const lbp_roi_t r = rois[n];
        uint8_t* st = gbase + s * Cfg::kStageBytes;
        mbar_arrive_expect_tx(&bars[s], HAS_DEPTH ? Cfg::kStageBytes : Cfg::kGreyBytes);
        tma_load_3d(st, &grey_map, &bars[s], r.x, r.y, r.img);
        if (HAS_DEPTH) tma_load_3d(st + Cfg::kGreyBytes, &depth_map, &bars[s], r.x, r.y, r.img);
    };

    // per-lane constants of the 4 columns 4l..4l+3: packed-histogram word offset of the cell,
    // depth-window bounds (border columns get an empty window: no code exists there)
    // increment of a valid pixel: +1 in the low half (cell rows 0..3) or the high half (4..7);
    // 0 for the 1-px ROI border (no code there) and for an empty depth window
    const uint32_t half_mult = (warp >= 4) ? 0x10000u : 1u;
    uint32_t cell_off[4];
    uint32_t mult[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = 4 * lane + k;             // column inside the ROI
        const bool inner = (x != 0) && (x != kFastTile - 1);
        const int cx = inner ? (8 * x - 1) / (kFastTile - 2) : 0;  // ((j+1)*Kx-1)/W', j=x-1
        cell_off[k] = (uint32_t)(((warp & 3) * kFastCells + cx) * BINS * 4);
        mult[k] = opaque((inner && !(HAS_DEPTH && win.none_valid)) ? half_mult : 0u);
    }
    // depth window on a u16 held in either half of a word w = d_hi:d_lo:
    //   lo <= d_lo <= lo+span  <=>  (w << 16) - (lo << 16)  <= (span << 16) | 0xFFFF  (u32)
    //   lo <= d_hi <= lo+span  <=>   w        - (lo << 16)  <= (span << 16) | 0xFFFF  (u32)
    const uint32_t lo16 = win.lo << 16;
    const uint32_t span16 = (win.span << 16) | 0xFFFFu;
    const int i0 = (warp * (kFastTile - 2)) / kFastCells;        // first interior row
    const int i1 = ((warp + 1) * (kFastTile - 2)) / kFastCells;  // end
    const uint32_t hist_addr0 = smem_u32(hist);
    const uint32_t lut_addr = smem_u32(lut);

    // prologue: fill the pipeline
    int32_t next_issue = gid;  // next crop index to be loaded (in this group's sequence)
    if (gtid == 0) {
        for (int s = 0; s < S; ++s) {
            while (next_issue < n_rois && !roi_is_fast(rois[next_issue], geom)) next_issue += n_groups;
            if (next_issue < n_rois) issue(next_issue, s);
            next_issue += n_groups;
        }
    }
    uint32_t phase_bits = 0;
    int stage = 0;
    int hbuf = 0;

    struct GroupSync {
        uint32_t id;
        __device__ __forceinline__ void operator()() const { named_barrier_sync(id, kFastGroupThreads); }
    };
    for (int32_t n = gid; n < n_rois; n += n_groups) {
        const lbp_roi_t r = rois[n];
        if (!roi_is_fast(r, geom)) {  // clamped / odd-sized ROI: generic path, same group
            named_barrier_sync(bar_id, kFastGroupThreads);  // previous epilogue finished
            extract_roi_generic<BINS, kFastGroupThreads>(
                CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                HAS_DEPTH ? depth : nullptr, geom, r, n, win, kFastCells, kFastCells, desc,
                desc_stride, roi_status, hist, 2 * Cfg::kHistWords, lut, BINS == 59 ? 2 : 0, gtid,
                GroupSync{bar_id});
            named_barrier_sync(bar_id, kFastGroupThreads);
            continue;
        }
        mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
        const uint8_t* st = gbase + stage * Cfg::kStageBytes;
        const uint32_t g_addr = smem_u32(st);
        const uint32_t d_addr = smem_u32(st + Cfg::kGreyBytes);
        const uint32_t hist_addr = hist_addr0 + hbuf * Cfg::kHistBytes;

        // ---- hot loop: rows of this warp's cell row (15 or 16 rows; fully unrolled so the
        // three rolling rows never move between registers)
        const uint32_t h_addr = opaque(hist_addr);
        uint32_t cell_addr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) cell_addr[k] = opaque(h_addr + cell_off[k]);
        const uint32_t g0 = opaque(g_addr + i0 * kFastTile + 4 * lane);   // this lane's word, row i0
        const uint32_t d_row = opaque(d_addr + (i0 + 1) * (kFastTile * 2) + 8 * lane);
        auto do_row = [&](const FastRow& top, const FastRow& mid, const FastRow& bot, int i) {
            // left pixel pair (4l, 4l+1) and right pair (4l+2, 4l+3)
            const uint32_t a0 = code2(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                      bot.lh0, mid.lh0);
            const uint32_t a1 = code2(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1, bot.h1,
                                      bot.mh, mid.mh);
            uint32_t val[4];
            if (HAS_DEPTH) {
                const uint2 d = ld_shared_u32x2(d_row + (i - i0) * (kFastTile * 2));
                const uint32_t x[4] = {d.x * 0x10000u - lo16, d.x - lo16, d.y * 0x10000u - lo16,
                                       d.y - lo16};
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult[k] : 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            }
            const uint32_t codes[4] = {prmt(a0, lut_addr, 0x7650), prmt(a0, lut_addr, 0x7652),
                                       prmt(a1, lut_addr, 0x7650), prmt(a1, lut_addr, 0x7652)};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // masked / border pixels add 0 (no branch, no predicate)
                const uint32_t off = (BINS == 59) ? ld_shared_u8(codes[k]) : (codes[k] & 0xFFu) * 4;
                red_shared_add(cell_addr[k] + off, val[k]);
            }
        };
        FastRow r0 = make_row(g0, lane), r1 = make_row(g0 + kFastTile, lane), r2;
        const int nrows = i1 - i0;  // 15 or 16, warp-uniform
#pragma unroll
        for (int j = 0; j < 16; j += 3) {
            if (j < nrows) { r2 = make_row(g0 + (j + 2) * kFastTile, lane); do_row(r0, r1, r2, i0 + j); }
            if (j + 1 < nrows) { r0 = make_row(g0 + (j + 3) * kFastTile, lane); do_row(r1, r2, r0, i0 + j + 1); }
            if (j + 2 < nrows) { r1 = make_row(g0 + (j + 4) * kFastTile, lane); do_row(r2, r0, r1, i0 + j + 2); }
        }
        // stage consumed, all increments of this crop done; also guarantees the epilogue of
        // the previous crop (other histogram buffer) has finished everywhere
        named_barrier_sync(bar_id, kFastGroupThreads);

        // refill this stage with the group's next fast crop
        if (gtid == 0) {
            while (next_issue < n_rois && !roi_is_fast(rois[next_issue], geom)) next_issue += n_groups;
            if (next_issue < n_rois) issue(next_issue, stage);
            next_issue += n_groups;
        }
        // ---- epilogue: packed u16 halves -> descriptor (16-B stores), re-zero this buffer.
        // Low halves are cells 0..31 (desc[0, 32*BINS)), high halves cells 32..63.
        uint4* out_lo = reinterpret_cast<uint4*>(desc + (int64_t)n * desc_stride);
        uint4* out_hi = reinterpret_cast<uint4*>(desc + (int64_t)n * desc_stride + Cfg::kHistWords);
        for (int c = gtid; c < Cfg::kHistWords / 8; c += kFastGroupThreads) {
            const uint4 w0 = ld_shared_u32x4(hist_addr + c * 32);
            const uint4 w1 = ld_shared_u32x4(hist_addr + c * 32 + 16);
            out_lo[c] = make_uint4(prmt(w0.x, w0.y, 0x5410), prmt(w0.z, w0.w, 0x5410),
                                   prmt(w1.x, w1.y, 0x5410), prmt(w1.z, w1.w, 0x5410));
            out_hi[c] = make_uint4(prmt(w0.x, w0.y, 0x7632), prmt(w0.z, w0.w, 0x7632),
                                   prmt(w1.x, w1.y, 0x7632), prmt(w1.z, w1.w, 0x7632));
            st_shared_u32x4(hist_addr + c * 32, make_uint4(0, 0, 0, 0));
            st_shared_u32x4(hist_addr + c * 32 + 16, make_uint4(0, 0, 0, 0));
        }
        if (gtid == 0 && roi_status) roi_status[n] = LBP_OK;
        stage = (stage + 1 == S) ? 0 : stage + 1;
        hbuf ^= 1;
    }
}

// ---------------------------------------------------------------------------- host side

inline bool fast_path_applicable(const lbp_images_t& g, const uint8_t* grey, const uint16_t* depth,
                                 int32_t cells_x, int32_t cells_y, int32_t bins,
                                 const uint16_t* desc) {
    if (cells_x != kFastCells || cells_y != kFastCells) return false;
    if (reinterpret_cast<uintptr_t>(desc) & 15) return false;
    if (bins != 59 && bins != 256) return false;
    if (g.width < kFastTile || g.height < kFastTile) return false;
    if (grey && ((reinterpret_cast<uintptr_t>(grey) & 15) || (g.grey_pitch & 15) ||
                 (g.grey_img_stride & 15)))
        return false;  // (grey == NULL: depth-source launch, grey unused)
    if (depth && ((reinterpret_cast<uintptr_t>(depth) & 15) || ((g.depth_pitch * 2) & 15) ||
                  ((g.depth_img_stride * 2) & 15)))
        return false;
    // TMA: strides < 2^40 bytes
    if ((grey && g.grey_img_stride >= (int64_t(1) << 39)) ||
        (depth && g.depth_img_stride >= (int64_t(1) << 38)))
        return false;
    return true;
}

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    // resolved once (thread-safe static init); immutable afterwards
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

inline bool encode_stack_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem,
                             const lbp_images_t& g, int64_t pitch, int64_t img_stride,
                             int box_w = kFastTile) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * elem), (cuuint64_t)(img_stride * elem)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, kFastTile, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BINS, bool HAS_DEPTH>
inline cudaError_t launch_fast_t(const CUtensorMap& gm, const CUtensorMap& dm, const uint8_t* grey,
                                 const uint16_t* depth,
                                 const lbp_images_t& geom, const lbp_roi_t* rois, int32_t n_rois,
                                 const DepthWindow& win, uint16_t* desc, int64_t desc_stride,
                                 int32_t* roi_status, int sms, cudaStream_t stream) {
    auto kern = lbp_hist_fast_kernel<BINS, HAS_DEPTH>;
    const int smem = FastCfg<BINS>::kSmemBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(sms, (n_rois + kFastGroups - 1) / kFastGroups));
    kern<<<grid, kFastThreads, smem, stream>>>(gm, dm, grey, depth, geom, rois, n_rois, win, desc,
                                               desc_stride, roi_status);
    return cudaGetLastError();
}

inline cudaError_t launch_lbp_hist_fast(const uint8_t* grey, const uint16_t* depth,
                                        const lbp_images_t& geom, const lbp_roi_t* rois,
                                        int32_t n_rois, const DepthWindow& win, int32_t bins,
                                        uint16_t* desc, int64_t desc_stride, int32_t* roi_status,
                                        int sms, cudaStream_t stream) {
    CUtensorMap gm, dm;
    if (!encode_stack_map(&gm, grey, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, geom, geom.grey_pitch,
                          geom.grey_img_stride))
        return cudaErrorNotSupported;
    if (depth) {
        if (!encode_stack_map(&dm, depth, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, geom,
                              geom.depth_pitch, geom.depth_img_stride))
            return cudaErrorNotSupported;
    } else {
        dm = gm;
    }
    if (bins == 59)
        return depth ? launch_fast_t<59, true>(gm, dm, grey, depth, geom, rois, n_rois, win, desc, desc_stride, roi_status, sms, stream)
                     : launch_fast_t<59, false>(gm, dm, grey, depth, geom, rois, n_rois, win, desc, desc_stride, roi_status, sms, stream);
    return depth ? launch_fast_t<256, true>(gm, dm, grey, depth, geom, rois, n_rois, win, desc, desc_stride, roi_status, sms, stream)
                 : launch_fast_t<256, false>(gm, dm, grey, depth, geom, rois, n_rois, win, desc, desc_stride, roi_status, sms, stream);
}

}  // namespace lbpf
