// lbp_hist_lane256.cuh -- the lane-private design of lbp_hist_lane59.cuh for the full 256-bin
// histogram ("0-255"; bins = 256, 8x8 cells, 128x128 ROIs at 16-px aligned x): no LUT --
// the code arithmetic produces the counter address itself.
//
//  * counters: u32 words [cell-row group g][bin 0..255 + dummy][lane], 4 cell rows per word
//    as bytes (as lane59), 2 x 257 x 128 B = 65,792 B per 8-warp group;
//  * codes: per 16-bit half t = 4 col + 128 code (col = the pixel's counter lane: its own
//    lane, or the first lane of the neighbouring cell for a spill-over column): TL, T, TR
//    (weights 128, 256, 512) on the FMA pipe as 1 - sat(g_c - g_p) accumulated down from
//    4 col + 896 in the fp16 SUBNORMAL range (bits = the integer, value = bits * 2^-24: exact,
//    < 1024 so bits 10-15 stay zero), R, BR, B, BL, L (1024 .. 16384) as HSET2 masks OR-ed
//    into bits 10-14 (no add); the counter address is group base + t, and a masked-out pixel
//    gets t of a dummy bin 256 in its own lane, so the update needs no select;
//  * 2 groups x 8 warps, 2 TMA stages (stage == group: grey 16 KB + depth 32 KB), the next
//    crop's boxes issued as soon as the rows are consumed; the 32-KB descriptor is staged
//    over the consumed counters (no room elsewhere): the epilogue reads a cell-row group's
//    counters into registers, and after a barrier writes the counts over them (cell rows of
//    512 B with the 16-B chunks XOR-swizzled by cell x, so the 8 cell-x lanes store to
//    distinct banks); the group copies the staging out with 16-B loads and coalesced 16-B
//    global stores, re-zeroing it;
//  * the per-pixel work is the code, one address op and one red.shared (lane59 also reads the
//    LUT byte and forms the counter address): 59 instructions per lane-row.
#pragma once
#include "lbp_hist_lane59.cuh"

namespace lbpf {

namespace l256 {
constexpr int kGroups = 2;
constexpr int kGroupThreads = 256;
constexpr int kThreads = kGroups * kGroupThreads;
constexpr int kTile = 128;
constexpr int kBins = 256;
constexpr int kRows = kBins + 1;                             // + the dummy bin row
constexpr int kStages = 2;
constexpr int kGreyBytes = kTile * kTile;                    // 16,384
constexpr int kStageBytes = kGreyBytes + 2 * kTile * kTile;  // 49,152
constexpr int kHistBytes = 2 * kRows * 32 * 4;               // 65,792
constexpr int kDescBytes = 64 * kBins * 2;                   // 32,768 (staged over g = 0)
constexpr int kGroupOff = kStages * kStageBytes;             // 98,304
constexpr int kLutOff = kGroupOff + kGroups * kHistBytes;    // 229,888: identity LUT (generic)
constexpr int kBarOff = kLutOff + 256;
constexpr int kSmemBytes = kBarOff + kStages * 12 + 128;     // barriers, fast flags, 128-B slack
static_assert(kSmemBytes <= 227 * 1024, "shared memory");
static_assert(kDescBytes <= kRows * 128, "staging fits over the first cell-row group");
static_assert(kStages == kGroups, "stage == group");
}  // namespace l256

// Eq. 2 as the counter-address half 4 col + 128 code (see the header)
__device__ __forceinline__ uint32_t lbp_addr2_256(uint32_t c, uint32_t tl, uint32_t t,
                                                  uint32_t tr, uint32_t r, uint32_t br,
                                                  uint32_t b, uint32_t bl, uint32_t l,
                                                  uint32_t top2) {
    // subnormal weights: -128, -256, -512 times 2^-24 (bits 0x8080, 0x8100, 0x8200)
    uint32_t f = f16_fma(hsub2_sat(c, tl), 0x80808080u, top2);  // TL -128
    f = f16_fma(hsub2_sat(c, t), 0x81008100u, f);                // T  -256
    f = f16_fma(hsub2_sat(c, tr), 0x82008200u, f);               // TR -512
    f |= hge2_mask(r, c) & 0x04000400u;                          // R  bit 10 (1024)
    f |= hge2_mask(br, c) & 0x08000800u;                         // BR bit 11
    f |= hge2_mask(b, c) & 0x10001000u;                          // B  bit 12
    f |= hge2_mask(bl, c) & 0x20002000u;                         // BL bit 13
    f |= hge2_mask(l, c) & 0x40004000u;                          // L  bit 14 (16384)
    return f;  // each half <= 124 + 32640
}

template <bool HAS_DEPTH, int WINM>
__global__ void __launch_bounds__(l256::kThreads, 1)
lbp_hist_lane256_kernel(const __grid_constant__ CUtensorMap grey_map,
                        const __grid_constant__ CUtensorMap depth_map,
                        const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                        lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                        DepthWindow win, uint16_t* __restrict__ desc, int64_t desc_stride,
                        int32_t* __restrict__ roi_status) {
    using namespace l256;
    constexpr bool FP16WIN = HAS_DEPTH && WINM != 0;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                               ~uintptr_t(127));
    const int tid = threadIdx.x;
    const int group = tid / kGroupThreads, gtid = tid % kGroupThreads;
    const int warp = gtid >> 5, lane = gtid & 31;
    const uint32_t stages0 = smem_u32(smem);
    const uint32_t hist0 = stages0 + kGroupOff + group * kHistBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    const uint32_t bar_id = 1 + group;
    // per-stage flag: the position staged there takes the fast path (written by the issuing
    // thread before its mbarrier arrive, read after the wait: lbp_hist_lane59.cuh)
    const uint32_t fastf = smem_u32(smem + kBarOff + kStages * 8);

    const int n_pos = (n_rois > (int)blockIdx.x) ? (n_rois - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto crop_of = [&](int i) -> int32_t { return (int32_t)blockIdx.x + i * (int32_t)gridDim.x; };
    // part bit 1: arrive + expect the stage's bytes + the grey box; bit 2: the depth box
    auto issue = [&](int i, int part) {
        if (i >= n_pos) return;
        const int s = i % kStages;
        const lbp_roi_t r = rois[crop_of(i)];
        const bool fast = roi_is_fast(r, geom);
        if (part & 1) st_shared_u32(fastf + 4 * s, fast ? 1u : 0u);
        if (fast) {
            uint8_t* st = smem + s * kStageBytes;
            if (part & 1) {
                mbar_arrive_expect_tx(&bars[s], HAS_DEPTH ? kStageBytes : kGreyBytes);
                tma_load_3d(st, &grey_map, &bars[s], r.x, r.y, r.img);
            }
            if (HAS_DEPTH && (part & 2))
                tma_load_3d(st + kGreyBytes, &depth_map, &bars[s], r.x, r.y, r.img);
        } else if (part & 1) {
            mbar_arrive(&bars[s]);
        }
    };

    // the dependent launch (the scorer) may be scheduled now (see lbp_hist_lane59.cuh)
    launch_dependents();
    // ---- one-time setup: identity LUT (generic path), zero counters, barriers, first stages
    if (tid < 256) smem[kLutOff + tid] = (uint8_t)tid;
    for (int i = gtid; i < kHistBytes / 16; i += kGroupThreads)
        st_shared_u32x4(hist0 + i * 16, make_uint4(0, 0, 0, 0));
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
        if (HAS_DEPTH) prefetch_tensormap(&depth_map);
        grid_dependency_wait();
        for (int i = 0; i < kStages; ++i) issue(i, 3);
    }
    // programmatic dependent launch: the setup above may overlap the tail of the previous
    // kernel on the stream; inputs and outputs are touched only after it has completed
    grid_dependency_wait();
    __syncthreads();

    // ---- per-lane / per-warp constants
    const uint32_t byte_mult = 1u << (8 * (warp & 3));
    uint32_t mult[4], colk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = 4 * lane + k;
        const bool inner = (x != 0) && (x != kTile - 1);  // the 1-px ROI border has no code
        const int cx = inner ? (8 * x - 1) / (kTile - 2) : (lane >> 2);
        colk[k] = 4 * cx + (lane & 3);  // the cell's quad, position lane & 3 (lbp_hist_lane59.cuh)
        mult[k] = opaque((inner && !(HAS_DEPTH && win.none_valid)) ? byte_mult : 0u);
    }
    // start values (all of TL, T, TR set) and dummy-bin addresses per pixel pair
    const uint32_t top_a = opaque((4u * colk[0] + 896u) | ((4u * colk[1] + 896u) << 16));
    const uint32_t top_b = opaque((4u * colk[2] + 896u) | ((4u * colk[3] + 896u) << 16));
    const uint32_t dum_a = (128u * kBins + 4u * colk[0]) | ((128u * kBins + 4u * colk[1]) << 16);
    const uint32_t dum_b = (128u * kBins + 4u * colk[2]) | ((128u * kBins + 4u * colk[3]) << 16);
    const uint32_t gbase = opaque(hist0 + (uint32_t)((warp >> 2) * kRows * 128));
    const uint32_t lo16 = win.lo << 16;
    const uint32_t span16 = (win.span << 16) | 0xFFFFu;
    const uint32_t lo2 = win.lo * 0x10001u, hi2 = (win.lo + win.span) * 0x10001u;  // WINM 1
    const uint32_t mid2 = ((2 * win.lo + win.span) / 2) * 0x10001u;                 // WINM 2
    const uint32_t half2 = (win.span / 2) * 0x10001u;
    const int i0 = (warp * (kTile - 2)) / 8;
    const int nrows = ((warp + 1) * (kTile - 2)) / 8 - i0;

    struct GroupSync {
        uint32_t id;
        __device__ __forceinline__ void operator()() const {
            named_barrier_sync(id, l256::kGroupThreads);
        }
    };

    for (int i = group; i < n_pos; i += kGroups) {
        const int32_t n = crop_of(i);
        const int s = i % kStages;
        mbar_wait(&bars[s], (uint32_t)(i / kStages) & 1u);
        if (ld_shared_u32(fastf + 4 * s) == 0u) {
            const lbp_roi_t roi = rois[n];
            // stage s was never filled: release it, once every thread of the group has
            // passed its wait on this phase (lbp_hist_lane59.cuh: an earlier plain arrive
            // completes the next phase and a late thread waits on the one after it)
            named_barrier_sync(bar_id, kGroupThreads);
            if (gtid == 0) issue(i + kStages, 3);
            extract_roi_generic<kBins, kGroupThreads>(
                CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                HAS_DEPTH ? depth : nullptr, geom, roi, n, win, 8, 8, desc, desc_stride,
                roi_status, reinterpret_cast<uint32_t*>(smem + (hist0 - stages0)),
                kHistBytes / 4, smem + kLutOff, 0, gtid, GroupSync{bar_id});
            named_barrier_sync(bar_id, kGroupThreads);
            continue;
        }
        const uint32_t st = stages0 + s * kStageBytes;
        const uint32_t g0 = opaque(st + i0 * kTile + 4 * lane);
        const uint32_t d0 = opaque(st + kGreyBytes + (i0 + 1) * (kTile * 2) + 8 * lane);

        auto do_row = [&](const LaneRow& top, const LaneRow& mid, const LaneRow& bot,
                          const uint2 d) {
            uint32_t t0 = lbp_addr2_256(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                        bot.lh0, mid.lh0, top_a);
            uint32_t t1 = lbp_addr2_256(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1, bot.h1,
                                        bot.mh, mid.mh, top_b);
            uint32_t val[4];
            if constexpr (FP16WIN) {  // (the window tests of lane59's WINM 1 / 2)
                uint32_t m0, m1;
                if constexpr (WINM == 2) {
                    m0 = hle2_mask(habsdiff2(d.x, mid2), half2);
                    m1 = hle2_mask(habsdiff2(d.y, mid2), half2);
                } else {
                    m0 = hge2_mask(d.x, lo2) & hle2_mask(d.x, hi2);
                    m1 = hge2_mask(d.y, lo2) & hle2_mask(d.y, hi2);
                }
                t0 = (t0 & m0) | (dum_a & ~m0);
                t1 = (t1 & m1) | (dum_b & ~m1);
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            } else if (HAS_DEPTH) {
                const uint32_t x[4] = {d.x * 0x10000u - lo16, d.x - lo16, d.y * 0x10000u - lo16,
                                       d.y - lo16};
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult[k] : 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            }
            const uint32_t a[4] = {gbase + (t0 & 0xFFFFu), __umulhi(t0, 0x10000u) + gbase,
                                   gbase + (t1 & 0xFFFFu), __umulhi(t1, 0x10000u) + gbase};
#pragma unroll
            for (int k = 0; k < 4; ++k) red_shared_add(a[k], val[k]);
        };
        // raw words one row ahead of use (as lbp_hist_lane59.cuh)
        LaneRow r0 = lane_row(g0), r1 = lane_row(g0 + kTile);
        uint32_t wn = ld_shared_u32(g0 + 2 * kTile);
        uint2 dn = make_uint2(0u, 0u);
        if constexpr (HAS_DEPTH) dn = ld_shared_u32x2(d0);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t wc = wn;
            const uint2 dc = dn;
            if (j < 15) {
                wn = ld_shared_u32(g0 + (j + 3) * kTile);
                if constexpr (HAS_DEPTH) dn = ld_shared_u32x2(d0 + (j + 1) * (kTile * 2));
            }
            if (j == 15 && nrows < 16) break;  // a 15-row cell row (warp-uniform)
            const LaneRow r2 = lane_row_w(wc);
            do_row(r0, r1, r2, dc);
            r0 = r1;
            r1 = r2;
        }

        named_barrier_sync(bar_id, kGroupThreads);  // A: stage read, counters complete
        if (gtid == 0) {
            issue(i + kStages, 3);  // the whole next stage: the staging is not in it
            if (roi_status) roi_status[n] = LBP_OK;
        }
        // ---- epilogue in two halves, the staging inside the consumed counters: quad q =
        // (bin, cx) of cell-row group g as lane59 (conflict-free 16-B loads) -> the 4 cells'
        // counts in registers; g = 0's counts are written (swizzled) over g = 0's own
        // counters once every thread has read them, g = 1's after them (cells 32..63)
        constexpr int kQ = kRows * 8;                      // quads per cell-row group
        constexpr int kQIter = (kQ + kGroupThreads - 1) / kGroupThreads;
        const uint32_t staging = hist0;
        auto counts = [&](uint32_t qa) {  // 4 cells' u16 counts of one quad, packed in 2 words
            const uint4 w = ld_shared_u32x4(qa);
            const uint32_t lo01 = prmt(w.x, w.y, 0x5140), hi01 = prmt(w.x, w.y, 0x7362);
            const uint32_t lo23 = prmt(w.z, w.w, 0x5140), hi23 = prmt(w.z, w.w, 0x7362);
            const uint32_t c0 = __dp4a(prmt(lo01, lo23, 0x5410), 0x01010101u, 0u);
            const uint32_t c1 = __dp4a(prmt(lo01, lo23, 0x7632), 0x01010101u, 0u);
            const uint32_t c2 = __dp4a(prmt(hi01, hi23, 0x5410), 0x01010101u, 0u);
            const uint32_t c3 = __dp4a(prmt(hi01, hi23, 0x7632), 0x01010101u, 0u);
            return make_uint2(c0 | (c1 << 16), c2 | (c3 << 16));
        };
        auto put = [&](int g, int q, uint2 c) {  // cells (4g + j, cx), j = 0..3
            const int bin = q >> 3, cx = q & 7;
            const uint32_t o = staging + ((4 * g) * 8 + cx) * (kBins * 2) +
                               ((2u * bin) ^ ((uint32_t)cx << 4));
            constexpr uint32_t kRow = 8 * kBins * 2;
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o), "h"((uint16_t)c.x) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + kRow), "h"((uint16_t)(c.x >> 16)) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 2 * kRow), "h"((uint16_t)c.y) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 3 * kRow), "h"((uint16_t)(c.y >> 16)) : "memory");
        };
        uint2 cnt[kQIter];
#pragma unroll
        for (int k = 0; k < kQIter; ++k) {  // g = 0: read (the dummy row is only re-zeroed)
            const int q = gtid + k * kGroupThreads;
            if (q < kQ) {
                if ((q >> 3) == kBins) st_shared_u32x4(hist0 + q * 16, make_uint4(0, 0, 0, 0));
                else cnt[k] = counts(hist0 + q * 16);
            }
        }
        named_barrier_sync(bar_id, kGroupThreads);  // every g = 0 counter read
#pragma unroll
        for (int k = 0; k < kQIter; ++k) {
            const int q = gtid + k * kGroupThreads;
            if (q < kQ && (q >> 3) < kBins) put(0, q, cnt[k]);
        }
        const uint32_t hist1 = hist0 + kRows * 128;
#pragma unroll
        for (int k = 0; k < kQIter; ++k) {  // g = 1: read and re-zero
            const int q = gtid + k * kGroupThreads;
            if (q < kQ) {
                const uint32_t qa = hist1 + q * 16;
                if ((q >> 3) < kBins) cnt[k] = counts(qa);
                st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
            }
        }
#pragma unroll
        for (int k = 0; k < kQIter; ++k) {
            const int q = gtid + k * kGroupThreads;
            if (q < kQ && (q >> 3) < kBins) put(1, q, cnt[k]);
        }
        named_barrier_sync(bar_id, kGroupThreads);  // B: staging complete
        {  // copy-out: 2,048 chunks of 16 B, un-swizzled, coalesced; each chunk re-zeroed
            uint16_t* out = desc + (int64_t)n * desc_stride;
#pragma unroll 4
            for (int idx = gtid; idx < kDescBytes / 16; idx += kGroupThreads) {
                const int cell = idx >> 5, chunk = idx & 31;
                const uint32_t sa = staging + cell * (kBins * 2) + ((chunk * 16) ^ ((cell & 7) << 4));
                const uint4 v = ld_shared_u32x4(sa);
                st_shared_u32x4(sa, make_uint4(0, 0, 0, 0));
                *reinterpret_cast<uint4*>(out + cell * kBins + chunk * 8) = v;
            }
        }
        named_barrier_sync(bar_id, kGroupThreads);  // C: counters zero for the next crop
    }
}

inline cudaError_t launch_lbp_hist_lane256(const uint8_t* grey, const uint16_t* depth,
                                           const lbp_images_t& geom, const lbp_roi_t* rois,
                                           int32_t n_rois, const DepthWindow& win,
                                           uint16_t* desc, int64_t desc_stride,
                                           int32_t* roi_status, int sms, cudaStream_t stream) {
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
    const bool fp16win = depth && !win.none_valid && win.lo + win.span <= 0x7BFEu;
    const uint32_t whi = win.lo + win.span;
    const bool centred = fp16win && whi < 2048u && ((win.lo + whi) & 1u) == 0;
    auto kern = !depth    ? lbp_hist_lane256_kernel<false, 0>
                : centred ? lbp_hist_lane256_kernel<true, 2>
                : fp16win ? lbp_hist_lane256_kernel<true, 1>
                          : lbp_hist_lane256_kernel<true, 0>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, l256::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(sms, n_rois));
    return launch_pdl(kern, grid, l256::kThreads, l256::kSmemBytes, stream, gm, dm, grey, depth,
                      geom, rois, n_rois, win, desc, desc_stride, roi_status);
}

}  // namespace lbpf
