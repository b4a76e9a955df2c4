// lbp_hist_lane59.cuh -- fused-depth LBP histogram kernel for 128x128 ROIs, 8x8 cells,
// 59 uniform bins (the headline workload, BASELINE configs[1..4]), with conflict-free
// shared memory in the hot loop.
//
// Why (profiles/r01/README.md): the first TMA kernel was bound by the shared-memory data
// pipe -- random-bin histogram atomics cost ~4 wavefronts each and byte loads from a 256-B
// LUT ~2.  Here:
//  * counters are lane-private: u32 word [cell-row group g][bin][lane] (g = w/4 for cell row
//    w), lane l always hits bank l; the four cell rows of a group share a word as its four
//    bytes (<= 80 per byte per crop: 4 px x 16 rows + one spill-over pixel per row).  The 4
//    lanes of a cell are summed in the epilogue (one 16-B load, a byte transpose, IDP4A);
//  * the uniform-bin LUT is lane-banked: bin(c) lives at byte (c>>2)*128 + 4*lane + (c&3),
//    so lane l reads bank l; the compare results are accumulated directly into that offset;
//  * only grey is staged by TMA (16 KB per crop, 3 stages per group); depth is read straight
//    from global memory, 8 B per lane per row (256 B coalesced per warp row), prefetched
//    8 rows ahead in registers and across crop boundaries.
// Structure: persistent, 1 CTA/SM, 2 independent groups of 8 warps; warp w of a group owns
// cell row w of its current crop; lane l owns columns 4l..4l+3.  One named barrier per crop
// per group (counters double-buffered); the epilogue writes the 7,552-B descriptor into a
// smem staging buffer (double-buffered) and a bulk async copy stores it.  ROIs that are not
// fully-inside 16-px-aligned 128x128 boxes take the generic path inside the same kernel.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"

namespace lbpf {

namespace l59 {
constexpr int kGroups = 2;
constexpr int kGroupThreads = 256;
constexpr int kThreads = kGroups * kGroupThreads;
constexpr int kTile = 128;
constexpr int kBins = 59;
constexpr int kStages = 3;
constexpr int kGreyBytes = kTile * kTile;                      // 16,384
constexpr int kHistBytes = 2 * kBins * 32 * 4;                 // [g][bin][lane] = 15,104
constexpr int kDescBytes = 64 * kBins * 2;                     // 7,552
constexpr int kGroupBytes = kStages * kGreyBytes + 2 * kHistBytes + 2 * kDescBytes;  // 94,464
constexpr int kLutOff = kGroups * kGroupBytes;                 // 188,928 (256-aligned)
constexpr int kLutBytes = 64 * 128;
constexpr int kPlainLutOff = kLutOff + kLutBytes;
constexpr int kBarOff = kPlainLutOff + 256;
constexpr int kSmemBytes = kBarOff + kGroups * kStages * 8 + 1024;
static_assert(kGroupBytes % 128 == 0 && kLutOff % 256 == 0, "alignment");
}  // namespace l59

__device__ __forceinline__ void bulk_store_s2g(void* gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(ssrc), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// read-only 8-B global load; plain (non-volatile) so the compiler can keep the destination
// in the prefetch-ring register (a volatile asm load was followed by a register move that
// stalled on the load and defeated the prefetch)
__device__ __forceinline__ uint2 ld_global_nc_v2(const void* p) {
    return __ldg(reinterpret_cast<const uint2*>(p));
}
__device__ __forceinline__ uint32_t f16_fma_sat(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.sat.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t f16_fma(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

struct LaneRow {
    uint32_t h0, h1;        // fp16x2 1024+g of columns (4l, 4l+1), (4l+2, 4l+3)
    uint32_t lh0, mh, rh1;  // (4l-1, 4l), (4l+1, 4l+2), (4l+3, 4l+4)
};

__device__ __forceinline__ LaneRow lane_row(uint32_t word_addr) {
    const uint32_t w = ld_shared_u32(word_addr);
    LaneRow r;
    r.h0 = prmt(w, 0x64646464u, 0x5140);
    r.h1 = prmt(w, 0x64646464u, 0x7362);
    const uint32_t left = __shfl_up_sync(0xFFFFFFFFu, r.h1, 1);
    const uint32_t right = __shfl_down_sync(0xFFFFFFFFu, r.h0, 1);
    r.lh0 = prmt(left, r.h0, 0x5432);
    r.mh = prmt(r.h0, r.h1, 0x5432);
    r.rh1 = prmt(r.h1, right, 0x5432);
    return r;
}

// Eq. 2 for the centre pair c as the lane-banked LUT offset, per 16-bit half:
// 0x6400 + (code & 3) + 128 * (code >> 2) with the Fig. 7 bits (TL 1, T 2, TR 4, R 8,
// BR 16, B 32, BL 64, L 128).  TL, T, TR, R: FMA pipe, sat(g_p - g_c + 1) in {0,1} scaled by
// 1, 2, 128, 256 onto 1024.0 (exact fp16 integers); BR, B, BL, L: ALU pipe, HSET2 masks at
// offsets 512..4096.  The bias 0x6400 is an arithmetic constant removed by the LUT base.
__device__ __forceinline__ uint32_t lbp_offset2(uint32_t c, uint32_t tl, uint32_t t, uint32_t tr,
                                                uint32_t r, uint32_t br, uint32_t b, uint32_t bl,
                                                uint32_t l) {
    constexpr uint32_t kOne = 0x3C003C00u, kMinusOne = 0xBC00BC00u, k1024 = 0x64006400u;
    const uint32_t negc1 = f16_fma(c, kMinusOne, kOne);                 // 1 - g_c
    uint32_t f = f16_fma(f16_fma_sat(tl, kOne, negc1), kOne, k1024);   // TL +1
    f = f16_fma(f16_fma_sat(t, kOne, negc1), 0x40004000u, f);          // T  +2
    f = f16_fma(f16_fma_sat(tr, kOne, negc1), 0x58005800u, f);         // TR +128
    f = f16_fma(f16_fma_sat(r, kOne, negc1), 0x5C005C00u, f);          // R  +256
    uint32_t a = hge2_mask(br, c) & 0x02000200u;                       // BR +512
    a |= hge2_mask(b, c) & 0x04000400u;                                // B  +1024
    a |= hge2_mask(bl, c) & 0x08000800u;                               // BL +2048
    a |= hge2_mask(l, c) & 0x10001000u;                                // L  +4096
    return f + a;  // no carry between halves (each half <= 0x6400 + 8067)
}

template <bool HAS_DEPTH>
__global__ void __launch_bounds__(l59::kThreads, 1)
lbp_hist_lane59_kernel(const __grid_constant__ CUtensorMap grey_map,
                       const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                       lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                       DepthWindow win, uint16_t* __restrict__ desc,
                       int32_t* __restrict__ roi_status) {
    using namespace l59;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int tid = threadIdx.x;
    const int group = tid / kGroupThreads, gtid = tid % kGroupThreads;
    const int warp = gtid >> 5, lane = gtid & 31;
    uint8_t* gbase = smem + group * kGroupBytes;
    const uint32_t stage0 = smem_u32(gbase);
    const uint32_t hist0 = stage0 + kStages * kGreyBytes;
    const uint32_t staging0 = hist0 + 2 * kHistBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff) + group * kStages;
    const uint32_t bar_id = 1 + group;

    // ---- one-time setup: LUTs, zero counters, barriers
    for (int i = tid; i < kLutBytes; i += kThreads) {
        const int code = (i >> 7) * 4 + (i & 3);
        smem[kLutOff + i] = kUniformLutDev.v[code];
    }
    if (tid < 256) smem[kPlainLutOff + tid] = kUniformLutDev.v[tid];
    for (int i = gtid; i < 2 * kHistBytes / 16; i += kGroupThreads)
        st_shared_u32x4(hist0 + i * 16, make_uint4(0, 0, 0, 0));
    if (gtid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
    }
    __syncthreads();

    const int G = gridDim.x * kGroups;
    const int gid = blockIdx.x * kGroups + group;
    auto next_fast = [&](int32_t n) {
        while (n < n_rois && !roi_is_fast(rois[n], geom)) n += G;
        return n;
    };
    auto issue = [&](int32_t n, int s) {
        const lbp_roi_t r = rois[n];
        mbar_arrive_expect_tx(&bars[s], kGreyBytes);
        tma_load_3d(gbase + s * kGreyBytes, &grey_map, &bars[s], r.x, r.y, r.img);
    };
    int32_t pn = next_fast(gid);  // producer cursor (used by gtid 0)
    if (gtid == 0)
        for (int s = 0; s < kStages && pn < n_rois; ++s) {
            issue(pn, s);
            pn = next_fast(pn + G);
        }

    // ---- per-lane / per-warp constants
    const uint32_t byte_mult = 1u << (8 * (warp & 3));
    uint32_t col_off[4], mult[4], mult_row[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = 4 * lane + k;
        const bool inner = (x != 0) && (x != kTile - 1);  // the 1-px ROI border has no code
        const int cx = inner ? (8 * x - 1) / (kTile - 2) : (lane >> 2);
        const int col = (cx == (lane >> 2)) ? lane : 4 * cx;  // spill-over -> next cell's lane
        col_off[k] = (uint32_t)(((warp >> 2) * kBins * 32 + col) * 4);
        mult[k] = opaque((inner && !(HAS_DEPTH && win.none_valid)) ? byte_mult : 0u);
        mult_row[k] = mult[k];
    }
    const uint32_t lo16 = win.lo << 16;
    const uint32_t span16 = (win.span << 16) | 0xFFFFu;
    const uint32_t lut_lane = opaque(smem_u32(smem + kLutOff) + 4 * lane - 0x6400u);
    const int i0 = (warp * (kTile - 2)) / 8;                   // first interior row of cell row
    const int nrows = ((warp + 1) * (kTile - 2)) / 8 - i0;     // 15 or 16

    // depth rows of this warp for crop `roi`: image rows y+i0+1 .. y+i0+nrows, 8 B per lane
    auto depth_row_ptr = [&](const lbp_roi_t& r, int j) -> const uint16_t* {
        return depth + (int64_t)r.img * geom.depth_img_stride +
               (int64_t)(r.y + i0 + 1 + j) * geom.depth_pitch + r.x + 4 * lane;
    };
    constexpr int kPre = 8;  // depth prefetch distance (rows)
    uint2 dq[kPre];  // prefetch ring (rows j .. j+kPre-1)
    bool prefetched = false;

    struct GroupSync {
        uint32_t id;
        __device__ __forceinline__ void operator()() const {
            named_barrier_sync(id, l59::kGroupThreads);
        }
    };

    int stage = 0, hb = 0;  // grey stage, counter/staging buffer parity
    uint32_t phase_bits = 0;
    int32_t prev_n = -1;    // crop whose descriptor waits in staging[hb ^ 1]

    for (int32_t n = gid; n < n_rois; n += G) {
        const lbp_roi_t roi = rois[n];
        if (!roi_is_fast(roi, geom)) {
            named_barrier_sync(bar_id, kGroupThreads);  // previous epilogue finished
            extract_roi_generic<kBins, kGroupThreads>(
                grey, HAS_DEPTH ? depth : nullptr, geom, roi, n, win, 8, 8, desc, roi_status,
                reinterpret_cast<uint32_t*>(smem + (hist0 - smem_u32(smem))), 2 * kHistBytes / 4,
                smem + kPlainLutOff, 0, gtid, GroupSync{bar_id});
            named_barrier_sync(bar_id, kGroupThreads);
            prefetched = false;
            continue;
        }
        // next crop of this group, for the cross-crop depth prefetch
        const int32_t nn = n + G;
        lbp_roi_t nroi{};
        bool next_ok = false;
        if (HAS_DEPTH && nn < n_rois) {
            nroi = rois[nn];
            next_ok = roi_is_fast(nroi, geom);
        }
        if (HAS_DEPTH && !prefetched) {
#pragma unroll
            for (int j = 0; j < kPre; ++j) dq[j] = ld_global_nc_v2(depth_row_ptr(roi, j));
        }

        mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
        const uint32_t g0 = opaque(stage0 + stage * kGreyBytes + i0 * kTile + 4 * lane);
        const uint32_t hbuf = hist0 + hb * kHistBytes;
        uint32_t colb[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) colb[k] = opaque(hbuf + col_off[k]);

        auto do_row = [&](const LaneRow& top, const LaneRow& mid, const LaneRow& bot, int j) {
            const uint32_t t0 = lbp_offset2(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                            bot.lh0, mid.lh0);
            const uint32_t t1 = lbp_offset2(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1,
                                            bot.h1, bot.mh, mid.mh);
            uint32_t val[4];
            if (HAS_DEPTH) {
                const uint2 d = dq[j % kPre];
                // refill the ring slot: row j+kPre of this crop; in the last kPre rows (which
                // cover every slot) row j % kPre of the group's next crop, read from that slot
                // (one unconditional load from a selected address, so that the compiler writes
                // the ring register directly; without a next crop it harmlessly re-reads row 0)
                const int jn = j + kPre;  // compile-time: rows 0..15 of every crop
                const uint16_t* src = (jn < 16) ? depth_row_ptr(roi, jn)
                                                : depth_row_ptr(next_ok ? nroi : roi,
                                                                next_ok ? j % kPre : 0);
                dq[j % kPre] = ld_global_nc_v2(src);
                // depth window on a u16 in either half of a word
                const uint32_t x[4] = {d.x * 0x10000u - lo16, d.x - lo16, d.y * 0x10000u - lo16,
                                       d.y - lo16};
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult_row[k] : 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult_row[k];
            }
            const uint32_t la[4] = {lut_lane + (t0 & 0xFFFFu), __umulhi(t0, 0x10000u) + lut_lane,
                                    lut_lane + (t1 & 0xFFFFu), __umulhi(t1, 0x10000u) + lut_lane};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t bin = ld_shared_u8(la[k]);
                red_shared_add(colb[k] + bin * (32 * 4), val[k]);
            }
        };
        // 16 rows, straight-line (no branches: a conditional row block made the compiler copy
        // prefetched registers at the block end, stalling on the load).  Cell rows with 15
        // rows run a 16th dummy row whose increments are 0 (its pixels belong to the next
        // warp's cell row; the rows it touches exist inside the crop).
        LaneRow r0 = lane_row(g0), r1 = lane_row(g0 + kTile), r2;
#pragma unroll
        for (int j = 0; j < 15; j += 3) {
            r2 = lane_row(g0 + (j + 2) * kTile); do_row(r0, r1, r2, j);
            r0 = lane_row(g0 + (j + 3) * kTile); do_row(r1, r2, r0, j + 1);
            r1 = lane_row(g0 + (j + 4) * kTile); do_row(r2, r0, r1, j + 2);
        }
        if (nrows < 16) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mult_row[k] = 0u;
        }
        r2 = lane_row(g0 + 17 * kTile);
        do_row(r0, r1, r2, 15);
#pragma unroll
        for (int k = 0; k < 4; ++k) mult_row[k] = mult[k];
        prefetched = next_ok;

        // staging writes of the previous epilogue -> visible to the bulk-copy engine; the
        // store issued one crop ago must be done reading before this epilogue reuses its buffer
        fence_proxy_async_smem();
        if (gtid == 0) bulk_wait_read_all();
        named_barrier_sync(bar_id, kGroupThreads);  // stage free, counters of crop n complete

        if (gtid == 0) {
            if (prev_n >= 0)
                bulk_store_s2g(desc + (int64_t)prev_n * (64 * kBins), staging0 + (hb ^ 1) * kDescBytes,
                               kDescBytes);
            if (pn < n_rois) {
                issue(pn, stage);
                pn = next_fast(pn + G);
            }
            if (roi_status) roi_status[n] = LBP_OK;
        }
        // ---- epilogue: quad q = (g, bin, cx) holds the 4 lane columns of cells (4g + j, cx),
        // j = byte.  Byte-transpose the 4 words and sum each byte column with IDP4A.
        const uint32_t stg = staging0 + hb * kDescBytes;
        for (int q = gtid; q < 2 * kBins * 8; q += kGroupThreads) {
            const uint32_t qa = hbuf + q * 16;
            const uint4 w = ld_shared_u32x4(qa);
            st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
            const uint32_t lo01 = prmt(w.x, w.y, 0x5140), hi01 = prmt(w.x, w.y, 0x7362);
            const uint32_t lo23 = prmt(w.z, w.w, 0x5140), hi23 = prmt(w.z, w.w, 0x7362);
            const uint32_t c0 = __dp4a(prmt(lo01, lo23, 0x5410), 0x01010101u, 0u);
            const uint32_t c1 = __dp4a(prmt(lo01, lo23, 0x7632), 0x01010101u, 0u);
            const uint32_t c2 = __dp4a(prmt(hi01, hi23, 0x5410), 0x01010101u, 0u);
            const uint32_t c3 = __dp4a(prmt(hi01, hi23, 0x7632), 0x01010101u, 0u);
            const int g = q / (kBins * 8), rem = q - g * (kBins * 8);
            const int bin = rem >> 3, cx = rem & 7;
            const uint32_t o = stg + (((4 * g) * 8 + cx) * kBins + bin) * 2;  // cell (4g, cx)
            constexpr uint32_t kRow = 8 * kBins * 2;                          // next cell row
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o), "h"((uint16_t)c0) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + kRow), "h"((uint16_t)c1) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 2 * kRow), "h"((uint16_t)c2) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 3 * kRow), "h"((uint16_t)c3) : "memory");
        }
        prev_n = n;
        hb ^= 1;
        stage = (stage + 1 == kStages) ? 0 : stage + 1;
    }
    // flush the last descriptor of this group
    fence_proxy_async_smem();
    named_barrier_sync(bar_id, kGroupThreads);
    if (gtid == 0) {
        if (prev_n >= 0)
            bulk_store_s2g(desc + (int64_t)prev_n * (64 * kBins), staging0 + (hb ^ 1) * kDescBytes,
                           kDescBytes);
        bulk_wait_all();
    }
}

inline cudaError_t launch_lbp_hist_lane59(const uint8_t* grey, const uint16_t* depth,
                                          const lbp_images_t& geom, const lbp_roi_t* rois,
                                          int32_t n_rois, const DepthWindow& win, uint16_t* desc,
                                          int32_t* roi_status, int sms, cudaStream_t stream) {
    CUtensorMap gm;
    if (!encode_stack_map(&gm, grey, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, geom, geom.grey_pitch,
                          geom.grey_img_stride))
        return cudaErrorNotSupported;
    auto kern = depth ? lbp_hist_lane59_kernel<true> : lbp_hist_lane59_kernel<false>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, l59::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(sms, (n_rois + l59::kGroups - 1) / l59::kGroups));
    kern<<<grid, l59::kThreads, l59::kSmemBytes, stream>>>(gm, grey, depth, geom, rois, n_rois,
                                                          win, desc, roi_status);
    return cudaGetLastError();
}

}  // namespace lbpf
