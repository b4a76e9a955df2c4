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
//  * grey and depth of a crop (48 KB) are staged by TMA into a ring of 3 stages shared by
//    the CTA's groups (crop position i of the CTA -> stage i%3, group i%kGroups); the group
//    that finishes position i refills its stage with position i+3.
// Structure: persistent, 1 CTA/SM, 3 groups of 8 warps (24 warps hide each group's barrier
// and load waits); warp w of a group owns cell row w
// of its crop (with Ky = 8 the floor partition of the 126 interior rows is exactly the
// warp's rows), lane l owns columns 4l..4l+3.  The epilogue writes the 7,552-B descriptor
// into a smem staging buffer and a bulk async copy (cp.async.bulk) stores it.  ROIs that are
// not fully-inside 16-px-aligned 128x128 boxes take the generic path inside the same kernel.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gather.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"
#include "tma_util.cuh"

namespace lbpf {

namespace l59 {
#ifndef LBPF_L59_GROUPS
#define LBPF_L59_GROUPS 3  // (2 groups with 113 registers: 10% slower -- fewer warps)
#endif
constexpr int kGroups = LBPF_L59_GROUPS;  // 8-warp groups per CTA, one crop each
constexpr int kGroupThreads = 256;
constexpr int kThreads = kGroups * kGroupThreads;
constexpr int kTile = 128;
constexpr int kBins = 59;
constexpr int kBinsAlloc = 60;  // + a dummy bin row that counts the masked-out pixels
constexpr int kStages = 3;
constexpr int kHistBytes = 2 * kBinsAlloc * 32 * 4;            // [g][bin][lane] = 15,360
constexpr int kDescBytes = 64 * kBins * 2;                     // 7,552
constexpr int kGroupBytes = (kHistBytes + kDescBytes + 255) / 256 * 256;  // 23,040 (+ staging)
constexpr int kLutBytes = 65 * 128;  // 64 lane-banked rows + the dummy row (bin 59 everywhere)
constexpr uint32_t kLutMod = 0x6000u;       // the LUT's shared address mod 2^16 (lut_placement)
constexpr uint32_t kDummyOff2 = 0x80008000u;  // LUT offset of the dummy row (64), both halves
static_assert(kStages >= kGroups, "every group has a staged crop");
// epilogue output modes of the kernel (template parameter OUTM)
constexpr int kOutU16 = 0;     // u16 row, one bulk store (lbp_fused_extract)
constexpr int kOutGather = 1;  // u16 row stored into every destination (lbp_extract_gather)
constexpr int kOutU8 = 2;      // compact row: u8 low bytes + exceptions (lbp_extract_u8)
constexpr int kOutFused = 3;   // u16 grey block then depth block from ONE staged tile
                               // (lbp_extract_source LBP_SRC_FUSED)

// Stage layout of the two variants.  FRAME (ROIs at any column of wider frames): the grey
// box is 144 px wide at x & ~15 and the depth box 136 px at x & ~7 (TMA needs 16-B aligned
// box starts), so each lane's 4 columns start og = x & 15 bytes (grey) / od = x & 7 pixels
// (depth) into the staged row; the 7,552-B descriptor is then staged over the group's
// consumed counters (no room for a separate buffer) and copied out by the group.
template <bool FRAME>
struct Layout {
    static constexpr int kGreyW = FRAME ? 144 : kTile;   // grey row bytes in a stage
    static constexpr int kDepthW = FRAME ? 136 : kTile;  // depth row pixels in a stage
    static constexpr int kGreyBytes = kGreyW * kTile;
    static constexpr int kStageBytes = kGreyBytes + 2 * kDepthW * kTile;
    static constexpr int kGroupOff = kStages * kStageBytes;
    static constexpr int kGroupBytes = FRAME ? kHistBytes : l59::kGroupBytes;
    // the lane-banked LUT goes at the first offset >= kLutMin whose shared-window address is
    // 0x6000 mod 2^16 (lut_placement): then the LUT address of a code offset t (a 16-bit half
    // 0x6000 + ...) is (address - 0x6000) | t, one LOP3 / IMAD.HI per half.  The plain LUT and
    // the stage barriers follow it.
    static constexpr int kLutMin = kGroupOff + kGroups * kGroupBytes;
    // LUT, plain LUT, stage barriers, stage-release counters, stage fast flags, align slack
    static constexpr int kTailBytes = kLutBytes + 256 + kStages * 8 + 2 * kStages * 4 + 128;
    // headline: stages 3 x 49,152, groups 3 x 23,040 (counters + staging), LUT >= 216,576;
    // FRAME: stages 3 x 53,248, groups 3 x 15,360, LUT >= 205,824
    static_assert(kStageBytes % 128 == 0 && kGreyBytes % 128 == 0 && kLutMin % 256 == 0,
                  "alignment");
    static_assert(kLutMin + kTailBytes <= 227 * 1024, "shared memory");
    static_assert(kDescBytes <= kBinsAlloc * 32 * 4, "FRAME staging fits over one cell-row group");
};
// the depth window as the packed words the row loop compares with (both fp16x2 halves, or
// the high u16 of a word): lo16 / span16 (WINM 0), lo2 / hi2 (WINM 1), mid2 / half2 (WINM 2:
// |d - mid| <= half), and DINT's clamp bounds lo - 1, lo + 1022 and offset 0x6401 - lo
struct WinWords {
    uint32_t lo16, span16, lo2, hi2, mid2, half2, dlo2m1, dhi2, doff2;
};
inline WinWords win_words(const DepthWindow& w) {
    WinWords r;
    r.lo16 = w.lo << 16;
    r.span16 = (w.span << 16) | 0xFFFFu;
    r.lo2 = w.lo * 0x10001u;
    r.hi2 = (w.lo + w.span) * 0x10001u;
    r.mid2 = ((2 * w.lo + w.span) / 2) * 0x10001u;
    r.half2 = (w.span / 2) * 0x10001u;
    r.dlo2m1 = (w.lo - 1u) * 0x10001u;
    r.dhi2 = (w.lo + 1022u) * 0x10001u;
    r.doff2 = ((0x6401u - w.lo) & 0xFFFFu) * 0x10001u;
    return r;
}
}  // namespace l59

// 4 bytes starting s = sel-encoded bytes into the word pair at addr (funnel shift by PRMT)
__device__ __forceinline__ uint32_t ld_shared_funnel1(uint32_t addr, uint32_t sel) {
    return prmt(ld_shared_u32(addr), ld_shared_u32(addr + 4), sel);
}
// 8 bytes starting 0 or 2 bytes into the three words at addr (sel 0x3210 / 0x5432)
__device__ __forceinline__ uint2 ld_shared_funnel2(uint32_t addr, uint32_t sel) {
    const uint32_t w0 = ld_shared_u32(addr), w1 = ld_shared_u32(addr + 4),
                   w2 = ld_shared_u32(addr + 8);
    return make_uint2(prmt(w0, w1, sel), prmt(w1, w2, sel));
}

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

__device__ __forceinline__ uint32_t hsub2_sat(uint32_t a, uint32_t b) {
    uint32_t r;  // sat(a - b) per half
    asm("sub.rn.sat.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// The compact descriptor of lbp_extract_u8 (include/lbpfused.h): packed[n][d] = count & 255
// (rows of `pitch` bytes), exc_n[n] = the number of entries above 255,
// exc[n * exc_cap + k] = (d << 16) | count for the first exc_cap of them.
struct U8Out {
    uint8_t* packed;
    int32_t* exc_n;
    uint32_t* exc;
    int32_t exc_cap;
    int64_t pitch;
};

__device__ __forceinline__ uint32_t atom_shared_add(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
// The halves' hand-off counters (stage release, exception count) are relaxed shared-memory
// atomics (acq_rel would add a MEMBAR after the bulk store): what they order is complete
// before them -- the stage rows were consumed before the half's barrier A, and the half's
// exception-count increments returned (their slots were used) before its barrier B -- and
// the atomics of one thread reach the CTA's shared memory in program order.
__device__ __forceinline__ uint32_t atom_shared_exch(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}

// entry d of row n holds count v: its low byte (staged; st.u8 keeps bits 0-7) ...
__device__ __forceinline__ void put_u8(uint32_t staging, uint32_t d, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(staging + d), "r"(v) : "memory");
}
// ... and, above 255, an exception record (rare: a 16x16 cell whose 256 pixels share a bin)
__device__ __forceinline__ void record_u8(const U8Out& o, int64_t n, uint32_t cnt_addr,
                                          uint32_t d, uint32_t v) {
    if (v > 255u) {
        const uint32_t k = atom_shared_add(cnt_addr, 1u);
        if ((int32_t)k < o.exc_cap) o.exc[n * o.exc_cap + k] = (d << 16) | v;
    }
}

struct LaneRow {
    uint32_t h0, h1;        // fp16x2 1024+g of columns (4l, 4l+1), (4l+2, 4l+3)
    uint32_t lh0, mh, rh1;  // (4l-1, 4l), (4l+1, 4l+2), (4l+3, 4l+4)
};

__device__ __forceinline__ LaneRow lane_row_w(uint32_t w) {
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
__device__ __forceinline__ LaneRow lane_row(uint32_t word_addr) {
    return lane_row_w(ld_shared_u32(word_addr));
}

// Eq. 2 for the centre pair c as the lane-banked LUT offset, per 16-bit half:
// 0x6000 + 4 lane + (code & 3) + 128 * (code >> 2) with the Fig. 7 bits (TL 1, T 2, TR 4,
// R 8, BR 16, B 32, BL 64, L 128).  fp16 values in [512, 1024) have ulp 0.5 and bits
// 0x6000 + m (value 512 + m/2, m < 1024), so bits 10-12 are zero there.  TL, T, TR, R, BR: FMA
// pipe, sat(g_c - g_p) in {0,1} scaled by -0.5, -1, -64, -128, -256 (offsets 1, 2, 128, 256,
// 512) onto top2 = base2 + 899/2 with base2 = 512 + 2 lane (exact: every value stays on the
// 0.5 grid in [512, 1024)); B, BL, L: ALU pipe, HSET2 masks OR-ed into bits 10, 11, 12 (offsets
// 1024, 2048, 4096) -- no carry, so no add: one LOP3 per bit.
__device__ __forceinline__ uint32_t lbp_offset2(uint32_t c, uint32_t tl, uint32_t t, uint32_t tr,
                                                uint32_t r, uint32_t br, uint32_t b, uint32_t bl,
                                                uint32_t l, uint32_t top2) {
    // [g_p >= g_c] = 1 - sat(g_c - g_p) (integers): start from top2 (all five bits set) and
    // subtract w_p sat(g_c - g_p) -- one HADD2.SAT per bit, no 1 - g_c term
    uint32_t f = f16_fma(hsub2_sat(c, tl), 0xB800B800u, top2);        // TL -0.5   (offset 1)
    f = f16_fma(hsub2_sat(c, t), 0xBC00BC00u, f);                      // T  -1     (2)
    f = f16_fma(hsub2_sat(c, tr), 0xD400D400u, f);                     // TR -64    (128)
    f = f16_fma(hsub2_sat(c, r), 0xD800D800u, f);                      // R  -128   (256)
    f = f16_fma(hsub2_sat(c, br), 0xDC00DC00u, f);                     // BR -256   (512)
    f |= hge2_mask(b, c) & 0x04000400u;                                // B  bit 10 (1024)
    f |= hge2_mask(bl, c) & 0x08000800u;                               // BL bit 11 (2048)
    f |= hge2_mask(l, c) & 0x10001000u;                                // L  bit 12 (4096)
    return f;
}

// ---- depth source: codes on the u16 depth plane.  A u16 d <= 0x7BFF read as
// fp16 bits is a non-negative finite half, and the bit order of those halves is their value
// order, so HSET2 on the raw bits is an exact unsigned compare.  Every depth word is clamped
// to 0x7BFF first (VIMNMX.U16x2); this is exact for the codes that are counted when
// dmax <= 0x7BFE: a counted centre c <= dmax < 0x7BFF, so min(n, 0x7BFF) >= c iff n >= c
// (the host takes the generic kernel otherwise).
struct DepthRow {
    uint32_t h0, h1;        // clamped (4l, 4l+1), (4l+2, 4l+3)
    uint32_t lh0, mh, rh1;  // (4l-1, 4l), (4l+1, 4l+2), (4l+3, 4l+4)
    uint32_t raw0, raw1;    // unclamped words, for the depth-window test of centre rows
};

__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t a, uint32_t b) {
    return __vminu2(a, b);  // VIMNMX.U16x2
}

__device__ __forceinline__ DepthRow depth_row_w(uint2 w) {
    DepthRow r;
    r.raw0 = w.x;
    r.raw1 = w.y;
    r.h0 = vmin_u16x2(w.x, 0x7BFF7BFFu);
    r.h1 = vmin_u16x2(w.y, 0x7BFF7BFFu);
    const uint32_t left = __shfl_up_sync(0xFFFFFFFFu, r.h1, 1);
    const uint32_t right = __shfl_down_sync(0xFFFFFFFFu, r.h0, 1);
    r.lh0 = prmt(left, r.h0, 0x5432);
    r.mh = prmt(r.h0, r.h1, 0x5432);
    r.rh1 = prmt(r.h1, right, 0x5432);
    return r;
}
__device__ __forceinline__ DepthRow depth_row(uint32_t addr) {
    return depth_row_w(ld_shared_u32x2(addr));
}

// DINT depth rows (window span <= 1022, lo <= 0x6400): every depth word clamped to
// [lo - 1, lo + 1022] and offset to the fp16 bits of the INTEGER 1025 + (d' - lo) in
// [1024, 2047] (one VIMNMX pair and one packed add per word: no carry between the halves).
// The order is preserved for the codes that are counted: a counted centre c is in
// [lo, lo + span], so d' >= c iff d >= c; and the values are exact fp16 integers, so the
// codes use the grey plane's HADD2.SAT arithmetic (FMA pipe) instead of HSET2 compares.
__device__ __forceinline__ DepthRow depth_row_int(uint2 w, uint32_t lo2m1, uint32_t hi2,
                                                  uint32_t off2) {
    DepthRow r;
    r.raw0 = w.x;
    r.raw1 = w.y;
    r.h0 = vmin_u16x2(__vmaxu2(w.x, lo2m1), hi2) + off2;
    r.h1 = vmin_u16x2(__vmaxu2(w.y, lo2m1), hi2) + off2;
    const uint32_t left = __shfl_up_sync(0xFFFFFFFFu, r.h1, 1);
    const uint32_t right = __shfl_down_sync(0xFFFFFFFFu, r.h0, 1);
    r.lh0 = prmt(left, r.h0, 0x5432);
    r.mh = prmt(r.h0, r.h1, 0x5432);
    r.rh1 = prmt(r.h1, right, 0x5432);
    return r;
}

__device__ __forceinline__ uint32_t hle2_mask(uint32_t a, uint32_t b) {
    uint32_t r;  // 0xFFFF / 0 per half
    asm("set.le.u32.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// |a - b| per half (exact where used: see the WINM == 2 window below)
__device__ __forceinline__ uint32_t habsdiff2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    asm("abs.f16x2 %0, %0;" : "+r"(d));
    return d;
}

__device__ __forceinline__ uint32_t hge2_one(uint32_t a, uint32_t b) {
    uint32_t r;  // 1.0 / 0.0 per half
    asm("set.ge.f16x2.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Same LUT offset as lbp_offset2, every bit from an exact compare: TL, T, TR, R, BR as
// 1.0/0.0 halves accumulated by HFMA2 onto base2 = 512 + 2 lane (weights 0.5, 1, 64, 128, 256:
// offsets 1, 2, 128, 256, 512 on the 0.5 grid of [512, 1024)), B, BL, L as HSET2 masks OR-ed
// into bits 10, 11, 12.
__device__ __forceinline__ uint32_t lbp_offset2_cmp(uint32_t c, uint32_t tl, uint32_t t,
                                                    uint32_t tr, uint32_t r, uint32_t br,
                                                    uint32_t b, uint32_t bl, uint32_t l,
                                                    uint32_t base2) {
    uint32_t f = f16_fma(hge2_one(tl, c), 0x38003800u, base2);        // TL +0.5 (offset 1)
    f = f16_fma(hge2_one(t, c), 0x3C003C00u, f);                       // T  +1   (2)
    f = f16_fma(hge2_one(tr, c), 0x54005400u, f);                      // TR +64  (128)
    f = f16_fma(hge2_one(r, c), 0x58005800u, f);                       // R  +128 (256)
    f = f16_fma(hge2_one(br, c), 0x5C005C00u, f);                      // BR +256 (512)
    f |= hge2_mask(b, c) & 0x04000400u;                                // B  bit 10
    f |= hge2_mask(bl, c) & 0x08000800u;                               // BL bit 11
    f |= hge2_mask(l, c) & 0x10001000u;                                // L  bit 12
    return f;
}

// WINM: how the depth window is tested.  0: integer compare per pixel; 1: both halves of a
// depth word at once as fp16 compares, dmax <= 0x7BFE (a u16 d read as fp16 bits is, for
// d <= 0x7BFF, a non-negative finite half whose bit order is its value order; larger bit
// patterns are +inf, NaN or negative and fail d >= dmin or d <= dmax, so the raw words are
// compared); 2: |d - mid| <= half with mid = (dmin + dmax) / 2 and half = (dmax - dmin) / 2,
// when dmax < 2048 and dmin + dmax is even -- below 2048 the halves are exact multiples of
// 2^-24 (value = bits * 2^-24), so the subtraction is exact there; for larger d either
// mid/2 <= d <= 2 mid (exact by Sterbenz) or d > 2 mid, where the rounded difference is still
// >= mid > half; NaN / inf / negative patterns fail the compare.
// OUTM == kOutGather (the fused database build, gather.cuh): the descriptor rows go from the
// staging buffer to every destination of `gd` (multicast or peer stores) instead of a bulk
// store to `desc`; `desc` is then local scratch for the ROIs that take the generic code path,
// whose rows are forwarded from there.  OUTM == kOutU8: the compact row (U8Out) is staged
// and bulk-stored; `desc` is unused (the generic path counts into the group's counters and
// stages its row the same way).
// WINM bit 2 (DINT, with WINM 1 or 2): depth-plane codes in the integer domain (depth_row_int).
template <bool HAS_DEPTH, bool DEPTH_SRC, int WINM, bool FRAME, int OUTM = l59::kOutU16>
__global__ void __launch_bounds__(l59::kThreads, 1)
lbp_hist_lane59_kernel(const __grid_constant__ CUtensorMap grey_map,
                       const __grid_constant__ CUtensorMap depth_map,
                       const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                       lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                       DepthWindow win, uint16_t* __restrict__ desc, int64_t desc_stride,
                       int32_t* __restrict__ roi_status, int32_t lut_off,
                       const __grid_constant__ lbp_gather_dst_t gd,
                       const int32_t* __restrict__ glabels, const __grid_constant__ U8Out u8o,
                       const __grid_constant__ l59::WinWords ww) {
    constexpr bool GATHER = OUTM == l59::kOutGather;
    constexpr bool U8 = OUTM == l59::kOutU8;
    constexpr bool FUSED = OUTM == l59::kOutFused;
    static_assert(!FUSED || (HAS_DEPTH && !DEPTH_SRC && (WINM & 3) != 0 && !FRAME),
                  "fused grey||depth: depth plane staged, fp16 depth window, crop stacks");
    static_assert(OUTM == l59::kOutU16 || !FRAME, "the gather / u8 outputs use the crop-stack epilogue");
    using namespace l59;
    using L = Layout<FRAME>;
    constexpr int WIN = WINM & 3;          // the window test
    constexpr bool DINT = (WINM & 4) != 0;  // depth codes in the integer domain
    constexpr bool FP16WIN = WIN != 0;
    constexpr int kGreyBytes = L::kGreyBytes, kStageBytes = L::kStageBytes;
    constexpr int kGroupOff = L::kGroupOff, kGroupBytes = L::kGroupBytes;
    const int kLutOff = lut_off, kPlainLutOff = lut_off + kLutBytes;  // (lut_placement)
    const int kBarOff = kPlainLutOff + 256;
    // FRAME with grey codes and a depth mask: the staging overwrites the stage's grey rows, so
    // the next grey box is loaded only once the descriptor store has read the staging (the
    // depth box goes first); without depth it uses the unused depth region, for the depth
    // source the unused grey region.
    // FRAME: no room for a staging buffer; the descriptor is staged over the group's consumed
    // counters (see the epilogue) and copied out by the group, so, as for crop stacks, both
    // boxes of the next crop are issued as soon as the rows are done
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                               ~uintptr_t(127));
    const int tid = threadIdx.x;
    const int group = tid / kGroupThreads, gtid = tid % kGroupThreads;
    const int warp = gtid >> 5, lane = gtid & 31;
    const uint32_t stages0 = smem_u32(smem);
    const uint32_t hist0 = stages0 + kGroupOff + group * kGroupBytes;
    const uint32_t staging = FRAME ? hist0 : hist0 + kHistBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    const uint32_t bar_id = 1 + group;
    // SUB (crop stacks): the two cell-row halves of a group -- warps 4 sub .. 4 sub + 3, one warp
    // per SMSP, whose counters are the cell-row group g = sub -- run the rows, the epilogue and
    // the store of their half of the descriptor row with 128-thread barriers of their own (the
    // scheduler's warp priorities no longer stall a whole 8-warp group at every barrier); the
    // stage is refilled by whichever half releases it second.  FRAME keeps 8-warp barriers.
    constexpr bool SUB = !FRAME;
    const int sub = warp >> 2, stid = gtid & 127;
    const uint32_t sub_bar = 4 + 2 * group + sub;  // named barriers 4..9 (0: CTA, 1..3: groups)
    const bool leader = SUB ? stid == 0 : gtid == 0;  // owns a bulk-store group
    // group slack words after the staging (crop stacks): [0..1] exception counts and [2..3]
    // halves-done counts by crop parity (U8)
    const uint32_t slack = staging + kDescBytes;
    // per-stage release counts (after the stage barriers): two halves release each position
    const uint32_t rel0 = smem_u32(smem + kBarOff + kStages * 8);
    // per-stage flag: the position staged there takes the fast path (written by the thread that
    // issues the stage's loads, before its mbarrier arrive; read after the wait), so only the
    // threads that issue loads (and, FRAME, every thread: the box offset) read the ROIs
    const uint32_t fastf = rel0 + kStages * 4;
    const bool loads_roi = FRAME || leader;

    // crop positions of this CTA: position i -> crop blockIdx.x + i * gridDim.x
    const int n_pos = (n_rois > (int)blockIdx.x) ? (n_rois - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto crop_of = [&](int i) -> int32_t { return (int32_t)blockIdx.x + i * (int32_t)gridDim.x; };
    // fill position i into stage i % 3: TMA for fast crops, a plain arrive otherwise (keeps the
    // stage barrier's phase count in step with the positions)
    auto is_fast = [&](const lbp_roi_t& r) {
        return FRAME ? roi_is_fast_frame(r, geom) : roi_is_fast(r, geom);
    };
    // fill position i into its stage
    // (r: the ROI of position i, already loaded by the caller)
    auto issue = [&](int i, const lbp_roi_t& r) {
        if (i >= n_pos) return;
        const int s = i % kStages;
        const bool fast = is_fast(r);
        st_shared_u32(fastf + 4 * s, fast ? 1u : 0u);
        if (fast) {
            uint8_t* st = smem + s * kStageBytes;
            const int gx = FRAME ? (r.x & ~15) : r.x, dx = FRAME ? (r.x & ~7) : r.x;
            mbar_arrive_expect_tx(&bars[s], DEPTH_SRC ? kStageBytes - kGreyBytes
                                                      : HAS_DEPTH ? kStageBytes : kGreyBytes);
            if (HAS_DEPTH) tma_load_3d(st + kGreyBytes, &depth_map, &bars[s], dx, r.y, r.img);
            if (!DEPTH_SRC) tma_load_3d(st, &grey_map, &bars[s], gx, r.y, r.img);
        } else {
            mbar_arrive(&bars[s]);
        }
    };
    // L2 prefetch of position i's boxes (crop stacks): the stage ring holds one crop per group,
    // so the load of position i + 3, issued when position i releases its stage, would wait for
    // HBM while the group idles; prefetching position i + 6 at the same moment lets that load
    // hit L2 (more bytes in flight per SM than the shared-memory ring can hold)
    auto prefetch = [&](int i, int32_t x, int32_t y, int32_t img) {
        if (FRAME || i >= n_pos) return;
        if (HAS_DEPTH) tma_prefetch_l2_3d(&depth_map, x, y, img);
        if (!DEPTH_SRC) tma_prefetch_l2_3d(&grey_map, x, y, img);
    };

    // the dependent launch (the scorer) may be scheduled now: its CTAs take SMs as these
    // CTAs exit, run their prologue, and wait for this grid's completion
    launch_dependents();
    // ---- one-time setup: barriers and the first positions' loads first (their latency
    // overlaps the table fills), then LUTs and zeroed counters
    if (tid == 0) {
        // the host placed the LUT from the device's reserved shared memory size; a mismatch
        // would misaddress every lookup, so it stops the kernel (LBP_E_CUDA) instead
        if ((smem_u32(smem + kLutOff) & 0xFFFFu) != kLutMod) __trap();
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
        if (HAS_DEPTH) prefetch_tensormap(&depth_map);
        grid_dependency_wait();  // (see below)
        for (int i = 0; i < kStages; ++i)
            if (i < n_pos) issue(i, rois[crop_of(i)]);
        for (int i = kStages; i < 2 * kStages; ++i)
            if (i < n_pos) {
                const lbp_roi_t r = rois[crop_of(i)];
                prefetch(i, r.x, r.y, r.img);
            }
    }
    for (int i = tid; i < kLutBytes; i += kThreads) {
        const int code = (i >> 7) * 4 + (i & 3);
        smem[kLutOff + i] = code < 256 ? kUniformLutDev.v[code] : (uint8_t)kBins;  // row 64: dummy
    }
    if (tid < 256) smem[kPlainLutOff + tid] = kUniformLutDev.v[tid];
    for (int i = gtid; i < kHistBytes / 16; i += kGroupThreads)
        st_shared_u32x4(hist0 + i * 16, make_uint4(0, 0, 0, 0));
    if (SUB && gtid < 4) st_shared_u32(slack + 4 * gtid, 0u);
    if (SUB && tid < kStages) st_shared_u32(rel0 + 4 * tid, 0u);
    // programmatic dependent launch: everything above may overlap the tail of the previous
    // kernel on the stream (e.g. the scorer of the previous batch); its inputs and the outputs
    // it reads (the descriptor rows) are touched only after it has completed
    grid_dependency_wait();
    __syncthreads();

    // ---- per-lane / per-warp constants
    const uint32_t byte_mult = 1u << (8 * (warp & 3));
    uint32_t colb[4], mult[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = 4 * lane + k;
        const bool inner = (x != 0) && (x != kTile - 1);  // the 1-px ROI border has no code
        const int cx = inner ? (8 * x - 1) / (kTile - 2) : (lane >> 2);
        // the cell's quad of slots 4 cx .. 4 cx + 3, position lane & 3: for one pixel index k
        // a cell (<= 16 px) spans <= 4 consecutive lanes, so a spill-over pixel never shares a
        // slot -- a bank -- with another lane's pixel of the same atomic
        const int col = 4 * cx + (lane & 3);
        colb[k] = opaque(hist0 + (uint32_t)(((warp >> 2) * kBinsAlloc * 32 + col) * 4));
        mult[k] = opaque((inner && !(HAS_DEPTH && win.none_valid)) ? byte_mult : 0u);
    }
    // depth-window words, computed on the host (WinWords): kernel parameters the row loop
    // reads as constant-bank operands instead of holding (or recomputing) them in registers
    const uint32_t lo16 = ww.lo16, span16 = ww.span16;        // WINM 0
    const uint32_t lo2 = ww.lo2, hi2 = ww.hi2;                // WINM 1
    const uint32_t mid2 = ww.mid2, half2 = ww.half2;          // WINM 2
    const uint32_t dlo2m1 = ww.dlo2m1, dhi2 = ww.dhi2, doff2 = ww.doff2;  // DINT
    // LUT address of an offset half t: lutb | t (the LUT sits at 0x6000 mod 2^16)
    const uint32_t lutb = opaque(smem_u32(smem + kLutOff) - kLutMod);
    const uint32_t base2 = opaque((kLutMod + 4u * lane) * 0x10001u);  // 512.0 + 2 lane
    const uint32_t top2 = opaque((kLutMod + 4u * lane + 899u) * 0x10001u);  // + TL..BR
    const int i0 = (warp * (kTile - 2)) / 8;                   // first interior row of cell row
    const int nrows = ((warp + 1) * (kTile - 2)) / 8 - i0;     // 15 or 16

    struct GroupSync {
        uint32_t id;
        __device__ __forceinline__ void operator()() const {
            named_barrier_sync(id, l59::kGroupThreads);
        }
    };

    int32_t pending = -1;  // last crop whose descriptor was bulk-stored
    // the group's next ROI is loaded one crop ahead (its latency hidden by the current crop);
    // with kStages == kGroups it is also the position whose TMA this group issues next
    lbp_roi_t roi_next = loads_roi && group < n_pos ? rois[crop_of(group)] : lbp_roi_t{};
    for (int i = group; i < n_pos; i += kGroups) {
        const int32_t n = crop_of(i);
        lbp_roi_t roi = roi_next;
        if (loads_roi && i + kGroups < n_pos) roi_next = rois[crop_of(i + kGroups)];
        // position i + kStages: its TMA is issued when this crop releases stage s
        lbp_roi_t roi_fill{};
        if constexpr (kStages == kGroups) roi_fill = roi_next;
        else if (loads_roi && i + kStages < n_pos) roi_fill = rois[crop_of(i + kStages)];
        // the box of position i + 6, prefetched to L2 when this crop releases its stage (read
        // now by the releasing threads, used after the rows)
        int32_t pf_x = 0, pf_y = 0, pf_img = 0;
        if (!FRAME && (SUB ? stid == 0 : gtid == 0) && i + 2 * kStages < n_pos) {
            const lbp_roi_t& rp = rois[crop_of(i + 2 * kStages)];
            pf_x = rp.x; pf_y = rp.y; pf_img = rp.img;
        }
        const int s = i % kStages;
        mbar_wait(&bars[s], (uint32_t)(i / kStages) & 1u);
        const uint32_t par = (uint32_t)(i / kGroups) & 1u;
        const uint32_t exc_cnt = slack + 4 * par;  // U8: the crop's exception count
        if (ld_shared_u32(fastf + 4 * s) == 0u) {
            if (!loads_roi) roi = rois[n];
            // stage s was never filled: release it at once -- but only once every thread of
            // the group has passed its wait on this position's phase (a plain arrive for
            // position i + 3 completes the NEXT phase at once, and a thread still polling the
            // parity of this phase would then wait for the phase after that: deadlock)
            named_barrier_sync(bar_id, kGroupThreads);
            if (gtid == 0) {
                issue(i + kStages, roi_fill);
                prefetch(i + 2 * kStages, pf_x, pf_y, pf_img);
            }
            if constexpr (U8) {
                // counts stay in the group's counters (KEEP; 64 cells x 59 bins fit one chunk),
                // then the row is staged as u8 + exceptions like the fast path's
                if (leader) bulk_wait_read_all();           // previous rows left the staging
                named_barrier_sync(bar_id, kGroupThreads);
                uint32_t* hist = reinterpret_cast<uint32_t*>(smem + (hist0 - stages0));
                uint16_t* zrow = reinterpret_cast<uint16_t*>(smem + (staging - stages0));
                extract_roi_generic<kBins, kGroupThreads, uint8_t, GroupSync, true>(
                    CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                    HAS_DEPTH ? depth : nullptr, geom, roi, 0, win, 8, 8, zrow, 0, nullptr,
                    hist, kHistBytes / 4, smem + kPlainLutOff, 0, gtid, GroupSync{bar_id});
                if (gtid == 0 && roi_status) roi_status[n] = clamp_roi(roi, geom, 8, 8).status;
                named_barrier_sync(bar_id, kGroupThreads);  // counts complete
                for (int d = gtid; d < 64 * kBins; d += kGroupThreads) {
                    const uint32_t v = hist[d];
                    hist[d] = 0u;
                    put_u8(staging, (uint32_t)d, v);
                    record_u8(u8o, n, exc_cnt, (uint32_t)d, v);
                }
                fence_proxy_async_smem();
                named_barrier_sync(bar_id, kGroupThreads);  // staging complete, counters zero
                if (gtid == 0) {
                    bulk_store_s2g(u8o.packed + (int64_t)n * u8o.pitch, staging, kDescBytes / 2);
                    u8o.exc_n[n] = (int32_t)ld_shared_u32(exc_cnt);
                    st_shared_u32(exc_cnt, 0u);
                    // the other half's leader does not wait on this thread's bulk group
                    bulk_wait_read_all();
                }
                pending = n;
                continue;
            }
            if constexpr (SUB) {  // both halves past the previous crop (counters zero)
                if (leader) bulk_wait_read_all();
                named_barrier_sync(bar_id, kGroupThreads);
            }
            if (DEPTH_SRC)
                extract_roi_generic<kBins, kGroupThreads>(
                    CodePlane<uint16_t>{depth, geom.depth_pitch, geom.depth_img_stride}, depth, geom,
                    roi, n, win, 8, 8, desc, desc_stride, roi_status,
                    reinterpret_cast<uint32_t*>(smem + (hist0 - stages0)), kHistBytes / 4,
                    smem + kPlainLutOff, 0, gtid, GroupSync{bar_id});
            else
            extract_roi_generic<kBins, kGroupThreads>(
                CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                HAS_DEPTH ? depth : nullptr, geom, roi, n, win, 8, 8, desc, desc_stride, roi_status,
                reinterpret_cast<uint32_t*>(smem + (hist0 - stages0)), kHistBytes / 4,
                smem + kPlainLutOff, 0, gtid, GroupSync{bar_id});
            if constexpr (FUSED)  // the depth block of the row
                extract_roi_generic<kBins, kGroupThreads>(
                    CodePlane<uint16_t>{depth, geom.depth_pitch, geom.depth_img_stride}, depth, geom,
                    roi, n, win, 8, 8, desc + 64 * kBins, desc_stride, nullptr,
                    reinterpret_cast<uint32_t*>(smem + (hist0 - stages0)), kHistBytes / 4,
                    smem + kPlainLutOff, 0, gtid, GroupSync{bar_id});
            named_barrier_sync(bar_id, kGroupThreads);
            if constexpr (GATHER) {  // forward the row written to the local scratch
                gather_row_from_global<kGroupThreads>(gd, n, desc + (int64_t)n * desc_stride,
                                                      kDescBytes / 2, gtid);
                if (gtid == 0) gather_label(gd, n, glabels);
            }
            continue;
        }
        // One code plane of the staged crop (FUSED: the grey plane, then the depth plane of the
        // same staged tile -- depth read from HBM once); `last` releases the stage.
        auto plane = [&](auto src_tag, uint16_t* out_row, bool last) {
        constexpr bool DS = decltype(src_tag)::value;  // codes on the depth plane
        const uint32_t st = stages0 + s * kStageBytes;
        // code plane rows: grey u8 (kGreyW B per row) or depth u16 (2 kDepthW B, DS).
        // FRAME: the lane's bytes start og (grey) / 2 od (depth) bytes past its aligned words.
        constexpr uint32_t kDRow = 2 * L::kDepthW;
        constexpr uint32_t kRowStep = DS ? kDRow : L::kGreyW;
        const uint32_t og = FRAME ? (uint32_t)roi.x & 15u : 0u;
        const uint32_t od2 = FRAME ? 2u * ((uint32_t)roi.x & 7u) : 0u;
        const uint32_t gsel = 0x3210u + (og & 3u) * 0x1111u;    // funnel by og & 3 bytes
        const uint32_t dsel = (od2 & 2u) ? 0x5432u : 0x3210u;  // funnel by 0 / 2 bytes
        const uint32_t g0 = DS ? opaque(st + kGreyBytes + i0 * kDRow + 8 * lane + (od2 & ~3u))
                                      : opaque(st + i0 * L::kGreyW + 4 * lane + (og & ~3u));
        const uint32_t d0 = opaque(st + kGreyBytes + (i0 + 1) * kDRow + 8 * lane + (od2 & ~3u));
        // Raw shared-memory words of a row are loaded one row AHEAD of their use (the loop
        // below is fully unrolled): a row's loads are issued before the previous row's
        // counter updates, so their latency overlaps a whole row of arithmetic.
        struct Raw { uint32_t a, b, c; };
        auto raw_depth = [&](uint32_t addr) {  // 8 depth bytes of the lane (FRAME: 3 words)
            Raw w{0u, 0u, 0u};
            if constexpr (FRAME) {
                w.a = ld_shared_u32(addr); w.b = ld_shared_u32(addr + 4); w.c = ld_shared_u32(addr + 8);
            } else {
                const uint2 v = ld_shared_u32x2(addr);
                w.a = v.x; w.b = v.y;
            }
            return w;
        };
        auto depth_words = [&](const Raw& w) {
            if constexpr (FRAME) return make_uint2(prmt(w.a, w.b, dsel), prmt(w.b, w.c, dsel));
            else return make_uint2(w.a, w.b);
        };
        auto raw_row = [&](uint32_t addr) {
            if constexpr (DS) return raw_depth(addr);
            Raw w{ld_shared_u32(addr), 0u, 0u};
            if constexpr (FRAME) w.b = ld_shared_u32(addr + 4);
            return w;
        };
        auto build_row = [&](const Raw& w) {
            if constexpr (DS && DINT) return depth_row_int(depth_words(w), dlo2m1, dhi2, doff2);
            else if constexpr (DS) return depth_row_w(depth_words(w));
            else if constexpr (FRAME) return lane_row_w(prmt(w.a, w.b, gsel));
            else return lane_row_w(w.a);
        };
        using Row = decltype(build_row(Raw{}));

        // a row's counter updates are issued one row later (Pend: its bins and increments),
        // so the LUT-byte loads' latency overlaps the next row's arithmetic
        struct Pend { uint32_t bin[4], val[4]; };
        auto do_row = [&](const Row& top, const Row& mid, const Row& bot, const Raw& dc) {
            uint32_t t0, t1;
            if constexpr (DS && !DINT) {
                t0 = lbp_offset2_cmp(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                     bot.lh0, mid.lh0, base2);
                t1 = lbp_offset2_cmp(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1, bot.h1,
                                     bot.mh, mid.mh, base2);
            } else {
                t0 = lbp_offset2(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                 bot.lh0, mid.lh0, top2);
                t1 = lbp_offset2(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1, bot.h1,
                                 bot.mh, mid.mh, top2);
            }
            uint32_t val[4];
            if constexpr (HAS_DEPTH && FP16WIN) {
                // depth window on both halves at once, on the raw words (see WINM above);
                // masked-out pixels are redirected to the dummy LUT row (-> dummy bin)
                // instead of adding 0
                uint32_t c0, c1;
                if constexpr (DS) {
                    c0 = mid.raw0;
                    c1 = mid.raw1;
                } else {
                    const uint2 d = depth_words(dc);
                    c0 = d.x;
                    c1 = d.y;
                }
                uint32_t m0, m1;
                if constexpr (WIN == 2) {
                    m0 = hle2_mask(habsdiff2(c0, mid2), half2);
                    m1 = hle2_mask(habsdiff2(c1, mid2), half2);
                } else {
                    m0 = hge2_mask(c0, lo2) & hle2_mask(c0, hi2);
                    m1 = hge2_mask(c1, lo2) & hle2_mask(c1, hi2);
                }
                t0 = (t0 & m0) | (kDummyOff2 & ~m0);
                t1 = (t1 & m1) | (kDummyOff2 & ~m1);
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            } else if (HAS_DEPTH) {
                uint2 d;
                if constexpr (DS) d = make_uint2(mid.raw0, mid.raw1);  // centre row
                else d = depth_words(dc);
                // depth window on a u16 in either half of a word
                const uint32_t x[4] = {d.x * 0x10000u - lo16, d.x - lo16, d.y * 0x10000u - lo16,
                                       d.y - lo16};
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult[k] : 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            }
            // (an IMAD.HI form of the high halves, to move them to the FMA pipe, needs a register
            // for 2^16 and costs more moves than it saves at 80 registers: LEA.HI stays)
            const uint32_t la[4] = {lutb | (t0 & 0xFFFFu), __umulhi(t0, 0x10000u) + lutb,
                                    lutb | (t1 & 0xFFFFu), __umulhi(t1, 0x10000u) + lutb};
            Pend p;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                p.bin[k] = ld_shared_u8(la[k]);
                p.val[k] = val[k];
            }
            return p;
        };
        auto flush = [&](const Pend& p) {
#pragma unroll
            for (int k = 0; k < 4; ++k) red_shared_add(colb[k] + p.bin[k] * (32 * 4), p.val[k]);
        };
        // 16 rows, straight-line (the 15-row cell rows stop before the 16th).
        constexpr bool kMaskRow = HAS_DEPTH && !DS;  // a separate depth centre row
        Row r0 = build_row(raw_row(g0)), r1 = build_row(raw_row(g0 + kRowStep));
        Raw wn = raw_row(g0 + 2 * kRowStep), dn{0u, 0u, 0u};
        Pend pend;
        if constexpr (kMaskRow) dn = raw_depth(d0);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const Raw wc = wn, dc = dn;
            if (j < 15) {
                wn = raw_row(g0 + (j + 3) * kRowStep);
                if constexpr (kMaskRow) dn = raw_depth(d0 + (j + 1) * kDRow);
            }
            if (j == 15 && nrows < 16) {  // a 15-row cell row: no 16th row (warp-uniform)
                flush(pend);
                break;
            }
            const Row r2 = build_row(wc);
            const Pend p = do_row(r0, r1, r2, dc);
            if (j > 0) flush(pend);
            pend = p;
            r0 = r1;
            r1 = r2;
            if (j == 15) flush(pend);
        }

        if (leader) bulk_wait_read_all();  // this thread's previous store left the staging
        if constexpr (SUB) {
            named_barrier_sync(sub_bar, 128);  // A: this half's counters complete, its rows read
            // the second half to release stage s refills it with position i + 3
            if (stid == 0 && last && (atom_shared_add(rel0 + 4 * s, 1u) & 1u)) {
                issue(i + kStages, roi_fill);
                prefetch(i + 2 * kStages, pf_x, pf_y, pf_img);
                if (roi_status) roi_status[n] = LBP_OK;
            }
        } else {
            named_barrier_sync(bar_id, kGroupThreads);  // A: stage read, counters complete
            if (gtid == 0 && last) {
                issue(i + kStages, roi_fill);
                if (roi_status) roi_status[n] = LBP_OK;
            }
        }
        // ---- epilogue: quad q = (g, bin, cx) holds the 4 lane columns of cells (4g + j, cx),
        // j = byte.  Byte-transpose the 4 words and sum each byte column with IDP4A.
        auto counts = [&](uint32_t qa) {
            const uint4 w = ld_shared_u32x4(qa);
            const uint32_t lo01 = prmt(w.x, w.y, 0x5140), hi01 = prmt(w.x, w.y, 0x7362);
            const uint32_t lo23 = prmt(w.z, w.w, 0x5140), hi23 = prmt(w.z, w.w, 0x7362);
            return make_uint4(__dp4a(prmt(lo01, lo23, 0x5410), 0x01010101u, 0u),
                              __dp4a(prmt(lo01, lo23, 0x7632), 0x01010101u, 0u),
                              __dp4a(prmt(hi01, hi23, 0x5410), 0x01010101u, 0u),
                              __dp4a(prmt(hi01, hi23, 0x7632), 0x01010101u, 0u));
        };
        auto put = [&](int g, int bin, int cx, uint4 c) {  // cells (4g + j, cx), j = 0..3
            const uint32_t o = staging + (((4 * g) * 8 + cx) * kBins + bin) * 2;
            constexpr uint32_t kRow = 8 * kBins * 2;  // next cell row
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o), "h"((uint16_t)c.x) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + kRow), "h"((uint16_t)c.y) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 2 * kRow), "h"((uint16_t)c.z) : "memory");
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o + 3 * kRow), "h"((uint16_t)c.w) : "memory");
        };
        if constexpr (FRAME) {
            // staging over the consumed counters: g = 0's counts to registers, barrier, then
            // written over g = 0's counters; g = 1's read (and re-zeroed) and written after
            // them; the group copies the row out with 16-B stores and re-zeroes g = 0
            constexpr int kQ = kBinsAlloc * 8;  // quads per cell-row group
            constexpr int kIt = (kQ + kGroupThreads - 1) / kGroupThreads;
            uint4 cnt[kIt];
#pragma unroll
            for (int k = 0; k < kIt; ++k) {
                const int q = gtid + k * kGroupThreads;
                if (q < kQ && (q >> 3) < kBins) cnt[k] = counts(hist0 + q * 16);
            }
            named_barrier_sync(bar_id, kGroupThreads);  // every g = 0 counter read
#pragma unroll
            for (int k = 0; k < kIt; ++k) {
                const int q = gtid + k * kGroupThreads;
                if (q < kQ && (q >> 3) < kBins) put(0, q >> 3, q & 7, cnt[k]);
            }
#pragma unroll
            for (int k = 0; k < kIt; ++k) {
                const int q = gtid + k * kGroupThreads;
                if (q < kQ) {
                    const uint32_t qa = hist0 + (kQ + q) * 16;
                    if ((q >> 3) < kBins) cnt[k] = counts(qa);
                    st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
                }
            }
#pragma unroll
            for (int k = 0; k < kIt; ++k) {
                const int q = gtid + k * kGroupThreads;
                if (q < kQ && (q >> 3) < kBins) put(1, q >> 3, q & 7, cnt[k]);
            }
            named_barrier_sync(bar_id, kGroupThreads);  // staging complete
            uint16_t* out = out_row;
            for (int idx = gtid; idx < kQ; idx += kGroupThreads) {  // g = 0 region: 480 x 16 B
                const uint32_t sa = hist0 + idx * 16;
                if (idx < kDescBytes / 16) {
                    const uint4 v = ld_shared_u32x4(sa);
                    *reinterpret_cast<uint4*>(out + idx * 8) = v;
                }
                st_shared_u32x4(sa, make_uint4(0, 0, 0, 0));
            }
            named_barrier_sync(bar_id, kGroupThreads);  // counters zero for the next crop
        } else {
            // thread -> quads: cx = gtid & 7, bin = bp + 16 k (bp = (gtid >> 3) & 15, k = 0..3),
            // g = gtid >> 7, so the counter quad and the staged entries are affine in k ([R +
            // imm] addressing, no per-quad index math) and each quarter-warp reads 128
            // contiguous bytes (8 cx of one bin).  Bins 60..63 do not exist (k = 3, bp >= 12);
            // bin 59 is the dummy (masked-out pixels): only re-zeroed.
            static_assert(kGroupThreads == 2 * 8 * 16 && kBins > 48 && kBins <= 60, "epilogue map");
            const int ecx = gtid & 7, ebp = (gtid >> 3) & 15, eg = gtid >> 7;
            const uint32_t qbase = hist0 + (uint32_t)(((eg * kBinsAlloc + ebp) * 8 + ecx) * 16);
            const uint32_t dbase = (uint32_t)(((4 * eg) * 8 + ecx) * kBins + ebp);
            uint4 cq[4];
            uint32_t any = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k == 3 && ebp >= 12) break;
                const uint32_t qa = qbase + k * (16 * 128);
                if (k == 3 && ebp == kBins - 48) {
                    st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
                    break;
                }
                const uint4 c = counts(qa);
                st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
                if constexpr (U8) {
                    constexpr uint32_t kRowE = 8 * kBins;  // next cell row
                    const uint32_t d0 = dbase + 16 * k;
                    put_u8(staging, d0, c.x);
                    put_u8(staging, d0 + kRowE, c.y);
                    put_u8(staging, d0 + 2 * kRowE, c.z);
                    put_u8(staging, d0 + 3 * kRowE, c.w);
                    cq[k] = c;
                    any |= c.x | c.y | c.z | c.w;
                } else {
                    put(eg, ebp + 16 * k, ecx, c);
                }
            }
            if constexpr (U8) {
                if (any > 255u) {  // rare: a 16x16 cell whose 256 pixels share a bin
                    constexpr uint32_t kRowE = 8 * kBins;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k == 3 && ebp >= kBins - 48) break;
                        const uint32_t d0 = dbase + 16 * k;
                        record_u8(u8o, n, exc_cnt, d0, cq[k].x);
                        record_u8(u8o, n, exc_cnt, d0 + kRowE, cq[k].y);
                        record_u8(u8o, n, exc_cnt, d0 + 2 * kRowE, cq[k].z);
                        record_u8(u8o, n, exc_cnt, d0 + 3 * kRowE, cq[k].w);
                    }
                }
            }
            // this half's part of the row: cell rows 4 sub .. 4 sub + 3 (contiguous)
            constexpr uint32_t kHalfB = kDescBytes / 2;  // u16 bytes (the u8 half: kHalfB / 2)
            if constexpr (U8) {
                fence_proxy_async_smem();          // staging writes -> async proxy
                named_barrier_sync(sub_bar, 128);  // B: this half's counters zero, staged
                if (stid == 0) {
                    bulk_store_s2g(u8o.packed + (int64_t)n * u8o.pitch + sub * (kHalfB / 2),
                                   staging + sub * (kHalfB / 2), kHalfB / 2);
                    // the second half done: the crop's exception count is final
                    if (atom_shared_add(slack + 8 + 4 * par, 1u) & 1u)
                        u8o.exc_n[n] = (int32_t)atom_shared_exch(exc_cnt, 0u);
                }
            } else if constexpr (GATHER) {
                // every thread of the half forwards 16-B chunks of its part of the staged row
                // to every destination (rewritten only after this half's next barrier A, which
                // its threads reach after their loads here); half 1 also writes the padding
                named_barrier_sync(sub_bar, 128);  // B: this half's counters zero, staged
                gather_row_from_smem<128>(gd, n, staging, sub * (kHalfB / 16),
                                          sub ? -1 : (int)(kHalfB / 16), kDescBytes / 16, stid);
                if (gtid == 0) gather_label(gd, n, glabels);
            } else {
                fence_proxy_async_smem();          // staging writes -> async proxy
                named_barrier_sync(sub_bar, 128);  // B: this half's counters zero, staged
                if (stid == 0)
                    bulk_store_s2g(out_row + sub * (kHalfB / 2), staging + sub * kHalfB, kHalfB);
            }
        }
        };
        if constexpr (FUSED) {
            plane(std::false_type{}, desc + (int64_t)n * desc_stride, false);
            plane(std::true_type{}, desc + (int64_t)n * desc_stride + 64 * kBins, true);
        } else {
            plane(std::integral_constant<bool, DEPTH_SRC>{}, desc + (int64_t)n * desc_stride, true);
        }
        pending = n;
    }
    if (leader && pending >= 0) bulk_wait_all();
    if constexpr (GATHER) __threadfence_system();  // before the caller's cross-rank barrier
}

// Offset of the lane-banked LUT in the dynamic shared memory: the first offset >= lut_min
// whose shared-window address is l59::kLutMod (0x6000) mod 2^16.  Dynamic shared memory starts at the
// device's reserved shared memory per block (these kernels have no static shared memory),
// and the kernel rounds its base up to 128 B.  False if the layout does not fit.
inline bool lut_placement(int lut_min, int tail_bytes, int* lut_off, int* smem_bytes) {
    static const int reserved = []() {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, dev) !=
                cudaSuccess)
            return -1;
        return v;
    }();
    if (reserved < 0) return false;
    const int base = (reserved + 127) & ~127;
    const int off = lut_min + ((((int)l59::kLutMod - base - lut_min) % 65536) + 65536) % 65536;
    *lut_off = off;
    *smem_bytes = off + tail_bytes;
    return *smem_bytes <= 227 * 1024;
}

inline cudaError_t launch_lbp_hist_lane59(const uint8_t* grey, const uint16_t* depth,
                                          const lbp_images_t& geom, const lbp_roi_t* rois,
                                          int32_t n_rois, const DepthWindow& win, uint16_t* desc,
                                          int64_t desc_stride, int32_t* roi_status, int sms,
                                          cudaStream_t stream, bool depth_source = false,
                                          bool frame = false,
                                          const lbp_gather_dst_t* gather = nullptr,
                                          const int32_t* glabels = nullptr,
                                          const U8Out* u8out = nullptr, bool fused = false) {
    if ((gather || u8out || fused) && (frame || depth_source)) return cudaErrorNotSupported;
    CUtensorMap gm, dm;
    if (!depth_source &&
        !encode_stack_map(&gm, grey, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, geom, geom.grey_pitch,
                          geom.grey_img_stride, frame ? l59::Layout<true>::kGreyW : kFastTile))
        return cudaErrorNotSupported;
    if (depth) {
        if (!encode_stack_map(&dm, depth, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, geom,
                              geom.depth_pitch, geom.depth_img_stride,
                              frame ? l59::Layout<true>::kDepthW : kFastTile))
            return cudaErrorNotSupported;
    } else {
        dm = gm;
    }
    if (depth_source) gm = dm;  // grey is not read
    // depth window as fp16 compares whenever dmax <= 0x7BFE (always for the depth source)
    const bool fp16win = depth && !win.none_valid && win.lo + win.span <= 0x7BFEu;
    const uint32_t whi = win.lo + win.span;
    const bool centred = fp16win && whi < 2048u && ((win.lo + whi) & 1u) == 0;  // WINM 2
    // depth-plane codes in the integer domain (WINM | 4): window span <= 1022, lo <= 0x6400
    const bool dint = fp16win && win.span <= 1022u && win.lo <= 0x6400u;
    auto pick = [&](auto frame_tag) {
        constexpr bool F = decltype(frame_tag)::value;
        if (depth_source)
            return dint ? (centred ? lbp_hist_lane59_kernel<true, true, 6, F>
                                   : lbp_hist_lane59_kernel<true, true, 5, F>)
                        : (centred ? lbp_hist_lane59_kernel<true, true, 2, F>
                                   : lbp_hist_lane59_kernel<true, true, 1, F>);
        if (depth)
            return centred   ? lbp_hist_lane59_kernel<true, false, 2, F>
                   : fp16win ? lbp_hist_lane59_kernel<true, false, 1, F>
                             : lbp_hist_lane59_kernel<true, false, 0, F>;
        return lbp_hist_lane59_kernel<false, false, 0, F>;
    };
    auto pick_out = [&](auto out_tag) {  // crop stacks, grey codes, gather or u8 output
        constexpr int O = decltype(out_tag)::value;
        if (depth)
            return centred   ? lbp_hist_lane59_kernel<true, false, 2, false, O>
                   : fp16win ? lbp_hist_lane59_kernel<true, false, 1, false, O>
                             : lbp_hist_lane59_kernel<true, false, 0, false, O>;
        return lbp_hist_lane59_kernel<false, false, 0, false, O>;
    };
    if (fused && !fp16win) return cudaErrorNotSupported;  // (the depth plane's compares)
    auto kern = fused   ? (dint ? (centred ? lbp_hist_lane59_kernel<true, false, 6, false, l59::kOutFused>
                                           : lbp_hist_lane59_kernel<true, false, 5, false, l59::kOutFused>)
                                : (centred ? lbp_hist_lane59_kernel<true, false, 2, false, l59::kOutFused>
                                           : lbp_hist_lane59_kernel<true, false, 1, false, l59::kOutFused>))
                : gather  ? pick_out(std::integral_constant<int, l59::kOutGather>{})
                : u8out ? pick_out(std::integral_constant<int, l59::kOutU8>{})
                : frame ? pick(std::true_type{})
                        : pick(std::false_type{});
    int lut_off = 0, smem = 0;
    if (!lut_placement(frame ? l59::Layout<true>::kLutMin : l59::Layout<false>::kLutMin,
                       l59::Layout<false>::kTailBytes, &lut_off, &smem))
        return cudaErrorNotSupported;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(sms, n_rois));
    lbp_gather_dst_t gd{};
    if (gather) gd = *gather;
    U8Out uo{};
    if (u8out) uo = *u8out;
    return launch_pdl(kern, grid, l59::kThreads, smem, stream, gm, dm, grey, depth, geom, rois,
                      n_rois, win, desc, desc_stride, roi_status, lut_off, gd, glabels, uo,
                      l59::win_words(win));
}

}  // namespace lbpf
