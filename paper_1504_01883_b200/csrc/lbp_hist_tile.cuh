// lbp_hist_tile.cuh -- the lane-private TMA extraction kernel (lbp_hist_lane59.cuh) for other
// crop sizes: stacks of T x T ROIs, 8x8 cells, 59 uniform bins, grey codes with the depth
// mask (Eq. 2; per-cell histograms; ROI sizes: the paper resizes every face to
// 200x200; BASELINE configs[0] uses 64x64 crops).
//
// The 128x128 kernel maps warp w to cell row w and lane l to columns 4l..4l+3 of a crop.  Here
// a TILE is what one 8-warp group processes between two barriers:
//  * T <= 64 (kP = 2): two crops side by side -- lanes 0-15 hold crop A's columns, lanes 16-31
//    crop B's; warp w = cell row w of both.  The shuffles across the 15|16 lane boundary only
//    feed border pixels, which have no code.
//  * T > 128 (kQ = 2): one QUADRANT of a crop (4x4 cells): the box of its interior plus the
//    1-px halo (101 x 101 for T = 200), processed by a 4-warp group (warp = cell row).  A
//    quadrant's cells are disjoint from the other quadrants', so its 16 cell histograms are
//    final at the end of the tile: no cross-tile merge.
// Boxes start 16-B aligned (TMA); a quadrant's box starts at its halo column rounded down to
// 16 px, so its counted pixels begin o = 0..15 columns in.  Which counter lane ("slot") each
// (lane, pixel) adds to is a host-built table (TileTab, build_tab): the cell's slot group at
// position lane & (m - 1) -- conflict-free shared atomics -- and the epilogue reads each cell's
// 2 / 4 / 8 slots as one 8-B pair / one or two 16-B quads (bytes = 4 cell rows) and stages u16
// counts.
#pragma once
#include "lbp_hist_lane59.cuh"

namespace lbpf {
namespace tile {

constexpr int kBins = 59;
constexpr int kBinsAlloc = 60;  // + the dummy bin of masked-out pixels

// floor partition of n interior pixels into 8 cells: first interior index of cell c
__host__ __device__ constexpr int cstart(int c, int n) { return (c * n) / 8; }
__host__ __device__ constexpr int up(int v, int m) { return (v + m - 1) / m * m; }

template <int T>
struct Geo {
    static_assert(T % 4 == 0 && T >= 32 && T <= 252,
                  "tile kernel: T <= 64 (two crops per tile), <= 128 (one), <= 252 (quadrants)");
    static constexpr int kQ = T > 128 ? 2 : 1;        // tiles per axis of a crop
    static constexpr int kP = T <= 64 ? 2 : 1;         // crops side by side in a tile
    static constexpr int kCT = 8 / kQ;                 // cells per tile axis
    static constexpr int kInt = T - 2;                 // interior pixels per axis
    // one warp per cell row of the tile: 8-warp groups x 3 with one stage each (64 px), x 2
    // with two stages each (65-128 px), 4-warp groups x 5 with one stage each (200 px: a
    // quadrant's 4 cell rows of 24-25 rows each -- twice the rows per warp of two warps per
    // cell row, half the per-tile head per crop, one warp per SMSP in each group barrier).
    // A second stage per group hides the refill (the group's next tile is loaded while it
    // works on the current one): 100 px 0.2055 -> 0.2030 ms per step; at 64 px three
    // single-stage groups measured faster than two double-buffered ones (0.1174 vs 0.1235 ms);
    // at 200 px two stages per group do not fit (3 groups x 2: 233,568 B)
    static constexpr int kWarps = kCT;
    static constexpr int kGT = kWarps * 32;
    static constexpr int kGroups = kQ == 2 ? 5 : kP == 2 ? 3 : 2;
    static constexpr int kThreads = kGroups * kGT;
    static constexpr int kG = kCT / 4 > 0 ? kCT / 4 : 1;  // counter words per (bin, lane)
    // halo column (= crop column of the tile's first interior pixel - 1) and aligned box start
    static constexpr int halo(int q) { return cstart(q * kCT, kInt); }
    static constexpr int bx(int q) { return halo(q) & ~15; }
    static constexpr int span(int q) { return cstart((q + 1) * kCT, kInt) - cstart(q * kCT, kInt); }
    static constexpr int need(int q) { return halo(q) - bx(q) + span(q) + 2; }  // box columns
    static constexpr int kNeed = need(0) > need(kQ - 1) ? need(0) : need(kQ - 1);
    static constexpr int kGW = up(kNeed, 16);           // grey box width (bytes)
    static constexpr int kDW = up(kNeed, 8);            // depth box width (pixels)
    static constexpr int kBH = (span(0) > span(kQ - 1) ? span(0) : span(kQ - 1)) + 2;  // rows
    // a crop in a stage: the grey box, then the depth box, each 128-B aligned (TMA destination)
    static constexpr int kGreyRegion = up(kBH * kGW, 128);
    static constexpr int kCropBytes = up(kGreyRegion + kBH * 2 * kDW, 128);
    static constexpr int kBoxBytesGrey = kBH * kGW, kBoxBytesDepth = kBH * 2 * kDW;
    static constexpr int kStageBytes = kP * kCropBytes;
    // kSPG stages per group: position i takes stage i % kStages and group i % kGroups, so a
    // group's positions always reuse ITS stages in turn and each stage barrier's phases are
    // consumed in order (stages shared between groups would let a fast group wait on a phase
    // two ahead, which mbarrier parity cannot tell from the last one)
    static constexpr int kSPG = kQ == 1 && kP == 1 ? 2 : 1;
    static constexpr int kStages = kGroups * kSPG;
    // staged row pitch (kQ = 1): 16 B more than the row, so the two rows' entries of one cell
    // land in different banks
    static constexpr int kRowPad = 64 * kBins + 8;
    static constexpr int kHistBytes = kG * kBinsAlloc * 32 * 4;
    // the tile's output staged as u16 before the coalesced copy-out: kP whole rows (kQ = 1)
    // or the quadrant's kCT x kCT cells (kQ = 2)
    static constexpr int kStageOut = kQ == 1 ? kP * kRowPad * 2 : kCT * kCT * kBins * 2;
    // + the ROIs of the tile this group's release will load next (kP x 20 B, cp.async)
    static constexpr int kGroupBytes = kHistBytes + up(kStageOut, 128) + 128;
    static constexpr int kGroupOff = kStages * kStageBytes;
    static constexpr int kLutMin = up(kGroupOff + kGroups * kGroupBytes, 256);
    // LUT, plain LUT, stage barriers, the lane tables (TileTab, copied to shared memory: the
    // lane-indexed reads of the kernel-parameter copy serialise in the constant cache), slack
    static constexpr int kTailBytes = l59::kLutBytes + 256 + kStages * 8 + 512 + kStages * 8 + 128;
    // rows of one warp: a cell row
    static constexpr int kMaxRows = (kInt + 7) / 8;
    static constexpr int kMinRows = kInt / 8;  // every warp has at least these rows
    static constexpr int kLanesPerCrop = 32 / kP;
    static_assert(kNeed <= 4 * kLanesPerCrop, "a tile row fits the lanes");
    static_assert(kLutMin + kTailBytes <= 227 * 1024, "shared memory");
};

// host-built lane tables of one tile column position qx (see the header)
struct TileTab {
    uint8_t slot[2][32][4];  // [qx][lane][pixel k]: counter lane, 0xFF = not counted
};

}  // namespace tile

template <int T, bool HAS_DEPTH, int WINM>
__global__ void __launch_bounds__(tile::Geo<T>::kThreads, 1)
lbp_hist_tile_kernel(const __grid_constant__ CUtensorMap grey_map,
                     const __grid_constant__ CUtensorMap depth_map,
                     const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                     lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                     DepthWindow win, uint16_t* __restrict__ desc, int64_t desc_stride,
                     int32_t* __restrict__ roi_status, int32_t lut_off,
                     const __grid_constant__ tile::TileTab tab) {
    using namespace tile;
    using G = Geo<T>;
    constexpr int kQ = G::kQ, kP = G::kP, kCT = G::kCT, kInt = G::kInt;
    constexpr int kStages = G::kStages, kGroups = G::kGroups, kGT = G::kGT;
    constexpr int kTilesPerCrop = kQ * kQ;
    constexpr int kDim = 64 * kBins;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                               ~uintptr_t(127));
    const int tid = threadIdx.x;
    const int group = tid / kGT, gtid = tid % kGT;
    const int warp = gtid >> 5, lane = gtid & 31;
    const uint32_t stages0 = smem_u32(smem);
    const uint32_t hist0 = stages0 + G::kGroupOff + group * G::kGroupBytes;
    const uint32_t staging = hist0 + G::kHistBytes;
    const uint32_t roi_slot = staging + up(G::kStageOut, 128);
    const int kLutOff = lut_off, kPlainLutOff = lut_off + l59::kLutBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPlainLutOff + 256);
    const uint32_t tab_s = smem_u32(smem + kPlainLutOff + 256 + kStages * 8);  // TileTab copy
    // 64 px (kQ = 1): the two 4-warp halves of a group (cell rows 0-3 / 4-7 = the counter
    // words g = 0 / 1, one warp per SMSP) sync among themselves and store their half of both
    // rows; the stage is refilled by the half that releases it second (per-stage counter)
    constexpr bool SUB = kQ == 1;
    const int sub = warp >> 2, stid = gtid & 127;
    const uint32_t sub_bar = 1 + kGroups + 2 * group + sub;  // after the group barriers
    const bool leader = SUB ? stid == 0 : gtid == 0;
    const uint32_t rel0 = tab_s + 512;  // per-stage release counts
    // per-stage flag: the tile staged there takes the fast path (written by the issuing thread
    // before its mbarrier arrive, read after the wait: lbp_hist_lane59.cuh), so the ROIs are
    // read only by the issuing leaders and on the generic path
    const uint32_t fastf = rel0 + kStages * 4;
    const uint32_t bar_id = 1 + group;

    // tiles: crop pairs (kP = 2: crops 2t, 2t+1) or quadrants (kQ = 2: crop t / 4, q = t % 4)
    const int64_t n_tiles = kP == 2 ? ((int64_t)n_rois + 1) / 2 : (int64_t)n_rois * kTilesPerCrop;
    // quadrant tiles (kQ = 2): a CTA takes all four quadrants of its crops at consecutive
    // positions (four groups at once), so the rows and columns the quadrant boxes share, and
    // the DRAM sectors their edges share, are read while still in L2 (the four quadrants of a
    // crop in four CTAs read 1.35x the crop's bytes from DRAM)
    const int n_pos = kQ == 2
        ? (n_rois > (int)blockIdx.x ? ((n_rois - 1 - (int)blockIdx.x) / (int)gridDim.x + 1) * 4 : 0)
        : (n_tiles > (int64_t)blockIdx.x) ? (int)((n_tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    auto tile_of = [&](int i) -> int64_t {
        if constexpr (kQ == 2)
            return ((int64_t)blockIdx.x + (int64_t)(i >> 2) * gridDim.x) * 4 + (i & 3);
        return (int64_t)blockIdx.x + (int64_t)i * gridDim.x;
    };
    auto crop_of = [&](int64_t t, int p) -> int64_t {
        return kP == 2 ? 2 * t + p : t / kTilesPerCrop;
    };
    auto fast_roi = [&](const lbp_roi_t& r) {
        return r.w == T && r.h == T && r.img >= 0 && r.img < geom.n_images && r.x >= 0 &&
               (r.x & 15) == 0 && r.y >= 0 && (int64_t)r.x + T <= geom.width &&
               (int64_t)r.y + T <= geom.height;
    };
    struct TileRois { lbp_roi_t r[kP]; bool valid[kP]; };
    auto load_tile = [&](int i) {
        TileRois tr{};
        if (i >= n_pos) return tr;
        const int64_t t = tile_of(i);
#pragma unroll
        for (int p = 0; p < kP; ++p) {
            const int64_t c = crop_of(t, p);
            tr.valid[p] = c < n_rois;
            if (tr.valid[p]) tr.r[p] = rois[c];
        }
        return tr;
    };
    auto tile_fast = [&](const TileRois& tr) {
        bool f = true;
#pragma unroll
        for (int p = 0; p < kP; ++p) f = f && (!tr.valid[p] || fast_roi(tr.r[p]));
        return f;
    };
    auto issue = [&](int i, const TileRois& tr) {
        if (i >= n_pos) return;
        const int s = i % kStages;
        const bool fast = tile_fast(tr);
        st_shared_u32(fastf + 4 * s, fast ? 1u : 0u);
        if (!fast) {
            mbar_arrive(&bars[s]);
            return;
        }
        const int q = kQ == 2 ? (int)(tile_of(i) % kTilesPerCrop) : 0;
        const int qx = q & 1, qy = q >> 1;
        uint32_t bytes = 0;
#pragma unroll
        for (int p = 0; p < kP; ++p)
            if (tr.valid[p]) bytes += G::kBoxBytesGrey + (HAS_DEPTH ? G::kBoxBytesDepth : 0);
        mbar_arrive_expect_tx(&bars[s], bytes);
        uint8_t* st = smem + s * G::kStageBytes;
#pragma unroll
        for (int p = 0; p < kP; ++p) {
            if (!tr.valid[p]) continue;
            const lbp_roi_t& r = tr.r[p];
            const int x = r.x + G::bx(qx), y = r.y + G::halo(qy);
            uint8_t* cp = st + p * G::kCropBytes;
            tma_load_3d(cp, &grey_map, &bars[s], x, y, r.img);
            if (HAS_DEPTH) tma_load_3d(cp + G::kGreyRegion, &depth_map, &bars[s], x, y, r.img);
        }
    };

    // the dependent launch (the scorer) may be scheduled now (see lbp_hist_lane59.cuh)
    launch_dependents();
    // ---- one-time setup: barriers and the first kStages positions' loads first (their
    // latency overlaps the table fills), then LUTs, lane table, zeroed counters
    if (tid == 0) {
        if ((smem_u32(smem + kLutOff) & 0xFFFFu) != l59::kLutMod) __trap();
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
        if (HAS_DEPTH) prefetch_tensormap(&depth_map);
        grid_dependency_wait();  // (see below)
        for (int i = 0; i < kStages; ++i) issue(i, load_tile(i));
    }
    for (int i = tid; i < l59::kLutBytes; i += G::kThreads) {
        const int code = (i >> 7) * 4 + (i & 3);
        smem[kLutOff + i] = code < 256 ? kUniformLutDev.v[code] : (uint8_t)kBins;
    }
    if (tid < 256) smem[kPlainLutOff + tid] = kUniformLutDev.v[tid];
    static_assert(sizeof(TileTab) % 4 == 0 && sizeof(TileTab) <= 512, "table copy");
    if (tid < (int)sizeof(TileTab) / 4)
        st_shared_u32(tab_s + 4 * tid, reinterpret_cast<const uint32_t*>(&tab)[tid]);
    if (tid < kStages) st_shared_u32(tab_s + 512 + 4 * tid, 0u);
    for (int i = gtid; i < G::kHistBytes / 16; i += kGT)
        st_shared_u32x4(hist0 + i * 16, make_uint4(0, 0, 0, 0));
    // programmatic dependent launch: the setup above may overlap the tail of the previous
    // kernel on the stream; inputs and outputs are touched only after it has completed
    grid_dependency_wait();
    __syncthreads();

    // ---- per-thread constants
    const uint32_t mid2 = ((2 * win.lo + win.span) / 2) * 0x10001u;  // WINM 2
    const uint32_t half2 = (win.span / 2) * 0x10001u;
    const uint32_t lo2 = win.lo * 0x10001u, hi2 = (win.lo + win.span) * 0x10001u;  // WINM 1
    const uint32_t lo16 = win.lo << 16, span16 = (win.span << 16) | 0xFFFFu;        // WINM 0
    const uint32_t lutb = opaque(smem_u32(smem + kLutOff) - l59::kLutMod);
    const uint32_t top2 = opaque((l59::kLutMod + 4u * lane + 899u) * 0x10001u);
    const int p_lane = lane / G::kLanesPerCrop, l_in = lane % G::kLanesPerCrop;
    // the warp's cell row in the tile and its share of that cell row's interior rows
    const int cr = warp;  // the warp's cell row in the tile
    const uint32_t byte_mult = 1u << (8 * (cr & 3));
    const uint32_t hist_g = hist0 + (uint32_t)((cr >> 2) * kBinsAlloc * 128);
    const bool none = HAS_DEPTH && win.none_valid;

    bool pending = false;  // leader: a bulk store of the staging is in flight
    for (int i = group; i < n_pos; i += kGroups) {
        const int64_t t = tile_of(i);
        bool valid[kP];
#pragma unroll
        for (int p = 0; p < kP; ++p) valid[p] = crop_of(t, p) < n_rois;
        // the ROIs of position i + kStages (loaded when this tile releases stage s): fetched
        // now by cp.async into the group's slot, so no registers hold them through the rows
        if (leader && i + kStages < n_pos) {  // each leader into its own slot
            const int64_t tf = tile_of(i + kStages);
#pragma unroll
            for (int p = 0; p < kP; ++p) {
                const int64_t c = crop_of(tf, p);
                if (c < n_rois)
                    for (int w = 0; w < 5; ++w)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                         roi_slot + (uint32_t)(sub * 64 + p * 20 + 4 * w)),
                                     "l"(reinterpret_cast<const int32_t*>(rois + c) + w)
                                     : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        auto fill_rois = [&]() {  // (a leader) the ROIs of position i + kStages, its own slot
            TileRois f{};
            if (i + kStages >= n_pos) return f;
            asm volatile("cp.async.wait_all;" ::: "memory");
            const int64_t tf = tile_of(i + kStages);
#pragma unroll
            for (int p = 0; p < kP; ++p) {
                f.valid[p] = crop_of(tf, p) < n_rois;
                if (f.valid[p]) {
                    int32_t* d = reinterpret_cast<int32_t*>(&f.r[p]);
                    for (int w = 0; w < 5; ++w)
                        d[w] = (int32_t)ld_shared_u32(roi_slot + (uint32_t)(sub * 64 + p * 20 + 4 * w));
                }
            }
            return f;
        };
        const int s = i % kStages;
        const int q = kQ == 2 ? (int)(t % kTilesPerCrop) : 0;
        const int qx = q & 1, qy = q >> 1;
        mbar_wait(&bars[s], (uint32_t)(i / kStages) & 1u);
        if (ld_shared_u32(fastf + 4 * s) == 0u) {
            const TileRois tr = load_tile(i);
            // release the unfilled stage only after every thread passed its wait on this
            // phase (see lbp_hist_lane59.cuh: an early plain arrive completes the next phase)
            named_barrier_sync(bar_id, kGT);
            if (gtid == 0) issue(i + kStages, fill_rois());
            else if (leader) asm volatile("cp.async.wait_all;" ::: "memory");  // its own copies
            uint32_t* hist = reinterpret_cast<uint32_t*>(smem + (hist0 - stages0));
#pragma unroll
            for (int p = 0; p < kP; ++p) {
                if (!tr.valid[p]) continue;
                const int64_t n = crop_of(t, p);
                if (kQ == 1) {
                    extract_roi_generic<kBins, kGT>(
                        CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                        HAS_DEPTH ? depth : nullptr, geom, tr.r[p], (int32_t)n, win, 8, 8, desc,
                        desc_stride, roi_status, hist, G::kHistBytes / 4, smem + kPlainLutOff,
                        0, gtid, [&]() { named_barrier_sync(bar_id, kGT); });
                } else {
                    for (int r = 0; r < kCT; ++r) {
                        const int c0 = (qy * kCT + r) * 8 + qx * kCT;
                        extract_roi_generic<kBins, kGT>(
                            CodePlane<uint8_t>{grey, geom.grey_pitch, geom.grey_img_stride},
                            HAS_DEPTH ? depth : nullptr, geom, tr.r[p], (int32_t)n, win, 8, 8,
                            desc, desc_stride, roi_status, hist, G::kHistBytes / 4,
                            smem + kPlainLutOff, 0, gtid,
                            [&]() { named_barrier_sync(bar_id, kGT); }, c0, c0 + kCT);
                    }
                }
            }
            named_barrier_sync(bar_id, kGT);
            continue;
        }
        // ---- per-tile lane setup: counter slots of the lane's 4 pixels (quadrant column qx)
        uint32_t colb[4], mult[4];
        // the lane's 4 slots (TileTab::slot[qx][lane][0..3]) in one conflict-free LDS
        const uint32_t slots4 = ld_shared_u32(tab_s + (uint32_t)(qx * 128 + lane * 4));
        const bool crop_ok = p_lane == 0 ? valid[0] : valid[kP - 1];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t sl = (slots4 >> (8 * k)) & 0xFFu;
            // uncounted pixels add 0 to their own lane's word (a shared dummy word would make
            // the idle lanes' atomics collide)
            colb[k] = hist_g + (sl == 0xFFu ? (uint32_t)lane : sl) * 4u;
            mult[k] = (sl != 0xFFu && crop_ok && !none) ? byte_mult : 0u;
        }
        // rows: interior rows [a, b) of the cell row
        const int cy = qy * kCT + cr;
        const int ra = cstart(cy, kInt), rb = cstart(cy + 1, kInt);
        const int i0 = ra, nrows = rb - ra;
        // box row of interior row i: i + 1 - halo(qy); the top neighbour of i0 is box row
        // i0 - halo(qy)
        const int br0 = i0 - G::halo(qy);
        const uint32_t st = stages0 + s * G::kStageBytes + p_lane * G::kCropBytes;
        const uint32_t g0 = st + br0 * G::kGW + 4 * l_in;
        const uint32_t d0 = st + G::kGreyRegion + (br0 + 1) * (2 * G::kDW) + 8 * l_in;

        struct Pend { uint32_t bin[4], val[4]; };
        auto do_row = [&](const LaneRow& top, const LaneRow& mid, const LaneRow& bot, uint2 dw) {
            uint32_t t0 = lbp_offset2(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh, bot.h0,
                                      bot.lh0, mid.lh0, top2);
            uint32_t t1 = lbp_offset2(mid.h1, top.mh, top.h1, top.rh1, mid.rh1, bot.rh1, bot.h1,
                                      bot.mh, mid.mh, top2);
            uint32_t val[4];
            if constexpr (HAS_DEPTH && WINM != 0) {
                uint32_t m0, m1;
                if constexpr (WINM == 2) {
                    m0 = hle2_mask(habsdiff2(dw.x, mid2), half2);
                    m1 = hle2_mask(habsdiff2(dw.y, mid2), half2);
                } else {
                    m0 = hge2_mask(dw.x, lo2) & hle2_mask(dw.x, hi2);
                    m1 = hge2_mask(dw.y, lo2) & hle2_mask(dw.y, hi2);
                }
                t0 = (t0 & m0) | (l59::kDummyOff2 & ~m0);
                t1 = (t1 & m1) | (l59::kDummyOff2 & ~m1);
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            } else if constexpr (HAS_DEPTH) {
                const uint32_t x[4] = {dw.x * 0x10000u - lo16, dw.x - lo16, dw.y * 0x10000u - lo16,
                                       dw.y - lo16};
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult[k] : 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) val[k] = mult[k];
            }
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
        LaneRow r0 = lane_row(g0), r1 = lane_row(g0 + G::kGW);
        uint32_t wn = ld_shared_u32(g0 + 2 * G::kGW);
        uint2 dn = make_uint2(0u, 0u);
        if (HAS_DEPTH) dn = ld_shared_u32x2(d0);
        Pend pend;
#pragma unroll
        // straight-line rows; only the last (kMaxRows - kMinRows) test the warp's row count, and
        // the look-ahead loads are unconditional (a row past the warp's band is read but not
        // used: still inside the CTA's shared memory)
        for (int j = 0; j < G::kMaxRows; ++j) {
            if (j >= G::kMinRows && j == nrows) {  // warp-uniform
                flush(pend);
                break;
            }
            const uint32_t wc = wn;
            const uint2 dc = dn;
            if (j + 1 < G::kMaxRows) {
                wn = ld_shared_u32(g0 + (j + 3) * G::kGW);
                if (HAS_DEPTH) dn = ld_shared_u32x2(d0 + (j + 1) * (2 * G::kDW));
            }
            const LaneRow r2 = lane_row_w(wc);
            const Pend p = do_row(r0, r1, r2, dc);
            if (j > 0) flush(pend);
            pend = p;
            r0 = r1;
            r1 = r2;
            if (j == G::kMaxRows - 1) flush(pend);
        }

        if (SUB && leader && pending) bulk_wait_read_all();  // staging half free again
        // A: this half's (SUB) / the group's counters complete and its stage rows read; the
        // second half to get here refills the stage
        named_barrier_sync(SUB ? sub_bar : bar_id, SUB ? 128 : kGT);
        if (leader && (!SUB || (atom_shared_add(rel0 + 4 * s, 1u) & 1u))) {
            issue(i + kStages, fill_rois());
            if (roi_status && q == 0) {
#pragma unroll
                for (int p = 0; p < kP; ++p)
                    if (valid[p]) roi_status[crop_of(t, p)] = LBP_OK;
            }
        } else if (leader) {
            // the half that released first: retire its own ROI copies too, so that they can
            // never land after the next tile's copies into the same slot
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        // ---- epilogue: the slots of each cell summed, counters re-zeroed, counts staged
        // as u16 ([row][cell][bin]), then copied out
        if constexpr (kQ == 1 && kP == 1) {
            // one crop (64 < T <= 128), quad slots (build_tab): this half's quads (bin, cell
            // x) of its counter word g = sub, as the 128-px kernel's epilogue -- thread ->
            // cx = stid & 7, bins bp + 16 k (bp = stid >> 3); one 16-B load, a byte transpose
            // and IDP4A give the cell's 4 cell rows
            const int ecx = stid & 7, ebp = stid >> 3;
            const uint32_t qbase = hist0 + (uint32_t)(((sub * kBinsAlloc + ebp) * 8 + ecx) * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int bin = ebp + 16 * k;
                if (bin > kBins) break;
                const uint32_t qa = qbase + k * (16 * 128);
                const uint4 w = ld_shared_u32x4(qa);
                st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
                if (bin == kBins) break;  // dummy bin: only re-zeroed
                const uint32_t lo01 = prmt(w.x, w.y, 0x5140), hi01 = prmt(w.x, w.y, 0x7362);
                const uint32_t lo23 = prmt(w.z, w.w, 0x5140), hi23 = prmt(w.z, w.w, 0x7362);
                const uint32_t c[4] = {__dp4a(prmt(lo01, lo23, 0x5410), 0x01010101u, 0u),
                                       __dp4a(prmt(lo01, lo23, 0x7632), 0x01010101u, 0u),
                                       __dp4a(prmt(hi01, hi23, 0x5410), 0x01010101u, 0u),
                                       __dp4a(prmt(hi01, hi23, 0x7632), 0x01010101u, 0u)};
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int e = ((4 * sub + b) * 8 + ecx) * kBins + bin;
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(staging + 2 * e),
                                 "h"((uint16_t)c[b])
                                 : "memory");
                }
            }
        } else if constexpr (kQ == 1) {
            // two crops, pair slots (build_tab: cell c of crop p = slots 16 p + 2 c, + 1): thread -> cell
            // column cc = bits 0-2, crop p = bit 3, bins bp + 8 k (bp = bits 4-6), counter
            // word g = bit 7 = the half -- affine in k; a quarter-warp's LDS.64 reads 64
            // contiguous B
            const int ecc = gtid & 7, ep = (gtid >> 3) & 1, ebp = (gtid >> 4) & 7, eg = gtid >> 7;
            const uint32_t q0 =
                hist0 + (uint32_t)((eg * kBinsAlloc + ebp) * 128 + (2 * ecc + 16 * ep) * 4);
            const uint32_t e0 = staging + 2u * (uint32_t)(ep * G::kRowPad +
                                                          ((4 * eg) * 8 + ecc) * kBins + ebp);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int bin = ebp + 8 * k;
                if (bin > kBins) break;
                const uint32_t qa = q0 + k * 8 * 128;
                const uint2 w = ld_shared_u32x2(qa);
                st_shared_u32x2(qa, make_uint2(0u, 0u));
                if (bin == kBins) break;  // dummy bin (masked-out pixels): only re-zeroed
                const uint32_t sum = w.x + w.y;  // bytewise: each byte <= 2 x 48
#pragma unroll
                for (int b = 0; b < 4; ++b)  // byte b zero-extended: one PRMT with a zero word
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(e0 + 2u * (8 * k + b * 8 * kBins)),
                                 "r"(prmt(sum, 0u, 0x4440u | (uint32_t)b))
                                 : "memory");
            }
        } else {
            // quadrant, octet slots (build_tab): thread -> quad lq = gtid & 7 (slots 4 lq ..
            // 4 lq + 3: half of cell lq >> 1), bins bp + 16 k (bp = gtid >> 3); a quarter-warp
            // reads one bin's 128 contiguous bytes; the two quads of a cell (adjacent lanes)
            // are combined by one shuffle of the packed 16-bit partial counts.  The loop runs
            // uniformly (the shuffles need the whole warp); bins past the dummy are predicated.
            static_assert(kGT == 128 && kCT == 4, "quadrant epilogue map");
            const int lq = gtid & 7, ebp = gtid >> 3;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int bin = ebp + 16 * k;
                const uint32_t qa = hist0 + (uint32_t)(bin * 128 + lq * 16);
                uint4 w = make_uint4(0, 0, 0, 0);
                if (bin <= kBins) {
                    w = ld_shared_u32x4(qa);
                    st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
                }
                const uint32_t lo01 = prmt(w.x, w.y, 0x5140), hi01 = prmt(w.x, w.y, 0x7362);
                const uint32_t lo23 = prmt(w.z, w.w, 0x5140), hi23 = prmt(w.z, w.w, 0x7362);
                const uint32_t p01 = __dp4a(prmt(lo01, lo23, 0x5410), 0x01010101u, 0u) |
                                     (__dp4a(prmt(lo01, lo23, 0x7632), 0x01010101u, 0u) << 16);
                const uint32_t p23 = __dp4a(prmt(hi01, hi23, 0x5410), 0x01010101u, 0u) |
                                     (__dp4a(prmt(hi01, hi23, 0x7632), 0x01010101u, 0u) << 16);
                // each partial <= 4 x 255: the 16-bit halves do not carry
                const uint32_t s01 = p01 + __shfl_xor_sync(0xFFFFFFFFu, p01, 1);
                const uint32_t s23 = p23 + __shfl_xor_sync(0xFFFFFFFFu, p23, 1);
                if (bin < kBins && (lq & 1) == 0) {
                    const int cc = lq >> 1;
                    const uint32_t c[4] = {s01 & 0xFFFFu, s01 >> 16, s23 & 0xFFFFu, s23 >> 16};
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int e = (b * kCT + cc) * kBins + bin;
                        asm volatile("st.shared.u16 [%0], %1;" ::"r"(staging + 2 * e),
                                     "h"((uint16_t)c[b])
                                     : "memory");
                    }
                }
            }
        }
        if constexpr (kQ == 1) {
            fence_proxy_async_smem();          // staged rows -> async proxy
            named_barrier_sync(sub_bar, 128);  // B: this half's counters zero, its half staged
            if (stid == 0) {  // cell rows 4 sub .. 4 sub + 3 of both rows: contiguous halves
                constexpr int kHalf = kDim / 2;
#pragma unroll
                for (int p = 0; p < kP; ++p)
                    if (p == 0 ? valid[0] : valid[kP - 1])
                        bulk_store_s2g(desc + crop_of(t, p) * desc_stride + sub * kHalf,
                                       staging + (p * G::kRowPad + sub * kHalf) * 2, kHalf * 2);
                pending = true;
            }
        } else {
            named_barrier_sync(bar_id, kGT);   // B: counters zero, quadrant staged
            // copy-out: kCT runs (cell rows) of kCT cells x 59 bins, 8-B aligned in the row
            constexpr int kRun8 = kCT * kBins * 2 / 8;  // u64 per run
            uint16_t* out = desc + crop_of(t, 0) * desc_stride;
            for (int v = gtid; v < kCT * kRun8; v += kGT) {
                const int r = v / kRun8, o = v - r * kRun8;
                const uint2 x = ld_shared_u32x2(staging + (uint32_t)(r * kRun8 + o) * 8);
                uint16_t* dst = out + ((qy * kCT + r) * 8 + qx * kCT) * kBins + 4 * o;
                *reinterpret_cast<uint2*>(dst) = x;
            }
        }
    }
    if (SUB && leader && pending) bulk_wait_all();
}

// ---- host side
namespace tile {

// the lane tables of crop size T (TileTab): pixel (lane, k) of tile column qx is crop column
// x = bx(qx) + 4 (lane % lanes_per_crop) + k; it is counted iff x is an interior column of the
// tile (halo < x <= halo + span), into a SLOT (counter lane) of its cell: for one pixel index k
// a cell of <= 4 m px spans <= m consecutive lanes, so slot m c + (lane & (m - 1)) never puts
// two lanes of one atomic on the same bank, and a cell's m slots are contiguous words for the
// epilogue -- m = 2 (two 64-px crops: 16 slots each), 4 (one crop of <= 128 px), 8 (200-px
// quadrants: 4 cells).  False when the cells are too wide for that (never for the
// instantiated T).
template <int T>
inline bool build_tab(TileTab* tab) {
    using G = Geo<T>;
    *tab = TileTab{};
    for (int qx = 0; qx < G::kQ; ++qx) {
        const int h = G::halo(qx), lo_x = h + 1, hi_x = h + G::span(qx);  // counted columns
        auto cell = [&](int x) { return (((x - 1) + 1) * 8 - 1) / G::kInt - qx * G::kCT; };
        if (G::kP == 2) {
            // two crops (cells <= 8 px): PAIR slots -- pixel (l, k) of cell c of crop p counts
            // into slot 16 p + 2 c + (l & 1): for one pixel index k a cell spans <= 2
            // consecutive lanes, so the atomics are conflict-free, and each cell's two slots
            // are the 8-B pair the epilogue reads
            for (int l = 0; l < 32; ++l) {
                const int li = l % G::kLanesPerCrop, base = l - li;
                for (int k = 0; k < 4; ++k) {
                    const int x = G::bx(qx) + 4 * li + k;
                    uint8_t sl = 0xFF;
                    if (x >= lo_x && x <= hi_x) sl = (uint8_t)(base + 2 * cell(x) + (l & 1));
                    tab->slot[qx][l][k] = sl;
                }
            }
            if (G::kInt / 8 + 1 > 8) return false;  // pair slots need cells of <= 8 px
            continue;
        }
        if (G::kQ == 2) {
            // quadrant (4 cells of ~25 px, <= 8 lanes each): OCTET slots -- pixel (l, k) of
            // tile cell c counts into slot 8 c + (l & 7): conflict-free atomics (a cell's
            // lanes are <= 8 consecutive lanes), each cell's slots two 16-B quads
            int first[4], last[4];
            for (int c = 0; c < 4; ++c) { first[c] = 99; last[c] = -1; }
            for (int l = 0; l < 32; ++l)
                for (int k = 0; k < 4; ++k) {
                    const int x = G::bx(qx) + 4 * l + k;
                    uint8_t sl = 0xFF;
                    if (x >= lo_x && x <= hi_x) {
                        const int c = cell(x);
                        sl = (uint8_t)(8 * c + (l & 7));
                        first[c] = first[c] < l ? first[c] : l;
                        last[c] = last[c] > l ? last[c] : l;
                    }
                    tab->slot[qx][l][k] = sl;
                }
            for (int c = 0; c < 4; ++c) {
                if (last[c] < 0 || last[c] - first[c] > 7) return false;
            }
            continue;
        }
        if (G::kP == 1 && G::kQ == 1) {
            // one crop, cells <= 13 px (<= 4 lanes): QUAD slots -- pixel (l, k) of cell c counts
            // into slot 4 c + (l & 3); the lanes of one cell are <= 4 consecutive lanes, so their
            // (l & 3) differ and the atomics stay conflict-free with no spill case, and each
            // cell's 4 slots are one 16-B quad for the epilogue (as the 128-px kernel)
            int first[8], last[8];
            for (int c = 0; c < 8; ++c) { first[c] = 99; last[c] = -1; }
            for (int l = 0; l < 32; ++l)
                for (int k = 0; k < 4; ++k) {
                    const int x = G::bx(qx) + 4 * l + k;
                    uint8_t sl = 0xFF;
                    if (x >= lo_x && x <= hi_x) {
                        const int c = cell(x);
                        sl = (uint8_t)(4 * c + (l & 3));
                        first[c] = first[c] < l ? first[c] : l;
                        last[c] = last[c] > l ? last[c] : l;
                    }
                    tab->slot[qx][l][k] = sl;
                }
            for (int c = 0; c < 8; ++c) {
                if (last[c] < 0 || last[c] - first[c] > 3) return false;
            }
            continue;
        }
        return false;  // (no slot scheme for this geometry)
    }
    return true;
}

inline bool encode_box_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem,
                           const lbp_images_t& g, int64_t pitch, int64_t img_stride, int box_w,
                           int box_h) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * elem), (cuuint64_t)(img_stride * elem)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace tile

// The tile kernel for crop size T (64 or 200) on a crop stack; cudaErrorNotSupported when the
// geometry does not allow it (the caller then takes the band kernel).
template <int T>
inline cudaError_t launch_lbp_hist_tile(const uint8_t* grey, const uint16_t* depth,
                                        const lbp_images_t& geom, const lbp_roi_t* rois,
                                        int32_t n_rois, const DepthWindow& win, uint16_t* desc,
                                        int64_t desc_stride, int32_t* roi_status, int sms,
                                        cudaStream_t stream) {
    using G = tile::Geo<T>;
    static tile::TileTab tab;
    static const bool tab_ok = tile::build_tab<T>(&tab);
    if (!tab_ok) return cudaErrorNotSupported;
    CUtensorMap gm, dm;
    if (!tile::encode_box_map(&gm, grey, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, geom, geom.grey_pitch,
                              geom.grey_img_stride, G::kGW, G::kBH))
        return cudaErrorNotSupported;
    if (depth) {
        if (!tile::encode_box_map(&dm, depth, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, geom,
                                  geom.depth_pitch, geom.depth_img_stride, G::kDW, G::kBH))
            return cudaErrorNotSupported;
    } else {
        dm = gm;
    }
    const bool fp16win = depth && !win.none_valid && win.lo + win.span <= 0x7BFEu;
    const uint32_t whi = win.lo + win.span;
    const bool centred = fp16win && whi < 2048u && ((win.lo + whi) & 1u) == 0;
    auto kern = depth ? (centred   ? lbp_hist_tile_kernel<T, true, 2>
                         : fp16win ? lbp_hist_tile_kernel<T, true, 1>
                                   : lbp_hist_tile_kernel<T, true, 0>)
                      : lbp_hist_tile_kernel<T, false, 0>;
    int lut_off = 0, smem = 0;
    if (!lut_placement(G::kLutMin, G::kTailBytes, &lut_off, &smem)) return cudaErrorNotSupported;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // CTAs: crop pairs (kP = 2), crops (one tile, or all four quadrants of a crop in one CTA)
    const int64_t n_units = G::kP == 2 ? ((int64_t)n_rois + 1) / 2 : (int64_t)n_rois;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, n_units));
    return launch_pdl(kern, grid, G::kThreads, smem, stream, gm, dm, grey, depth, geom, rois,
                      n_rois, win, desc, desc_stride, roi_status, lut_off, tab);
}

}  // namespace lbpf
