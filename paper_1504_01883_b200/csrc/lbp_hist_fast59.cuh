// lbp_hist_fast59.cuh -- bank-conflict-free fused-depth LBP histogram kernel for 128x128
// ROIs, 8x8 cells, 59 uniform bins (BASELINE configs[1..4], the headline workload).
//
// Round-1 profiling of the previous kernel (profiles/r01/README.md) showed the shared-memory
// data pipe saturated by bank conflicts of the histogram atomics (random bins over random
// banks, ~4 wavefronts per ATOMS) and of the 256-B LUT (~2 wavefronts per byte load).  This
// kernel makes every shared access of the hot loop conflict-free:
//  * lane-private counters: word [bin][cell row][lane] -- lane l always hits bank l.  The 4
//    lanes of a cell (cells are 16 px = 4 lanes wide; 3 lanes spill one pixel into the next
//    cell, routed to that cell's first column) and the 4 warps sharing a cell row (each adds
//    1 << 8*sub_block: bytes of the same word, <= 16 per byte per task) are summed in the
//    epilogue with one 16-B load and one IDP4A;
//  * lane-banked LUT: bin(c) stored at byte (c>>2)*128 + 4*lane + (c&3), so lane l reads bank
//    l; the compare results are accumulated directly into that offset (Fig. 7 bits p0,p1 at
//    offsets 1,2 and p2..p7 at 128..4096);
//  * a task is HALF a crop (4 cell rows = image rows 0..65 or 62..127): one TMA stage is
//    66 x (128 + 256) B = 24.75 KB, so 4 stages, 2 counter buffers, the LUT and the output
//    staging fit in shared memory with 16 warps per SM.
// Per task: 16 warps = 4 cell rows x 4 row blocks of 3-4 rows; one named barrier; the
// epilogue writes the task's 3,776-B half descriptor to smem and a bulk async copy
// (cp.async.bulk) stores it.  Non-fast ROIs take the generic path inside the same kernel.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "lbp_hist_generic.cuh"
#include "ptx.cuh"

namespace lbpf {

namespace f59 {
constexpr int kThreads = 512;                 // 16 warps
constexpr int kTile = 128;                    // crop edge
constexpr int kBoxRows = 66;                  // rows per half-crop task (incl. halo)
constexpr int kStages = 4;
constexpr int kGreyBytes = kBoxRows * kTile;           // 8,448
constexpr int kDepthBytes = kBoxRows * kTile * 2;      // 16,896
constexpr int kStageBytes = kGreyBytes + kDepthBytes;  // 25,344 (multiple of 128)
constexpr int kBins = 59;
constexpr int kHalfCells = 32;
constexpr int kHistBytes = kBins * 4 * 32 * 4;         // [bin][cell row][lane] u32 = 30,208
constexpr int kLutBytes = 64 * 128;                    // lane-banked LUT, 8 KB
constexpr int kHalfDescBytes = kHalfCells * kBins * 2; // 3,776
constexpr int kStageOff = 0;
constexpr int kHistOff = kStages * kStageBytes;                     // 101,376
constexpr int kLutOff = kHistOff + 2 * kHistBytes;                  // 161,792
constexpr int kStagingOff = kLutOff + kLutBytes;                    // 169,984
constexpr int kPlainLutOff = kStagingOff + 2 * kHalfDescBytes;      // 177,536 (generic path)
constexpr int kBarOff = kPlainLutOff + 256;
constexpr int kSmemBytes = kBarOff + kStages * 8 + 1024;            // + align slack
static_assert(kStageBytes % 128 == 0 && kHistOff % 16 == 0 && kStagingOff % 16 == 0, "align");
}  // namespace f59

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

// Rows of fp16x2 pixels, as in lbp_hist_fast.cuh (1024+g).
struct Row59 {
    uint32_t h0, h1, lh0, mh, rh1;
};

__device__ __forceinline__ Row59 make_row59(uint32_t word_addr) {
    const uint32_t w = ld_shared_u32(word_addr);
    Row59 r;
    r.h0 = prmt(w, 0x64646464u, 0x5140);
    r.h1 = prmt(w, 0x64646464u, 0x7362);
    const uint32_t left = __shfl_up_sync(0xFFFFFFFFu, r.h1, 1);
    const uint32_t right = __shfl_down_sync(0xFFFFFFFFu, r.h0, 1);
    r.lh0 = prmt(left, r.h0, 0x5432);
    r.mh = prmt(r.h0, r.h1, 0x5432);
    r.rh1 = prmt(r.h1, right, 0x5432);
    return r;
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

// Eq. 2 for the two pixels of centre pair c, returned per 16-bit half as the lane-banked
// LUT offset 0x6400 + (code & 3) + 128 * (code >> 2), with the Fig. 7 bit order
// (TL 1, T 2, TR 4, R 8, BR 16, B 32, BL 64, L 128).  TL, T, TR, R run on the FMA pipe as
// sat(g_p - g_c + 1) in {0,1} scaled by 1, 2, 128, 256 and accumulated onto 1024.0 (exact
// integers below 2048 in fp16); BR, B, BL, L run on the ALU pipe as HSET2 masks at bits
// 9..12; the two partial words are added (the fp16 bias 0x6400 overlaps bit 10 only as an
// arithmetic constant).
__device__ __forceinline__ uint32_t code_offset2(uint32_t c, uint32_t tl, uint32_t t, uint32_t tr,
                                                 uint32_t r, uint32_t br, uint32_t b,
                                                 uint32_t bl, uint32_t l) {
    constexpr uint32_t kOne = 0x3C003C00u, kMinusOne = 0xBC00BC00u, k1024 = 0x64006400u;
    const uint32_t negc1 = f16_fma(c, kMinusOne, kOne);                         // 1 - g_c
    uint32_t f = f16_fma(f16_fma_sat(tl, kOne, negc1), kOne, k1024);           // TL -> +1
    f = f16_fma(f16_fma_sat(t, kOne, negc1), 0x40004000u, f);                  // T  -> +2
    f = f16_fma(f16_fma_sat(tr, kOne, negc1), 0x58005800u, f);                 // TR -> +128
    f = f16_fma(f16_fma_sat(r, kOne, negc1), 0x5C005C00u, f);                  // R  -> +256
    uint32_t a = hge2_mask(br, c) & 0x02000200u;                               // BR -> +512
    a |= hge2_mask(b, c) & 0x04000400u;                                        // B  -> +1024
    a |= hge2_mask(bl, c) & 0x08000800u;                                       // BL -> +2048
    a |= hge2_mask(l, c) & 0x10001000u;                                        // L  -> +4096
    return f + a;  // per half: 0x6400 + offset, offset <= 8067 (no carry between halves)
}

template <bool HAS_DEPTH>
__global__ void __launch_bounds__(f59::kThreads, 1)
lbp_hist_fast59_kernel(const __grid_constant__ CUtensorMap grey_map,
                       const __grid_constant__ CUtensorMap depth_map,
                       const uint8_t* __restrict__ grey, const uint16_t* __restrict__ depth,
                       lbp_images_t geom, const lbp_roi_t* __restrict__ rois, int32_t n_rois,
                       DepthWindow win, uint16_t* __restrict__ desc,
                       int32_t* __restrict__ roi_status) {
    using namespace f59;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cr = warp >> 2, sb = warp & 3;  // cell row within the half, row block

    // ---- one-time setup: lane-banked LUT, zero counters, barriers
    for (int i = tid; i < kLutBytes; i += kThreads) {
        const int row = i >> 7, ln_byte = i & 127;
        const int code = row * 4 + (ln_byte & 3);
        smem[kLutOff + i] = kUniformLutDev.v[code];
    }
    if (tid < 256) smem[kPlainLutOff + tid] = kUniformLutDev.v[tid];
    for (int i = tid; i < 2 * kHistBytes / 16; i += kThreads)
        st_shared_u32x4(smem_u32(smem + kHistOff) + i * 16, make_uint4(0, 0, 0, 0));
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        prefetch_tensormap(&grey_map);
        if (HAS_DEPTH) prefetch_tensormap(&depth_map);
    }
    __syncthreads();

    // ---- task sequence of this CTA: fast ROIs n = blockIdx.x + k*gridDim.x, halves 0, 1
    const int G = gridDim.x;
    auto next_fast = [&](int32_t n) {
        while (n < n_rois && !roi_is_fast(rois[n], geom)) n += G;
        return n;
    };
    auto issue = [&](int32_t n, int half, int s) {
        const lbp_roi_t r = rois[n];
        uint8_t* st = smem + kStageOff + s * kStageBytes;
        mbar_arrive_expect_tx(&bars[s], HAS_DEPTH ? kStageBytes : kGreyBytes);
        tma_load_3d(st, &grey_map, &bars[s], r.x, r.y + 62 * half, r.img);
        if (HAS_DEPTH) tma_load_3d(st + kGreyBytes, &depth_map, &bars[s], r.x, r.y + 62 * half, r.img);
    };
    // producer cursor (thread 0 only)
    int32_t pn = next_fast(blockIdx.x);
    int ph = 0;
    if (tid == 0) {
        for (int s = 0; s < kStages && pn < n_rois; ++s) {
            issue(pn, ph, s);
            if (ph == 1) pn = next_fast(pn + G);
            ph ^= 1;
        }
    }

    // ---- per-lane constants
    // columns 4l..4l+3: counter column (own lane, or the next cell's first lane for the one
    // spill-over pixel of lanes 19/23/27) and validity multiplier (0 on the 1-px ROI border)
    uint32_t col_off[4], mult[4];
    const uint32_t byte_mult = 1u << (8 * sb);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int x = 4 * lane + k;
        const bool inner = (x != 0) && (x != kTile - 1);
        const int cx = inner ? (8 * x - 1) / (kTile - 2) : (lane >> 2);
        const int col = (cx == (lane >> 2)) ? lane : 4 * cx;
        col_off[k] = (uint32_t)(cr * 128 + col * 4);
        mult[k] = (inner && !(HAS_DEPTH && win.none_valid)) ? byte_mult : 0u;
    }
    const uint32_t lo16 = win.lo << 16;
    const uint32_t span16 = (win.span << 16) | 0xFFFFu;
    const uint32_t lut_lane = opaque(smem_u32(smem + kLutOff) + 4 * lane - 0x6400u);
    const uint32_t hist0 = smem_u32(smem + kHistOff);
    const uint32_t staging0 = smem_u32(smem + kStagingOff);

    struct Sync512 {
        __device__ __forceinline__ void operator()() const { named_barrier_sync(1, f59::kThreads); }
    };

    int stage = 0;
    uint32_t phase_bits = 0;
    int task = 0;                    // fast tasks completed (counter buffer / staging parity)
    int32_t prev_n = -1;             // task whose half descriptor waits in staging[(task-1)&1]
    int prev_half = 0;

    for (int32_t n = blockIdx.x; n < n_rois; n += G) {
        const lbp_roi_t roi = rois[n];
        if (!roi_is_fast(roi, geom)) {
            named_barrier_sync(1, kThreads);  // previous epilogue complete, buffers zero
            extract_roi_generic<kBins, kThreads>(
                grey, HAS_DEPTH ? depth : nullptr, geom, roi, n, win, kFastCells, kFastCells, desc,
                roi_status, reinterpret_cast<uint32_t*>(smem + kHistOff), 2 * kHistBytes / 4,
                smem + kPlainLutOff, 0, tid, Sync512{});
            named_barrier_sync(1, kThreads);
            continue;
        }
        for (int half = 0; half < 2; ++half) {
            mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
            phase_bits ^= 1u << stage;
            const uint32_t st = smem_u32(smem + kStageOff + stage * kStageBytes);
            const uint32_t hbuf = hist0 + (task & 1) * kHistBytes;

            // rows of this warp: cell row R = 4*half + cr, row block sb of its 15/16 rows
            const int R = 4 * half + cr;
            const int ra = (R * (kTile - 2)) / 8, rn = ((R + 1) * (kTile - 2)) / 8 - ra;
            const int i_first = ra + (rn * sb) / 4;
            const int nrows = ra + (rn * (sb + 1)) / 4 - i_first;  // 3 or 4
            // local stage row of interior row i is i + 1 - 62*half; first needed row = that - 1
            const int lrow0 = i_first - 62 * half;
            const uint32_t g0 = opaque(st + lrow0 * kTile + 4 * lane);
            const uint32_t d0 = opaque(st + kGreyBytes + (lrow0 + 1) * (kTile * 2) + 8 * lane);
            uint32_t colb[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) colb[k] = opaque(hbuf + col_off[k]);

            auto do_row = [&](const Row59& top, const Row59& mid, const Row59& bot, int j) {
                const uint32_t t0 = code_offset2(mid.h0, top.lh0, top.h0, top.mh, mid.mh, bot.mh,
                                                 bot.h0, bot.lh0, mid.lh0);
                const uint32_t t1 = code_offset2(mid.h1, top.mh, top.h1, top.rh1, mid.rh1,
                                                 bot.rh1, bot.h1, bot.mh, mid.mh);
                uint32_t val[4];
                if (HAS_DEPTH) {
                    const uint2 d = ld_shared_u32x2(d0 + j * (kTile * 2));
                    const uint32_t x[4] = {d.x * 0x10000u - lo16, d.x - lo16, d.y * 0x10000u - lo16,
                                           d.y - lo16};
#pragma unroll
                    for (int k = 0; k < 4; ++k) val[k] = (x[k] <= span16) ? mult[k] : 0u;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) val[k] = mult[k];
                }
                const uint32_t lut_addr[4] = {lut_lane + (t0 & 0xFFFFu), __umulhi(t0, 0x10000u) + lut_lane,
                                              lut_lane + (t1 & 0xFFFFu), __umulhi(t1, 0x10000u) + lut_lane};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t bin = ld_shared_u8(lut_addr[k]);
                    red_shared_add(colb[k] + bin * (4 * 32 * 4), val[k]);
                }
            };
            Row59 r0 = make_row59(g0), r1 = make_row59(g0 + kTile), r2;
            r2 = make_row59(g0 + 2 * kTile);
            do_row(r0, r1, r2, 0);
            r0 = make_row59(g0 + 3 * kTile);
            do_row(r1, r2, r0, 1);
            r1 = make_row59(g0 + 4 * kTile);
            do_row(r2, r0, r1, 2);
            if (nrows > 3) {
                r2 = make_row59(g0 + 5 * kTile);
                do_row(r0, r1, r2, 3);
            }

            // make the previous epilogue's staging writes visible to the bulk copy engine and
            // make sure the bulk store issued one task ago has finished reading its staging
            fence_proxy_async_smem();
            if (tid == 0) bulk_wait_read_all();
            named_barrier_sync(1, kThreads);  // stage free, counters complete, staging ready

            if (tid == 0) {
                if (prev_n >= 0)
                    bulk_store_s2g(reinterpret_cast<uint8_t*>(desc + (int64_t)prev_n * (64 * kBins)) +
                                       prev_half * kHalfDescBytes,
                                   staging0 + ((task - 1) & 1) * kHalfDescBytes, kHalfDescBytes);
                if (pn < n_rois) {
                    issue(pn, ph, stage);
                    if (ph == 1) pn = next_fast(pn + G);
                    ph ^= 1;
                }
                if (half == 0 && roi_status) roi_status[n] = LBP_OK;
            }
            // ---- epilogue: 32 cells x 59 bins of this half; quad o = (bin, cell row, cell x)
            // holds the 4 lane columns of the cell; bytes = the 4 row blocks.
            const uint32_t stg = staging0 + (task & 1) * kHalfDescBytes;
            for (int o = tid; o < kBins * kHalfCells; o += kThreads) {
                const uint32_t qa = hbuf + o * 16;
                const uint4 q = ld_shared_u32x4(qa);
                const uint32_t count = __dp4a(q.x + q.y + q.z + q.w, 0x01010101u, 0u);
                const int bin = o >> 5, cell = o & 31;
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(stg + (cell * kBins + bin) * 2),
                             "h"((uint16_t)count)
                             : "memory");
                st_shared_u32x4(qa, make_uint4(0, 0, 0, 0));
            }
            prev_n = n;
            prev_half = half;
            ++task;
            stage = (stage + 1 == kStages) ? 0 : stage + 1;
        }
    }
    // flush the last half descriptor
    fence_proxy_async_smem();
    named_barrier_sync(1, kThreads);
    if (tid == 0) {
        if (prev_n >= 0)
            bulk_store_s2g(reinterpret_cast<uint8_t*>(desc + (int64_t)prev_n * (64 * kBins)) +
                               prev_half * kHalfDescBytes,
                           staging0 + ((task - 1) & 1) * kHalfDescBytes, kHalfDescBytes);
        bulk_wait_all();
    }
}

inline bool encode_stack_map_rows(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                                  int elem, const lbp_images_t& g, int64_t pitch,
                                  int64_t img_stride, uint32_t box_rows) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.width, (cuuint64_t)g.height, (cuuint64_t)g.n_images};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * elem), (cuuint64_t)(img_stride * elem)};
    cuuint32_t box[3] = {(cuuint32_t)f59::kTile, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline cudaError_t launch_lbp_hist_fast59(const uint8_t* grey, const uint16_t* depth,
                                          const lbp_images_t& geom, const lbp_roi_t* rois,
                                          int32_t n_rois, const DepthWindow& win, uint16_t* desc,
                                          int32_t* roi_status, int sms, cudaStream_t stream) {
    CUtensorMap gm, dm;
    if (!encode_stack_map_rows(&gm, grey, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, geom, geom.grey_pitch,
                               geom.grey_img_stride, f59::kBoxRows))
        return cudaErrorNotSupported;
    if (depth) {
        if (!encode_stack_map_rows(&dm, depth, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, geom,
                                   geom.depth_pitch, geom.depth_img_stride, f59::kBoxRows))
            return cudaErrorNotSupported;
    } else {
        dm = gm;
    }
    auto kern = depth ? lbp_hist_fast59_kernel<true> : lbp_hist_fast59_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         f59::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(sms, n_rois));
    kern<<<grid, f59::kThreads, f59::kSmemBytes, stream>>>(gm, dm, grey, depth, geom, rois, n_rois,
                                                          win, desc, roi_status);
    return cudaGetLastError();
}

}  // namespace lbpf
