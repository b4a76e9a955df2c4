// gather.cuh -- the fused database build (way 2; "online database generation",
// P:154): the extraction epilogue writes every descriptor row ONCE into the gathered training
// matrix of every rank -- through an NVLS multicast address (multimem.st: NVSwitch replicates
// the store to every rank's copy) or, without multicast, as one store per peer-mapped rank
// buffer (NVLink P2P) -- instead of a local write followed by an all-gather collective.
//
// Destination layout (lbp_gather_dst_t, include/lbpfused.h): at byte desc_offset of each
// destination base, rows of desc_pitch u16 (16-B aligned, entries past dim are zero); at
// labels_offset, int32 labels.  This rank's ROI n is global row row_base + n.  Every store is
// 16 B (rows) or 4 B (labels); the kernel ends with a system-scope fence and the caller runs
// a cross-rank barrier before reading other ranks' rows.
#pragma once
#include "common.cuh"

namespace lbpf {

__device__ __forceinline__ void multimem_st16(uint64_t addr, uint4 v) {
    // a multicast address: the NVSwitch replicates the store to every bound rank buffer
    // (SASS: STG.E.128.STRONG.SYS on the multicast range)
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void multimem_st4(uint64_t addr, uint32_t v) {
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_global16(uint64_t addr, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_global4(uint64_t addr, uint32_t v) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

// 16 B at byte offset `off` of every destination
__device__ __forceinline__ void gather_st16(const lbp_gather_dst_t& g, int64_t off, uint4 v) {
    if (g.mode == LBP_GATHER_MULTIMEM) {
        multimem_st16(g.base[0] + (uint64_t)off, v);
    } else {
#pragma unroll 1
        for (int r = 0; r < g.n_dst; ++r) st_global16(g.base[r] + (uint64_t)off, v);
    }
}
__device__ __forceinline__ void gather_st4(const lbp_gather_dst_t& g, int64_t off, uint32_t v) {
    if (g.mode == LBP_GATHER_MULTIMEM) {
        multimem_st4(g.base[0] + (uint64_t)off, v);
    } else {
#pragma unroll 1
        for (int r = 0; r < g.n_dst; ++r) st_global4(g.base[r] + (uint64_t)off, v);
    }
}

__device__ __forceinline__ int64_t gather_row_off(const lbp_gather_dst_t& g, int64_t row) {
    return g.desc_offset + (row + g.row_base) * g.desc_pitch * 2;
}

// Chunks [c0, c1) (c1 < 0: to the end of the padded row) of the row of ROI n from a 16-B
// aligned shared-memory staging buffer of `chunks16` chunks (the lane kernel's epilogue), by
// the t-th of NT threads; pad chunks up to desc_pitch are zero.
template <int NT>
__device__ __forceinline__ void gather_row_from_smem(const lbp_gather_dst_t& g, int64_t n,
                                                     uint32_t staging, int c0, int c1,
                                                     int chunks16, int t) {
    const int64_t base = gather_row_off(g, n);
    const int total = c1 < 0 ? (int)(g.desc_pitch / 8) : c1;
    for (int c = c0 + t; c < total; c += NT) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (c < chunks16)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(staging + 16 * c));
        gather_st16(g, base + 16 * c, v);
    }
}

// Row of ROI n from a u16 global row of `dim` entries (any alignment), zero padded.
template <int NT>
__device__ __forceinline__ void gather_row_from_global(const lbp_gather_dst_t& g, int64_t n,
                                                       const uint16_t* src, int32_t dim, int t) {
    const int64_t base = gather_row_off(g, n);
    const int total = (int)(g.desc_pitch / 8);
    for (int c = t; c < total; c += NT) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = 8 * c + 2 * k;
            const uint32_t lo = e < dim ? src[e] : 0u, hi = e + 1 < dim ? src[e + 1] : 0u;
            w[k] = lo | (hi << 16);
        }
        gather_st16(g, base + 16 * c, make_uint4(w[0], w[1], w[2], w[3]));
    }
}

__device__ __forceinline__ void gather_label(const lbp_gather_dst_t& g, int64_t n,
                                             const int32_t* labels) {
    if (labels && g.labels_offset >= 0)
        gather_st4(g, g.labels_offset + 4 * (n + g.row_base), (uint32_t)labels[n]);
}

// Fallback when the extraction ran in its own kernel (geometries off the TMA fast path, small
// batches): forward the local rows to every destination.  One warp per row.
__global__ void __launch_bounds__(256)
lbp_gather_forward_kernel(const uint16_t* __restrict__ scratch, int32_t n_rois, int32_t dim,
                          const int32_t* __restrict__ labels, lbp_gather_dst_t g) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int n_warps = (gridDim.x * blockDim.x) >> 5;
    for (int64_t n = warp; n < n_rois; n += n_warps) {
        gather_row_from_global<32>(g, n, scratch + n * dim, dim, lane);
        if (lane == 0) gather_label(g, n, labels);
    }
    __threadfence_system();  // the stores before the caller's cross-rank barrier
}

}  // namespace lbpf
