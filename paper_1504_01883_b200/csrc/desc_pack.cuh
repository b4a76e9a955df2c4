// desc_pack.cuh -- descriptor compaction for the database all-gather (DESIGN.md
// R21; include/lbpfused.h lbp_desc_pack_u8 / lbp_desc_unpack_u8):
//   packed = min(count, 255) per entry, exceptions = (row, index, count) of counts > 255.
// Both directions are streaming, HBM-bound kernels (pack: 2 B read + 1 B written per entry;
// unpack: 1 B read + 2 B written): 8 entries per thread iteration (16-B u16 / 8-B u8
// vectors, evict-first loads and stores), grid-stride over a grid of 8 CTAs per SM.  The
// saturation is one VIMNMX.U16x2 per word and the narrowing one PRMT per 4 entries; the
// exception test is a single mask of the high bytes, so the rare slow path (a 16x16 cell
// whose 256 pixels share one bin) costs nothing when unused.
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace lbpf {

constexpr int kPackThreads = 256;
constexpr int kPackUnroll = 4;
static_assert(sizeof(lbp_desc_exc_t) == 16, "exception record layout (include/lbpfused.h)");

__device__ __forceinline__ void record_exception(uint32_t h, int64_t e, int32_t dim,
                                                 int64_t row_base, lbp_desc_exc_t* exc,
                                                 int32_t cap, int32_t* count) {
    const int32_t k = atomicAdd(count, 1);
    if (k < cap) {
        lbp_desc_exc_t x;
        x.row = row_base + e / dim;
        x.index = (int32_t)(e % dim);
        x.value = (int32_t)h;
        exc[k] = x;
    }
}

template <bool VEC>
__global__ void __launch_bounds__(kPackThreads)
desc_pack_u8_kernel(const uint16_t* __restrict__ desc, int64_t total, int32_t dim,
                    int64_t row_base, uint8_t* __restrict__ packed,
                    lbp_desc_exc_t* __restrict__ exc, int32_t cap, int32_t* __restrict__ count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tail = 0;
    if constexpr (VEC) {
        const int64_t n8 = total >> 3;
        auto one = [&](const uint4& w, int64_t v) {
            const uint32_t lo = prmt(__vminu2(w.x, 0x00FF00FFu), __vminu2(w.y, 0x00FF00FFu), 0x6420);
            const uint32_t hi = prmt(__vminu2(w.z, 0x00FF00FFu), __vminu2(w.w, 0x00FF00FFu), 0x6420);
            __stcs(reinterpret_cast<uint2*>(packed) + v, make_uint2(lo, hi));
            if ((w.x | w.y | w.z | w.w) & 0xFF00FF00u) {
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t h = (ws[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
                    if (h > 255u) record_exception(h, 8 * v + k, dim, row_base, exc, cap, count);
                }
            }
        };
        // kPackUnroll independent 16-B loads in flight per thread (bytes in flight for HBM)
        int64_t v = t;
        for (; v + (kPackUnroll - 1) * stride < n8; v += kPackUnroll * stride) {
            uint4 w[kPackUnroll];
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u)
                w[u] = __ldcs(reinterpret_cast<const uint4*>(desc) + v + u * stride);
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) one(w[u], v + u * stride);
        }
        for (; v < n8; v += stride) one(__ldcs(reinterpret_cast<const uint4*>(desc) + v), v);
        tail = n8 << 3;
    }
    for (int64_t e = tail + t; e < total; e += stride) {
        const uint32_t h = desc[e];
        packed[e] = (uint8_t)(h > 255u ? 255u : h);
        if (h > 255u) record_exception(h, e, dim, row_base, exc, cap, count);
    }
}

template <bool VEC>
__global__ void __launch_bounds__(kPackThreads)
desc_unpack_u8_kernel(const uint8_t* __restrict__ packed, int64_t total,
                      uint16_t* __restrict__ desc) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t tail = 0;
    if constexpr (VEC) {
        const int64_t n8 = total >> 3;
        auto one = [&](const uint2& b, int64_t v) {
            __stcs(reinterpret_cast<uint4*>(desc) + v,
                   make_uint4(prmt(b.x, 0u, 0x4140), prmt(b.x, 0u, 0x4342),
                              prmt(b.y, 0u, 0x4140), prmt(b.y, 0u, 0x4342)));
        };
        // (one load in flight per thread: the unrolled form measured slower for this
        // write-heavy direction)
        for (int64_t v = t; v < n8; v += stride)
            one(__ldcs(reinterpret_cast<const uint2*>(packed) + v), v);
        tail = n8 << 3;
    }
    for (int64_t e = tail + t; e < total; e += stride) desc[e] = packed[e];
}

// exceptions of n_lists lists (list l: exc + l * cap, min(counts[l], cap) valid records)
__global__ void __launch_bounds__(kPackThreads)
desc_exc_scatter_kernel(const lbp_desc_exc_t* __restrict__ exc,
                        const int32_t* __restrict__ counts, int32_t n_lists, int32_t cap,
                        int64_t row_base, int64_t n, int32_t dim, uint16_t* __restrict__ desc) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (int64_t)n_lists * cap;
         j += stride) {
        const int32_t l = (int32_t)(j / cap), k = (int32_t)(j - (int64_t)l * cap);
        if (k >= min(counts[l], cap)) continue;
        const lbp_desc_exc_t x = exc[j];
        const int64_t r = x.row - row_base;
        if (r < 0 || r >= n || x.index < 0 || x.index >= dim) continue;
        desc[r * dim + x.index] = (uint16_t)x.value;
    }
}

// Per-row compact form of lbp_extract_u8 (include/lbpfused.h) from a u16 descriptor: one warp
// per row, the entries' low bytes, the entries above 255 listed in the row's own record slots
// (warp-aggregated slot indices; the caller guarantees cap >= the row's count).
__global__ void __launch_bounds__(256)
desc_pack_rows_kernel(const uint16_t* __restrict__ desc, int64_t n, int32_t dim,
                      uint8_t* __restrict__ packed, int64_t pitch, int32_t* __restrict__ exc_n,
                      uint32_t* __restrict__ exc, int32_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n;
         row += warps) {
        const uint16_t* src = desc + row * dim;
        uint8_t* dst = packed + row * pitch;
        int32_t count = 0;
        for (int32_t d0 = 0; d0 < dim; d0 += 32) {
            const int32_t d = d0 + lane;
            const uint32_t v = d < dim ? src[d] : 0u;
            if (d < dim) dst[d] = (uint8_t)(v & 255u);
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, v > 255u);
            if (v > 255u) {
                const int32_t k = count + __popc(m & ((1u << lane) - 1u));
                if (k < cap) exc[row * cap + k] = ((uint32_t)d << 16) | v;
            }
            count += __popc(m);
        }
        if (lane == 0) exc_n[row] = count;
    }
}

}  // namespace lbpf
