// synth_gen.cu -- GPU twin of synthgen/__init__.py (seeded synthetic inputs ONLY).
//
// Same integer recipe, bit for bit (checked by tests/test_synth_gpu.py), so
// that large benchmark batches (up to 2^20 crops = 51 GB) can be drawn in HBM
// without a host round trip.  Holds none of the method's arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t hash5(uint32_t seed, int64_t n, int64_t a, int64_t b,
                                          uint32_t salt) {
    uint32_t h = lowbias32(seed + 0x9E3779B9u * salt);
    h = lowbias32(h ^ (uint32_t)n);
    h = lowbias32(h ^ (uint32_t)a);
    h = lowbias32(h ^ (uint32_t)b);
    return h;
}

__device__ __forceinline__ int64_t value_noise(uint32_t seed, int64_t n, int64_t y, int64_t x,
                                               int shift, uint32_t mask, uint32_t salt) {
    const int64_t cell = 1ll << shift;
    const int64_t Y = y >> shift, X = x >> shift;
    const int64_t fy = y & (cell - 1), fx = x & (cell - 1);
    const int64_t v00 = hash5(seed, n, Y, X, salt) & mask;
    const int64_t v01 = hash5(seed, n, Y, X + 1, salt) & mask;
    const int64_t v10 = hash5(seed, n, Y + 1, X, salt) & mask;
    const int64_t v11 = hash5(seed, n, Y + 1, X + 1, salt) & mask;
    const int64_t acc = v00 * (cell - fx) * (cell - fy) + v01 * fx * (cell - fy) +
                        v10 * (cell - fx) * fy + v11 * fx * fy;
    return acc >> (2 * shift);
}

__global__ void synth_kernel(uint8_t* __restrict__ grey, uint16_t* __restrict__ depth, int64_t n_crops,
                             int32_t H, int32_t W, uint32_t seed, int64_t first, int32_t dist) {
    const int64_t total = n_crops * H * W;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = t % W, y = (t / W) % H, k = t / ((int64_t)W * H);
        const int64_t n = first + k;
        if (dist == 1) {  // constant
            grey[t] = 128;
            depth[t] = 1000;
            continue;
        }
        if (dist == 2) {  // iid noise
            grey[t] = (uint8_t)(hash5(seed, n, y, x, 8) & 255u);
            depth[t] = 1000;
            continue;
        }
        const int64_t v16 = value_noise(seed, n, y, x, 4, 255u, 1);
        const int64_t v4 = value_noise(seed, n, y, x, 2, 63u, 2);
        const int64_t base = 60 + (int64_t)(hash5(seed, n, 0, 0, 3) % 141u);
        int64_t g = base + (((v16 - 128) * 3) >> 2) + (v4 - 32);
        g = g < 0 ? 0 : (g > 255 ? 255 : g);
        grey[t] = (uint8_t)(g & ~3ll);

        const int64_t bg = 2000 + (int64_t)(hash5(seed, n, 0, 0, 4) % 1001u);
        const int64_t cx = W / 2 + (int64_t)(hash5(seed, n, 0, 0, 5) % (uint32_t)(W / 8 + 1)) - W / 16;
        const int64_t cy = H / 2 + (int64_t)(hash5(seed, n, 0, 0, 9) % (uint32_t)(H / 8 + 1)) - H / 16;
        const int64_t a = ((int64_t)W * 36) / 100, b = ((int64_t)H * 43) / 100;
        const int64_t a2 = a * a, b2 = b * b, R = a2 * b2;
        const int64_t fd = 900 + (int64_t)(hash5(seed, n, 0, 0, 6) % 201u);
        const int64_t dx = x - cx, dy = y - cy;
        const int64_t e = dx * dx * b2 + dy * dy * a2;
        const int64_t rn = W / 8 > 1 ? W / 8 : 1;
        const int64_t r2 = dx * dx + dy * dy;
        const int64_t relief = r2 < rn * rn ? 40 - (40 * r2) / (rn * rn) : 0;
        int64_t d = e <= R ? fd - relief : bg;
        const int64_t by = y / 3, bx = x / 3;
        const int64_t ecx = 3 * bx + 1 - cx, ecy = 3 * by + 1 - cy;
        const int64_t ec = ecx * ecx * b2 + ecy * ecy * a2;
        const int64_t diff = ec - R < 0 ? R - ec : ec - R;
        const int64_t p = diff * 100 < 15 * R ? 200 : 10;
        if ((int64_t)(hash5(seed, n, by, bx, 7) % 1000u) < p) d = 0;
        depth[t] = (uint16_t)d;
    }
}

}  // namespace

extern "C" int32_t synth_face_crops(uint8_t* grey, uint16_t* depth, int64_t n_crops, int32_t H,
                                    int32_t W, uint32_t seed, int64_t first_index, int32_t dist,
                                    void* stream) {
    if (!grey || !depth || n_crops < 0 || H < 1 || W < 1 || dist < 0 || dist > 2) return -1;
    if (n_crops == 0) return 0;
    const int64_t total = n_crops * H * W;
    const int threads = 256;
    const int64_t blocks64 = (total + threads - 1) / threads;
    const int blocks = (int)(blocks64 < 148 * 64 ? blocks64 : 148 * 64);
    synth_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(grey, depth, n_crops, H, W, seed,
                                                               first_index, dist);
    return cudaGetLastError() == cudaSuccess ? 0 : -6;
}
