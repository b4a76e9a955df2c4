// micro_smem_hist.cu -- microbenchmark of shared-memory histogram update
// strategies on B200 (informs the lbp_hist fast-path design).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro tools/micro_smem_hist.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kThreads = 512;

template <int MODE>
__global__ void __launch_bounds__(kThreads) micro(uint32_t* out, uint32_t seed) {
    __shared__ uint32_t h[64 * 64 + 64];
    for (int i = threadIdx.x; i < 64 * 64 + 64; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
    uint32_t acc = 0;
#pragma unroll 8
    for (int it = 0; it < kIters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t bin = x >> 26;  // 0..63
        if (MODE == 0) {  // baseline: no memory op
            acc += bin;
        } else if (MODE == 1) {  // ATOMS, [bin][lane]: distinct addresses, conflict-free banks
            atomicAdd(&h[bin * 32 + lane], 1u);
        } else if (MODE == 2) {  // ATOMS, [cell=lane][bin] stride 59: distinct addr, random banks
            atomicAdd(&h[lane * 59 + (bin % 59)], 1u);
        } else if (MODE == 3) {  // ATOMS, whole warp same address
            atomicAdd(&h[0], 1u);
        } else if (MODE == 4) {  // ATOMS, one cell's 64 bins shared by the warp (collisions)
            atomicAdd(&h[bin], 1u);
        } else if (MODE == 5) {  // RED (no return) [bin][lane]
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&h[bin * 32 + lane])));
        } else if (MODE == 6) {  // lane-private RMW (LDS+IADD+STS), dependent through smem
            h[bin * 32 + lane] += 1u;
        } else if (MODE == 7) {  // match_any aggregation into one cell's bins (warp-owned)
            const uint32_t m = __match_any_sync(0xFFFFFFFFu, bin);
            if (lane == __ffs(m) - 1) h[bin] += __popc(m);
        } else if (MODE == 8) {  // ATOMS [bin][lane] with 16-bit packed lanes (2 lanes per word)
            atomicAdd(&h[bin * 16 + (lane >> 1)], 1u << ((lane & 1) * 16));
        } else if (MODE == 9) {  // ATOMS, per-warp private [bin][lane] region (warp w offset)
            atomicAdd(&h[((threadIdx.x >> 5) & 1) * 2048 + bin * 32 + lane], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) acc += h[i];
    if (acc == 0x12345678u) out[0] = acc;  // keep everything live
}

template <int MODE>
float run(uint32_t* out, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    micro<MODE><<<blocks, kThreads>>>(out, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) micro<MODE><<<blocks, kThreads>>>(out, r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4;  // 4 x 512 threads = 64 warps per SM
    const double ops = (double)blocks * kThreads * kIters;  // thread-updates
    const char* names[] = {"baseline(no mem)", "ATOMS [bin][lane]", "ATOMS [lane][bin59]",
                           "ATOMS same-address", "ATOMS one-cell 64 bins", "RED [bin][lane]",
                           "LDS+IADD+STS private", "match_any aggregated", "ATOMS u16x2 packed",
                           "ATOMS 2 warp-private"};
    float t[10];
    t[0] = run<0>(out, blocks);
    t[1] = run<1>(out, blocks);
    t[2] = run<2>(out, blocks);
    t[3] = run<3>(out, blocks);
    t[4] = run<4>(out, blocks);
    t[5] = run<5>(out, blocks);
    t[6] = run<6>(out, blocks);
    t[7] = run<7>(out, blocks);
    t[8] = run<8>(out, blocks);
    t[9] = run<9>(out, blocks);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sms=%d clock(kHz)=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
    printf("%-26s %10s %14s %18s\n", "mode", "ms", "Gupd/s chip", "warp-upd/SM/cycle@1.9G");
    for (int m = 0; m < 10; ++m) {
        const double rate = ops / (t[m] * 1e-3);
        printf("%-26s %10.3f %14.1f %18.3f\n", names[m], t[m], rate / 1e9,
               rate / 32 / sms / 1.9e9);
    }
    return 0;
}
