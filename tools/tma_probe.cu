// tma_probe.cu -- does a 3-D tiled TMA load accept an innermost start coordinate that is
// not 16-byte aligned?  Loads a 128x8 u8 box at x = 0, 16, 40, 47, 1 from a pitched
// 640-wide image and checks the bytes.  Each case runs in its own process (argv[1]).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__global__ void probe(const __grid_constant__ CUtensorMap map, int x, int y, uint8_t* out) {
    __shared__ alignas(128) uint8_t buf[128 * 8];
    __shared__ uint64_t bar;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(128 * 8));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((uint32_t)__cvta_generic_to_shared(buf)),
            "l"((uint64_t)&map), "r"(x), "r"(y), "r"(0), "r"(b)
            : "memory");
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(b));
    for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    int x = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 640, H = 64, P = 704;
    uint8_t* h = (uint8_t*)malloc(P * H);
    for (int i = 0; i < P * H; ++i) h[i] = (uint8_t)(i * 7 + (i / P) * 13);
    uint8_t *d, *o;
    cudaMalloc(&d, P * H);
    cudaMalloc(&o, 128 * 8);
    cudaMemcpy(d, h, P * H, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[3] = {W, H, 1};
    cuuint64_t strides[2] = {P, (cuuint64_t)P * H};
    cuuint32_t box[3] = {128, 8, 1}, es[3] = {1, 1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(
        &map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    probe<<<1, 128>>>(map, x, 3, o);
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t res[128 * 8];
    cudaMemcpy(res, o, sizeof(res), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int yy = 0; yy < 8; ++yy)
        for (int xx = 0; xx < 128; ++xx) bad += res[yy * 128 + xx] != h[(3 + yy) * P + x + xx];
    printf("x=%d encode=%d err=%s mismatches=%d\n", x, (int)r, cudaGetErrorString(e), bad);
    return 0;
}
