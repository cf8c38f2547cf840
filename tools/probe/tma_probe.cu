// Standalone probe of the TMA building blocks used by k_fused_tma
// (tensor-map encode via the driver entry point, mbarrier, 3-D box load).
// Usage: tma_probe <bits>: 1 prefetch.tensormap, 4 descriptor in global
// memory, 8 fp32 element type, 16 no L2 promotion, 64 encode through the
// versioned entry point, 128 box of 16 elements, 256 16-byte aligned start.
// versioned entry point, 128 box of 16 elements.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>

typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, void* out,
                      int bytes, int c0, int c1, int c2, int variant) {
    __shared__ __align__(1024) double buf[128];
    __shared__ __align__(8) uint64_t bar;
    const CUtensorMap* m = (variant & 4) ? gmap : &map;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (variant & 1)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(buf)),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar)),
        "r"(0)
        : "memory");
    if (threadIdx.x * 8 < bytes) ((double*)out)[threadIdx.x] = buf[threadIdx.x];
}

int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    const bool f32 = variant & 8;
    const int es = f32 ? 4 : 8;
    const int pitch = 32, Y = 10, Zq = 19 * 8;
    size_t n = (size_t)pitch * Y * Zq;
    char* h = (char*)malloc(n * 8);
    for (size_t i = 0; i < n; ++i) {
        if (f32) ((float*)h)[i] = (float)i; else ((double*)h)[i] = (double)i;
    }
    void *d, *o;
    CUtensorMap* gm;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 128 * 8);
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(d, h, n * es, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (variant & 64)
        cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    else
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (!fn) { printf("no entry point\n"); return 1; }
    int bw = (variant & 128) ? 16 : 10;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)Y, (cuuint64_t)Zq};
    cuuint64_t str[2] = {(cuuint64_t)pitch * es, (cuuint64_t)pitch * Y * es};
    cuuint32_t box[3] = {(cuuint32_t)bw, 1, 1}, est[3] = {1, 1, 1};
    CUresult r = ((enc_t)fn)(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             3, d, dims, str, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE,
                             (variant & 16) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
    int c0 = (variant & 256) ? 14 : 15, c1 = 3, c2 = 40;
    probe<<<1, 128>>>(map, gm, o, bw * es, c0, c1, c2, variant);
    cudaError_t e = cudaDeviceSynchronize();
    char ho[1024];
    cudaMemcpy(ho, o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < bw; ++i) {
        int x = c0 + i;
        double want = x < pitch ? (double)(((size_t)c2 * Y + c1) * pitch + x) : 0.0;
        double got = f32 ? ((float*)ho)[i] : ((double*)ho)[i];
        if (got != want) bad++;
    }
    printf("variant %3d: encode=%d kernel=%s data=%s\n", variant, (int)r, cudaGetErrorString(e),
           bad ? "MISMATCH" : "ok");
    return e != cudaSuccess || bad;
}
