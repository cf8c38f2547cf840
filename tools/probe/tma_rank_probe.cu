// Probe: tensor TMA of rank 1/2/3, fp32, 64-element box; descriptor by value.
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

__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int rank) {
    __shared__ __align__(1024) float buf[64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(256) : "memory");
        uint64_t d = reinterpret_cast<uint64_t>(&map);
        if (rank == 1)
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                         ::"r"(su32(buf)), "l"(d), "r"(64), "r"(su32(&bar)) : "memory");
        else if (rank == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"(d), "r"(0), "r"(1), "r"(su32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(buf)), "l"(d), "r"(0), "r"(1), "r"(1), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(su32(&bar)), "r"(0) : "memory");
    out[threadIdx.x] = buf[threadIdx.x];
}

int main(int argc, char** argv) {
    int rank = argc > 1 ? atoi(argv[1]) : 1;
    const int n = 64 * 4 * 4;
    float h[n];
    for (int i = 0; i < n; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 1024);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    printf("entry: %s q=%d fn=%p\n", cudaGetErrorString(ge), (int)q, fn);
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    cuuint64_t dims[3] = {256, 4, 1};
    cuuint64_t str[2] = {1024, 4096};
    if (rank == 2) { dims[0] = 64; dims[1] = 16; str[0] = 256; }
    if (rank == 3) { dims[0] = 64; dims[1] = 4; dims[2] = 4; str[0] = 256; str[1] = 1024; }
    cuuint32_t box[3] = {64, 1, 1}, est[3] = {1, 1, 1};
    CUresult r = ((enc_t)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, est,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 64>>>(map, o, rank);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[64];
    cudaMemcpy(ho, o, 256, cudaMemcpyDeviceToHost);
    float want0 = rank == 1 ? 64 : (rank == 2 ? 64 : 64 + 256);
    printf("rank %d: encode=%d kernel=%s first=%g want %g\n", rank, (int)r, cudaGetErrorString(e), ho[0], want0);
    return 0;
}
