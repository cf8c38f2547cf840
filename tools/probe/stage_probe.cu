// Probe: streaming bandwidth of the D3Q19 pull pattern (19 shifted row reads +
// 19 row writes per cell, (z, slot, y, x) layout) staged through shared memory
// by 1-D bulk copies (cp.async.bulk + mbarrier ring) against plain LDG pulls.
// Not product code: sizes the tile / stage ring of a bulk-staged k_fused.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stage_probe.cu -o stage_probe
//   ./stage_probe            (sweeps W, stages, CTAs/SM, element size)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__constant__ int c_cx[19] = {0, 0, 0, -1, 1, 0, 0, -1, 1, -1, 1, 0, 0, -1, 1, 0, 0, -1, 1};
__constant__ int c_cy[19] = {0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, -1, 0, 0, 1, -1, 0, 0};
__constant__ int c_cz[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, 1, 1, 1, -1, -1, -1, -1};

struct G { int nx, ny, nz, pitch, xoff; long long plane, zstride; };

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

template <typename T>
__device__ __forceinline__ T work(T acc, int n) {
    for (int k = 0; k < n; ++k) acc = acc * (T)0.999 + (T)1e-3;
    return acc;
}

// ---- bulk-staged: W cells per tile, CPT cells per consumer thread, S stages
template <typename T, int W, int CPT, int S>
__global__ void __launch_bounds__(W / CPT + 32) k_bulk(G g, const T* __restrict__ src, T* __restrict__ dst,
                                                       int ntiles, int nseg, int wk) {
    constexpr int M = 16 / sizeof(T);
    constexpr int SW = ((W + 2 * M) * sizeof(T) + 127) / 128 * 128 / sizeof(T);
    constexpr int NC = W / CPT;
    extern __shared__ __align__(128) unsigned char sm[];
    T* st = (T*)sm;
    uint64_t* full = (uint64_t*)(sm + (size_t)S * 19 * SW * sizeof(T));
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nmine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (tid >= NC) {
        const int lane = tid - NC;
        for (int k = 0; k < nmine; ++k) {
            const int s = k % S;
            if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
            const int t = blockIdx.x + k * gridDim.x;
            const int xs = t % nseg, r = t / nseg, y = r % g.ny, z = r / g.ny;
            if (lane == 0) mbar_expect(&full[s], 19 * (W + 2 * M) * sizeof(T));
            __syncwarp();
            if (lane < 19) {
                int ys = y - c_cy[lane]; ys = ys < 0 ? g.ny - 1 : (ys >= g.ny ? 0 : ys);
                int zs = z - c_cz[lane]; zs = zs < 0 ? g.nz - 1 : (zs >= g.nz ? 0 : zs);
                const T* p = src + zs * g.zstride + lane * g.plane + (long long)ys * g.pitch + g.xoff + xs * W - M;
                bulk_g2s(st + ((size_t)s * 19 + lane) * SW, p, (W + 2 * M) * sizeof(T), &full[s]);
            }
        }
        return;
    }
    for (int k = 0; k < nmine; ++k) {
        const int s = k % S;
        const int t = blockIdx.x + k * gridDim.x;
        const int xs = t % nseg, r = t / nseg, y = r % g.ny, z = r / g.ny;
        mbar_wait(&full[s], (k / S) & 1);
        T v[CPT][19];
#pragma unroll
        for (int c = 0; c < CPT; ++c)
#pragma unroll
            for (int i = 0; i < 19; ++i) v[c][i] = st[((size_t)s * 19 + i) * SW + M + c * NC + tid - c_cx[i]];
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            T acc = 0;
#pragma unroll
            for (int i = 0; i < 19; ++i) acc += v[c][i];
            acc = work(acc, wk);
            T* d = dst + z * g.zstride + (long long)y * g.pitch + g.xoff + xs * W + c * NC + tid;
#pragma unroll
            for (int i = 0; i < 19; ++i) d[i * g.plane] = v[c][i] + acc * (T)1e-30;
        }
    }
}

// ---- plain LDG pulls, one cell per thread, 128-thread blocks along x
template <typename T>
__global__ void __launch_bounds__(128) k_ldg(G g, const T* __restrict__ src, T* __restrict__ dst, int wk) {
    const int x = blockIdx.x * 128 + threadIdx.x, y = blockIdx.y, z = blockIdx.z;
    const T* o = src + z * g.zstride + (long long)y * g.pitch + g.xoff + x;
    T v[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) {
        int ys = y - c_cy[i]; ys = ys < 0 ? g.ny - 1 : (ys >= g.ny ? 0 : ys);
        int zs = z - c_cz[i]; zs = zs < 0 ? g.nz - 1 : (zs >= g.nz ? 0 : zs);
        v[i] = __ldg(src + zs * g.zstride + i * g.plane + (long long)ys * g.pitch + g.xoff + x - c_cx[i]);
    }
    (void)o;
    T acc = 0;
#pragma unroll
    for (int i = 0; i < 19; ++i) acc += v[i];
    acc = work(acc, wk);
    T* d = dst + z * g.zstride + (long long)y * g.pitch + g.xoff + x;
#pragma unroll
    for (int i = 0; i < 19; ++i) d[i * g.plane] = v[i] + acc * (T)1e-30;
}

template <typename T>
double run_ldg(G g, T* a, T* b, int wk) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dim3 grid(g.nx / 128, g.ny, g.nz);
    for (int r = 0; r < 3; ++r) k_ldg<T><<<grid, 128>>>(g, a, b, wk);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int R = 10;
    for (int r = 0; r < R; ++r) { k_ldg<T><<<grid, 128>>>(g, (r & 1) ? b : a, (r & 1) ? a : b, wk); }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return 2.0 * 19 * sizeof(T) * (double)g.nx * g.ny * g.nz / (ms / R * 1e-3) / 1e9;
}

template <typename T, int W, int CPT, int S>
double run_bulk(G g, T* a, T* b, int ctas_per_sm, int wk) {
    constexpr int M = 16 / sizeof(T);
    constexpr int SW = ((W + 2 * M) * sizeof(T) + 127) / 128 * 128 / sizeof(T);
    const size_t smem = (size_t)S * 19 * SW * sizeof(T) + 2 * S * 8;
    auto kern = k_bulk<T, W, CPT, S>;
    if (smem > 227 * 1024) return -1;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W / CPT + 32, smem));
    if (occ < ctas_per_sm) return -2;
    const int nseg = g.nx / W, ntiles = nseg * g.ny * g.nz;
    const int grid = 148 * ctas_per_sm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) kern<<<grid, W / CPT + 32, smem>>>(g, a, b, ntiles, nseg, wk);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int R = 10;
    for (int r = 0; r < R; ++r) kern<<<grid, W / CPT + 32, smem>>>(g, (r & 1) ? b : a, (r & 1) ? a : b, ntiles, nseg, wk);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return 2.0 * 19 * sizeof(T) * (double)g.nx * g.ny * g.nz / (ms / R * 1e-3) / 1e9;
}

template <typename T>
void sweep(const char* name) {
    G g;
    g.nx = 512; g.ny = 512; g.nz = sizeof(T) == 8 ? 256 : 512;
    g.pitch = g.nx + 2 * 128 / (int)sizeof(T);
    g.xoff = 128 / sizeof(T);
    g.plane = (long long)g.ny * g.pitch;
    g.zstride = 19 * g.plane;
    const size_t n = (size_t)g.zstride * g.nz + 4096;
    T *a, *b;
    CK(cudaMalloc(&a, n * sizeof(T))); CK(cudaMalloc(&b, n * sizeof(T)));
    CK(cudaMemset(a, 0, n * sizeof(T))); CK(cudaMemset(b, 0, n * sizeof(T)));
    for (int wk : {0, 40}) {
        printf("%s wk=%d ldg: %.0f GB/s\n", name, wk, run_ldg<T>(g, a, b, wk));
#define B(W, CPT, S, C) printf("%s wk=%d bulk W=%d cpt=%d S=%d ctas=%d: %.0f GB/s\n", name, wk, W, CPT, S, C, run_bulk<T, W, CPT, S>(g, a, b, C, wk))
        B(128, 1, 4, 4); B(128, 1, 6, 3);
        B(256, 1, 3, 2); B(256, 1, 4, 2); B(256, 2, 4, 2); B(256, 2, 6, 1);
        B(512, 2, 3, 1); B(512, 2, 4, 1); B(512, 4, 4, 1); B(512, 4, 5, 1);
#undef B
    }
    cudaFree(a); cudaFree(b);
}

int main() {
    sweep<float>("f32");
    sweep<double>("f64");
    return 0;
}
