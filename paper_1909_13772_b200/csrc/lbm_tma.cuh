// TMA-staged fused sweep for sm_100a (k_fused_tma).
//
// Same step as k_fused (pull -> bounce-back -> collide, G-form in and out,
// identical arithmetic), but the pulls do not go through the LSU: for every
// tile of 128 cells of one (y, z) row a producer warp issues one TMA box
// load per direction i - the row segment shifted by -c_i, taken from slot i
// of plane z - cz_i (cp.async.bulk.tensor.3d over the field viewed as
// (x, y, q*(z+2)) rows) - into a shared-memory stage, completing on an
// mbarrier.  Consumer warps read their cell's Q values from the stage
// (conflict-free: lane-contiguous), release the stage, and compute while the
// producer already streams the next tiles: memory-level parallelism comes
// from the stage ring, not from occupancy, and a pull costs one LDS instead
// of an address computation plus an LDG.
//
// What the boxes cannot express goes through the LDG path of lbm_kernels.cuh:
//   * bounce-back links (the own cell's opposite direction), per lane;
//   * warps touching a periodic edge owned by this rank (index wrap);
//   * UBB / Pressure corrections (pull_finish).
// Non-periodic ghosts and halo planes are read raw by the boxes, exactly as
// the reference's uncovered / exchanged ghost cells.
//
// Status: correct (the whole GPU parity suite passes bitwise with it) but
// slower than the LDG kernel on B200, so it is only compiled into variant
// libraries (-DLBM_TMA_VARIANT; LBM_B200_FUSED=ldg|tma picks at run time).
// Measured (MLUPS, fraction of the HBM roofline; LDG kernel in brackets):
//   config 4 fp64  11.9k 0.55 (19.9k 0.92)   without the edge path 14.4k
//   config 4 fp32  21.4k 0.50 (37.7k 0.88)
//   config 2       18.8k 0.62 (25.9k 0.85)
// Hardware facts learnt on the way: a box must start 16-byte aligned and
// land 128-byte aligned in shared memory (else "illegal instruction" /
// "misaligned address"), hence the aligned windows; prefetching the next
// tile's cell mask did not help.  One-row boxes (~1 KB) appear to be the
// limit: 19-27 TMA ops per 128 cells.  Next attempt: multi-row boxes.
#pragma once
#include <cuda.h>

#include "lbm_kernels.cuh"

namespace lbm {

constexpr int kTmaW = 128;         // cells per tile = consumer threads per CTA
constexpr int kTmaThreads = kTmaW + 32;   // + one producer warp

template <typename Real>
constexpr int tma_stages() {
#ifdef LBM_TMA_STAGES
    return LBM_TMA_STAGES;
#else
    return sizeof(Real) == 8 ? 2 : 3;
#endif
}

// A TMA box must start on a 16-byte boundary (a misaligned start faults with
// "illegal instruction" on B200, measured), so every direction loads the
// same aligned window [x0 - A, x0 + 128 + A) with A = 16 bytes of cells and
// a lane picks its shifted element inside it.
template <typename Real>
constexpr int tma_margin() {
    return 16 / (int)sizeof(Real);
}
template <typename Real>
constexpr int tma_stride() {   // elements per direction in a stage (each box
                               // destination 128-byte aligned, also required)
    constexpr int line = 128 / (int)sizeof(Real);
    return (kTmaW + 2 * tma_margin<Real>() + line - 1) / line * line;
}

template <int Q, typename Real>
constexpr int tma_smem_bytes() {
    return tma_stages<Real>() * Q * tma_stride<Real>() * (int)sizeof(Real) + 2 * tma_stages<Real>() * 8;
}

// resident CTAs per SM the shared-memory ring allows (228 KB per SM, 1 KB
// reserved per CTA), capped at 8
template <int Q, typename Real>
constexpr int tma_minb() {
    constexpr int m = 233472 / (tma_smem_bytes<Q, Real>() + 1024);
    return m > 8 ? 8 : (m < 1 ? 1 : m);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// warps on a periodic edge: the LDG pull with index wrap, out of line so the
// common path keeps its registers
template <int Q, typename Real, typename Acc>
__device__ __noinline__ void pull_generic(const KGrid& g, const KParams& p,
                                          const Real* __restrict__ src, int x, int y, int z,
                                          uint32_t code, const uint32_t* __restrict__ typemask,
                                          Acc (&f)[Q]) {
    pull_cell<Q, Real, Acc, 0>(g, p, src, x, y, z, code, typemask, true, f);
}

// tile -> (x tile, row y, plane z)
struct TmaTile {
    int xt, y, z;
};
__device__ __forceinline__ TmaTile tma_tile(uint32_t tile, uint32_t nxt, uint32_t ny, int z0) {
    TmaTile t;
    const uint32_t r = tile / nxt;
    t.xt = (int)(tile - r * nxt);
    const uint32_t zz = r / ny;
    t.y = (int)(r - zz * ny);
    t.z = z0 + (int)zz;
    return t;
}

// Persistent: CTA b processes tiles b, b + gridDim.x, ... (consecutive CTAs
// hold neighbouring row segments at any time, like the plain grid order).
// bw: box width in cells: the 128-cell tile (or nx rounded up to 16 bytes
// when narrower) plus the two margins.
template <int Q, typename Real, int MODEL, int FORCE>
__global__ void __launch_bounds__(kTmaThreads, tma_minb<Q, Real>())
    k_fused_tma(const __grid_constant__ CUtensorMap tmap, KGrid g, KParams p,
                const Real* __restrict__ src, Real* __restrict__ dst,
                const uint32_t* __restrict__ cellmask, const uint32_t* __restrict__ typemask,
                int z0, int nxt, int64_t ntiles, int bw) {
    using D = Dirs<Q>;
    constexpr int S = tma_stages<Real>();
    constexpr int A = tma_margin<Real>();
    constexpr int SW = tma_stride<Real>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Real* stage = reinterpret_cast<Real*>(smem_raw);  // [S][Q][SW]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + S * Q * SW * sizeof(Real));
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTmaW / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int nmine = first < ntiles ? (int)((ntiles - 1 - first) / stride + 1) : 0;

    if (warp == kTmaW / 32) {
        // ---- producer: one elected lane streams the tiles into the ring
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                         : "memory");
            for (int k = 0; k < nmine; ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
                const TmaTile t = tma_tile((uint32_t)(first + (int64_t)k * stride), nxt, g.ny, z0);
                mbar_expect_tx(&full[s], Q * bw * sizeof(Real));
                Real* dstage = stage + (size_t)s * Q * SW;
                static_for<0, Q>([&](auto I_) {
                    constexpr int i = decltype(I_)::value;
                    constexpr int cy = D::cy[i], cz = D::cz[i];
                    constexpr int slot = slot_of<Q>(i);
                    tma_load_3d(dstage + i * SW, &tmap, &full[s], g.xoff + t.xt * kTmaW - A,
                                1 + t.y - cy, (t.z + 1 - cz) * Q + slot);
                });
            }
        }
        return;
    }

    // ---- consumers: one cell per thread per tile
    using Acc = AccOf<Real>;
    // the cell mask of the next tile is loaded one iteration ahead (it gates
    // the link loads and would otherwise put a DRAM latency on every tile)
    auto mask_of = [&](int kk) -> uint32_t {
        if (kk >= nmine) return 0u;
        const TmaTile u = tma_tile((uint32_t)(first + (int64_t)kk * stride), nxt, g.ny, z0);
        const int xx = u.xt * kTmaW + tid;
        return xx < g.nx ? __ldg(cellmask + ((int64_t)u.z * g.ny + u.y) * g.nx + xx) : 0u;
    };
    uint32_t code_next = mask_of(0);
    for (int k = 0; k < nmine; ++k) {
        const int s = k % S;
        const TmaTile t = tma_tile((uint32_t)(first + (int64_t)k * stride), nxt, g.ny, z0);
        const int x = t.xt * kTmaW + tid;
        const int y = t.y, z = t.z;
        const bool active = x < g.nx;
        const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
        const uint32_t code = code_next;
        code_next = mask_of(k + 1);
        const int xw0 = t.xt * kTmaW + (tid & ~31);
        const bool edge_x = g.wrap_x && (xw0 == 0 || xw0 + 32 >= g.nx);
        const bool edge_y = g.wrap_y && (y == 0 || y == g.ny - 1);
        const bool edge_z =
            (g.zlo == LBM_ZFACE_WRAP && z == 0) || (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1);
        const bool generic = edge_x || edge_y || edge_z;
        mbar_wait(&full[s], (k / S) & 1);
        Real raw[Q];
        const Real* sst = stage + (size_t)s * Q * SW + A + tid;
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            constexpr int cx = D::cx[i];
            raw[i] = sst[i * SW - cx];
        });
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (!active) continue;
        Acc f[Q];
#ifdef LBM_TMA_NO_GENERIC
        if (false) {   // timing experiment only: wrong at periodic edges
#else
        if (generic) {
#endif
            // only this array's address escapes to the out-of-line call; f
            // itself stays in registers
            Acc fg[Q];
            pull_generic<Q, Real, Acc>(g, p, src, x, y, z, code, typemask, fg);
            static_for<0, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                f[i] = fg[i];
            });
        } else {
            const int64_t own = lidx(g, z, 0, y, x);
            const Real* sp = opaque(src + own);
            static_for<1, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                if ((code >> i) & 1u) raw[i] = __ldg(sp + g.dlink[i]);
            });
            uint2 tm = make_uint2(0u, 0u);
            if (code & (LBM_MASK_UBB | LBM_MASK_PRESSURE))
                tm = __ldg(reinterpret_cast<const uint2*>(typemask) + cell);
            pull_finish<Q, Real, Acc, 0>(g, p, src, x, y, z, own, code, tm, raw, f);
        }
        if (code & LBM_MASK_FLUID) collide_any<Q, MODEL, FORCE>(f, p, cell);
        Real* dp = opaque(dst + lidx(g, z, 0, y, x));
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            store_any<Q, i>(dp + g.dslot[i], f[i]);
        });
    }
}

}  // namespace lbm
