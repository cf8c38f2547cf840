// Vectorised fused sweep (k_fused_vec): V consecutive cells of a row per
// thread, every pull one aligned V-wide load along x.
//
// Same step and arithmetic as k_fused (pull -> bounce-back -> collide,
// G-form).  For direction i a thread loads the UNSHIFTED V-cell group of the
// source row (slot i, row y - cy_i, plane z - cz_i) as one 64/128-bit load;
// the x shift of the pull (-cx_i) is a warp shuffle of the group edge
// (__shfl_up / __shfl_down), and only lane 0 / lane 31 (or a lane whose
// neighbour is past the row end) loads the one element outside the warp's
// groups.  Per V cells that is Q vector loads + 2 x (directions with
// c_x != 0) single-lane loads instead of V Q scalar loads, and one address
// computation per direction instead of V.  Links, typed corrections,
// collision and stores stay per cell (pull_finish / collide_any), and warps
// on a periodic edge take the scalar index-wrap path.
//
// Status: bitwise correct (GPU parity suite) but slower than the scalar
// kernel on B200, so it is compiled only into variant libraries
// (-DLBM_VEC_VARIANT).  Measured (fraction of the HBM roofline, scalar
// kernel in brackets): config 4 fp64 0.73 (0.92), config 4 fp32 0.73 (0.88),
// config 2 0.78 (0.85); per-cell scalar stores instead of V-wide stores
// 0.64 / 0.62 / 0.68 (half-written sectors); register caps of 3 or 5
// blocks/SM instead of 4/6 lower still.  Holding V cells' populations costs
// occupancy and spills that the saved load instructions do not repay - the
// scalar kernel's 19 loads per thread already saturate HBM in fp64.
#pragma once
#include "lbm_kernels.cuh"

namespace lbm {

#ifndef LBM_VEC_WIDTH
#define LBM_VEC_WIDTH 2
#endif

template <typename Real, int V>
struct VecT;
template <>
struct VecT<double, 2> {
    using T = double2;
};
template <>
struct VecT<float, 2> {
    using T = float2;
};
template <>
struct VecT<float, 4> {
    using T = float4;
};
template <>
struct VecT<uint32_t, 2> {
    using T = uint2;
};
template <>
struct VecT<uint32_t, 4> {
    using T = uint4;
};

template <typename Real, int V>
__device__ __forceinline__ void vload(const Real* p, Real (&out)[V]) {
    using VT = typename VecT<Real, V>::T;
    const VT v = __ldg(reinterpret_cast<const VT*>(p));
    out[0] = v.x;
    out[1] = v.y;
    if constexpr (V == 4) {
        out[2] = v.z;
        out[3] = v.w;
    }
}

template <int Q, typename Real, int MODEL>
constexpr int vec_minb() {
#ifdef LBM_VEC_MINB
    return LBM_VEC_MINB;
#else
    if constexpr (std::is_same_v<Real, double>) return Q == 19 ? 4 : 2;
    else return MODEL == 3 ? 4 : 6;
#endif
}

template <int Q, typename Real, int MODEL, int FORCE, int V>
__global__ void __launch_bounds__(128, vec_minb<Q, Real, MODEL>())
    k_fused_vec(KGrid g, KParams p, const Real* __restrict__ src, Real* __restrict__ dst,
                const uint32_t* __restrict__ cellmask, const uint32_t* __restrict__ typemask,
                int z0) {
    using D = Dirs<Q>;
    using Acc = AccOf<Real>;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * V;
    const int y = blockIdx.y;
    const int z = z0 + blockIdx.z;
    const int xw0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * V;
    const bool edge_x = g.wrap_x && (xw0 == 0 || xw0 + 32 * V >= g.nx);
    const bool edge_y = g.wrap_y && (y == 0 || y == g.ny - 1);
    const bool edge_z = (g.zlo == LBM_ZFACE_WRAP && z == 0) || (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1);
    const bool active = x0 < g.nx;   // the launcher requires nx % V == 0
    const int64_t cell0 = ((int64_t)z * g.ny + y) * g.nx + x0;
    uint32_t code[V];
    if (active) {
        vload<uint32_t, V>(cellmask + cell0, code);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) code[j] = 0u;
    }
    if (edge_x || edge_y || edge_z) {   // warp-uniform: index wrap, per cell
        if (!active) return;
#pragma unroll 1
        for (int j = 0; j < V; ++j) {
            const uint32_t cj = __ldg(cellmask + cell0 + j);   // (no dynamic index into code[])
            Acc f[Q];
            pull_cell<Q, Real, Acc, 0>(g, p, src, x0 + j, y, z, cj, typemask, true, f);
            if (cj & LBM_MASK_FLUID) collide_any<Q, MODEL, FORCE>(f, p, cell0 + j);
            Real* dp = opaque(dst + lidx(g, z, 0, y, x0 + j));
            static_for<0, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                store_any<Q, i>(dp + g.dslot[i], f[i]);
            });
        }
        return;
    }
    // all lanes stay for the shuffles; inactive lanes load nothing
    const Real* sp = opaque(src + lidx(g, z, 0, y, x0));
    const bool lo_direct = lane == 0 || x0 == 0;
    const bool hi_direct = lane == 31 || x0 + V >= g.nx;
    Real raw[V][Q];
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        constexpr int cx = D::cx[i];
        const Real* rowp = sp + (g.dpull[i] + cx);   // the group's own x, source row of i
        Real L[V];
        if (active) {
            vload<Real, V>(rowp, L);
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j) L[j] = Real(0);
        }
        if constexpr (cx == 0) {
#pragma unroll
            for (int j = 0; j < V; ++j) raw[j][i] = L[j];
        } else if constexpr (cx == 1) {   // source x - 1
            Real prev = __shfl_up_sync(FULL, L[V - 1], 1);
            if (lo_direct && active) prev = __ldg(rowp - 1);
            raw[0][i] = prev;
#pragma unroll
            for (int j = 1; j < V; ++j) raw[j][i] = L[j - 1];
        } else {                          // source x + 1
            Real next = __shfl_down_sync(FULL, L[0], 1);
            if (hi_direct && active) next = __ldg(rowp + V);
            raw[V - 1][i] = next;
#pragma unroll
            for (int j = 0; j < V - 1; ++j) raw[j][i] = L[j + 1];
        }
    });
    if (!active) return;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        // bounce-back links: the own cell's opposite direction
        static_for<1, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            constexpr int k = D::opp[i];
            if ((code[j] >> i) & 1u) raw[j][i] = __ldg(sp + j + g.dslot[k]);
        });
    }
    Acc f[V][Q];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int x = x0 + j;
        const int64_t own = lidx(g, z, 0, y, x);
        uint2 tm = make_uint2(0u, 0u);
        if (code[j] & (LBM_MASK_UBB | LBM_MASK_PRESSURE))
            tm = __ldg(reinterpret_cast<const uint2*>(typemask) + cell0 + j);
        pull_finish<Q, Real, Acc, 0>(g, p, src, x, y, z, own, code[j], tm, raw[j], f[j]);
        if (code[j] & LBM_MASK_FLUID) collide_any<Q, MODEL, FORCE>(f[j], p, cell0 + j);
    }
    // V-wide stores: per-cell scalar stores would leave every sector half
    // written per instruction (measured: 0.64 of the roofline on config 4)
    Real* dp = opaque(dst + lidx(g, z, 0, y, x0));
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        Real o[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            if constexpr (std::is_same_v<Acc, double> && std::is_same_v<Real, float>)
                o[j] = (float)(f[j][i] - wt<Q, i>());
            else
                o[j] = (Real)f[j][i];
        }
        using VT = typename VecT<Real, V>::T;
        VT v;
        v.x = o[0];
        v.y = o[1];
        if constexpr (V == 4) {
            v.z = o[2];
            v.w = o[3];
        }
        *reinterpret_cast<VT*>(dp + g.dslot[i]) = v;
    });
}

}  // namespace lbm
