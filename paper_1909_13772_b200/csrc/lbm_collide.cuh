// Per-cell collision, fp64 registers, reference op order.
//
// Mirrors impl.collide (/root/reference/pkg/src/blocksim/_kernels/_core_py.py:70-200)
// expression by expression: every value is rounded separately (the fp64
// translation unit is compiled with -fmad=false) and reductions run in the
// same fixed direction order, so the result is bitwise identical to the numpy
// kernel.  Value-safe restatements (validated bitwise, see tests/):
//   * c_a * f with c_a = +-1 becomes +-f, zero-velocity terms are skipped
//     (x + (+-0) == x for the non-zero values the populations take);
//   * TRT pairs (i, opp(i)) share f+ / feq+ and negate f- / feq- (exact);
//   * the equilibrium of opp(i) reuses 3cu and (4.5cu)cu with cu -> -cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "lbm_stencil.cuh"

namespace lbm {

// kernel-side copy of lbm_params_t (by value in the launch)
struct KParams {
    double rem, hw;               // SRT
    double omega_e, omega_o;      // TRT
    double he_half, ho_half;      // TRT Guo weights
    double fx, fy, fz;            // body force
    double sfx, sfy, sfz;         // 0.5 F (Guo) or tau F (SimpleShift)
    double ubb[27];               // per link direction k
    double pw[27];                // (2 w_k) rho_w, Pressure links
    // fp32-storage path: the same constants rounded once on the host
    float frem, fhw, fomega_e, fomega_o, fhe_half, fho_half;
    float ffx, ffy, ffz, fsfx, fsfy, fsfz;
    float fubb[27];
    // fp32 TRT Guo pair constants: fcF = c_i . F, fguo_p = he_half 6 w_i
    // (fguo_p[0] = 2 he_half 3 w_0), fguo_q = ho_half 6 w_i (c_i . F)
    float fcF[27], fguo_p[27], fguo_q[27];
    int mrt_fast;                 // fp32 D3Q27 MRT: factorised raw-moment form
    const double* omega;          // SRT per-cell rates (nz, ny, nx), model 4
    // moving-body walls (lbm_moving_t), read only on cells with LBM_MASK_MOVING
    const int* mv_owner;          // (nz+2, ny+2, nx+2) body slot or -1
    const uint32_t* mv_link;      // (nz, ny, nx) pulled directions from covered cells
    const double* mv_bodies;      // (blocks * slots, 9) p, v, omega per block's copy
    const double* mv_cell0;       // (blocks, 3) first-cell centres
    double* mv_forces;            // (blocks * slots, 6) force, torque accumulators
    int mv_slots, mv_bx, mv_by, mv_cx, mv_cy, mv_cz;
    double mv_rho0;
    // fused z-face halo (lbm_fused_step_peer): the z-block (all q slots) of
    // the lower / upper neighbour's receiving ghost plane, in its own memory
    // (same device, or a peer GPU's HBM mapped over NVLink); NULL otherwise
    void* peer_lo;
    void* peer_hi;
};

// MRT tables in constant memory: M, Minv, S, G (q <= 27).  One private copy
// per translation unit (no -rdc) and per device (constant memory belongs to
// the device's context); each unit exposes a setter that uploads only when
// the device does not already hold the same content (tables are per model,
// not per step).  The record of what each device holds is keyed by the
// current device and guarded by a mutex, so rank threads driving different
// GPUs (or one GPU) never skip an upload they need.  Captured CUDA graphs
// do not capture constant memory: lbm_bind_params re-runs the setter before
// a replay.
#define LBM_MRT_MAXQ 27
static __constant__ double c_mrt_M[LBM_MRT_MAXQ * LBM_MRT_MAXQ];
static __constant__ double c_mrt_Minv[LBM_MRT_MAXQ * LBM_MRT_MAXQ];
static __constant__ double c_mrt_S[LBM_MRT_MAXQ];
static __constant__ double c_mrt_G[LBM_MRT_MAXQ * LBM_MRT_MAXQ];

// per-device record of the last uploaded table content (+ one derived int)
struct DeviceTableCache {
    std::mutex mu;
    std::vector<std::vector<double>> content;  // indexed by device ordinal
    std::vector<int> derived;
    // true (and *derived_out set) when device `dev` already holds `tables`
    bool hit(int dev, const double* tables, size_t n, int* derived_out) {
        if ((size_t)dev >= content.size()) {
            content.resize(dev + 1);
            derived.resize(dev + 1, 0);
        }
        const std::vector<double>& c = content[dev];
        if (c.size() != n || memcmp(c.data(), tables, n * sizeof(double)) != 0) return false;
        if (derived_out) *derived_out = derived[dev];
        return true;
    }
    void store(int dev, const double* tables, size_t n, int d) {
        content[dev].assign(tables, tables + n);
        derived[dev] = d;
    }
};

// tables: M[q*q] Minv[q*q] S[q] G[q*q] (G may be absent: pass zeros)
#define LBM_DEFINE_MRT_SETTER(NAME)                                                       \
    cudaError_t NAME(int q, const double* tables, cudaStream_t s) {                       \
        static DeviceTableCache cache;                                                    \
        const size_t n = (size_t)3 * q * q + q;                                           \
        int dev = 0;                                                                      \
        cudaError_t e = cudaGetDevice(&dev);                                              \
        if (e != cudaSuccess) return e;                                                   \
        std::lock_guard<std::mutex> lock(cache.mu);                                       \
        if (cache.hit(dev, tables, n, nullptr)) return cudaSuccess;                       \
        const size_t qq = (size_t)q * q * sizeof(double);                                 \
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_M, tables, qq, 0,                          \
                                         cudaMemcpyHostToDevice, s)) != cudaSuccess)       \
            return e;                                                                     \
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_Minv, tables + q * q, qq, 0,               \
                                         cudaMemcpyHostToDevice, s)) != cudaSuccess)       \
            return e;                                                                     \
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_S, tables + 2 * q * q, q * sizeof(double), \
                                         0, cudaMemcpyHostToDevice, s)) != cudaSuccess)    \
            return e;                                                                     \
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_G, tables + 2 * q * q + q, qq, 0,          \
                                         cudaMemcpyHostToDevice, s)) != cudaSuccess)       \
            return e;                                                                     \
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;                      \
        cache.store(dev, tables, n, 0);                                                   \
        return cudaSuccess;                                                               \
    }

// term c * u for c in {-1, 0, 1}, appended to a left-assoc sum
template <int C, typename T>
__device__ __forceinline__ T add_cu(T acc, T u, bool& started) {
    if constexpr (C == 1) {
        if (started) return acc + u;
        started = true;
        return u;
    } else if constexpr (C == -1) {
        if (started) return acc - u;
        started = true;
        return -u;
    } else {
        return acc;
    }
}

// cu_i = (cx ux + cy uy) + cz uz with zero terms dropped (_core_py.py:127)
template <int Q, int I, typename T = double>
__device__ __forceinline__ T cu_of(T ux, T uy, T uz) {
    using D = Dirs<Q>;
    bool started = false;
    T acc = T(0);
    acc = add_cu<D::cx[I]>(acc, ux, started);
    acc = add_cu<D::cy[I]>(acc, uy, started);
    acc = add_cu<D::cz[I]>(acc, uz, started);
    return acc;  // rest direction: 0.0
}

// (c - u + (3 cu) c) for one axis (_core_py.py:176-178)
template <int C>
__device__ __forceinline__ double guo_axis(double u, double cu3) {
    if constexpr (C == 1) return (1.0 - u) + cu3;
    else if constexpr (C == -1) return (-1.0 - u) - cu3;
    else return -u;
}

// XONLY: force along x only (fy == fz == 0): the y/z terms of t are +-0 and
// adding them leaves A fx unchanged, so dropping them is value-identical.
template <int Q, int I, bool XONLY = false>
__device__ __forceinline__ double guo_F(double ux, double uy, double uz, double cu,
                                        const KParams& p) {
    using D = Dirs<Q>;
    const double cu3 = 3.0 * cu;
    double t;
    if constexpr (XONLY)
        t = guo_axis<D::cx[I]>(ux, cu3) * p.fx;
    else
        t = (guo_axis<D::cx[I]>(ux, cu3) * p.fx + guo_axis<D::cy[I]>(uy, cu3) * p.fy) +
            guo_axis<D::cz[I]>(uz, cu3) * p.fz;
    constexpr double w3 = 3.0 * D::w[I];
    return w3 * t;
}

// MODEL: 0 SRT, 1 TRT, 2 MRT, 4 SRT with the per-cell rate `om`
// (rem = 1 - om, hw = 1 - 0.5 om as _core_py.py:133-134,181 compute them).
// FORCE: 0 none, 1 Guo, 2 SimpleShift, 3 Guo with the force along x only.
// MOUT: also hand back rho and the (shifted) velocity the collision used -
// the macroscopic readout of the pre-collision state (k_fused_mom).
template <int Q, int MODEL, int FORCE, bool MOUT = false>
__device__ __forceinline__ void collide_cell(double (&f)[Q], const KParams& p, double om = 0.0,
                                             double* mout = nullptr) {
    using D = Dirs<Q>;
    constexpr bool GUO = FORCE == 1 || FORCE == 3;
    constexpr bool XO = FORCE == 3;
    // density: sequential sum (_core_py.py:91-93)
    double rho = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) rho = rho + f[i];
    // momentum: 0 + sum c f in index order (_core_py.py:94-103)
    double mx = 0.0, my = 0.0, mz = 0.0;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        if constexpr (D::cx[i] == 1) mx = mx + f[i];
        if constexpr (D::cx[i] == -1) mx = mx - f[i];
        if constexpr (D::cy[i] == 1) my = my + f[i];
        if constexpr (D::cy[i] == -1) my = my - f[i];
        if constexpr (D::cz[i] == 1) mz = mz + f[i];
        if constexpr (D::cz[i] == -1) mz = mz - f[i];
    });
    const double inv_rho = 1.0 / rho;
    double ux = mx * inv_rho;
    double uy = my * inv_rho;
    double uz = mz * inv_rho;
    if constexpr (FORCE != 0) {  // Guo half shift / SimpleShift (_core_py.py:113-122)
        ux = ux + p.sfx * inv_rho;
        uy = uy + p.sfy * inv_rho;
        uz = uz + p.sfz * inv_rho;
    }
    if constexpr (MOUT) {
        mout[0] = rho;
        mout[1] = ux;
        mout[2] = uy;
        mout[3] = uz;
    }
    const double usq15 = 1.5 * ((ux * ux + uy * uy) + uz * uz);

    if constexpr (MODEL == 0 || MODEL == 4) {
        // SRT (_core_py.py:130-136) + Guo source (:180-183)
        const double rem = MODEL == 0 ? p.rem : 1.0 - om;
        const double hw = MODEL == 0 ? p.hw : 1.0 - 0.5 * om;
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            const double cu = cu_of<Q, i>(ux, uy, uz);
            const double feq =
                (wt<Q, i>() * rho) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - usq15);
            double v = feq + rem * (f[i] - feq);
            if constexpr (GUO) v = v + hw * guo_F<Q, i, XO>(ux, uy, uz, cu, p);
            f[i] = v;
        });
    } else if constexpr (MODEL == 1) {
        // TRT (_core_py.py:137-148) + Guo source (:184-190), pairs shared
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            constexpr int j = D::opp[i];
            if constexpr (i == 0) {
                const double feq0 = (wt<Q, 0>() * rho) * (1.0 - usq15);
                const double fp = 0.5 * (f[0] + f[0]);
                const double fm = 0.5 * (f[0] - f[0]);
                const double ep = 0.5 * (feq0 + feq0);
                const double em = 0.5 * (feq0 - feq0);
                double v = (f[0] - p.omega_e * (fp - ep)) - p.omega_o * (fm - em);
                if constexpr (GUO) {
                    const double F0 = guo_F<Q, 0, XO>(ux, uy, uz, 0.0, p);
                    v = (v + p.he_half * (F0 + F0)) + p.ho_half * (F0 - F0);
                }
                f[0] = v;
            } else if constexpr (i < j) {
                const double cu = cu_of<Q, i>(ux, uy, uz);
                const double a = 3.0 * cu;
                const double b = (4.5 * cu) * cu;
                const double wr = wt<Q, i>() * rho;
                const double feq_i = wr * (((1.0 + a) + b) - usq15);
                const double feq_j = wr * (((1.0 - a) + b) - usq15);
                const double fp = 0.5 * (f[i] + f[j]);
                const double fm = 0.5 * (f[i] - f[j]);
                const double ep = 0.5 * (feq_i + feq_j);
                const double em = 0.5 * (feq_i - feq_j);
                const double A = p.omega_e * (fp - ep);
                const double B = p.omega_o * (fm - em);
                double vi = (f[i] - A) - B;
                double vj = (f[j] - A) + B;
                if constexpr (GUO) {
                    const double Fi = guo_F<Q, i, XO>(ux, uy, uz, cu, p);
                    const double Fj = guo_F<Q, j, XO>(ux, uy, uz, -cu, p);
                    const double P = p.he_half * (Fi + Fj);
                    const double Qd = p.ho_half * (Fi - Fj);
                    vi = (vi + P) + Qd;
                    vj = (vj + P) - Qd;
                }
                f[i] = vi;
                f[j] = vj;
            }
        });
    } else {
        // MRT, dense tables exactly as _core_py.py:149-169 and :191-197
        double feq[Q];
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            const double cu = cu_of<Q, i>(ux, uy, uz);
            feq[i] = (wt<Q, i>() * rho) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - usq15);
        });
        double m[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
            double acc = c_mrt_M[a * Q] * f[0];
            double acq = c_mrt_M[a * Q] * feq[0];
#pragma unroll
            for (int i = 1; i < Q; ++i) {
                acc = acc + c_mrt_M[a * Q + i] * f[i];
                acq = acq + c_mrt_M[a * Q + i] * feq[i];
            }
            m[a] = c_mrt_S[a] * (acc - acq);
        }
        double Fi[Q];
        if constexpr (GUO) {
            static_for<0, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                Fi[i] = guo_F<Q, i, XO>(ux, uy, uz, cu_of<Q, i>(ux, uy, uz), p);
            });
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            double acc = c_mrt_Minv[i * Q] * m[0];
#pragma unroll
            for (int a = 1; a < Q; ++a) acc = acc + c_mrt_Minv[i * Q + a] * m[a];
            f[i] = f[i] - acc;
        }
        if constexpr (GUO) {
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                double acc = c_mrt_G[i * Q] * Fi[0];
#pragma unroll
                for (int a = 1; a < Q; ++a) acc = acc + c_mrt_G[i * Q + a] * Fi[a];
                f[i] = f[i] + acc;
            }
        }
    }
}

}  // namespace lbm
