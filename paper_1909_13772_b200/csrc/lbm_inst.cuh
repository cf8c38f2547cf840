// Launchers for one storage type.  Included by lbm_inst_f64.cu (REAL=double,
// compiled with -fmad=false: bitwise reference arithmetic) and
// lbm_inst_f32.cu (REAL=float storage, fp64 registers, FMA allowed).
#pragma once
#include <stdlib.h>
#include "lbm_kernels.cuh"
#include "lbm_launch.h"

#ifndef LBM_REAL
#error "define LBM_REAL before including lbm_inst.cuh"
#endif

namespace lbm {
namespace {

inline dim3 cell_block(int nx) {
    int bx = nx >= 128 ? 128 : ((nx + 31) / 32) * 32;
    return dim3(bx, 1, 1);
}

inline dim3 fused_block(int nx) {
    int bx = nx >= LBM_FUSED_BX ? LBM_FUSED_BX : ((nx + 31) / 32) * 32;
    return dim3(bx, 1, 1);
}

template <int Q, int MODEL, int FORCE>
cudaError_t fused_t(const KGrid& g, const KParams& p, const void* src, void* dst,
                    const uint32_t* cm, const uint32_t* tmk, int z0, int z1, cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    dim3 b = fused_block(g.nx);
    dim3 grid((g.nx + b.x - 1) / b.x, g.ny, z1 - z0);
    const bool peer = p.peer_lo != nullptr || p.peer_hi != nullptr;
    if (p.mv_link) {
        // moving-body walls: a separate instantiation, so the standard sweep
        // keeps its register allocation (3D stencils, SRT/TRT/dense MRT)
        if constexpr (Q != 9 && MODEL <= 2 && FORCE != 2) {
            if (peer)
                k_fused<Q, LBM_REAL, MODEL, FORCE, true, true><<<grid, b, 0, s>>>(
                    g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0);
            else
                k_fused<Q, LBM_REAL, MODEL, FORCE, true><<<grid, b, 0, s>>>(
                    g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0);
            return cudaGetLastError();
        } else {
            return cudaErrorInvalidValue;
        }
    }
    if constexpr (Q != 9) {
        if (peer) {
            k_fused<Q, LBM_REAL, MODEL, FORCE, false, true><<<grid, b, 0, s>>>(
                g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0);
            return cudaGetLastError();
        }
    }
    k_fused<Q, LBM_REAL, MODEL, FORCE><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src,
                                                         (LBM_REAL*)dst, cm, tmk, z0);
    return cudaGetLastError();
}

template <int Q, int MODEL, int FORCE>
cudaError_t collide_t(const KGrid& g, const KParams& p, void* pdf, const uint32_t* cm,
                      cudaStream_t s) {
    dim3 b = cell_block(g.nx);
    dim3 grid((g.nx + b.x - 1) / b.x, g.ny, g.nz);
    k_collide_only<Q, LBM_REAL, MODEL, FORCE><<<grid, b, 0, s>>>(g, p, (LBM_REAL*)pdf, cm);
    return cudaGetLastError();
}

// (model, force) -> template; SimpleShift only with SRT (collision.py:431-435).
// Model 3 = MRT in the factorised raw-moment form (fp32 storage, D3Q27 only).
template <int Q, class F>
cudaError_t by_model(int model, int force, F&& fn) {
    if constexpr (std::is_same_v<LBM_REAL, float> && Q == 27) {
        if (model == 3 && force == 0) return fn(std::integral_constant<int, 3>{}, std::integral_constant<int, 0>{});
        if (model == 3 && force == 1) return fn(std::integral_constant<int, 3>{}, std::integral_constant<int, 1>{});
        if (model == 3 && force == 3) return fn(std::integral_constant<int, 3>{}, std::integral_constant<int, 3>{});
    }
    // ABI model 3 (SRT with a per-cell rate field) is kernel model 4
    if (model == 4 && force == 0) return fn(std::integral_constant<int, 4>{}, std::integral_constant<int, 0>{});
    if (model == 4 && force == 1) return fn(std::integral_constant<int, 4>{}, std::integral_constant<int, 1>{});
    if (model == 4 && force == 3) return fn(std::integral_constant<int, 4>{}, std::integral_constant<int, 3>{});
    if (model == 0 && force == 0) return fn(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{});
    if (model == 0 && force == 1) return fn(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
    if (model == 0 && force == 2) return fn(std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{});
    if (model == 1 && force == 0) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{});
    if (model == 1 && force == 1) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
    if (model == 2 && force == 0) return fn(std::integral_constant<int, 2>{}, std::integral_constant<int, 0>{});
    if (model == 2 && force == 1) return fn(std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{});
    if (model == 0 && force == 3) return fn(std::integral_constant<int, 0>{}, std::integral_constant<int, 3>{});
    if (model == 1 && force == 3) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 3>{});
    if (model == 2 && force == 3) return fn(std::integral_constant<int, 2>{}, std::integral_constant<int, 3>{});
    return cudaErrorInvalidValue;
}

template <class F>
cudaError_t by_q(int q, F&& fn) {
    if (q == 9) return fn(std::integral_constant<int, 9>{});
    if (q == 19) return fn(std::integral_constant<int, 19>{});
    if (q == 27) return fn(std::integral_constant<int, 27>{});
    return cudaErrorInvalidValue;
}

}  // namespace

namespace LBM_UNIT {

cudaError_t fused(int q, int model, int force, const KGrid& g, const KParams& p, const void* src,
                  void* dst, const uint32_t* cm, const uint32_t* tmk, int z0, int z1,
                  cudaStream_t s) {
    if (model == LBM_SRT_FIELD) model = 4;
    else if (model == LBM_MRT && p.mrt_fast && !p.mv_link) model = 3;  // moving walls: dense MRT
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        return by_model<Q>(model, force, [&](auto Mc, auto Fc) {
            return fused_t<Q, decltype(Mc)::value, decltype(Fc)::value>(g, p, src, dst, cm, tmk, z0,
                                                                        z1, s);
        });
    });
}

cudaError_t collide_only(int q, int model, int force, const KGrid& g, const KParams& p, void* pdf,
                         const uint32_t* cm, cudaStream_t s) {
    if (model == LBM_SRT_FIELD) model = 4;
    else if (model == LBM_MRT && p.mrt_fast) model = 3;
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        return by_model<Q>(model, force, [&](auto Mc, auto Fc) {
            return collide_t<Q, decltype(Mc)::value, decltype(Fc)::value>(g, p, pdf, cm, s);
        });
    });
}

cudaError_t stream_only(int q, const KGrid& g, const KParams& p, const void* src,
                        const uint32_t* cm, const uint32_t* tmk, double* out, cudaStream_t s) {
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx);
        dim3 grid((g.nx + b.x - 1) / b.x, g.ny, g.nz);
        k_stream_only<Q, LBM_REAL><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src, cm, tmk, out);
        return cudaGetLastError();
    });
}

cudaError_t moments(int q, int guo, const KGrid& g, const KParams& p, const void* src,
                    const uint32_t* cm, const uint32_t* tmk, int stream_form, double* rho,
                    double* u, int* bad, cudaStream_t s) {
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx);
        dim3 grid((g.nx + b.x - 1) / b.x, g.ny, g.nz);
        if (guo)
            k_moments<Q, LBM_REAL, 1><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src, cm, tmk,
                                                         stream_form, rho, u, bad);
        else
            k_moments<Q, LBM_REAL, 0><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src, cm, tmk,
                                                         stream_form, rho, u, bad);
        return cudaGetLastError();
    });
}

cudaError_t convert(int q, int to_layout, const KGrid& g, double* dense, void* pdf,
                    cudaStream_t s) {
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx + 2);
        dim3 grid((g.nx + 2 + b.x - 1) / b.x, g.ny + 2, g.nz + 2);
        if (to_layout)
            k_convert<Q, LBM_REAL, 1><<<grid, b, 0, s>>>(g, dense, (LBM_REAL*)pdf);
        else
            k_convert<Q, LBM_REAL, 0><<<grid, b, 0, s>>>(g, dense, (LBM_REAL*)pdf);
        return cudaGetLastError();
    });
}

cudaError_t fill_eq(int q, const KGrid& g, const double* rho, const double* u, void* pdf,
                    cudaStream_t s) {
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx + 2);
        dim3 grid((g.nx + 2 + b.x - 1) / b.x, g.ny + 2, g.nz + 2);
        k_fill_eq<Q, LBM_REAL><<<grid, b, 0, s>>>(g, rho, u, (LBM_REAL*)pdf);
        return cudaGetLastError();
    });
}

}  // namespace LBM_UNIT
}  // namespace lbm
