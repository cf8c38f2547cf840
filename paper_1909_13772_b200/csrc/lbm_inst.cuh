// Launchers for one storage type.  Included by lbm_inst_f64.cu (REAL=double,
// compiled with -fmad=false: bitwise reference arithmetic) and
// lbm_inst_f32.cu (REAL=float storage of f - w_i, fp32 registers on the centred
// populations, FMA allowed; readouts widen to fp64).
#pragma once
#include <stdlib.h>
#include <string.h>
#include "lbm_kernels.cuh"
#include "lbm_launch.h"
#ifdef LBM_TMA_VARIANT
#include "lbm_tma.cuh"
#endif
#ifdef LBM_VEC_VARIANT
#include "lbm_vec.cuh"
#endif


#ifndef LBM_REAL
#error "define LBM_REAL before including lbm_inst.cuh"
#endif

namespace lbm {
namespace {

inline dim3 cell_block(int nx) {
    int bx = nx >= 128 ? 128 : ((nx + 31) / 32) * 32;
    return dim3(bx, 1, 1);
}

inline bool use_z2() {
    const char* e = getenv("LBM_B200_Z2");
    return !(e && e[0] == '0');
}

inline dim3 fused_block(int nx) {
    int bx = nx >= LBM_FUSED_BX ? LBM_FUSED_BX : ((nx + 31) / 32) * 32;
    return dim3(bx, 1, 1);
}

#ifdef LBM_TMA_VARIANT
// ---------------------------------------------------------------- TMA path
// Built only into variant libraries (-DLBM_TMA_VARIANT, see lbm_tma.cuh for
// the design and the B200 measurements that keep it out of the default
// build).  In such a build LBM_B200_FUSED=ldg selects the LDG kernel.
inline bool use_tma() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("LBM_B200_FUSED");
        v = (e && strcmp(e, "ldg") == 0) ? 0 : 1;
    }
    return v == 1;
}

typedef CUresult (*pfn_tmap_encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The field as a 3-D tensor (x: pitch, y: ny+2 rows, q*(nz+2) z-slot planes),
// box = one 128-cell row segment.  Encoded once per (buffer, geometry).
inline int tma_box_width(const KGrid& g) {
    constexpr int a = tma_margin<LBM_REAL>();   // 16 bytes of cells
    return (g.nx >= kTmaW ? kTmaW : (g.nx + a - 1) / a * a) + 2 * a;
}

inline cudaError_t field_tmap(CUtensorMap* out, const void* base, const KGrid& g, int q) {
    static pfn_tmap_encode_t enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) !=
                cudaSuccess ||
            qr != cudaDriverEntryPointSuccess || !fn)
            return cudaErrorNotSupported;
        enc = (pfn_tmap_encode_t)fn;
    }
    struct Entry {
        const void* base;
        int nx, ny, nz, pitch, q;
        CUtensorMap map;
    };
    static thread_local Entry cache[4];
    static thread_local int next = 0;
    for (auto& e : cache)
        if (e.base == base && e.nx == g.nx && e.ny == g.ny && e.nz == g.nz && e.pitch == g.pitch &&
            e.q == q) {
            *out = e.map;
            return cudaSuccess;
        }
    const cuuint64_t dims[3] = {(cuuint64_t)g.pitch, (cuuint64_t)(g.ny + 2),
                                (cuuint64_t)q * (g.nz + 2)};
    const cuuint64_t strides[2] = {(cuuint64_t)g.pitch * sizeof(LBM_REAL),
                                   (cuuint64_t)g.plane * sizeof(LBM_REAL)};
    const cuuint32_t box[3] = {(cuuint32_t)tma_box_width(g), 1, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(out,
                     sizeof(LBM_REAL) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    Entry& e = cache[next];
    next = (next + 1) % 4;
    e = Entry{base, g.nx, g.ny, g.nz, g.pitch, q, *out};
    return cudaSuccess;
}

template <int Q, int MODEL, int FORCE>
cudaError_t fused_tma_t(const KGrid& g, const KParams& p, const void* src, void* dst,
                        const uint32_t* cm, const uint32_t* tmk, int z0, int z1, cudaStream_t s) {
    auto kern = k_fused_tma<Q, LBM_REAL, MODEL, FORCE>;
    constexpr int smem = tma_smem_bytes<Q, LBM_REAL>();
    static int ctas = 0;   // persistent grid: SMs x resident CTAs
    if (ctas == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        int occ = 0, dev = 0, sms = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTmaThreads, smem)) !=
            cudaSuccess)
            return e;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ctas = sms * (occ > 0 ? occ : 1);
    }
    CUtensorMap map;
    cudaError_t e = field_tmap(&map, src, g, Q);
    if (e != cudaSuccess) return e;
    const int nxt = (g.nx + kTmaW - 1) / kTmaW;
    const int64_t ntiles = (int64_t)nxt * g.ny * (z1 - z0);
    if (ntiles >= (int64_t)1 << 31) return cudaErrorInvalidValue;   // 32-bit tile indices
    const int grid = (int)(ntiles < ctas ? ntiles : ctas);
    kern<<<grid, kTmaThreads, smem, s>>>(map, g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0,
                                         nxt, ntiles, tma_box_width(g));
    return cudaGetLastError();
}

#endif  // LBM_TMA_VARIANT

#ifdef LBM_VEC_VARIANT
// ------------------------------------------------------- vectorised path
// Variant builds only (-DLBM_VEC_VARIANT; lbm_vec.cuh has the B200
// measurements).  LBM_B200_VEC=0|1 overrides the build default at run time.
#ifndef LBM_VEC_DEFAULT
#define LBM_VEC_DEFAULT 1
#endif
inline bool use_vec() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("LBM_B200_VEC");
        v = e ? (atoi(e) != 0) : LBM_VEC_DEFAULT;
    }
    return v == 1;
}

template <int Q, int MODEL, int FORCE>
cudaError_t fused_vec_t(const KGrid& g, const KParams& p, const void* src, void* dst,
                        const uint32_t* cm, const uint32_t* tmk, int z0, int z1, cudaStream_t s) {
    constexpr int V = std::is_same_v<LBM_REAL, double> ? 2 : LBM_VEC_WIDTH;
    const int groups = g.nx / V;
    const int bx = groups >= 128 ? 128 : ((groups + 31) / 32) * 32;
    dim3 grid((groups + bx - 1) / bx, g.ny, z1 - z0);
    k_fused_vec<Q, LBM_REAL, MODEL, FORCE, V><<<grid, bx, 0, s>>>(
        g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0);
    return cudaGetLastError();
}
#endif  // LBM_VEC_VARIANT

// launches that may read the link-bit map instead of the cell mask: D3Q19
// SRT / TRT (configs 0, 1, 3, 4) and the factorised D3Q27 MRT, NoSlip-only
// (no typemask), no moving walls, no fused halo
template <int Q, int MODEL, int FORCE>
constexpr bool bits_variant() {
    return (Q == 19 && MODEL <= 1 && FORCE != 2) || (Q == 27 && MODEL == 3);
}

inline bool use_bits() {
    const char* e = getenv("LBM_B200_LINKBITS");
    return !(e && e[0] == '0');
}

template <int Q, int MODEL, int FORCE>
cudaError_t fused_t(const KGrid& g, const KParams& p, const void* src, void* dst,
                    const uint32_t* cm, const uint32_t* tmk, const uint64_t* lb, int z0, int z1,
                    cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    const bool bits = lb && cm && !tmk && !p.mv_link && !p.peer_lo && !p.peer_hi && use_bits();
    // TMA staging for the 3-D SRT / TRT / factorised-MRT sweeps (the dense
    // MRT tables and SimpleShift keep the LDG kernel)
#ifdef LBM_VEC_VARIANT
    if constexpr (Q != 9 && MODEL != 2 && FORCE != 2) {
        constexpr int V = std::is_same_v<LBM_REAL, double> ? 2 : LBM_VEC_WIDTH;
        if (!p.mv_link && !p.peer_lo && !p.peer_hi && cm && g.nx % V == 0 && use_vec())
            return fused_vec_t<Q, MODEL, FORCE>(g, p, src, dst, cm, tmk, z0, z1, s);
    }
#endif
#ifdef LBM_TMA_VARIANT
    if constexpr (Q != 9 && MODEL != 2 && FORCE != 2) {
        if (!p.mv_link && !p.peer_lo && !p.peer_hi && cm && use_tma())
            return fused_tma_t<Q, MODEL, FORCE>(g, p, src, dst, cm, tmk, z0, z1, s);
    }
#endif
    dim3 b = fused_block(g.nx);
    dim3 grid((g.nx + b.x - 1) / b.x, g.ny, z1 - z0);
    const bool peer = p.peer_lo != nullptr || p.peer_hi != nullptr;
    // fp32 D3Q19 SRT / TRT without typed (UBB / Pressure) links: two cells
    // per thread along z (k_fused_z2, spill-free at 80 registers; the typed
    // corrections' register demand would make it spill, so typed launches
    // keep k_fused).  LBM_B200_Z2=0 selects k_fused (A/B runs).
    if constexpr (std::is_same_v<LBM_REAL, float> && Q == 19 && (MODEL == 0 || MODEL == 1)) {
        if (!p.mv_link && !peer && !tmk && use_z2()) {
            dim3 grid2(grid.x, grid.y, (z1 - z0 + 1) / 2);
            if (bits)
                k_fused_z2<Q, LBM_REAL, MODEL, FORCE, false, true><<<grid2, b, 0, s>>>(
                    g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, (const uint32_t*)lb, nullptr, z0, z1);
            else
                k_fused_z2<Q, LBM_REAL, MODEL, FORCE, false><<<grid2, b, 0, s>>>(
                    g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, cm, tmk, z0, z1);
            return cudaGetLastError();
        }
    }
    if constexpr (bits_variant<Q, MODEL, FORCE>()) {
        if (bits) {
            k_fused<Q, LBM_REAL, MODEL, FORCE, false, false, true><<<grid, b, 0, s>>>(
                g, p, (const LBM_REAL*)src, (LBM_REAL*)dst, (const uint32_t*)lb, nullptr, z0);
            return cudaGetLastError();
        }
    }
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
cudaError_t collide_t(const KGrid& g, const KParams& p, void* pdf, const uint32_t* cm, int z0,
                      int z1, cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    dim3 b = cell_block(g.nx);
    dim3 grid((g.nx + b.x - 1) / b.x, g.ny, z1 - z0);
    k_collide_only<Q, LBM_REAL, MODEL, FORCE><<<grid, b, 0, s>>>(g, p, (LBM_REAL*)pdf, cm, z0);
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
                  void* dst, const uint32_t* cm, const uint32_t* tmk, const uint64_t* lb, int z0,
                  int z1, cudaStream_t s) {
    if (model == LBM_SRT_FIELD) model = 4;
    else if (model == LBM_MRT && p.mrt_fast && !p.mv_link) model = 3;  // moving walls: dense MRT
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        return by_model<Q>(model, force, [&](auto Mc, auto Fc) {
            return fused_t<Q, decltype(Mc)::value, decltype(Fc)::value>(g, p, src, dst, cm, tmk, lb,
                                                                        z0, z1, s);
        });
    });
}

// fused sweep + readout of the pulled state (k_fused_mom): fp64 D3Q19 SRT /
// TRT, unforced or Guo; cudaErrorNotSupported elsewhere (the caller then
// runs the sweep and lbm_moments_planes as two launches).  A template on the
// storage type, so the fp32 unit (built with -fmad=true) never instantiates
// k_fused_mom: an `if constexpr` in a plain function still instantiates its
// discarded branch, and a kernel compiled into both units shares one host
// stub - which copy a launch resolves to then depends on which module the
// lazy loader brought in first (measured: the contracted copy gave 1-ulp
// velocity differences after fp32 kernels had run in the same process).
template <typename R>
static cudaError_t fused_mom_t(int q, int model, int force, const KGrid& g, const KParams& p,
                               const void* src, void* dst, const uint32_t* cm,
                               const uint32_t* tmk, int z0, int z1, double* rho, double* u,
                               int* bad, cudaStream_t s) {
    if constexpr (std::is_same_v<R, double>) {
        if (q != 19 || (model != 0 && model != 1) || (force != 0 && force != 1 && force != 3) ||
            p.mv_link || p.peer_lo || p.peer_hi)
            return cudaErrorNotSupported;
        if (z1 <= z0) return cudaSuccess;
        dim3 b = fused_block(g.nx);
        dim3 grid((g.nx + b.x - 1) / b.x, g.ny, z1 - z0);
        auto go = [&](auto Mc, auto Fc) {
            k_fused_mom<19, decltype(Mc)::value, decltype(Fc)::value><<<grid, b, 0, s>>>(
                g, p, (const double*)src, (double*)dst, cm, tmk, z0, rho, u, bad);
            return cudaGetLastError();
        };
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        using I3 = std::integral_constant<int, 3>;
        if (model == 0) return force == 0 ? go(I0{}, I0{}) : force == 1 ? go(I0{}, I1{}) : go(I0{}, I3{});
        return force == 0 ? go(I1{}, I0{}) : force == 1 ? go(I1{}, I1{}) : go(I1{}, I3{});
    } else {
        return cudaErrorNotSupported;
    }
}

cudaError_t fused_mom(int q, int model, int force, const KGrid& g, const KParams& p,
                      const void* src, void* dst, const uint32_t* cm, const uint32_t* tmk, int z0,
                      int z1, double* rho, double* u, int* bad, cudaStream_t s) {
    return fused_mom_t<LBM_REAL>(q, model, force, g, p, src, dst, cm, tmk, z0, z1, rho, u, bad, s);
}

cudaError_t collide_only(int q, int model, int force, const KGrid& g, const KParams& p, void* pdf,
                         const uint32_t* cm, int z0, int z1, cudaStream_t s) {
    if (model == LBM_SRT_FIELD) model = 4;
    else if (model == LBM_MRT && p.mrt_fast) model = 3;
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        return by_model<Q>(model, force, [&](auto Mc, auto Fc) {
            return collide_t<Q, decltype(Mc)::value, decltype(Fc)::value>(g, p, pdf, cm, z0, z1, s);
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
                    double* u, int* bad, int z0, int z1, cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx);
        dim3 grid((g.nx + b.x - 1) / b.x, g.ny, z1 - z0);
        if (guo)
            k_moments<Q, LBM_REAL, 1><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src, cm, tmk,
                                                         stream_form, rho, u, bad, z0);
        else
            k_moments<Q, LBM_REAL, 0><<<grid, b, 0, s>>>(g, p, (const LBM_REAL*)src, cm, tmk,
                                                         stream_form, rho, u, bad, z0);
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

cudaError_t fill_eq_dense(int q, const KGrid& g, const double* rho, const double* u, int zg0,
                          int zg1, void* pdf, void* shell, cudaStream_t s) {
    if (zg1 <= zg0) return cudaSuccess;
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        dim3 b = cell_block(g.nx + 2);
        dim3 grid((g.nx + 2 + b.x - 1) / b.x, g.ny + 2, zg1 - zg0);
        k_fill_eq_dense<Q, LBM_REAL><<<grid, b, 0, s>>>(g, rho, u, zg0, (LBM_REAL*)pdf,
                                                        (LBM_REAL*)shell);
        return cudaGetLastError();
    });
}

cudaError_t fill_collide(int q, int model, int force, const KGrid& g, const KParams& p,
                         const double* rho, const double* u, int zg0, int zg1, void* pdf,
                         void* shell, const uint32_t* cm, cudaStream_t s) {
    if (zg1 <= zg0) return cudaSuccess;
    if (model == LBM_SRT_FIELD) model = 4;
    else if (model == LBM_MRT && p.mrt_fast) model = 3;
    return by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        return by_model<Q>(model, force, [&](auto Mc, auto Fc) {
            dim3 b = cell_block(g.nx + 2);
            dim3 grid((g.nx + 2 + b.x - 1) / b.x, g.ny + 2, zg1 - zg0);
            k_fill_collide<Q, LBM_REAL, decltype(Mc)::value, decltype(Fc)::value>
                <<<grid, b, 0, s>>>(g, p, rho, u, zg0, (LBM_REAL*)pdf, (LBM_REAL*)shell, cm);
            return cudaGetLastError();
        });
    });
}

}  // namespace LBM_UNIT
}  // namespace lbm
