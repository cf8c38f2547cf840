// Launcher declarations shared by the instantiation units and the C-ABI.
// unit_f64 lives in lbm_inst_f64.cu, unit_f32 in lbm_inst_f32.cu; both have
// the same signatures (declared once through the macro below).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lbm {
struct KGrid;
struct KParams;

#define LBM_DECLARE_UNIT(NS)                                                                     \
    namespace NS {                                                                               \
    cudaError_t fused(int q, int model, int force, const KGrid& g, const KParams& p,             \
                      const void* src, void* dst, const uint32_t* cm, const uint32_t* tmk,       \
                      const uint64_t* lb, int z0, int z1, cudaStream_t s);                       \
    cudaError_t fused_mom(int q, int model, int force, const KGrid& g, const KParams& p,         \
                          const void* src, void* dst, const uint32_t* cm, const uint32_t* tmk,   \
                          int z0, int z1, double* rho, double* u, int* bad, cudaStream_t s);     \
    cudaError_t collide_only(int q, int model, int force, const KGrid& g, const KParams& p,      \
                             void* pdf, const uint32_t* cm, int z0, int z1, cudaStream_t s);     \
    cudaError_t stream_only(int q, const KGrid& g, const KParams& p, const void* src,            \
                            const uint32_t* cm, const uint32_t* tmk, double* out, cudaStream_t s); \
    cudaError_t moments(int q, int guo, const KGrid& g, const KParams& p, const void* src,       \
                        const uint32_t* cm, const uint32_t* tmk, int stream_form, double* rho,    \
                        double* u, int* bad, int z0, int z1, cudaStream_t s);                    \
    cudaError_t convert(int q, int to_layout, const KGrid& g, double* dense, void* pdf,          \
                        cudaStream_t s);                                                         \
    cudaError_t fill_eq(int q, const KGrid& g, const double* rho, const double* u, void* pdf,    \
                        cudaStream_t s);                                                         \
    cudaError_t fill_eq_dense(int q, const KGrid& g, const double* rho, const double* u, int zg0, \
                              int zg1, void* pdf, void* shell, cudaStream_t s);                  \
    cudaError_t fill_collide(int q, int model, int force, const KGrid& g, const KParams& p,      \
                             const double* rho, const double* u, int zg0, int zg1, void* pdf,    \
                             void* shell, const uint32_t* cm, cudaStream_t s);                   \
    }

LBM_DECLARE_UNIT(unit_f64)
LBM_DECLARE_UNIT(unit_f32)

// MRT constant tables of each unit (M, Minv, S, G packed, q <= 27)
cudaError_t set_mrt_tables_f64(int q, const double* tables, cudaStream_t s);
cudaError_t set_mrt_tables_f32(int q, const double* tables, cudaStream_t s);
cudaError_t set_mrt_tables_capi(int q, const double* tables, cudaStream_t s);
// fp32 unit: derive K = R Minv S M Rinv (raw-moment space) and enable the
// factorised D3Q27 MRT when K has the supported structure (*fast = 1)
cudaError_t set_mrt_fast_f32(int q, const double* tables, cudaStream_t s, int* fast);
}  // namespace lbm
