// extern "C" boundary of the LBM hot path (declared in include/lbm_b200.h).
//
// Converts the plain-C geometry/parameter structs into kernel structs,
// validates arguments, dispatches to the fp64 / fp32 instantiation units and
// turns CUDA errors into status codes + a thread-local message.  Also hosts
// the flag-validation / link-mask kernel and the flat-cell utilities
// (compiled with -fmad=false like the fp64 unit).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda.h>

#include "../../include/lbm_b200.h"
#include "lbm_kernels.cuh"
#include "lbm_launch.h"

namespace lbm {
LBM_DEFINE_MRT_SETTER(set_mrt_tables_capi)
}

using namespace lbm;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LBM_OK;
    if (e == cudaErrorInvalidValue)
        return fail(LBM_EINVAL, "%s: unsupported configuration", what);
    return fail(LBM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool q_ok(int q) { return q == 9 || q == 19 || q == 27; }

int check_grid(const lbm_grid_t* g, KGrid* k) {
    if (!g) return fail(LBM_EINVAL, "grid is NULL");
    if (!q_ok(g->q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", g->q);
    if (g->real_bytes != 8 && g->real_bytes != 4)
        return fail(LBM_EINVAL, "real_bytes must be 8 or 4, got %d", g->real_bytes);
    if (g->nx < 1 || g->ny < 1 || g->nz < 1)
        return fail(LBM_EINVAL, "box must be non-empty, got %dx%dx%d", g->nx, g->ny, g->nz);
    if (g->xoff < 1 || g->pitch < g->xoff + g->nx + 1)
        return fail(LBM_EINVAL, "pitch %d / xoff %d cannot hold %d cells + ghosts", g->pitch,
                    g->xoff, g->nx);
    if (g->zface_lo < 0 || g->zface_lo > 2 || g->zface_hi < 0 || g->zface_hi > 2)
        return fail(LBM_EINVAL, "bad z-face mode");
    if ((g->zface_lo == LBM_ZFACE_WRAP) != (g->zface_hi == LBM_ZFACE_WRAP))
        return fail(LBM_EINVAL, "z wrap must apply to both faces");
    if (g->ny + 2 > 65535 || g->nz + 2 > 65535)
        return fail(LBM_EINVAL, "ny/nz too large for the launch grid");
    k->nx = g->nx;
    k->ny = g->ny;
    k->nz = g->nz;
    k->pitch = g->pitch;
    k->xoff = g->xoff;
    k->wrap_x = g->wrap_x ? 1 : 0;
    k->wrap_y = g->wrap_y ? 1 : 0;
    k->zlo = g->zface_lo;
    k->zhi = g->zface_hi;
    k->plane = (int64_t)(g->ny + 2) * g->pitch;
    k->zstride = (int64_t)g->q * k->plane;
    // the kernels address a cell's sources and stores as int32 deltas from
    // the cell (KGrid::dpull/dlink/dslot, peer stores): every delta is
    // computed in int64 below and range-checked before it is narrowed; the
    // plane and z-stride themselves must fit too
    const int64_t lim = ((int64_t)1 << 31) - 1;
    if (k->zstride > lim)
        return fail(LBM_EINVAL, "x-y plane of %lld elements too large for 32-bit in-plane offsets",
                    (long long)k->plane);
    k->plane32 = (int)k->plane;
    k->zstride32 = (int)k->zstride;
    // keep-in-L2 hints for the bounce-back re-reads only where a z-plane of
    // the field is large against L2 (measured: +1.9 % on config 4 at 512^2,
    // -1.2 % on config 1 at 128^2 where the re-reads hit anyway)
    k->link_hint = k->zstride * g->real_bytes >= ((int64_t)16 << 20) ? 1 : 0;
    // LBM_B200_LINK_HINT=0|1 forces the choice (tests run the evict_last
    // path on small grids; it changes cache policy only, never a value)
    if (const char* h = getenv("LBM_B200_LINK_HINT")) {
        if (h[0] == '0' || h[0] == '1') k->link_hint = h[0] - '0';
    }
    // cell-mask rows prefetched into L2 ahead of the sweep (prefetch_mask).
    // Measured on B200, config 4 (rows ahead -> fraction of the HBM roofline):
    // fp32 0: 0.861, 32: 0.897, 64: 0.904, 128: 0.905, 300: 0.895, 600: 0.867;
    // fp64 0: 0.942, 32: 0.946, 64: 0.947, 128: 0.944, 600: 0.925;
    // config 2 (D3Q27 fp32, 256^2 planes) 0: 0.923, 4: 0.935, 16: 0.941,
    // 32: 0.946, 64: 0.936, 128: 0.935.
    // LBM_B200_MASK_AHEAD=n overrides (0: off).
    // (Packed into KGrid::link_hint bits 1.. so the kernel argument layout -
    // and with it the register allocation of the D3Q27 kernels - is unchanged:
    // a separate field cost config 2 9 % through a changed spill placement.)
    int ahead = g->real_bytes == 8 ? 64 : (g->q == 27 ? 32 : 128);
    if (const char* h = getenv("LBM_B200_MASK_AHEAD")) ahead = atoi(h) > 0 ? atoi(h) : 0;
    if (ahead > (1 << 20)) ahead = 1 << 20;
    k->link_hint |= ahead << 1;
    bool fits = true;
    auto narrow = [&](int64_t v) {
        if (v > lim || v < -lim) fits = false;
        return (int)v;
    };
    auto fill = [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        using D = Dirs<Q>;
        for (int i = 0; i < 27; ++i) k->dpull[i] = k->dlink[i] = k->dslot[i] = 0;
        for (int i = 0; i < Q; ++i) {
            const int64_t slot = (int64_t)slot_of<Q>(i) * k->plane;
            k->dslot[i] = narrow(slot);
            k->dpull[i] = narrow(slot - D::cz[i] * k->zstride - D::cy[i] * (int64_t)g->pitch - D::cx[i]);
            k->dlink[i] = narrow((int64_t)slot_of<Q>(D::opp[i]) * k->plane);
        }
    };
    if (g->q == 9) fill(std::integral_constant<int, 9>{});
    else if (g->q == 19) fill(std::integral_constant<int, 19>{});
    else fill(std::integral_constant<int, 27>{});
    // (peer stores add dslot < zstride to an int64 row offset: covered above)
    if (!fits)
        return fail(LBM_EINVAL, "x-y plane of %lld elements too large for 32-bit in-plane offsets",
                    (long long)k->plane);
    return LBM_OK;
}

int check_params(const lbm_params_t* p, int q, KParams* k, cudaStream_t s, int real_bytes) {
    if (!p) return fail(LBM_EINVAL, "params is NULL");
    if (p->model < 0 || p->model > 3) return fail(LBM_EINVAL, "bad model %d", p->model);
    if (p->model == LBM_SRT_FIELD && !p->omega_cells)
        return fail(LBM_EINVAL, "per-cell SRT rates need omega_cells");
    if (p->model == LBM_SRT_FIELD && p->force_mode == LBM_FORCE_SHIFT)
        return fail(LBM_EINVAL, "SimpleShift needs an SRT model with one global rate");
    k->omega = p->omega_cells;
    k->mv_owner = nullptr;
    k->mv_link = nullptr;
    k->mv_bodies = k->mv_cell0 = nullptr;
    k->mv_forces = nullptr;
    k->mv_slots = k->mv_bx = k->mv_by = 0;
    k->mv_cx = k->mv_cy = k->mv_cz = 1;
    k->mv_rho0 = 1.0;
    k->peer_lo = k->peer_hi = nullptr;
    if (p->moving) {
        const lbm_moving_t* m = p->moving;
        if (!m->owner || !m->linkmask || (!m->bodies && m->n_slots > 0) || !m->cell0)
            return fail(LBM_EINVAL, "moving walls: NULL array");
        if (m->n_slots < 0 || m->blocks[0] < 1 || m->blocks[1] < 1 || m->blocks[2] < 1 ||
            m->block_cells[0] < 1 || m->block_cells[1] < 1 || m->block_cells[2] < 1)
            return fail(LBM_EINVAL, "moving walls: bad block grid");
        k->mv_owner = m->owner;
        k->mv_link = m->linkmask;
        k->mv_bodies = m->bodies;
        k->mv_cell0 = m->cell0;
        k->mv_forces = m->forces;
        k->mv_slots = m->n_slots;
        k->mv_bx = m->blocks[0];
        k->mv_by = m->blocks[1];
        k->mv_cx = m->block_cells[0];
        k->mv_cy = m->block_cells[1];
        k->mv_cz = m->block_cells[2];
        k->mv_rho0 = m->rho0;
    }
    if (p->force_mode < 0 || p->force_mode > 3)
        return fail(LBM_EINVAL, "bad force mode %d", p->force_mode);
    if (p->force_mode == LBM_FORCE_SHIFT && p->model != LBM_SRT)
        return fail(LBM_EINVAL, "SimpleShift needs an SRT model with one global rate");
    k->rem = p->rem;
    k->hw = p->hw;
    k->omega_e = p->omega_e;
    k->omega_o = p->omega_o;
    k->he_half = p->he_half;
    k->ho_half = p->ho_half;
    k->fx = p->fx;
    k->fy = p->fy;
    k->fz = p->fz;
    k->sfx = p->shift_fx;
    k->sfy = p->shift_fy;
    k->sfz = p->shift_fz;
    for (int i = 0; i < 27; ++i) {
        k->ubb[i] = p->ubb[i];
        k->pw[i] = p->pressure[i];
        k->fubb[i] = (float)p->ubb[i];
    }
    k->frem = (float)p->rem;
    k->fhw = (float)p->hw;
    k->fomega_e = (float)p->omega_e;
    k->fomega_o = (float)p->omega_o;
    k->fhe_half = (float)p->he_half;
    k->fho_half = (float)p->ho_half;
    k->ffx = (float)p->fx;
    k->ffy = (float)p->fy;
    k->ffz = (float)p->fz;
    k->fsfx = (float)p->shift_fx;
    k->fsfy = (float)p->shift_fy;
    k->fsfz = (float)p->shift_fz;
    for (int i = 0; i < 27; ++i) k->fcF[i] = k->fguo_p[i] = k->fguo_q[i] = 0.f;
    for (int i = 0; i < q; ++i) {
        int cx, cy, cz;
        double w;
        if (q == 9) { cx = Dirs<9>::cx[i]; cy = Dirs<9>::cy[i]; cz = Dirs<9>::cz[i]; w = Dirs<9>::w[i]; }
        else if (q == 19) { cx = Dirs<19>::cx[i]; cy = Dirs<19>::cy[i]; cz = Dirs<19>::cz[i]; w = Dirs<19>::w[i]; }
        else { cx = Dirs<27>::cx[i]; cy = Dirs<27>::cy[i]; cz = Dirs<27>::cz[i]; w = Dirs<27>::w[i]; }
        const double cF = cx * p->fx + cy * p->fy + cz * p->fz;
        k->fcF[i] = (float)cF;
        k->fguo_p[i] = (float)(p->he_half * 6.0 * w);
        k->fguo_q[i] = (float)(p->ho_half * 6.0 * w * cF);
    }
    k->mrt_fast = 0;
    if (p->model == LBM_MRT) {
        if (!p->mrt) return fail(LBM_EINVAL, "MRT needs its tables");
        cudaError_t e = real_bytes == 8 ? set_mrt_tables_f64(q, p->mrt, s)
                                        : set_mrt_tables_f32(q, p->mrt, s);
        if (e == cudaSuccess && real_bytes == 4) e = set_mrt_fast_f32(q, p->mrt, s, &k->mrt_fast);
        if (e != cudaSuccess) return cuda_status(e, "MRT tables");
    }
    return LBM_OK;
}

// ------------------------------------------------------------------ masks
struct MaskBits {
    uint32_t fluid, noslip, ubb, pressure, solid, known;
};

// neighbour flag source with the same covered/uncovered rule as pull_cell
__device__ __forceinline__ uint32_t flag_at(const KGrid& g, const uint32_t* flags, int x, int y,
                                            int z, int cx, int cy, int cz, bool* uncovered) {
    const int X = g.nx + 2, Y = g.ny + 2;
    int xs = x + cx, ys = y + cy, zs = z + cz;
    bool unc = false;
    int xw = xs, yw = ys, zw = zs;
    if (xs < 0 || xs >= g.nx) {
        if (g.wrap_x) xw = xs < 0 ? g.nx - 1 : 0;
        else unc = true;
    }
    if (ys < 0 || ys >= g.ny) {
        if (g.wrap_y) yw = ys < 0 ? g.ny - 1 : 0;
        else unc = true;
    }
    if (zs < 0) {
        if (g.zlo == LBM_ZFACE_WRAP) zw = g.nz - 1;
        else if (g.zlo == LBM_ZFACE_GHOST) unc = true;
    } else if (zs >= g.nz) {
        if (g.zhi == LBM_ZFACE_WRAP) zw = 0;
        else if (g.zhi == LBM_ZFACE_GHOST) unc = true;
    }
    if (unc) { xw = xs; yw = ys; zw = zs; }
    *uncovered = unc;
    return flags[((int64_t)(zw + 1) * Y + (yw + 1)) * X + (xw + 1)];
}

__device__ __forceinline__ void note_first(int* slot, int64_t cell) {
    atomicMin(slot, (int)(cell + 1));
}

template <int Q>
__global__ void k_build_mask(KGrid g, const uint32_t* __restrict__ flags, MaskBits b,
                             uint32_t* __restrict__ cellmask, uint32_t* __restrict__ typemask,
                             int* err) {
    using D = Dirs<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const int X = g.nx + 2, Y = g.ny + 2;
    const uint32_t f = flags[((int64_t)(z + 1) * Y + (y + 1)) * X + (x + 1)];
    const uint32_t flagged = f & b.known;
    if (flagged & (flagged - 1u)) note_first(&err[0], cell);
    if (flagged == 0u) note_first(&err[3], cell);
    uint32_t code = 0, um = 0, pmk = 0;
    int n_ubb = 0, n_ns = 0, n_pr = 0;
    if (f & b.fluid) {
        code = LBM_MASK_FLUID;
        static_for<1, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            // pulled direction i reads x - c_i: the reference link (x, opp(i))
            bool unc;
            const uint32_t nb = flag_at(g, flags, x, y, z, -D::cx[i], -D::cy[i], -D::cz[i], &unc);
            if (nb & b.solid) note_first(&err[1], cell);
            if ((nb & b.known) == 0u) note_first(&err[2], cell);
            if (unc && (nb & b.fluid)) note_first(&err[7], cell);
            if (nb & b.noslip) { code |= 1u << i; ++n_ns; }
            if (nb & b.ubb) { code |= 1u << i; um |= 1u << i; ++n_ubb; }
            if (nb & b.pressure) { code |= 1u << i; pmk |= 1u << i; ++n_pr; }
        });
        if (um) code |= LBM_MASK_UBB;
        if (pmk) code |= LBM_MASK_PRESSURE;
    }
    cellmask[cell] = code;
    typemask[2 * cell] = um;
    typemask[2 * cell + 1] = pmk;
    if (n_ubb) atomicAdd(&err[4], n_ubb);
    if (n_ns) atomicAdd(&err[5], n_ns);
    if (n_pr) atomicAdd(&err[6], n_pr);
}

// combined masks of a moving-body sweep (lbm_build_moving_masks)
template <int Q>
__global__ void k_moving_masks(KGrid g, const uint32_t* __restrict__ cm_in,
                               const int32_t* __restrict__ owner, uint32_t* __restrict__ cm_out,
                               uint32_t* __restrict__ linkmask, int* n_links) {
    using D = Dirs<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const int X = g.nx + 2, Y = g.ny + 2;
    uint32_t code = cm_in[cell];
    uint32_t lm = 0;
    int n = 0;
    if (owner[((int64_t)(z + 1) * Y + (y + 1)) * X + (x + 1)] >= 0) {
        code &= ~LBM_MASK_FLUID;          // covered: keeps its static links, skips collision
    } else if (code & LBM_MASK_FLUID) {
        static_for<1, Q>([&](auto J_) {
            constexpr int j = decltype(J_)::value;
            // pulled direction j reads x - c_j (raw ghost-inclusive neighbour)
            const int64_t nb = ((int64_t)(z + 1 - D::cz[j]) * Y + (y + 1 - D::cy[j])) * X +
                               (x + 1 - D::cx[j]);
            if (owner[nb] >= 0) {
                lm |= 1u << j;
                ++n;
            }
        });
        if (lm) code |= lm | LBM_MASK_MOVING;
    }
    cm_out[cell] = code;
    linkmask[cell] = lm;
    if (n) atomicAdd(n_links, n);
}

// Body coverage of ghost-inclusive blocks (coupling/mapping.py:100-140): the
// cell centre c = c0 + h (i - 1) (per axis, the reference's numpy
// expression, every op rounded) is covered by the first sphere in uid order
// with p - r <= c < p + r on every axis (the reference's searchsorted
// window) and ((cx-px)^2 + (cy-py)^2) + (cz-pz)^2 < r r, provided the cell
// is static fluid (flags & fluid_bits, or no flags at all).
__global__ void k_map_spheres(int ncx, int ncy, int ncz, const double* __restrict__ frame,
                              const int* __restrict__ first, const double* __restrict__ spheres,
                              const int64_t* __restrict__ uids, const uint32_t* __restrict__ flags,
                              uint32_t fluid_bits, int64_t* __restrict__ owner) {
    const int X = ncx + 2, Y = ncy + 2, Z = ncz + 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int b = blockIdx.z / Z;
    const int k = blockIdx.z % Z;
    if (i >= X) return;
    const int64_t cell = (((int64_t)b * Z + k) * Y + j) * X + i;
    const double* fr = frame + 6 * b;
    const double x = fr[0] + fr[3] * (double)(i - 1);
    const double y = fr[1] + fr[4] * (double)(j - 1);
    const double z = fr[2] + fr[5] * (double)(k - 1);
    int64_t who = -1;
    for (int s = first[b]; s < first[b + 1]; ++s) {
        const double* sp = spheres + 4 * s;
        const double r = sp[3];
        if (!(x >= sp[0] - r && x < sp[0] + r && y >= sp[1] - r && y < sp[1] + r &&
              z >= sp[2] - r && z < sp[2] + r))
            continue;
        const double ex = x - sp[0], ey = y - sp[1], ez = z - sp[2];
        if ((ex * ex + ey * ey) + ez * ez < r * r) {
            who = uids[s];
            break;
        }
    }
    if (who >= 0 && flags && (flags[cell] & fluid_bits) == 0u) who = -1;
    owner[cell] = who;
}

// Ghost shell copy (all q slots of every ghost cell of the box: the two
// z ghost planes, and the y ghost rows / x ghost columns of each interior
// plane).  Element type T = the storage word (8 or 4 bytes).
template <typename T>
__global__ void k_copy_shell(KGrid g, int q, const T* __restrict__ src, T* __restrict__ dst) {
    const int X = g.nx + 2, Y = g.ny + 2;
    const int zg = blockIdx.z;                       // ghost-inclusive plane
    const int slot = blockIdx.y;
    const bool ghost_plane = zg == 0 || zg == g.nz + 1;
    // a ghost plane copies all Y rows; an interior plane its 2 ghost rows
    // (y = 0, Y-1, full width) and 2 ghost columns (x = 0, X-1, Y-2 rows)
    const int64_t n = ghost_plane ? (int64_t)X * Y : (int64_t)2 * X + 2 * (Y - 2);
    const int64_t base = (int64_t)zg * g.zstride + (int64_t)slot * g.plane + g.xoff - 1;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int x, y;
        if (ghost_plane) {
            y = (int)(k / X);
            x = (int)(k % X);
        } else if (k < 2 * X) {
            y = k < X ? 0 : Y - 1;
            x = (int)(k % X);
        } else {
            const int r = (int)(k - 2 * X);
            y = 1 + r / 2;
            x = (r & 1) ? X - 1 : 0;
        }
        const int64_t e = base + (int64_t)y * g.pitch + x;
        dst[e] = src[e];
    }
}

// Sweep-time fluid mask (lbm/sweep.py:124-136): links stay as frozen at
// freeze() (boundary.py:128-131), the collision mask follows the CURRENT
// flags; err[0] = first unflagged interior cell + 1.
__global__ void k_refresh_fluid(KGrid g, const uint32_t* __restrict__ flags, uint32_t fluid,
                                uint32_t known, const uint32_t* __restrict__ cm_in,
                                uint32_t* __restrict__ cm_out, int* err) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const uint32_t f = flags[((int64_t)(z + 1) * (g.ny + 2) + (y + 1)) * (g.nx + 2) + (x + 1)];
    if ((f & known) == 0u) note_first(&err[0], cell);
    cm_out[cell] = (cm_in[cell] & ~LBM_MASK_FLUID) | ((f & fluid) ? LBM_MASK_FLUID : 0u);
}

// ------------------------------------------------------------ flat cells
template <int Q, int MODEL, int FORCE>
__global__ void k_collide_cells(KParams p, double* __restrict__ f, int64_t n) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = f[c * Q + i];
    collide_cell<Q, MODEL, FORCE>(v, p);
#pragma unroll
    for (int i = 0; i < Q; ++i) f[c * Q + i] = v[i];
}

// Kernel-slot collide (impl.collide, _core_py.py:70-200): every cell of a
// dense (n, q) population array whose flags & fluid_bits != 0, ghost ring
// included; MODEL 4 reads the per-cell rate (the omega_window of an SRT
// rate field).
template <int Q, int MODEL, int FORCE>
__global__ void k_slot_collide(KParams p, double* __restrict__ f, const uint32_t* __restrict__ flags,
                               uint32_t fluid_bits, const double* __restrict__ omega, int64_t n) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n || (flags[c] & fluid_bits) == 0u) return;
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = f[c * Q + i];
    double om = 0.0;
    if constexpr (MODEL == 4) om = omega[c];
    collide_cell<Q, MODEL, FORCE>(v, p, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) f[c * Q + i] = v[i];
}

// Kernel-slot pull (impl.stream_pull, _core_py.py:203-218): dense (Z, Y, X, q)
// ghost-inclusive src with `gl` ghost layers -> interior (nz, ny, nx, q),
// out[z, y, x, i] = src[z + gl - cz_i, y + gl - cy_i, x + gl - cx_i, i] for
// the caller's velocity set (passed as given, not assumed).
struct SlotStencil {
    int cx[27], cy[27], cz[27];
};

__global__ void k_slot_stream_pull(SlotStencil c, int q, const double* __restrict__ src,
                                   double* __restrict__ out, int X, int Y, int gl, int nx, int ny,
                                   int nz) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= nx) return;
    const int64_t o = (((int64_t)z * ny + y) * nx + x) * q;
    for (int i = 0; i < q; ++i) {
        const int64_t s = (((int64_t)(z + gl - c.cz[i]) * Y + (y + gl - c.cy[i])) * X +
                           (x + gl - c.cx[i])) * q + i;
        out[o + i] = src[s];
    }
}

// BoundaryHandling.apply (lbm/boundary.py:154-195) on dense (n, q) arrays:
// one thread per link (kind 0 NoSlip, 1 UBB, 2 Pressure; direction i from
// the fluid cell into the wall), dst[cell, opp(i)] from post-collision src.
template <int Q>
__global__ void k_apply_links(KParams p, const int32_t* __restrict__ kind,
                              const int32_t* __restrict__ dir, const int64_t* __restrict__ cell,
                              const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
    using D = Dirs<Q>;
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n) return;
    const int i = dir[l];
    const double* s = src + cell[l] * Q;
    double v = s[i];
    if (kind[l] == 1) {
        v = v - p.ubb[i];
    } else if (kind[l] == 2) {
        double rho = s[0];
        for (int k = 1; k < Q; ++k) rho = rho + s[k];
        double mx = 0.0, my = 0.0, mz = 0.0;
        static_for<0, Q>([&](auto K_) {
            constexpr int k = decltype(K_)::value;
            if constexpr (D::cx[k] == 1) mx = mx + s[k];
            if constexpr (D::cx[k] == -1) mx = mx - s[k];
            if constexpr (D::cy[k] == 1) my = my + s[k];
            if constexpr (D::cy[k] == -1) my = my - s[k];
            if constexpr (D::cz[k] == 1) mz = mz + s[k];
            if constexpr (D::cz[k] == -1) mz = mz - s[k];
        });
        const double ux = mx / rho, uy = my / rho, uz = mz / rho;
        double cu = 0.0;
        static_for<0, Q>([&](auto K_) {
            constexpr int k = decltype(K_)::value;
            if (k == i) cu = cu_of<Q, k>(ux, uy, uz);
        });
        const double usq = (ux * ux + uy * uy) + uz * uz;
        v = -v + p.pw[i] * ((1.0 + (4.5 * cu) * cu) - 1.5 * usq);
    }
    int o = 0;
    static_for<0, Q>([&](auto K_) {
        constexpr int k = decltype(K_)::value;
        constexpr int ok = D::opp[k];
        if (k == i) o = ok;
    });
    dst[cell[l] * Q + o] = v;
}

template <int Q>
__global__ void k_equilibrium_cells(const double* __restrict__ rho, const double* __restrict__ u,
                                    double* __restrict__ f, int64_t n) {
    using D = Dirs<Q>;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double r = rho[c];
    const double ux = u[c * 3], uy = u[c * 3 + 1], uz = u[c * 3 + 2];
    const double usq = (ux * ux + uy * uy) + uz * uz;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        const double cu = cu_of<Q, i>(ux, uy, uz);
        f[c * Q + i] = (wt<Q, i>() * r) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - 1.5 * usq);
    });
}

template <int Q, int GUO>
__global__ void k_macroscopic_cells(KParams p, const double* __restrict__ f,
                                    double* __restrict__ rho, double* __restrict__ u, int* bad,
                                    int64_t n) {
    using D = Dirs<Q>;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = f[c * Q + i];
    double r = v[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) r = r + v[i];
    if (r <= 0.0) atomicAdd(bad, 1);
    double mx = 0.0, my = 0.0, mz = 0.0;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        if constexpr (D::cx[i] == 1) mx = mx + v[i];
        if constexpr (D::cx[i] == -1) mx = mx - v[i];
        if constexpr (D::cy[i] == 1) my = my + v[i];
        if constexpr (D::cy[i] == -1) my = my - v[i];
        if constexpr (D::cz[i] == 1) mz = mz + v[i];
        if constexpr (D::cz[i] == -1) mz = mz - v[i];
    });
    const double inv = 1.0 / r;
    double ux = mx * inv, uy = my * inv, uz = mz * inv;
    if constexpr (GUO) {
        ux = ux + p.sfx * inv;
        uy = uy + p.sfy * inv;
        uz = uz + p.sfz * inv;
    }
    rho[c] = r;
    u[c * 3] = ux;
    u[c * 3 + 1] = uy;
    u[c * 3 + 2] = uz;
}

template <class F>
cudaError_t by_q(int q, F&& fn) {
    if (q == 9) return fn(std::integral_constant<int, 9>{});
    if (q == 19) return fn(std::integral_constant<int, 19>{});
    if (q == 27) return fn(std::integral_constant<int, 27>{});
    return cudaErrorInvalidValue;
}

dim3 cell_block(int nx) { return dim3(nx >= 128 ? 128 : ((nx + 31) / 32) * 32, 1, 1); }

}  // namespace

// ================================================================== C-ABI
// ------------------------------------------------------- link-bit map
// (layout and rule: code_from_bits in lbm_kernels.cuh)
__device__ __forceinline__ void set_bit(const KGrid& g, uint64_t* bits, int xg, int yg, int zg) {
    const int64_t bw = (g.nx + 31) >> 5;
    const int64_t row = ((int64_t)zg * (g.ny + 2) + yg) * bw;
    const int w = xg >> 5;
    if (w < bw) atomicOr((unsigned long long*)(bits + row + w), 1ull << (xg & 31));
    if (w >= 1 && w - 1 < bw) atomicOr((unsigned long long*)(bits + row + w - 1), 1ull << ((xg & 31) + 32));
}

// N of every interior cell from its own code; N of ghost cells from the
// links that pull from them
template <int Q>
__global__ void k_linkbits_set(KGrid g, const uint32_t* __restrict__ cellmask, uint64_t* bits) {
    using D = Dirs<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const uint32_t code = cellmask[((int64_t)z * g.ny + y) * g.nx + x];
    if (!(code & LBM_MASK_FLUID)) set_bit(g, bits, x + 1, y + 1, z + 1);
    static_for<1, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        const int xs = x - D::cx[i], ys = y - D::cy[i], zs = z - D::cz[i];
        const bool ghost = xs < 0 || xs >= g.nx || ys < 0 || ys >= g.ny || zs < 0 || zs >= g.nz;
        if (ghost && ((code >> i) & 1u)) set_bit(g, bits, xs + 1, ys + 1, zs + 1);
    });
}

// every interior cell: the derived code must equal the mask bit for bit
template <int Q>
__global__ void k_linkbits_check(KGrid g, const uint32_t* __restrict__ cellmask,
                                 const uint64_t* __restrict__ bits, int* mismatch) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    if (mask_code_of_nb<Q>(code_from_bits<Q>(g, bits, x, y, z)) != cellmask[cell]) atomicMin(mismatch, (int)(cell + 1 < 0x7fffffff ? cell + 1 : 0x7fffffff));
}

extern "C" {

int lbm_abi_version(void) { return LBM_B200_ABI_VERSION; }

size_t lbm_struct_size(int which) {
    return which == 0 ? sizeof(lbm_grid_t)
                      : which == 1 ? sizeof(lbm_params_t) : which == 2 ? sizeof(lbm_moving_t) : 0;
}

const char* lbm_last_error(void) { return g_err; }

int lbm_slot_of(int q, int i) {
    if (!q_ok(q) || i < 0 || i >= q) return -1;
    if (q == 9) return slot_of<9>(i);
    if (q == 19) return slot_of<19>(i);
    return slot_of<27>(i);
}

int64_t lbm_field_elems(const lbm_grid_t* g) {
    KGrid k;
    if (check_grid(g, &k) != LBM_OK) return -1;
    return (int64_t)(g->nz + 2) * k.zstride;
}

int lbm_face_span(const lbm_grid_t* g, int face, int64_t* send_off, int64_t* recv_off,
                  int64_t* count) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (face != 0 && face != 1) return fail(LBM_EINVAL, "face must be 0 (low z) or 1 (high z)");
    int nm, np;  // directions with c_z = -1, +1
    if (g->q == 9) { nm = 0; np = 0; }
    else if (g->q == 19) { nm = count_cz<19>(-1); np = count_cz<19>(1); }
    else { nm = count_cz<27>(-1); np = count_cz<27>(1); }
    if (face == 0) {
        // receive into ghost plane z=-1 the directions pulled upward (c_z=+1);
        // send interior plane z=0's c_z=-1 run (the lower peer's high ghost)
        *recv_off = (int64_t)0 * k.zstride + (int64_t)(g->q - np) * k.plane;
        *send_off = (int64_t)1 * k.zstride + 0;
        *count = (int64_t)np * k.plane;
        if (np != nm) return fail(LBM_EINVAL, "asymmetric stencil");
    } else {
        *recv_off = (int64_t)(g->nz + 1) * k.zstride + 0;
        *send_off = (int64_t)g->nz * k.zstride + (int64_t)(g->q - np) * k.plane;
        *count = (int64_t)nm * k.plane;
    }
    return LBM_OK;
}

int lbm_fused_step(const lbm_grid_t* g, const lbm_params_t* p, const void* src, void* dst,
                   const uint32_t* cellmask, const uint32_t* typemask, int z_begin, int z_end,
                   void* stream) {
    return lbm_fused_step_bits(g, p, src, dst, cellmask, typemask, nullptr, z_begin, z_end, stream);
}

int lbm_fused_step_bits(const lbm_grid_t* g, const lbm_params_t* p, const void* src, void* dst,
                        const uint32_t* cellmask, const uint32_t* typemask,
                        const uint64_t* linkbits, int z_begin, int z_end, void* stream) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!src || !dst) return fail(LBM_EINVAL, "NULL buffer");
    if (src == dst) return fail(LBM_EINVAL, "fused step needs two fields (src != dst)");
    if (z_begin < 0 || z_end > g->nz || z_begin > z_end)
        return fail(LBM_EINVAL, "plane range [%d, %d) outside 0..%d", z_begin, z_end, g->nz);
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::fused(g->q, p->model, p->force_mode, k, kp, src, dst, cellmask,
                                          typemask, linkbits, z_begin, z_end, s)
                        : unit_f32::fused(g->q, p->model, p->force_mode, k, kp, src, dst, cellmask,
                                          typemask, linkbits, z_begin, z_end, s);
    return cuda_status(e, "lbm_fused_step");
}

int lbm_fused_step_peer(const lbm_grid_t* g, const lbm_params_t* p, const void* src, void* dst,
                        const uint32_t* cellmask, const uint32_t* typemask, int z_begin,
                        int z_end, void* peer_lo, void* peer_hi, void* stream) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!src || !dst) return fail(LBM_EINVAL, "NULL buffer");
    if (src == dst) return fail(LBM_EINVAL, "fused step needs two fields (src != dst)");
    if (z_begin < 0 || z_end > g->nz || z_begin > z_end)
        return fail(LBM_EINVAL, "plane range [%d, %d) outside 0..%d", z_begin, z_end, g->nz);
    if (peer_lo && g->zface_lo != LBM_ZFACE_HALO)
        return fail(LBM_EINVAL, "peer_lo given but the low z face is not a halo face");
    if (peer_hi && g->zface_hi != LBM_ZFACE_HALO)
        return fail(LBM_EINVAL, "peer_hi given but the high z face is not a halo face");
    if (g->q == 9 && (peer_lo || peer_hi)) return fail(LBM_EINVAL, "D2Q9 has no z faces");
    kp.peer_lo = peer_lo;
    kp.peer_hi = peer_hi;
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::fused(g->q, p->model, p->force_mode, k, kp, src, dst, cellmask,
                                          typemask, nullptr, z_begin, z_end, s)
                        : unit_f32::fused(g->q, p->model, p->force_mode, k, kp, src, dst, cellmask,
                                          typemask, nullptr, z_begin, z_end, s);
    return cuda_status(e, "lbm_fused_step_peer");
}

int lbm_ghost_block_offset(const lbm_grid_t* g, int face, int64_t* offset) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (face != 0 && face != 1) return fail(LBM_EINVAL, "face must be 0 (low z) or 1 (high z)");
    if (!offset) return fail(LBM_EINVAL, "offset is NULL");
    *offset = face == 0 ? 0 : (int64_t)(g->nz + 1) * k.zstride;
    return LBM_OK;
}

// Stream-ordered flag signalling for the fused halo (driver stream memory
// operations, resolved at run time so the library needs no -lcuda).  A wait
// blocks the stream's front end, never an SM.
namespace {
typedef CUresult (*pfn_write_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*pfn_wait_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
pfn_write_t g_write32 = nullptr;
pfn_wait_t g_wait32 = nullptr;
int g_flush_ok = -1;

int memops_init() {
    if (g_write32 && g_wait32) return LBM_OK;
    cudaDriverEntryPointQueryResult q1, q2;
    void* w = nullptr;
    void* v = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || !w)
        return fail(LBM_ECUDA, "driver entry point cuStreamWriteValue32 unavailable");
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) != cudaSuccess ||
        q2 != cudaDriverEntryPointSuccess || !v)
        return fail(LBM_ECUDA, "driver entry point cuStreamWaitValue32 unavailable");
    g_write32 = (pfn_write_t)w;
    g_wait32 = (pfn_wait_t)v;
    int dev = 0, flush = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, dev) == cudaSuccess)
        g_flush_ok = flush ? 1 : 0;
    else
        g_flush_ok = 0;
    return LBM_OK;
}
}  // namespace

// CUDA IPC for the fused halo: export a (possibly sub-allocated) device
// buffer as handle + offset from its allocation base, and open a peer's
// export in the CURRENT device's context with lazy peer access, so a
// kernel on this GPU can store into a neighbour GPU's HBM over NVLink
// without a second context on the neighbour's device.
namespace {
typedef CUresult (*pfn_range_t)(CUdeviceptr*, size_t*, CUdeviceptr);
}  // namespace

int lbm_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
    if (!ptr || !handle_out || !offset_out) return fail(LBM_EINVAL, "NULL argument");
    static pfn_range_t range = nullptr;
    if (!range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(LBM_ECUDA, "driver entry point cuMemGetAddressRange unavailable");
        range = (pfn_range_t)fn;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
        return fail(LBM_EINVAL, "pointer is not device memory");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((CUdeviceptr)ptr - base);
    return LBM_OK;
}

int lbm_ipc_open(const void* handle, void** base_out) {
    if (!handle || !base_out) return fail(LBM_EINVAL, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "cudaIpcOpenMemHandle");
    *base_out = base;
    return LBM_OK;
}

int lbm_ipc_close(void* base) {
    if (!base) return LBM_OK;
    return cuda_status(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
}

int lbm_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(LBM_EINVAL, "bad copy");
    if (bytes == 0) return LBM_OK;
    return cuda_status(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream),
                       "lbm_copy_async");
}

int lbm_stream_signal(void* flag, uint32_t value, void* stream) {
    if (!flag) return fail(LBM_EINVAL, "flag is NULL");
    int st = memops_init();
    if (st != LBM_OK) return st;
    // default flags: a memory barrier orders every earlier write of the
    // stream (the fused kernel's peer stores) before the flag write
    CUresult r = g_write32((CUstream)stream, (CUdeviceptr)flag, (cuuint32_t)value, 0);
    if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    return LBM_OK;
}

int lbm_can_flush_remote_writes(void) {
    int dev = 0, flush = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, dev) != cudaSuccess)
        return 0;
    return flush ? 1 : 0;
}

int lbm_stream_wait(const void* flag, uint32_t value, void* stream) {
    if (!flag) return fail(LBM_EINVAL, "flag is NULL");
    int st = memops_init();
    if (st != LBM_OK) return st;
    unsigned int fl = CU_STREAM_WAIT_VALUE_GEQ | (g_flush_ok == 1 ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
    CUresult r = g_wait32((CUstream)stream, (CUdeviceptr)flag, (cuuint32_t)value, fl);
    if (r != CUDA_SUCCESS) return fail(LBM_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
    return LBM_OK;
}

static int collide_only_range(const lbm_grid_t* g, const lbm_params_t* p, void* pdf,
                              const uint32_t* cellmask, int z0, int z1, void* stream,
                              const char* who) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!pdf || !cellmask) return fail(LBM_EINVAL, "NULL buffer");
    if (z0 < 0 || z1 > g->nz || z0 > z1) return fail(LBM_EINVAL, "bad plane range [%d, %d)", z0, z1);
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::collide_only(g->q, p->model, p->force_mode, k, kp, pdf,
                                                 cellmask, z0, z1, s)
                        : unit_f32::collide_only(g->q, p->model, p->force_mode, k, kp, pdf,
                                                 cellmask, z0, z1, s);
    return cuda_status(e, who);
}

int lbm_collide_only(const lbm_grid_t* g, const lbm_params_t* p, void* pdf,
                     const uint32_t* cellmask, void* stream) {
    return collide_only_range(g, p, pdf, cellmask, 0, g ? g->nz : 0, stream, "lbm_collide_only");
}

int lbm_collide_only_planes(const lbm_grid_t* g, const lbm_params_t* p, void* pdf,
                            const uint32_t* cellmask, int z0, int z1, void* stream) {
    return collide_only_range(g, p, pdf, cellmask, z0, z1, stream, "lbm_collide_only_planes");
}

int lbm_stream_only(const lbm_grid_t* g, const lbm_params_t* p, const void* src,
                    const uint32_t* cellmask, const uint32_t* typemask, double* out,
                    void* stream) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!src || !cellmask || !typemask || !out) return fail(LBM_EINVAL, "NULL buffer");
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::stream_only(g->q, k, kp, src, cellmask, typemask, out, s)
                        : unit_f32::stream_only(g->q, k, kp, src, cellmask, typemask, out, s);
    return cuda_status(e, "lbm_stream_only");
}

static int moments_range(const lbm_grid_t* g, const lbm_params_t* p, const void* src,
                         const uint32_t* cellmask, const uint32_t* typemask, int stream_form,
                         int z0, int z1, double* rho, double* u, int* bad_count, void* stream,
                         const char* who) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!src || !rho || !u || !bad_count) return fail(LBM_EINVAL, "NULL buffer");
    if (stream_form && (!cellmask || !typemask)) return fail(LBM_EINVAL, "NULL mask");
    if (z0 < 0 || z1 > g->nz || z0 > z1) return fail(LBM_EINVAL, "bad plane range [%d, %d)", z0, z1);
    const int guo = p->force_mode == LBM_FORCE_GUO || p->force_mode == LBM_FORCE_GUO_X;
    cudaError_t e = g->real_bytes == 8 ? unit_f64::moments(g->q, guo, k, kp, src, cellmask, typemask,
                                                           stream_form, rho, u, bad_count, z0, z1, s)
                                       : unit_f32::moments(g->q, guo, k, kp, src, cellmask, typemask,
                                                           stream_form, rho, u, bad_count, z0, z1, s);
    return cuda_status(e, who);
}

int lbm_fused_step_moments(const lbm_grid_t* g, const lbm_params_t* p, const lbm_params_t* p_moments,
                           const void* src, void* dst, const uint32_t* cellmask,
                           const uint32_t* typemask, int z_begin, int z_end, double* rho, double* u,
                           int* bad_count, void* stream) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!p_moments || !src || !dst || !rho || !u || !bad_count) return fail(LBM_EINVAL, "NULL buffer");
    if (src == dst) return fail(LBM_EINVAL, "fused step needs two fields (src != dst)");
    if (z_begin < 0 || z_end > g->nz || z_begin > z_end)
        return fail(LBM_EINVAL, "plane range [%d, %d) outside 0..%d", z_begin, z_end, g->nz);
    // one pass where the sweep's own rho / u ARE the readout's: the readout
    // is Guo-shifted exactly when the sweep is, by the same shift
    auto guo = [](const lbm_params_t* q) {
        return q->force_mode == LBM_FORCE_GUO || q->force_mode == LBM_FORCE_GUO_X;
    };
    const bool same = guo(p) == guo(p_moments) && (p->force_mode == LBM_FORCE_NONE || guo(p)) &&
                      (!guo(p) || (p->shift_fx == p_moments->shift_fx &&
                                   p->shift_fy == p_moments->shift_fy &&
                                   p->shift_fz == p_moments->shift_fz));
    if (same && g->real_bytes == 8) {
        cudaError_t e = unit_f64::fused_mom(g->q, p->model, p->force_mode, k, kp, src, dst, cellmask,
                                            typemask, z_begin, z_end, rho, u, bad_count, s);
        if (e != cudaErrorNotSupported) return cuda_status(e, "lbm_fused_step_moments");
    }
    // elsewhere: the readout of src, then the sweep (stream order)
    if (cellmask && typemask) {
        st = moments_range(g, p_moments, src, cellmask, typemask, 1, z_begin, z_end, rho, u,
                           bad_count, stream, "lbm_fused_step_moments");
        if (st != LBM_OK) return st;
    } else {
        return fail(LBM_EINVAL, "this lattice needs cellmask and typemask for the readout");
    }
    return lbm_fused_step(g, p, src, dst, cellmask, typemask, z_begin, z_end, stream);
}

int lbm_moments(const lbm_grid_t* g, const lbm_params_t* p, const void* src,
                const uint32_t* cellmask, const uint32_t* typemask, int stream_form, double* rho,
                double* u, int* bad_count, void* stream) {
    return moments_range(g, p, src, cellmask, typemask, stream_form, 0, g ? g->nz : 0, rho, u,
                         bad_count, stream, "lbm_moments");
}

int lbm_moments_planes(const lbm_grid_t* g, const lbm_params_t* p, const void* src,
                       const uint32_t* cellmask, const uint32_t* typemask, int stream_form, int z0,
                       int z1, double* rho, double* u, int* bad_count, void* stream) {
    return moments_range(g, p, src, cellmask, typemask, stream_form, z0, z1, rho, u, bad_count,
                         stream, "lbm_moments_planes");
}

int lbm_pack_rform(const lbm_grid_t* g, const double* dense, void* pdf, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!dense || !pdf) return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = g->real_bytes == 8 ? unit_f64::convert(g->q, 1, k, (double*)dense, pdf, s)
                                       : unit_f32::convert(g->q, 1, k, (double*)dense, pdf, s);
    return cuda_status(e, "lbm_pack_rform");
}

int lbm_unpack_rform(const lbm_grid_t* g, const void* pdf, double* dense, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!dense || !pdf) return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = g->real_bytes == 8 ? unit_f64::convert(g->q, 0, k, dense, (void*)pdf, s)
                                       : unit_f32::convert(g->q, 0, k, dense, (void*)pdf, s);
    return cuda_status(e, "lbm_unpack_rform");
}

int lbm_fill_equilibrium(const lbm_grid_t* g, const double* rho, const double* u, void* pdf,
                         void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!rho || !u || !pdf) return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = g->real_bytes == 8 ? unit_f64::fill_eq(g->q, k, rho, u, pdf, s)
                                       : unit_f32::fill_eq(g->q, k, rho, u, pdf, s);
    return cuda_status(e, "lbm_fill_equilibrium");
}

int lbm_fill_equilibrium_planes(const lbm_grid_t* g, const double* rho, const double* u, int z0,
                                int z1, void* pdf, void* pdf_shell, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!rho || !u || !pdf) return fail(LBM_EINVAL, "NULL buffer");
    if (pdf == pdf_shell) return fail(LBM_EINVAL, "pdf_shell must be the other field");
    if (z0 < 0 || z1 > g->nz || z0 > z1) return fail(LBM_EINVAL, "bad plane range [%d, %d)", z0, z1);
    // ghost-inclusive planes: interior z0..z1-1 are zg = z0+1 .. z1, plus the
    // z ghost planes at either end of the box
    const int zg0 = z0 == 0 ? 0 : z0 + 1;
    const int zg1 = z1 == g->nz ? g->nz + 2 : z1 + 1;
    if (z0 == z1) return LBM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::fill_eq_dense(g->q, k, rho, u, zg0, zg1, pdf, pdf_shell, s)
                        : unit_f32::fill_eq_dense(g->q, k, rho, u, zg0, zg1, pdf, pdf_shell, s);
    return cuda_status(e, "lbm_fill_equilibrium_planes");
}

int lbm_fill_collide_planes(const lbm_grid_t* g, const lbm_params_t* p, const double* rho,
                            const double* u, int z0, int z1, void* pdf, void* pdf_shell,
                            const uint32_t* cellmask, void* stream) {
    KGrid k;
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if ((st = check_params(p, g->q, &kp, s, g->real_bytes)) != LBM_OK) return st;
    if (!rho || !u || !pdf || !cellmask) return fail(LBM_EINVAL, "NULL buffer");
    if (pdf == pdf_shell) return fail(LBM_EINVAL, "pdf_shell must be the other field");
    if (z0 < 0 || z1 > g->nz || z0 > z1) return fail(LBM_EINVAL, "bad plane range [%d, %d)", z0, z1);
    if (z0 == z1) return LBM_OK;
    const int zg0 = z0 == 0 ? 0 : z0 + 1;
    const int zg1 = z1 == g->nz ? g->nz + 2 : z1 + 1;
    cudaError_t e = g->real_bytes == 8
                        ? unit_f64::fill_collide(g->q, p->model, p->force_mode, k, kp, rho, u, zg0,
                                                 zg1, pdf, pdf_shell, cellmask, s)
                        : unit_f32::fill_collide(g->q, p->model, p->force_mode, k, kp, rho, u, zg0,
                                                 zg1, pdf, pdf_shell, cellmask, s);
    return cuda_status(e, "lbm_fill_collide_planes");
}

int lbm_build_cellmask(const lbm_grid_t* g, const uint32_t* flags, const uint32_t bits[5],
                       uint32_t* cellmask, uint32_t* typemask, int* err, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!flags || !bits || !cellmask || !typemask || !err) return fail(LBM_EINVAL, "NULL buffer");
    MaskBits b{bits[0], bits[1], bits[2], bits[3], bits[4], 0};
    b.known = b.fluid | b.noslip | b.ubb | b.pressure | b.solid;
    cudaStream_t s = (cudaStream_t)stream;
    dim3 blk = cell_block(g->nx);
    dim3 grid((g->nx + blk.x - 1) / blk.x, g->ny, g->nz);
    cudaError_t e = by_q(g->q, [&](auto Qc) {
        k_build_mask<decltype(Qc)::value><<<grid, blk, 0, s>>>(k, flags, b, cellmask, typemask, err);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_build_cellmask");
}

int64_t lbm_linkbits_words(const lbm_grid_t* g) {
    KGrid k;
    if (check_grid(g, &k) != LBM_OK) return -1;
    return (int64_t)(g->nz + 2) * (g->ny + 2) * ((g->nx + 31) / 32);
}

int lbm_build_linkbits(const lbm_grid_t* g, const uint32_t* cellmask, uint64_t* linkbits,
                       int* mismatch, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!cellmask || !linkbits || !mismatch) return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t words = (int64_t)(g->nz + 2) * (g->ny + 2) * ((g->nx + 31) / 32);
    cudaError_t e = cudaMemsetAsync(linkbits, 0, (size_t)words * sizeof(uint64_t), s);
    if (e != cudaSuccess) return cuda_status(e, "lbm_build_linkbits");
    dim3 blk = cell_block(g->nx);
    dim3 grid((g->nx + blk.x - 1) / blk.x, g->ny, g->nz);
    e = by_q(g->q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        k_linkbits_set<Q><<<grid, blk, 0, s>>>(k, cellmask, linkbits);
        k_linkbits_check<Q><<<grid, blk, 0, s>>>(k, cellmask, linkbits, mismatch);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_build_linkbits");
}

int lbm_map_spheres(int n_blocks, const int32_t cells[3], const double* frame, const int32_t* first,
                    const double* spheres, const int64_t* uids, const uint32_t* flags,
                    uint32_t fluid_bits, int64_t* owner, void* stream) {
    if (n_blocks < 0 || !cells || cells[0] < 1 || cells[1] < 1 || cells[2] < 1)
        return fail(LBM_EINVAL, "bad block geometry");
    if (n_blocks == 0) return LBM_OK;
    if (!frame || !first || !owner) return fail(LBM_EINVAL, "NULL buffer");
    const int X = cells[0] + 2, Y = cells[1] + 2, Z = cells[2] + 2;
    if (Y > 65535 || (int64_t)Z * n_blocks > 65535)
        return fail(LBM_EINVAL, "block grid too large for one launch");
    cudaStream_t s = (cudaStream_t)stream;
    dim3 blk = cell_block(X);
    dim3 grid((X + blk.x - 1) / blk.x, Y, Z * n_blocks);
    k_map_spheres<<<grid, blk, 0, s>>>(cells[0], cells[1], cells[2], frame, first, spheres, uids,
                                       flags, fluid_bits, owner);
    return cuda_status(cudaGetLastError(), "lbm_map_spheres");
}

int lbm_refresh_fluid_mask(const lbm_grid_t* g, const uint32_t* flags, const uint32_t bits[5],
                           const uint32_t* cellmask_in, uint32_t* cellmask_out, int* err,
                           void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!flags || !bits || !cellmask_in || !cellmask_out || !err)
        return fail(LBM_EINVAL, "NULL buffer");
    const uint32_t known = bits[0] | bits[1] | bits[2] | bits[3] | bits[4];
    cudaStream_t s = (cudaStream_t)stream;
    dim3 blk = cell_block(g->nx);
    dim3 grid((g->nx + blk.x - 1) / blk.x, g->ny, g->nz);
    k_refresh_fluid<<<grid, blk, 0, s>>>(k, flags, bits[0], known, cellmask_in, cellmask_out, err);
    return cuda_status(cudaGetLastError(), "lbm_refresh_fluid_mask");
}

int lbm_build_moving_masks(const lbm_grid_t* g, const uint32_t* cellmask_in, const int32_t* owner,
                           uint32_t* cellmask_out, uint32_t* linkmask, int* n_links, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!cellmask_in || !owner || !cellmask_out || !linkmask || !n_links)
        return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    dim3 blk = cell_block(g->nx);
    dim3 grid((g->nx + blk.x - 1) / blk.x, g->ny, g->nz);
    cudaError_t e = by_q(g->q, [&](auto Qc) {
        k_moving_masks<decltype(Qc)::value><<<grid, blk, 0, s>>>(k, cellmask_in, owner, cellmask_out,
                                                                 linkmask, n_links);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_build_moving_masks");
}

int lbm_collide_cells(int q, const lbm_params_t* p, double* f, int64_t n, void* stream) {
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    if (!q_ok(q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", q);
    if (!p) return fail(LBM_EINVAL, "params is NULL");
    if (p->model == LBM_MRT) {
        if (!p->mrt) return fail(LBM_EINVAL, "MRT needs its tables");
        cudaError_t e = set_mrt_tables_capi(q, p->mrt, s);
        if (e != cudaSuccess) return cuda_status(e, "MRT tables");
    }
    lbm_params_t copy = *p;
    copy.model = p->model == LBM_MRT ? LBM_SRT : p->model;  // tables already set above
    int st = check_params(&copy, q, &kp, s, 8);
    if (st != LBM_OK) return st;
    if (n <= 0) return LBM_OK;
    if (!f) return fail(LBM_EINVAL, "NULL buffer");
    const int threads = 128;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    cudaError_t e = by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        const int m = p->model, fm = p->force_mode == LBM_FORCE_GUO_X ? LBM_FORCE_GUO : p->force_mode;
        if (m == 0 && fm == 0) k_collide_cells<Q, 0, 0><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 0 && fm == 1) k_collide_cells<Q, 0, 1><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 0 && fm == 2) k_collide_cells<Q, 0, 2><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 1 && fm == 0) k_collide_cells<Q, 1, 0><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 1 && fm == 1) k_collide_cells<Q, 1, 1><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 2 && fm == 0) k_collide_cells<Q, 2, 0><<<blocks, threads, 0, s>>>(kp, f, n);
        else if (m == 2 && fm == 1) k_collide_cells<Q, 2, 1><<<blocks, threads, 0, s>>>(kp, f, n);
        else return cudaErrorInvalidValue;
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_collide_cells");
}

int lbm_equilibrium_cells(int q, const double* rho, const double* u, double* f, int64_t n,
                          void* stream) {
    if (!q_ok(q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", q);
    if (n <= 0) return LBM_OK;
    if (!rho || !u || !f) return fail(LBM_EINVAL, "NULL buffer");
    cudaStream_t s = (cudaStream_t)stream;
    const int threads = 128;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    cudaError_t e = by_q(q, [&](auto Qc) {
        k_equilibrium_cells<decltype(Qc)::value><<<blocks, threads, 0, s>>>(rho, u, f, n);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_equilibrium_cells");
}

int lbm_macroscopic_cells(int q, const lbm_params_t* p, const double* f, double* rho, double* u,
                          int* bad_count, int64_t n, void* stream) {
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    if (!q_ok(q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", q);
    if (!p) return fail(LBM_EINVAL, "params is NULL");
    lbm_params_t copy = *p;
    copy.model = LBM_SRT;
    if (copy.force_mode == LBM_FORCE_SHIFT) copy.force_mode = LBM_FORCE_NONE;
    int st = check_params(&copy, q, &kp, s, 8);
    if (st != LBM_OK) return st;
    if (n <= 0) return LBM_OK;
    if (!f || !rho || !u || !bad_count) return fail(LBM_EINVAL, "NULL buffer");
    const int threads = 128;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    const int guo = p->force_mode == LBM_FORCE_GUO || p->force_mode == LBM_FORCE_GUO_X;
    cudaError_t e = by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        if (guo) k_macroscopic_cells<Q, 1><<<blocks, threads, 0, s>>>(kp, f, rho, u, bad_count, n);
        else k_macroscopic_cells<Q, 0><<<blocks, threads, 0, s>>>(kp, f, rho, u, bad_count, n);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_macroscopic_cells");
}

int lbm_copy_shell(const lbm_grid_t* g, const void* src, void* dst, void* stream) {
    KGrid k;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    if (!src || !dst) return fail(LBM_EINVAL, "NULL buffer");
    if (src == dst) return LBM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    dim3 grid(64, g->q, g->nz + 2);
    if (g->real_bytes == 8)
        k_copy_shell<uint64_t><<<grid, 256, 0, s>>>(k, g->q, (const uint64_t*)src, (uint64_t*)dst);
    else
        k_copy_shell<uint32_t><<<grid, 256, 0, s>>>(k, g->q, (const uint32_t*)src, (uint32_t*)dst);
    return cuda_status(cudaGetLastError(), "lbm_copy_shell");
}

int lbm_bind_params(const lbm_grid_t* g, const lbm_params_t* p, void* stream) {
    KGrid k;
    KParams kp;
    int st = check_grid(g, &k);
    if (st != LBM_OK) return st;
    return check_params(p, g->q, &kp, (cudaStream_t)stream, g->real_bytes);
}

int lbm_slot_collide(int q, const lbm_params_t* p, double* f, const uint32_t* flags,
                     uint32_t fluid_bits, int64_t n, void* stream) {
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    if (!q_ok(q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", q);
    if (!p) return fail(LBM_EINVAL, "params is NULL");
    if (p->model == LBM_MRT) {
        if (!p->mrt) return fail(LBM_EINVAL, "MRT needs its tables");
        cudaError_t e = set_mrt_tables_capi(q, p->mrt, s);
        if (e != cudaSuccess) return cuda_status(e, "MRT tables");
    }
    lbm_params_t copy = *p;
    if (p->model == LBM_MRT) copy.model = LBM_SRT;   // tables already set above
    int st = check_params(&copy, q, &kp, s, 8);
    if (st != LBM_OK) return st;
    if (n <= 0) return LBM_OK;
    if (!f || !flags) return fail(LBM_EINVAL, "NULL buffer");
    const int threads = 128;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    const double* om = p->omega_cells;
    cudaError_t e = by_q(q, [&](auto Qc) {
        constexpr int Q = decltype(Qc)::value;
        const int m = p->model == LBM_SRT_FIELD ? 4 : p->model;
        const int fm = p->force_mode;
#define LBM_SLOT(M, F)                                                                        \
    if (m == M && fm == F) {                                                                  \
        k_slot_collide<Q, M, F><<<blocks, threads, 0, s>>>(kp, f, flags, fluid_bits, om, n);  \
        return cudaGetLastError();                                                            \
    }
        LBM_SLOT(0, 0) LBM_SLOT(0, 1) LBM_SLOT(0, 2) LBM_SLOT(0, 3)
        LBM_SLOT(1, 0) LBM_SLOT(1, 1) LBM_SLOT(1, 3)
        LBM_SLOT(2, 0) LBM_SLOT(2, 1) LBM_SLOT(2, 3)
        LBM_SLOT(4, 0) LBM_SLOT(4, 1) LBM_SLOT(4, 3)
#undef LBM_SLOT
        return cudaErrorInvalidValue;
    });
    return cuda_status(e, "lbm_slot_collide");
}

int lbm_slot_apply_links(int q, const lbm_params_t* p, const int32_t* kind, const int32_t* dir,
                         const int64_t* cell, int64_t n_links, const double* src, double* dst,
                         void* stream) {
    KParams kp;
    cudaStream_t s = (cudaStream_t)stream;
    if (!q_ok(q)) return fail(LBM_EINVAL, "q must be 9, 19 or 27, got %d", q);
    if (!p) return fail(LBM_EINVAL, "params is NULL");
    lbm_params_t copy = *p;
    copy.model = LBM_SRT;
    copy.force_mode = LBM_FORCE_NONE;
    copy.mrt = nullptr;
    copy.moving = nullptr;
    int st = check_params(&copy, q, &kp, s, 8);
    if (st != LBM_OK) return st;
    if (n_links <= 0) return LBM_OK;
    if (!kind || !dir || !cell || !src || !dst) return fail(LBM_EINVAL, "NULL buffer");
    const int threads = 128;
    const unsigned blocks = (unsigned)((n_links + threads - 1) / threads);
    cudaError_t e = by_q(q, [&](auto Qc) {
        k_apply_links<decltype(Qc)::value><<<blocks, threads, 0, s>>>(kp, kind, dir, cell, src, dst,
                                                                     n_links);
        return cudaGetLastError();
    });
    return cuda_status(e, "lbm_slot_apply_links");
}

int lbm_slot_stream_pull(int q, const int32_t* cx, const int32_t* cy, const int32_t* cz,
                         const double* src, double* out, int nxg, int nyg, int nzg, int gl,
                         void* stream) {
    if (q < 1 || q > 27) return fail(LBM_EINVAL, "q must be 1..27, got %d", q);
    if (!cx || !cy || !cz || !src || !out) return fail(LBM_EINVAL, "NULL argument");
    if (gl < 1) return fail(LBM_EINVAL, "stream_pull needs a ghost layer, got %d", gl);
    const int nx = nxg - 2 * gl, ny = nyg - 2 * gl, nz = nzg - 2 * gl;
    SlotStencil c;
    for (int i = 0; i < q; ++i) {
        if (cx[i] < -gl || cx[i] > gl || cy[i] < -gl || cy[i] > gl || cz[i] < -gl || cz[i] > gl)
            return fail(LBM_EINVAL, "velocity %d reaches past %d ghost layer(s)", i, gl);
        c.cx[i] = cx[i];
        c.cy[i] = cy[i];
        c.cz[i] = cz[i];
    }
    if (nx <= 0 || ny <= 0 || nz <= 0) return LBM_OK;
    if (ny > 65535 || nz > 65535) return fail(LBM_EINVAL, "ny/nz too large for the launch grid");
    cudaStream_t s = (cudaStream_t)stream;
    dim3 blk = cell_block(nx);
    dim3 grid((nx + blk.x - 1) / blk.x, ny, nz);
    k_slot_stream_pull<<<grid, blk, 0, s>>>(c, q, src, out, nxg, nyg, gl, nx, ny, nz);
    return cuda_status(cudaGetLastError(), "lbm_slot_stream_pull");
}

}  // extern "C"
