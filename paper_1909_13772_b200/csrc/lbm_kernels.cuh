// LBM sweep kernels for sm_100a (templated; instantiated in lbm_inst_*.cu).
//
// State on the device is the post-collision "G-form" G_n = C(R_n) where R_n is
// the reference's stored state after n calls of stream_collide
// (lbm/sweep.py:93-151: collide src in place -> stream_pull -> boundary
// links -> swap).  One reference step R_{n+1} = S(C(R_n)) is re-bracketed as
// G_{n+1} = C(S(G_n)): pull, bounce-back and collision of a cell happen in one
// pass over HBM (2 q sizeof(real) bytes per cell + a 4-byte cell mask).
//
// Pull sources follow the reference's ghost semantics exactly:
//   * a source inside the box is read directly;
//   * a source on a periodic axis owned by this rank wraps (the reference's
//     periodic self-exchange, field/ghost.py:112-124);
//   * a source in a z ghost plane filled by the per-step exchange is read
//     from that plane (x/y wrapped inside it like any interior plane);
//   * a source outside the domain on a non-periodic axis ("uncovered") is
//     the ghost cell itself at its raw index - the reference never writes
//     those (exchange targets only images of the interior) so they keep the
//     value written at fill time.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lbm_b200.h"
#include "lbm_collide.cuh"
#include "lbm_collide_f32.cuh"

namespace lbm {

struct KGrid {
    int nx, ny, nz, pitch, xoff;
    int wrap_x, wrap_y, zlo, zhi;  // zlo/zhi: LBM_ZFACE_*
    int64_t plane;                 // (ny+2) * pitch
    int64_t zstride;               // q * plane
    int plane32, zstride32;        // the same as int (check_grid range-checks every delta)
    int link_hint;                 // bit 0: z-planes large against L2 (see ldg_keep);
                                   // bits 1..: cell-mask rows prefetched ahead (prefetch_mask)
    // own-relative element deltas, indexed by reference direction i (host-computed):
    int dpull[27];   // source of the pull of direction i: slot(i) plane - c_i . (1, pitch, zstride)
    int dlink[27];   // bounce-back source: own cell, slot(opp(i)) plane
    int dslot[27];   // slot(i) plane (stores)
};

// Opaque copy of a pointer: keeps `base + int32 delta` as one wide
// multiply-add per access instead of a re-associated 64-bit index sum.
template <typename T>
__device__ __forceinline__ T* opaque(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}

template <typename Real>
struct Store;
// fp64: stored as is
template <>
struct Store<double> {
    template <int Q, int I>
    __device__ __forceinline__ static double widen(double v) { return v; }
    template <int Q, int I>
    __device__ __forceinline__ static double load(const double* p) { return __ldg(p); }
    template <int Q, int I>
    __device__ __forceinline__ static void store(double* p, double v) { *p = v; }
};
// fp32: stored zero-centred (f - w_i).  These widening accessors serve the
// fp64-register readout kernels (stream-only, moments, convert); the fused
// and collide-only kernels keep fp32 registers (AccOf<float>, lbm_collide_f32.cuh)
template <>
struct Store<float> {
    template <int Q, int I>
    __device__ __forceinline__ static double widen(float v) { return (double)v + wt<Q, I>(); }
    template <int Q, int I>
    __device__ __forceinline__ static double load(const float* p) {
        return (double)__ldg(p) + wt<Q, I>();
    }
    template <int Q, int I>
    __device__ __forceinline__ static void store(float* p, double v) {
        *p = (float)(v - wt<Q, I>());
    }
};

// read-only load whose line should survive in L2 until a second reader
// (L2 evict_last policy).  Used by the fp64 pulls only: measured on B200,
// config 4 fp64 92.8 -> 94.6 % of the roofline; fp32 storage -4.7 % and
// config 2 -3.7 % (the split loads cost issue slots those kernels lack).
// -DLBM_LINK_HINT=0|1 forces it off / on for every storage type.
template <typename Real>
constexpr bool link_hint() {
#ifdef LBM_LINK_HINT
    return LBM_LINK_HINT != 0;
#else
    return std::is_same_v<Real, double>;
#endif
}
template <typename T>
__device__ __forceinline__ T ldg_keep(const T* p) {
    if constexpr (sizeof(T) == 8) {
        double v;
        asm volatile("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                     "ld.global.nc.L2::cache_hint.f64 %0, [%1], pol;\n}" : "=d"(v) : "l"(p));
        return (T)v;
    } else {
        float v;
        asm volatile("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                     "ld.global.nc.L2::cache_hint.f32 %0, [%1], pol;\n}" : "=f"(v) : "l"(p));
        return (T)v;
    }
}

// L2 prefetch of the cell-mask words `rows` rows ahead of this cell (same
// x, plane order): the block that reads them is launched about one resident
// window later, so its mask load - which every pull address waits on - hits
// L2 instead of paying a DRAM round trip.
__device__ __forceinline__ void prefetch_mask(const KGrid& g, const uint32_t* cellmask, int64_t cell,
                                              int64_t ncells) {
    const int ahead = g.link_hint >> 1;
    if (ahead > 0 && cellmask) {
        const int64_t c = cell + (int64_t)ahead * g.nx;
        if (c < ncells) asm volatile("prefetch.global.L2 [%0];" ::"l"(cellmask + c));
    }
}

// ---------------------------------------------------------------- link bits
// A NoSlip-only lattice's cell mask is a function of one bit per cell: with
// N(c) = "c is not collided and a fluid neighbour pulling from it takes a
// bounce-back link", code(x) = 0 if N(x), else FLUID | sum_i N(x - c_i) << i.
// The link-bit map (lbm_build_linkbits) stores N over the ghost-inclusive box
// as uint64 words [(zg * (ny + 2) + yg) * bw + w], bw = ceil(nx / 32): bit b of
// word w is cell xg = 32 w + b.  Consecutive words overlap by 32 cells, so the
// 34 cells a warp of 32 reads (x - 1 .. x + 32) sit in ONE word per row and
// every lane of the warp loads the same address (one broadcast per row).  At
// 512^3 the map is 34 MB (0.25 B per cell) against the 4 B/cell mask; the
// map is built only when the derivation reproduces the full mask on every
// cell (typed links, flags edited after freeze() etc. keep the mask).
template <int Q>
constexpr bool bits_row_used(int dz, int dy) {
    for (int i = 0; i < Q; ++i)
        if (-Dirs<Q>::cz[i] == dz && -Dirs<Q>::cy[i] == dy) return true;
    return false;
}

// link-bit words are re-read by the rows y +- 1 / planes z +- 1 of the sweep,
// about two planes of field traffic later: keep them in L2 (evict_last)
__device__ __forceinline__ uint64_t ldg_bits(const uint64_t* p) {
    uint64_t v;
    asm("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
        "ld.global.nc.L2::cache_hint.u64 %0, [%1], pol;\n}" : "=l"(v) : "l"(p));
    return v;
}

// With the map, a fused kernel works on the NEIGHBOURHOOD word of a cell
// instead of the mask's code: bits 3 r + b, row r = (dz + 1) * 3 + (dy + 1),
// b = 0..2 for x - 1 .. x + 1, hold N of the 27 cells around it.  Direction
// i's link is then bit nb_pos(i) = the bit of x - c_i, and the cell itself
// (bit 13) replaces LBM_MASK_FLUID: code = N(x) ? 0 : nb | bit 13.  Building
// it costs one funnel shift + one bit-field insert per row (no per-direction
// gather); CodeBits<Q, BITS> tells the pull which bit is whose.
template <int Q>
__host__ __device__ constexpr int nb_pos(int i) {
    return 3 * ((1 - Dirs<Q>::cz[i]) * 3 + (1 - Dirs<Q>::cy[i])) + 1 - Dirs<Q>::cx[i];
}
constexpr uint32_t kNbCentre = 1u << 13;

template <int Q, bool BITS>
struct CodeBits {
    static constexpr uint32_t fluid = BITS ? kNbCentre : LBM_MASK_FLUID;
    __host__ __device__ static constexpr int link(int i) { return BITS ? nb_pos<Q>(i) : i; }
};

// bits x .. x + 2 of row word v (lane offset l = x & 31) inserted at 3 r
template <int R>
__device__ __forceinline__ uint32_t nb_insert(uint32_t nb, uint64_t v, int l) {
    const uint32_t s = __funnelshift_r((uint32_t)v, (uint32_t)(v >> 32), l);
    uint32_t d;
    asm("bfi.b32 %0, %1, %2, %3, 3;" : "=r"(d) : "r"(s), "r"(nb), "n"(3 * R));
    return d;
}

__device__ __forceinline__ uint32_t nb_code(uint32_t nb) {
    return (nb & kNbCentre) ? 0u : (nb | kNbCentre);
}

// address of the word holding cell (x - 1 .. x + 1, y, z) of the map
__device__ __forceinline__ const uint64_t* bits_row(const KGrid& g, const uint64_t* bits, int x,
                                                    int y, int z) {
    const int64_t bw = (g.nx + 31) >> 5;
    return bits + ((int64_t)(z + 1) * (g.ny + 2) + (y + 1)) * bw + (x >> 5);
}

// L2 prefetch of the map word `ahead` rows (of the plane-major row order)
// after `w`: the words a block reads first-hand are those of the planes no
// earlier block touched; the blocks `ahead` rows later read these.
__device__ __forceinline__ void prefetch_bits(const KGrid& g, const uint64_t* w,
                                              const uint64_t* end) {
    const int ahead = g.link_hint >> 1;
    if (ahead > 0) {
        const uint64_t* q = w + (int64_t)ahead * ((g.nx + 31) >> 5);
        if (q < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
    }
}

template <int Q>
__device__ __forceinline__ uint32_t code_from_bits(const KGrid& g, const uint64_t* __restrict__ bits,
                                                   int x, int y, int z) {
    const int64_t bw = (g.nx + 31) >> 5;
    const int64_t ps = (int64_t)(g.ny + 2) * bw;
    const uint64_t* c = bits_row(g, bits, x, y, z);
    const int l = x & 31;
    uint64_t v[9];
    static_for<0, 9>([&](auto R_) {
        constexpr int r = decltype(R_)::value;
        v[r] = ldg_bits(c + (r / 3 - 1) * ps + (r % 3 - 1) * bw);
    });
    prefetch_bits(g, c + ps + bw, bits + (int64_t)(g.nz + 2) * ps);
    uint32_t nb = 0u;
    static_for<0, 9>([&](auto R_) {
        constexpr int r = decltype(R_)::value;
        nb = nb_insert<r>(nb, v[r], l);
    });
    return nb_code(nb);
}

// the cell-mask code a neighbourhood word stands for (the map's device check)
template <int Q>
__device__ __forceinline__ uint32_t mask_code_of_nb(uint32_t code) {
    if (!(code & kNbCentre)) return 0u;
    uint32_t m = LBM_MASK_FLUID;
    static_for<1, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        m |= ((code >> nb_pos<Q>(i)) & 1u) << i;
    });
    return m;
}

// the cell code a fused kernel works with: full mask, neighbourhood word or none
template <int Q, bool BITS>
__device__ __forceinline__ uint32_t cell_code(const KGrid& g, const uint32_t* __restrict__ cellmask,
                                              int x, int y, int z, int64_t cell) {
    if constexpr (BITS) return code_from_bits<Q>(g, reinterpret_cast<const uint64_t*>(cellmask), x, y, z);
    else return cellmask ? __ldg(cellmask + cell) : LBM_MASK_FLUID;
}

// both cells of a z-pair (za, za + 1) from the 12 words of planes
// za - 1 .. za + 2 (k_fused_z2)
template <int Q>
__device__ __forceinline__ void codes_from_bits_z2(const KGrid& g, const uint64_t* __restrict__ bits,
                                                   int x, int y, int za, bool two, uint32_t& ca,
                                                   uint32_t& cb) {
    const int64_t bw = (g.nx + 31) >> 5;
    const int64_t ps = (int64_t)(g.ny + 2) * bw;
    const uint64_t* c = bits_row(g, bits, x, y, za);
    const int l = x & 31;
    uint64_t v[12];
    static_for<0, 12>([&](auto R_) {
        constexpr int r = decltype(R_)::value;
        if (r < 9 || two) v[r] = ldg_bits(c + (r / 3 - 1) * ps + (r % 3 - 1) * bw);
        else v[r] = 0;
    });
    {   // the two planes this block reads first-hand
        const uint64_t* end = bits + (int64_t)(g.nz + 2) * ps;
        prefetch_bits(g, c + ps + bw, end);
        prefetch_bits(g, c + 2 * ps + bw, end);
    }
    uint32_t na = 0u, nb = 0u;
    static_for<0, 9>([&](auto R_) {
        constexpr int r = decltype(R_)::value;
        na = nb_insert<r>(na, v[r], l);
        nb = nb_insert<r>(nb, v[r + 3], l);
    });
    ca = nb_code(na);
    cb = two ? nb_code(nb) : 0u;
}

// (Measured and dropped: L2::128B / L2::256B prefetch-size qualifiers on the
// pulls - within noise on configs 4 fp64 / fp32 and 2.)
// (Measured and dropped: choosing the keep policy per warp - any wall lane
// or link in the warp - so each direction stays one load instruction: the
// extra evict_last lines cost 9 % in fp32 and nothing was gained in fp64.)
// per-axis source coordinate for a pull along -c (c in {-1,0,1})
struct AxisSrc {
    int lo_raw, hi_raw;    // coordinate - 1, coordinate + 1 (ghost-inclusive: may be -1 / n)
    int lo_w, hi_w;        // wrapped (or raw when the axis does not wrap)
    bool lo_unc, hi_unc;   // source outside the domain on a non-periodic axis
};

__device__ __forceinline__ AxisSrc make_axis(int c, int n, bool wrap, bool lo_unc_face,
                                             bool hi_unc_face) {
    AxisSrc a;
    a.lo_raw = c - 1;
    a.hi_raw = c + 1;
    a.lo_w = (c == 0 && wrap) ? n - 1 : c - 1;
    a.hi_w = (c == n - 1 && wrap) ? 0 : c + 1;
    a.lo_unc = (c == 0) && lo_unc_face;
    a.hi_unc = (c == n - 1) && hi_unc_face;
    return a;
}

// offset of direction I's slot within a cell's z-plane block.  (A "write-
// shifted" row layout, f_i(x) stored at x + c_x(i) so that every pull is
// 128-byte aligned and only stores straddle sectors, was measured on B200 and
// rejected: config 4 fp64 90.0 % vs 92.9 %, config 2 fp32 74 % vs 85 %.)
template <int Q, int I>
__device__ __forceinline__ int64_t dir_off(const KGrid& g) {
    return (int64_t)slot_of<Q>(I) * g.plane;
}

// element offset (relative to the field base) of (z, slot, y, x)
__device__ __forceinline__ int64_t lidx(const KGrid& g, int z, int slot, int y, int x) {
    return (int64_t)(z + 1) * g.zstride + (int64_t)slot * g.plane + (int64_t)(y + 1) * g.pitch +
           g.xoff + x;
}

// Pressure anti-bounce-back for the pulled directions in `pm`
// (boundary.py:171-195): rho, u from the cell's own post-collision state
// (sequential sums, u = m / rho), then
//   R[x, i] = -G[x, k] + (2 w_k rho_w) ((1 + (4.5 cu) cu) - 1.5 usq),  k = opp(i).
template <int Q, typename Real, typename Acc>
__device__ __forceinline__ void pressure_links(const KGrid& g, const KParams& p,
                                            const Real* __restrict__ src, int64_t own,
                                            uint32_t pm, Acc (&f)[Q]) {
    using D = Dirs<Q>;
    double c[Q];
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        c[i] = Store<Real>::template load<Q, i>(src + own + dir_off<Q, i>(g));
    });
    double rho = c[0];
#pragma unroll
    for (int k = 1; k < Q; ++k) rho = rho + c[k];
    double mx = 0.0, my = 0.0, mz = 0.0;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        if constexpr (D::cx[i] == 1) mx = mx + c[i];
        if constexpr (D::cx[i] == -1) mx = mx - c[i];
        if constexpr (D::cy[i] == 1) my = my + c[i];
        if constexpr (D::cy[i] == -1) my = my - c[i];
        if constexpr (D::cz[i] == 1) mz = mz + c[i];
        if constexpr (D::cz[i] == -1) mz = mz - c[i];
    });
    const double ux = mx / rho, uy = my / rho, uz = mz / rho;
    const double usq15 = 1.5 * ((ux * ux + uy * uy) + uz * uz);
    static_for<1, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        constexpr int k = D::opp[i];
        if ((pm >> i) & 1u) {
            const double cu = cu_of<Q, k>(ux, uy, uz);
            const double v = -c[k] + p.pw[k] * ((1.0 + (4.5 * cu) * cu) - usq15);
            if constexpr (std::is_same_v<Acc, double>) f[i] = v;
            else f[i] = (float)(v - wt<Q, i>());  // fp32 path: centred
        }
    });
}

// Moving-body walls (coupling/sweep.py:113-143) on the pulled directions of
// p.mv_link: the link (x, i = opp(j)) points into a covered cell; the pulled
// value becomes G[x, i] - ((6 w_i) rho0) (c_i . u_w) with u_w the body's
// surface velocity at the link midpoint x + c_i / 2, in the reference's
// operation order (fp64, every op rounded); FORCES adds the momentum
// dp = 2 G[x, i] - corr and its torque to the (block, body) accumulators.
template <int Q, typename Acc, bool FORCES>
__device__ __forceinline__ void moving_links(const KGrid& g, const KParams& p, int x, int y, int z,
                                             int64_t cell, Acc (&f)[Q]) {
    using D = Dirs<Q>;
    const uint32_t lm = __ldg(p.mv_link + cell);
    const int bx = x / p.mv_cx, by = y / p.mv_cy, bz = z / p.mv_cz;
    const int blk = (bz * p.mv_by + by) * p.mv_bx + bx;
    const double* c0 = p.mv_cell0 + 3 * blk;
    const double px = c0[0] + (double)(x - bx * p.mv_cx);
    const double py = c0[1] + (double)(y - by * p.mv_cy);
    const double pz = c0[2] + (double)(z - bz * p.mv_cz);
    const int X = g.nx + 2, Y = g.ny + 2;
    double fa[3] = {0.0, 0.0, 0.0}, ta[3] = {0.0, 0.0, 0.0};
    int last = -1;
    static_for<1, Q>([&](auto J_) {
        constexpr int j = decltype(J_)::value;
        constexpr int i = D::opp[j];
        constexpr double ci0 = D::cx[i], ci1 = D::cy[i], ci2 = D::cz[i];
        if ((lm >> j) & 1u) {
            const int slot = __ldg(p.mv_owner + ((int64_t)(z + 1 + D::cz[i]) * Y + (y + 1 + D::cy[i])) * X +
                                   (x + 1 + D::cx[i]));
            const int bi = blk * p.mv_slots + slot;
            const double* b = p.mv_bodies + 9 * bi;
            const double rx = (px + 0.5 * ci0) - b[0];
            const double ry = (py + 0.5 * ci1) - b[1];
            const double rz = (pz + 0.5 * ci2) - b[2];
            const double uwx = (b[3] + b[7] * rz) - b[8] * ry;
            const double uwy = (b[4] + b[8] * rx) - b[6] * rz;
            const double uwz = (b[5] + b[6] * ry) - b[7] * rx;
            const double cu = (ci0 * uwx + ci1 * uwy) + ci2 * uwz;
            const double corr = ((6.0 * wt<Q, i>()) * p.mv_rho0) * cu;
            double fi;
            if constexpr (std::is_same_v<Acc, double>) fi = f[j];
            else fi = (double)f[j] + wt<Q, i>();
            if constexpr (std::is_same_v<Acc, double>) f[j] = fi - corr;
            else f[j] = (float)((fi - corr) - wt<Q, j>());
            if constexpr (FORCES) {
                if (p.mv_forces) {
                    if (last >= 0 && last != bi) {   // a second body at this cell: flush
                        double* acc = p.mv_forces + 6 * last;
                        for (int k = 0; k < 3; ++k) {
                            atomicAdd(acc + k, fa[k]);
                            atomicAdd(acc + 3 + k, ta[k]);
                            fa[k] = ta[k] = 0.0;
                        }
                    }
                    last = bi;
                    const double dp = 2.0 * fi - corr;
                    fa[0] += ci0 * dp;
                    fa[1] += ci1 * dp;
                    fa[2] += ci2 * dp;
                    ta[0] += (ry * ci2 - rz * ci1) * dp;
                    ta[1] += (rz * ci0 - rx * ci2) * dp;
                    ta[2] += (rx * ci1 - ry * ci0) * dp;
                }
            }
        }
    });
    if constexpr (FORCES) {
        if (last >= 0) {
            double* acc = p.mv_forces + 6 * last;
            for (int k = 0; k < 3; ++k) {
                atomicAdd(acc + k, fa[k]);
                atomicAdd(acc + 3 + k, ta[k]);
            }
        }
    }
}

template <int Q, typename Real, typename Acc, int MV, bool TYPED = true>
__device__ __forceinline__ void pull_finish(const KGrid& g, const KParams& p,
                                            const Real* __restrict__ src, int x, int y, int z,
                                            int64_t own, uint32_t code, uint2 t, const Real (&raw)[Q],
                                            Acc (&f)[Q]);

// Load the 19/27/9 pulled populations of cell (x,y,z) with the fused
// bounce-back substitution R[x,i] = G[x,opp(i)] (- UBB term) for masked
// directions (boundary.py:163-170).
// Element offsets of the pulled sources.  GENERIC (warp-uniform: only warps
// touching a wrapping edge) applies the covered / uncovered ghost rules;
// otherwise the source is own - cz*zstride - cy*pitch - cx (+ slot plane).
template <int Q, bool GENERIC>
__device__ __forceinline__ void pull_offsets(const KGrid& g, int x, int y, int z, int64_t own,
                                             int64_t (&off)[Q]) {
    using D = Dirs<Q>;
    static_assert(GENERIC, "the fast path uses the host delta tables (KGrid::dpull)");
    {
        const AxisSrc ax = make_axis(x, g.nx, g.wrap_x, !g.wrap_x, !g.wrap_x);
        const AxisSrc ay = make_axis(y, g.ny, g.wrap_y, !g.wrap_y, !g.wrap_y);
        AxisSrc az = make_axis(z, g.nz, false, g.zlo == LBM_ZFACE_GHOST, g.zhi == LBM_ZFACE_GHOST);
        if (g.zlo == LBM_ZFACE_WRAP && z == 0) az.lo_w = g.nz - 1;
        if (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1) az.hi_w = 0;
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            constexpr int cx = D::cx[i], cy = D::cy[i], cz = D::cz[i];
            bool unc = false;
            int xs = x, ys = y, zs = z, xr = x, yr = y, zr = z;
            if constexpr (cx == 1) { xs = ax.lo_w; xr = ax.lo_raw; unc |= ax.lo_unc; }
            if constexpr (cx == -1) { xs = ax.hi_w; xr = ax.hi_raw; unc |= ax.hi_unc; }
            if constexpr (cy == 1) { ys = ay.lo_w; yr = ay.lo_raw; unc |= ay.lo_unc; }
            if constexpr (cy == -1) { ys = ay.hi_w; yr = ay.hi_raw; unc |= ay.hi_unc; }
            if constexpr (cz == 1) { zs = az.lo_w; zr = az.lo_raw; unc |= az.lo_unc; }
            if constexpr (cz == -1) { zs = az.hi_w; zr = az.hi_raw; unc |= az.hi_unc; }
            xs = unc ? xr : xs;
            ys = unc ? yr : ys;
            zs = unc ? zr : zs;
            off[i] = lidx(g, zs, 0, ys, xs) + dir_off<Q, i>(g);
        });
    }
}

// Three phases so every load of a cell is in flight at once: (1) source
// offsets with the link substitution folded in as a select, (2) all loads,
// (3) conversion + the rare UBB / Pressure corrections under one branch.
// Acc = double: widened populations f (fp64 storage, or fp32 readout);
// Acc = float (fp32 storage only): the stored centred g = f - w as is.
// MV: 0 no moving-body walls (the standard sweep kernels), 1 moving walls
// without force accumulation (readouts), 2 moving walls + forces (fused step).
// Phases 1 + 2 of a pull: source offsets (link substitution as a select)
// and all Q loads in flight.
// BITS: `code` is a neighbourhood word (code_from_bits), see CodeBits.
template <int Q, typename Real, bool BITS = false>
__device__ __forceinline__ void pull_load(const KGrid& g, const Real* __restrict__ src, int x,
                                          int y, int z, uint32_t code, bool generic,
                                          Real (&raw)[Q]) {
    using D = Dirs<Q>;
    using CB = CodeBits<Q, BITS>;
    const int64_t own = lidx(g, z, 0, y, x);
    // link: read the own cell's direction k = opp(i) instead (w_k == w_i, so
    // the fp32 zero-centring offset is the same)
    if (!generic) {
        // own-relative 32-bit element deltas: launch-uniform except for the
        // link select, so each pull costs one select + one address multiply-add
        const Real* sp = opaque(src + own);
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            int d = g.dpull[i];
            // link source = own cell, slot opp(i) (KGrid::dlink)
            if constexpr (i > 0) d = ((code >> CB::link(i)) & 1u) ? g.dlink[i] : d;
            // A bounce-back link of a fluid cell x reads G[x, opp(i)], which
            // the wall cell across the link also pulls.  For directions with
            // c_z = -1 the FIRST of the two reads is either x's link (wall one
            // plane later) or a wall cell's pull (fluid cell one plane
            // later); that read keeps the line in L2 (evict_last) for the
            // second one instead of leaving it to a whole plane of traffic.
            if constexpr (link_hint<Real>() && D::cz[i] == -1) {
                if ((g.link_hint & 1) && ((((code >> CB::link(i)) & 1u) != 0u) || !(code & CB::fluid)))
                    raw[i] = ldg_keep(sp + d);
                else
                    raw[i] = __ldg(sp + d);
            } else {
                raw[i] = __ldg(sp + d);
            }
        });
    } else {
        int64_t off[Q];
        pull_offsets<Q, true>(g, x, y, z, own, off);
        static_for<1, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            off[i] = ((code >> CB::link(i)) & 1u) ? own + dir_off<Q, D::opp[i]>(g) : off[i];
        });
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            raw[i] = __ldg(src + off[i]);
        });
    }
}

// typed-link words of a cell (read only where the cell has UBB / Pressure links)
__device__ __forceinline__ uint2 type_words(const KGrid& g, const uint32_t* __restrict__ typemask,
                                            int x, int y, int z, uint32_t code) {
    if (!(code & (LBM_MASK_UBB | LBM_MASK_PRESSURE))) return make_uint2(0u, 0u);
    return __ldg(reinterpret_cast<const uint2*>(typemask) + (((int64_t)z * g.ny + y) * g.nx + x));
}

template <int Q, typename Real, typename Acc, int MV = 0, bool BITS = false>
__device__ __forceinline__ void pull_cell(const KGrid& g, const KParams& p,
                                          const Real* __restrict__ src, int x, int y, int z,
                                          uint32_t code, const uint32_t* __restrict__ typemask,
                                          bool generic, Acc (&f)[Q]) {
    static_assert(std::is_same_v<Acc, double> || std::is_same_v<Real, float>,
                  "fp32 registers only for fp32 storage");
    const uint2 t = type_words(g, typemask, x, y, z, code);
    Real raw[Q];
    pull_load<Q, Real, BITS>(g, src, x, y, z, code, generic, raw);
    pull_finish<Q, Real, Acc, MV>(g, p, src, x, y, z, lidx(g, z, 0, y, x), code, t, raw, f);
}

// Phase 3 of a pull: widen the raw pulled values and apply the rare UBB /
// Pressure / moving-wall corrections (shared by the LDG and TMA kernels).
// TYPED = false compiles the corrections out (launches whose masks carry no
// UBB / Pressure link, where no typemask exists).
template <int Q, typename Real, typename Acc, int MV, bool TYPED>
__device__ __forceinline__ void pull_finish(const KGrid& g, const KParams& p,
                                            const Real* __restrict__ src, int x, int y, int z,
                                            int64_t own, uint32_t code, uint2 t, const Real (&raw)[Q],
                                            Acc (&f)[Q]) {
    using D = Dirs<Q>;
    constexpr uint32_t kTyped = LBM_MASK_UBB | LBM_MASK_PRESSURE | (MV ? LBM_MASK_MOVING : 0u);
    const bool typed = (code & kTyped) != 0u;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        if constexpr (std::is_same_v<Acc, double>) f[i] = Store<Real>::template widen<Q, i>(raw[i]);
        else f[i] = raw[i];
    });
    if (TYPED && typed) {
        if (t.x) {
            static_for<1, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                constexpr int k = D::opp[i];
                if constexpr (std::is_same_v<Acc, double>) {
                    if ((t.x >> i) & 1u) f[i] = f[i] - p.ubb[k];
                } else {
                    if ((t.x >> i) & 1u) f[i] = f[i] - p.fubb[k];
                }
            });
        }
        if (t.y) pressure_links<Q, Real, Acc>(g, p, src, own, t.y, f);
        if constexpr (MV != 0) {
            if (code & LBM_MASK_MOVING)
                moving_links<Q, Acc, MV == 2>(g, p, x, y, z, ((int64_t)z * g.ny + y) * g.nx + x, f);
        }
    }
}

// Fused pull -> bounce-back -> collide over interior planes [z0, z0+gridDim.z).
// Resident 128-thread blocks per SM requested from ptxas (caps registers at
// 65536 / (128 * minb)).  The kernel is latency-bound on its 19/27 pulls, so
// occupancy beats the few L1-resident spills it costs (measured on B200,
// config 4 D3Q19 TRT fp64: minb 1 -> 83 %, 5 -> 89 %, 6 -> 91.9 %,
// 7 -> 92.4 %, 8 -> 89.7 % of the HBM roofline).  MRT keeps all registers.
// -DLBM_FUSED_MINB=n overrides for tuning builds.
template <int Q, typename Real, int MODEL, int FORCE = 0>
constexpr int fused_minb() {
    if constexpr (std::is_same_v<Real, float>) {
        if constexpr (MODEL == 3) {
#ifdef LBM_FUSED_MINB_F32MRT
            return LBM_FUSED_MINB_F32MRT;
#else
            return 7;  // measured on B200 (config 2): 4 -> 68 %, 5 -> 69 %, 6 -> 74.5 %, 7 -> 75.6 %, 10 -> 45 %
#endif
        }
#ifdef LBM_FUSED_MINB_F32
        return LBM_FUSED_MINB_F32;
#else
        // D3Q19 config 4 fp32: 6 -> 74 %, 7 -> 76 %, 8 -> 80.8 %, 9 -> 82 %, 10 -> 69 %
        return MODEL == 2 ? 1 : (Q == 9 ? 8 : (Q == 19 ? 9 : 6));
#endif
    } else {
#ifdef LBM_FUSED_MINB
        return LBM_FUSED_MINB;
#else
        // D3Q19 SRT/TRT fp64: 6 (config 3, no force); with Guo 7 (config 4:
        // 6 -> 93.3 %, 7 -> 94.3 %, 5 -> 89.6 %, measured with the link hint)
        constexpr bool guo = FORCE == 1 || FORCE == 3;
        return MODEL == 2 ? 1 : (Q == 9 ? 8 : (Q == 19 ? (guo && MODEL <= 1 ? 7 : 6) : 4));
#endif
    }
}

// register type of the fused / collide-only kernels: fp32 storage computes in
// fp32 on centred populations (lbm_collide_f32.cuh), fp64 bitwise otherwise
template <typename Real>
using AccOf = std::conditional_t<std::is_same_v<Real, float>, float, double>;

template <int Q, int MODEL, int FORCE, typename Acc>
__device__ __forceinline__ void collide_any(Acc (&f)[Q], const KParams& p, int64_t cell) {
    double om = 0.0;
    if constexpr (MODEL == 4) om = __ldg(p.omega + cell);
    if constexpr (std::is_same_v<Acc, double>) collide_cell<Q, MODEL, FORCE>(f, p, om);
    else collide_cell_c32<Q, MODEL, FORCE>(f, p, om);
}

// (Measured on B200 and dropped: st.global.cs and an L2 evict_first policy on
// these stores, to keep re-read lines in L2 - within noise on configs 4 / 2,
// -1.3 % in fp32.)
template <int Q, int I, typename Real, typename Acc>
__device__ __forceinline__ void store_any(Real* p, Acc v) {
    if constexpr (std::is_same_v<Acc, double>) Store<Real>::template store<Q, I>(p, v);
    else *p = v;  // already centred fp32
}

// threads per block of the fused kernel (x extent of a block's row segment).
// Measured on B200 (config 4 / 3 / 2): 64 and 128 equal within noise, 256 -1..-9 %,
// 512 -12..-25 % (fewer resident blocks, coarser tail).
#ifndef LBM_FUSED_BX
#define LBM_FUSED_BX 128
#endif
template <int Q, typename Real, int MODEL, int FORCE = 0>
constexpr int fused_minb_bx() {
    constexpr int m = fused_minb<Q, Real, MODEL, FORCE>() * 128 / LBM_FUSED_BX;
    return m < 1 ? 1 : m;
}

// PEER: the launch carries the fused z-face halo (KParams::peer_lo / peer_hi,
// boundary planes of a multi-rank step only); a separate instantiation so
// the interior / single-rank kernels keep their register allocation.
// (Measured and rejected: visiting rows in tiles of 8..64 rows, all planes of
// a tile first, to bring the z-neighbour that re-reads a bounce-back source
// closer in time: -1..-8 % on configs 4 fp64 / fp32 and 2.)
// BITS: `cellmask` is a link-bit map (code_from_bits), not the 4 B/cell mask.
template <int Q, typename Real, int MODEL, int FORCE, bool MOVING = false, bool PEER = false,
          bool BITS = false>
__global__ void __launch_bounds__(LBM_FUSED_BX, fused_minb_bx<Q, Real, MODEL, FORCE>())
    k_fused(KGrid g, KParams p, const Real* __restrict__ src,
                                               Real* __restrict__ dst,
                                               const uint32_t* __restrict__ cellmask,
                                               const uint32_t* __restrict__ typemask, int z0) {
    using D = Dirs<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = z0 + blockIdx.z;
    const int xw0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    const bool edge_x = g.wrap_x && (xw0 == 0 || xw0 + 32 >= g.nx);
    const bool edge_y = g.wrap_y && (y == 0 || y == g.ny - 1);
    const bool edge_z = (g.zlo == LBM_ZFACE_WRAP && z == 0) || (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1);
    const bool generic = edge_x || edge_y || edge_z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    // cellmask == NULL: every cell fluid, no links (periodic runs without a
    // boundary handling) - saves the 4 B/cell mask read
    const uint32_t code = cell_code<Q, BITS>(g, cellmask, x, y, z, cell);
    if constexpr (!BITS) prefetch_mask(g, cellmask, cell, (int64_t)g.nx * g.ny * g.nz);
    using Acc = AccOf<Real>;
    Acc f[Q];
    pull_cell<Q, Real, Acc, MOVING ? 2 : 0, BITS>(g, p, src, x, y, z, code, typemask, generic, f);
    if (code & CodeBits<Q, BITS>::fluid) collide_any<Q, MODEL, FORCE>(f, p, cell);
    Real* dp = opaque(dst + lidx(g, z, 0, y, x));
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        store_any<Q, i>(dp + g.dslot[i], f[i]);
    });
    // Fused halo: a boundary plane also writes the directions that leave the
    // box through its face straight into the neighbour's ghost plane (peer
    // HBM over NVLink, or another slab on this device) - the per-step
    // exchange of field/ghost.py:202-264 without a separate send/recv.
    // Block-uniform (z is per block), so interior planes pay one test.
    if constexpr (PEER) {
    if (z == 0 && p.peer_lo != nullptr) {
        Real* pp = opaque(static_cast<Real*>(p.peer_lo) + (int64_t)(y + 1) * g.pitch + g.xoff + x);
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            if constexpr (D::cz[i] == -1) store_any<Q, i>(pp + g.dslot[i], f[i]);
        });
    }
    if (z == g.nz - 1 && p.peer_hi != nullptr) {
        Real* pp = opaque(static_cast<Real*>(p.peer_hi) + (int64_t)(y + 1) * g.pitch + g.xoff + x);
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            if constexpr (D::cz[i] == 1) store_any<Q, i>(pp + g.dslot[i], f[i]);
        });
    }
    }
}

// k_fused that also writes the macroscopic readout of the state it pulls:
// rho / u of R = S(src) per interior cell, exactly what k_moments with
// stream_form = 1 gives for src (moments of the last sweep's pull instead of
// a separate pass over the field).  Fluid cells take rho / u from the
// collision itself (the same operations: sequential sums, u = m (1 / rho),
// the Guo half shift when the sweep is Guo-forced); other cells sum their
// pulled values.  fp64 storage, no moving walls, no fused halo.
template <int Q, int MODEL, int FORCE>
__global__ void __launch_bounds__(LBM_FUSED_BX, fused_minb_bx<Q, double, MODEL, FORCE>())
    k_fused_mom(KGrid g, KParams p, const double* __restrict__ src, double* __restrict__ dst,
                const uint32_t* __restrict__ cellmask, const uint32_t* __restrict__ typemask,
                int z0, double* __restrict__ rho_out, double* __restrict__ u_out, int* bad) {
    using D = Dirs<Q>;
    constexpr bool GUO = FORCE == 1 || FORCE == 3;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = z0 + blockIdx.z;
    const int xw0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    const bool edge_x = g.wrap_x && (xw0 == 0 || xw0 + 32 >= g.nx);
    const bool edge_y = g.wrap_y && (y == 0 || y == g.ny - 1);
    const bool edge_z = (g.zlo == LBM_ZFACE_WRAP && z == 0) || (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1);
    const bool generic = edge_x || edge_y || edge_z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const uint32_t code = cellmask ? __ldg(cellmask + cell) : LBM_MASK_FLUID;
    prefetch_mask(g, cellmask, cell, (int64_t)g.nx * g.ny * g.nz);
    double f[Q];
    pull_cell<Q, double, double, 0>(g, p, src, x, y, z, code, typemask, generic, f);
    double mo[4];
    if (code & LBM_MASK_FLUID) {
        collide_cell<Q, MODEL, FORCE, true>(f, p, 0.0, mo);
    } else {
        double rho = f[0];
#pragma unroll
        for (int i = 1; i < Q; ++i) rho = rho + f[i];
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
        const double inv = 1.0 / rho;
        mo[0] = rho;
        mo[1] = mx * inv;
        mo[2] = my * inv;
        mo[3] = mz * inv;
        if constexpr (GUO) {
            mo[1] = mo[1] + p.sfx * inv;
            mo[2] = mo[2] + p.sfy * inv;
            mo[3] = mo[3] + p.sfz * inv;
        }
    }
    if (mo[0] <= 0.0) atomicAdd(bad, 1);
    rho_out[cell] = mo[0];
    u_out[cell * 3 + 0] = mo[1];
    u_out[cell * 3 + 1] = mo[2];
    u_out[cell * 3 + 2] = mo[3];
    double* dp = opaque(dst + lidx(g, z, 0, y, x));
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        store_any<Q, i>(dp + g.dslot[i], f[i]);
    });
}

// Two cells per thread, stacked in z (fp32 storage): both cells' 2Q pulls
// are issued before the first cell is finished, so each warp keeps twice the
// bytes in flight of k_fused with far fewer than twice the registers (the
// fp32 populations take one register each).  The kernel is latency-bound on
// its pulls (ncu: long_scoreboard dominates), so more loads in flight per
// resident warp is the lever; the collision and stores of cell a overlap
// the tail of cell b's loads.  Plane pairs [z0 + 2k, z0 + 2k + 1] per block
// row; an odd range's last plane runs alone.
template <int Q, typename Real, int MODEL, int FORCE>
constexpr int fused_z2_minb() {
#ifdef LBM_FUSED_Z2_MINB
    return LBM_FUSED_Z2_MINB;
#else
    return 6;
#endif
}

__device__ __forceinline__ bool plane_wraps(const KGrid& g, int z) {
    return (g.zlo == LBM_ZFACE_WRAP && z == 0) || (g.zhi == LBM_ZFACE_WRAP && z == g.nz - 1);
}

template <int Q, typename Real, int MODEL, int FORCE, bool TYPED, bool BITS = false>
__global__ void __launch_bounds__(LBM_FUSED_BX, fused_z2_minb<Q, Real, MODEL, FORCE>())
    k_fused_z2(KGrid g, KParams p, const Real* __restrict__ src, Real* __restrict__ dst,
               const uint32_t* __restrict__ cellmask, const uint32_t* __restrict__ typemask,
               int z0, int z1) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int za = z0 + 2 * blockIdx.z;
    const bool two = za + 1 < z1;                      // block-uniform
    const int xw0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    const bool edge_xy = (g.wrap_x && (xw0 == 0 || xw0 + 32 >= g.nx)) ||
                         (g.wrap_y && (y == 0 || y == g.ny - 1));
    if (x >= g.nx) return;
    const int64_t plane_cells = (int64_t)g.ny * g.nx;
    const int64_t cell_a = ((int64_t)za * g.ny + y) * g.nx + x;
    uint32_t code_a, code_b;
    if constexpr (BITS) {
        codes_from_bits_z2<Q>(g, reinterpret_cast<const uint64_t*>(cellmask), x, y, za, two, code_a,
                              code_b);
    } else {
        code_a = cell_code<Q, false>(g, cellmask, x, y, za, cell_a);
        code_b = !two ? 0u : cell_code<Q, false>(g, cellmask, x, y, za + 1, cell_a + plane_cells);
        // both planes of the pair, (link_hint >> 1) pair-rows ahead; a row
        // index beyond ny continues in the next plane pair
        const int64_t ncells = (int64_t)g.nx * g.ny * g.nz;
        const int64_t c = (g.link_hint >> 1) > g.ny - 1 - y ? cell_a + plane_cells : cell_a;
        prefetch_mask(g, cellmask, c, ncells);
        prefetch_mask(g, cellmask, c + plane_cells, ncells);
    }
    using Acc = AccOf<Real>;
    Real ra[Q], rb[Q];
    pull_load<Q, Real, BITS>(g, src, x, y, za, code_a, edge_xy || plane_wraps(g, za), ra);
    if (two) pull_load<Q, Real, BITS>(g, src, x, y, za + 1, code_b, edge_xy || plane_wraps(g, za + 1), rb);
    auto finish = [&](int z, int64_t cell, uint32_t code, const Real (&raw)[Q]) {
        Acc f[Q];
        const uint2 t = TYPED ? type_words(g, typemask, x, y, z, code) : make_uint2(0u, 0u);
        pull_finish<Q, Real, Acc, 0, TYPED>(g, p, src, x, y, z, lidx(g, z, 0, y, x), code, t, raw,
                                            f);
        if (code & CodeBits<Q, BITS>::fluid) collide_any<Q, MODEL, FORCE>(f, p, cell);
        Real* dp = opaque(dst + lidx(g, z, 0, y, x));
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            store_any<Q, i>(dp + g.dslot[i], f[i]);
        });
    };
    finish(za, cell_a, code_a, ra);
    if (two) finish(za + 1, cell_a + plane_cells, code_b, rb);
}

// G_0 = C(R_0): collide fluid interior cells in place.
template <int Q, typename Real, int MODEL, int FORCE>
__global__ void __launch_bounds__(128) k_collide_only(KGrid g, KParams p, Real* __restrict__ pdf,
                                                      const uint32_t* __restrict__ cellmask, int z0) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = z0 + blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const uint32_t code = cellmask[cell];
    if (!(code & LBM_MASK_FLUID)) return;
    const int64_t own = lidx(g, z, 0, y, x);
    using Acc = AccOf<Real>;
    Acc f[Q];
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        if constexpr (std::is_same_v<Acc, double>)
            f[i] = Store<Real>::template load<Q, i>(pdf + own + dir_off<Q, i>(g));
        else
            f[i] = pdf[own + dir_off<Q, i>(g)];
    });
    collide_any<Q, MODEL, FORCE>(f, p, cell);
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        store_any<Q, i>(pdf + own + dir_off<Q, i>(g), f[i]);
    });
}

// R = S(G) to dense fp64 (q, nz, ny, nx), reference direction order.
template <int Q, typename Real>
__global__ void __launch_bounds__(128) k_stream_only(KGrid g, KParams p, const Real* __restrict__ src,
                                                     const uint32_t* __restrict__ cellmask,
                                                     const uint32_t* __restrict__ typemask,
                                                     double* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    const uint32_t code = cellmask[cell];
    double f[Q];
    pull_cell<Q, Real, double, 1>(g, p, src, x, y, z, code, typemask, true, f);
    const int64_t n = (int64_t)g.nx * g.ny * g.nz;
#pragma unroll
    for (int i = 0; i < Q; ++i) out[(int64_t)i * n + cell] = f[i];
}

// rho/u (collision.py:167-184) of R = S(G) (stream_form) or of the stored R.
template <int Q, typename Real, int GUO>
__global__ void __launch_bounds__(128) k_moments(KGrid g, KParams p, const Real* __restrict__ src,
                                                 const uint32_t* __restrict__ cellmask,
                                                 const uint32_t* __restrict__ typemask,
                                                 int stream_form, double* __restrict__ rho_out,
                                                 double* __restrict__ u_out, int* bad, int z0) {
    using D = Dirs<Q>;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = z0 + blockIdx.z;
    if (x >= g.nx) return;
    const int64_t cell = ((int64_t)z * g.ny + y) * g.nx + x;
    double f[Q];
    if (stream_form) {
        pull_cell<Q, Real, double, 1>(g, p, src, x, y, z, cellmask[cell], typemask, true, f);
    } else {
        const int64_t own = lidx(g, z, 0, y, x);
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            f[i] = Store<Real>::template load<Q, i>(src + own + dir_off<Q, i>(g));
        });
    }
    double rho = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) rho = rho + f[i];
    if (rho <= 0.0) atomicAdd(bad, 1);
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
    const double inv = 1.0 / rho;
    double ux = mx * inv, uy = my * inv, uz = mz * inv;
    if constexpr (GUO) {
        ux = ux + p.sfx * inv;
        uy = uy + p.sfy * inv;
        uz = uz + p.sfz * inv;
    }
    rho_out[cell] = rho;
    u_out[cell * 3 + 0] = ux;
    u_out[cell * 3 + 1] = uy;
    u_out[cell * 3 + 2] = uz;
}

// dense ghost-inclusive (q, Z, Y, X) fp64 <-> layout
template <int Q, typename Real, int TO_LAYOUT>
__global__ void k_convert(KGrid g, double* __restrict__ dense, Real* __restrict__ pdf) {
    const int X = g.nx + 2, Y = g.ny + 2, Z = g.nz + 2;
    const int xg = blockIdx.x * blockDim.x + threadIdx.x;
    const int yg = blockIdx.y;
    const int zg = blockIdx.z;
    if (xg >= X) return;
    const int64_t n = (int64_t)X * Y * Z;
    const int64_t cell = ((int64_t)zg * Y + yg) * X + xg;
    const int64_t own = lidx(g, zg - 1, 0, yg - 1, xg - 1);
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        Real* pp = pdf + own + dir_off<Q, i>(g);
        if constexpr (TO_LAYOUT) Store<Real>::template store<Q, i>(pp, dense[i * n + cell]);
        else dense[i * n + cell] = Store<Real>::template load<Q, i>(pp);
    });
}

// equilibrium() (collision.py:150-154) into the layout, ghosts included
template <int Q, typename Real>
__global__ void k_fill_eq(KGrid g, const double* __restrict__ rho, const double* __restrict__ u,
                          Real* __restrict__ pdf) {
    using D = Dirs<Q>;
    const int X = g.nx + 2, Y = g.ny + 2;
    const int xg = blockIdx.x * blockDim.x + threadIdx.x;
    const int yg = blockIdx.y;
    const int zg = blockIdx.z;
    if (xg >= X) return;
    const int64_t cell = ((int64_t)zg * Y + yg) * X + xg;
    const double r = rho[cell];
    const double ux = u[cell * 3], uy = u[cell * 3 + 1], uz = u[cell * 3 + 2];
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const int64_t own = lidx(g, zg - 1, 0, yg - 1, xg - 1);
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        const double cu = cu_of<Q, i>(ux, uy, uz);
        const double feq = (wt<Q, i>() * r) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - 1.5 * usq);
        Store<Real>::template store<Q, i>(pdf + own + dir_off<Q, i>(g), feq);
    });
}

// equilibrium of dense interior arrays rho (nz, ny, nx), u (nz, ny, nx, 3)
// into the ghost-inclusive planes zg0 .. zg0 + gridDim.z - 1 of the layout;
// a ghost cell takes the nearest interior cell's rho / u (each coordinate
// clamped: the values fill_equilibrium_arrays gives the ghost shell, so the
// result is bitwise that of k_fill_eq).  `shell` (optional) receives the
// ghost cells too: the second buffer's shell (what lbm_copy_shell gives it).
template <int Q, typename Real>
__global__ void k_fill_eq_dense(KGrid g, const double* __restrict__ rho, const double* __restrict__ u,
                                int zg0, Real* __restrict__ pdf, Real* __restrict__ shell) {
    const int X = g.nx + 2;
    const int xg = blockIdx.x * blockDim.x + threadIdx.x;
    const int yg = blockIdx.y;
    const int zg = zg0 + blockIdx.z;
    if (xg >= X) return;
    const int xi = min(max(xg - 1, 0), g.nx - 1);
    const int yi = min(max(yg - 1, 0), g.ny - 1);
    const int zi = min(max(zg - 1, 0), g.nz - 1);
    const int64_t cell = ((int64_t)zi * g.ny + yi) * g.nx + xi;
    const double r = rho[cell];
    const double ux = u[cell * 3], uy = u[cell * 3 + 1], uz = u[cell * 3 + 2];
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const int64_t own = lidx(g, zg - 1, 0, yg - 1, xg - 1);
    const bool ghost = xg == 0 || xg == X - 1 || yg == 0 || yg == g.ny + 1 || zg == 0 || zg == g.nz + 1;
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        const double cu = cu_of<Q, i>(ux, uy, uz);
        const double feq = (wt<Q, i>() * r) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - 1.5 * usq);
        Store<Real>::template store<Q, i>(pdf + own + dir_off<Q, i>(g), feq);
        if (ghost && shell) Store<Real>::template store<Q, i>(shell + own + dir_off<Q, i>(g), feq);
    });
}

// k_fill_eq_dense followed by k_collide_only in one pass (a pipelined job's
// first touch of a plane chunk): interior fluid cells are collided before
// they are stored (G_0 = C(R_0)), every other cell keeps R_0; ghost cells
// also go to `shell`.  The collision starts from the STORED representation
// of feq (fp32: the centred float), so the result is bitwise that of the two
// separate passes.
template <int Q, typename Real, int MODEL, int FORCE>
__global__ void __launch_bounds__(128) k_fill_collide(KGrid g, KParams p, const double* __restrict__ rho,
                                                      const double* __restrict__ u, int zg0,
                                                      Real* __restrict__ pdf, Real* __restrict__ shell,
                                                      const uint32_t* __restrict__ cellmask) {
    const int X = g.nx + 2;
    const int xg = blockIdx.x * blockDim.x + threadIdx.x;
    const int yg = blockIdx.y;
    const int zg = zg0 + blockIdx.z;
    if (xg >= X) return;
    const int xi = min(max(xg - 1, 0), g.nx - 1);
    const int yi = min(max(yg - 1, 0), g.ny - 1);
    const int zi = min(max(zg - 1, 0), g.nz - 1);
    const int64_t cell = ((int64_t)zi * g.ny + yi) * g.nx + xi;
    const double r = rho[cell];
    const double ux = u[cell * 3], uy = u[cell * 3 + 1], uz = u[cell * 3 + 2];
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const int64_t own = lidx(g, zg - 1, 0, yg - 1, xg - 1);
    const bool ghost = xg == 0 || xg == X - 1 || yg == 0 || yg == g.ny + 1 || zg == 0 || zg == g.nz + 1;
    using Acc = AccOf<Real>;
    Acc f[Q];
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        const double cu = cu_of<Q, i>(ux, uy, uz);
        const double feq = (wt<Q, i>() * r) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - 1.5 * usq);
        if constexpr (std::is_same_v<Acc, double>) {
            f[i] = feq;
        } else {
            f[i] = (float)(feq - wt<Q, i>());   // Store<float>::store's rounding
        }
    });
    if (ghost) {
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            store_any<Q, i>(pdf + own + dir_off<Q, i>(g), f[i]);
            if (shell) store_any<Q, i>(shell + own + dir_off<Q, i>(g), f[i]);
        });
        return;
    }
    if (cellmask[cell] & LBM_MASK_FLUID) collide_any<Q, MODEL, FORCE>(f, p, cell);
    static_for<0, Q>([&](auto I_) {
        constexpr int i = decltype(I_)::value;
        store_any<Q, i>(pdf + own + dir_off<Q, i>(g), f[i]);
    });
}

}  // namespace lbm
