/*
 * lbm_oracle.c - CPU restatement of the reference LBM sweep.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product
 * path (paper_1909_13772_b200/ fails loudly without its CUDA library).
 *
 * Restates, in plain C with the reference's exact operation order (compile
 * with -ffp-contract=off, no fast-math), the numpy code of
 *   impl.collide        /root/reference/pkg/src/blocksim/_kernels/_core_py.py:70-200
 *   impl.stream_pull    _core_py.py:203-218
 *   BoundaryHandling.apply   lbm/boundary.py:154-195
 *   exchange_ghosts on one global block: a ghost cell receives the value of
 *     the interior cell it images iff every axis on which it lies outside
 *     the domain is periodic (field/ghost.py:112-124,176-184: receiver box
 *     grown by w, intersected with the sender's interior)
 *   stream_collide step order  lbm/sweep.py:93-151
 * Because every step is a pure copy or a pointwise update, one global block
 * reproduces any block/rank decomposition bit for bit (the reference's own
 * rank-invariance property, pkg/tests/test_lbm.py:452-471).
 *
 * Layout: the reference "fzyx" raw array, pdf[i][Z][Y][X] with one ghost
 * layer (Z = nz + 2, ...), i in reference direction order.
 * Pinned against golden vectors made by the reference itself
 * (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct orc_stencil {
    int q;
    int cx[27], cy[27], cz[27], opp[27];
    double w[27];
} orc_stencil;

typedef struct orc_params {
    int mode;          /* 0 SRT, 1 TRT, 2 MRT */
    int force_mode;    /* 0 none, 1 Guo, 2 SimpleShift */
    double omega;      /* SRT global rate */
    const double* omega_field; /* SRT per-cell rate (Z,Y,X) or NULL (omega_window) */
    double omega_e, omega_o;
    const double* M;    /* q*q row-major */
    const double* Minv; /* q*q */
    const double* S;    /* q */
    const double* G;    /* q*q guo_matrix */
    double fx, fy, fz;
    double shift_tau;
} orc_params;

typedef struct orc_links {
    uint32_t fluid, noslip, ubb, pressure;
    double uwx, uwy, uwz;   /* ubb_velocity */
    double rho0;            /* reference_density */
    double rho_w;           /* pressure_density */
} orc_links;

#define IDX(z, y, x) (((int64_t)(z) * Y + (y)) * X + (x))

/* impl.collide on every cell (ghosts included) with flags & fluid_bits */
void orc_collide(const orc_stencil* st, double* pdf, const uint32_t* flags, uint32_t fluid_bits,
                 int X, int Y, int Z, const orc_params* p) {
    const int q = st->q;
    const int64_t n = (int64_t)X * Y * Z;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
        if (!(flags[c] & fluid_bits)) continue;
        double f[27], feq[27], m[27], meq[27], Fi[27], out[27];
        for (int i = 0; i < q; ++i) f[i] = pdf[(int64_t)i * n + c];
        double rho = f[0];
        for (int i = 1; i < q; ++i) rho = rho + f[i];
        double mx = 0.0, my = 0.0, mz = 0.0;
        for (int i = 0; i < q; ++i) {
            if (st->cx[i]) mx = mx + (double)st->cx[i] * f[i];
            if (st->cy[i]) my = my + (double)st->cy[i] * f[i];
            if (st->cz[i]) mz = mz + (double)st->cz[i] * f[i];
        }
        const double inv_rho = 1.0 / rho;
        double ux = mx * inv_rho, uy = my * inv_rho, uz = mz * inv_rho;
        const double fx = p->force_mode ? p->fx : 0.0;
        const double fy = p->force_mode ? p->fy : 0.0;
        const double fz = p->force_mode ? p->fz : 0.0;
        if (p->force_mode == 1) {
            ux = ux + (0.5 * fx) * inv_rho;
            uy = uy + (0.5 * fy) * inv_rho;
            uz = uz + (0.5 * fz) * inv_rho;
        } else if (p->force_mode == 2) {
            ux = ux + (p->shift_tau * fx) * inv_rho;
            uy = uy + (p->shift_tau * fy) * inv_rho;
            uz = uz + (p->shift_tau * fz) * inv_rho;
        }
        const double usq = (ux * ux + uy * uy) + uz * uz;
        for (int i = 0; i < q; ++i) {
            const double cu = ((double)st->cx[i] * ux + (double)st->cy[i] * uy) + (double)st->cz[i] * uz;
            feq[i] = (st->w[i] * rho) * (((1.0 + 3.0 * cu) + (4.5 * cu) * cu) - 1.5 * usq);
        }
        double omega = p->omega;
        if (p->mode == 0) {
            if (p->omega_field) omega = p->omega_field[c];
            const double rem = 1.0 - omega;
            for (int i = 0; i < q; ++i) f[i] = feq[i] + rem * (f[i] - feq[i]);
        } else if (p->mode == 1) {
            for (int i = 0; i < q; ++i) {
                const int j = st->opp[i];
                const double fp = 0.5 * (f[i] + f[j]);
                const double fm = 0.5 * (f[i] - f[j]);
                const double ep = 0.5 * (feq[i] + feq[j]);
                const double em = 0.5 * (feq[i] - feq[j]);
                out[i] = (f[i] - p->omega_e * (fp - ep)) - p->omega_o * (fm - em);
            }
            for (int i = 0; i < q; ++i) f[i] = out[i];
        } else {
            for (int a = 0; a < q; ++a) {
                double acc = p->M[a * q] * f[0];
                for (int i = 1; i < q; ++i) acc = acc + p->M[a * q + i] * f[i];
                m[a] = acc;
            }
            for (int a = 0; a < q; ++a) {
                double acc = p->M[a * q] * feq[0];
                for (int i = 1; i < q; ++i) acc = acc + p->M[a * q + i] * feq[i];
                meq[a] = acc;
            }
            for (int a = 0; a < q; ++a) m[a] = p->S[a] * (m[a] - meq[a]);
            for (int i = 0; i < q; ++i) {
                double acc = p->Minv[i * q] * m[0];
                for (int a = 1; a < q; ++a) acc = acc + p->Minv[i * q + a] * m[a];
                f[i] = f[i] - acc;
            }
        }
        if (p->force_mode == 1) {
            for (int i = 0; i < q; ++i) {
                const double cxi = (double)st->cx[i], cyi = (double)st->cy[i], czi = (double)st->cz[i];
                const double cu = (cxi * ux + cyi * uy) + czi * uz;
                const double t = (((cxi - ux) + (3.0 * cu) * cxi) * fx +
                                  ((cyi - uy) + (3.0 * cu) * cyi) * fy) +
                                 ((czi - uz) + (3.0 * cu) * czi) * fz;
                Fi[i] = (3.0 * st->w[i]) * t;
            }
            if (p->mode == 0) {
                const double hw = 1.0 - 0.5 * omega;
                for (int i = 0; i < q; ++i) f[i] = f[i] + hw * Fi[i];
            } else if (p->mode == 1) {
                const double he = 1.0 - 0.5 * p->omega_e;
                const double ho = 1.0 - 0.5 * p->omega_o;
                const double he2 = he * 0.5, ho2 = ho * 0.5;
                for (int i = 0; i < q; ++i) {
                    const int j = st->opp[i];
                    f[i] = (f[i] + he2 * (Fi[i] + Fi[j])) + ho2 * (Fi[i] - Fi[j]);
                }
            } else {
                for (int i = 0; i < q; ++i) {
                    double acc = p->G[i * q] * Fi[0];
                    for (int a = 1; a < q; ++a) acc = acc + p->G[i * q + a] * Fi[a];
                    f[i] = f[i] + acc;
                }
            }
        }
        for (int i = 0; i < q; ++i) pdf[(int64_t)i * n + c] = f[i];
    }
}

/* impl.stream_pull: dst_i(x) = src_i(x - c_i) over the interior (g = 1) */
void orc_stream_pull(const orc_stencil* st, const double* src, double* dst, int X, int Y, int Z) {
    const int64_t n = (int64_t)X * Y * Z;
    for (int i = 0; i < st->q; ++i) {
        const double* s = src + (int64_t)i * n;
        double* d = dst + (int64_t)i * n;
        const int cx = st->cx[i], cy = st->cy[i], cz = st->cz[i];
#pragma omp parallel for schedule(static)
        for (int z = 1; z < Z - 1; ++z)
            for (int y = 1; y < Y - 1; ++y)
                for (int x = 1; x < X - 1; ++x) d[IDX(z, y, x)] = s[IDX(z - cz, y - cy, x - cx)];
    }
}

/* BoundaryHandling.apply: links from fluid interior cells into NoSlip/UBB/
 * Pressure neighbours (flags must hold exchanged ghost flags). */
void orc_apply_links(const orc_stencil* st, const double* src, double* dst, const uint32_t* flags,
                     int X, int Y, int Z, const orc_links* L) {
    const int q = st->q;
    const int64_t n = (int64_t)X * Y * Z;
#pragma omp parallel for schedule(static)
    for (int z = 1; z < Z - 1; ++z)
        for (int y = 1; y < Y - 1; ++y)
            for (int x = 1; x < X - 1; ++x) {
                const int64_t c = IDX(z, y, x);
                if (!(flags[c] & L->fluid)) continue;
                for (int i = 1; i < q; ++i) {
                    const uint32_t nb = flags[IDX(z + st->cz[i], y + st->cy[i], x + st->cx[i])];
                    const int o = st->opp[i];
                    if (nb & L->noslip) {
                        dst[(int64_t)o * n + c] = src[(int64_t)i * n + c];
                    } else if (nb & L->ubb) {
                        const double cu = ((double)st->cx[i] * L->uwx + (double)st->cy[i] * L->uwy) +
                                          (double)st->cz[i] * L->uwz;
                        dst[(int64_t)o * n + c] =
                            src[(int64_t)i * n + c] - ((6.0 * st->w[i]) * L->rho0) * cu;
                    } else if (nb & L->pressure) {
                        double rho = src[c];
                        for (int k = 1; k < q; ++k) rho += src[(int64_t)k * n + c];
                        double mx = 0.0, my = 0.0, mz = 0.0;
                        for (int k = 0; k < q; ++k) {
                            const double v = src[(int64_t)k * n + c];
                            if (st->cx[k]) mx += (double)st->cx[k] * v;
                            if (st->cy[k]) my += (double)st->cy[k] * v;
                            if (st->cz[k]) mz += (double)st->cz[k] * v;
                        }
                        const double ux = mx / rho, uy = my / rho, uz = mz / rho;
                        const double cu = ((double)st->cx[i] * ux + (double)st->cy[i] * uy) +
                                          (double)st->cz[i] * uz;
                        const double usq = (ux * ux + uy * uy) + uz * uz;
                        dst[(int64_t)o * n + c] =
                            -src[(int64_t)i * n + c] +
                            ((2.0 * st->w[i]) * L->rho_w) * (((1.0 + (4.5 * cu) * cu)) - 1.5 * usq);
                    }
                }
            }
}

static inline int covered(int v, int nint, int periodic, int* wrapped) {
    /* v is a ghost-inclusive coordinate 0..nint+1; interior is 1..nint */
    if (v >= 1 && v <= nint) { *wrapped = v; return 1; }
    if (!periodic) return 0;
    *wrapped = v == 0 ? nint : 1;
    return 1;
}

/* exchange_ghosts on one global block: fill covered ghost cells.
 * nf components, data[f][Z][Y][X]; periodic = (x, y, z). */
void orc_exchange(double* data, int nf, int X, int Y, int Z, const int periodic[3]) {
    const int64_t n = (int64_t)X * Y * Z;
    for (int z = 0; z < Z; ++z)
        for (int y = 0; y < Y; ++y)
            for (int x = 0; x < X; ++x) {
                const int ghost = (x == 0 || x == X - 1 || y == 0 || y == Y - 1 || z == 0 || z == Z - 1);
                if (!ghost) continue;
                int xw, yw, zw;
                if (!covered(x, X - 2, periodic[0], &xw)) continue;
                if (!covered(y, Y - 2, periodic[1], &yw)) continue;
                if (!covered(z, Z - 2, periodic[2], &zw)) continue;
                for (int f = 0; f < nf; ++f)
                    data[(int64_t)f * n + IDX(z, y, x)] = data[(int64_t)f * n + IDX(zw, yw, xw)];
            }
}

void orc_exchange_u32(uint32_t* data, int X, int Y, int Z, const int periodic[3]) {
    for (int z = 0; z < Z; ++z)
        for (int y = 0; y < Y; ++y)
            for (int x = 0; x < X; ++x) {
                const int ghost = (x == 0 || x == X - 1 || y == 0 || y == Y - 1 || z == 0 || z == Z - 1);
                if (!ghost) continue;
                int xw, yw, zw;
                if (!covered(x, X - 2, periodic[0], &xw)) continue;
                if (!covered(y, Y - 2, periodic[1], &yw)) continue;
                if (!covered(z, Z - 2, periodic[2], &zw)) continue;
                data[IDX(z, y, x)] = data[IDX(zw, yw, xw)];
            }
}

/* `steps` calls of stream_collide (lbm/sweep.py:93-151) on one global block.
 * a: src field (R-form in/out), b: dst scratch.  flags must already hold
 * exchanged ghost flags (BoundaryHandling.freeze).  links may be NULL
 * (fully periodic, no handling: every cell collides, sweep.py:333-334).
 * Returns 0. */
/* link_flags: the flags the links were frozen from (BoundaryHandling.freeze,
 * boundary.py:128-131); `flags` are the current ones the collision reads
 * (lbm/sweep.py:124-136).  NULL: the same array. */
int orc_run(const orc_stencil* st, double* a, double* b, const uint32_t* flags,
            const uint32_t* link_flags, uint32_t fluid_bits, int X, int Y, int Z,
            const int periodic[3], const orc_params* p, const orc_links* links, int steps) {
    if (!link_flags) link_flags = flags;
    for (int s = 0; s < steps; ++s) {
        orc_exchange(a, st->q, X, Y, Z, periodic);
        orc_collide(st, a, flags, fluid_bits, X, Y, Z, p);
        orc_stream_pull(st, a, b, X, Y, Z);
        if (links) orc_apply_links(st, a, b, link_flags, X, Y, Z, links);
        /* swap: copy back so `a` stays the src handle for the caller */
        double* t = a;
        a = b;
        b = t;
    }
    /* after an odd number of steps the result lives in the caller's b */
    return steps & 1;
}
