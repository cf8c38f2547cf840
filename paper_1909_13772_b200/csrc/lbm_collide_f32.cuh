// Per-cell collision of the fp32-storage path, fp32 registers.
//
// The fp32 field stores zero-centred populations g_i = f_i - w_i (SURVEY
// hard part 8).  This path keeps them centred through the collision, so
// every fp32 rounding error is relative to |f - w| (~1e-2 w) instead of |f|:
//   drho = sum g_i,   rho = 1 + drho,   j = sum c_i g_i   (sum c_i w_i = 0)
//   g_i^eq = w_i drho + (w_i rho) ((3 cu + 4.5 cu^2) - 1.5 u^2)
// which is feq_i - w_i of impl.collide (_core_py.py:124-128) regrouped.
// SRT/TRT/Guo follow _core_py.py:130-148,171-190 (w_i = w_opp(i), so the TRT
// pair algebra is unchanged in g).  Results are checked against the fp64
// oracle at BASELINE's 1e-5 relative tolerance, not bitwise, so sums are
// reassociated for ILP and FMA contraction is allowed.
//
// D3Q27 MRT uses the raw-moment factorisation instead of the dense q x q
// products of _core_py.py:149-169 / :191-197:
//   f' = f - Minv S M (f - feq) + G F,  G = Minv (I - S/2) M
//      = f + F - Rinv K R (d + F/2),    d = f - feq,  K = R Minv S M Rinv
// where R is the tensor-product raw-moment transform (per axis: 1, c, c^2;
// 3 passes of 9 three-point butterflies).  For bases that are raw monomials
// up to a mixing of the second-order pure moments (the shear-separated basis
// of BASELINE config 2), K is diagonal plus one 3x3 block on (xx, yy, zz);
// the host checks that structure (set_mrt_fast_f32) before enabling it.
#pragma once
#include <type_traits>

#include "lbm_collide.cuh"

namespace lbm {

static __constant__ float c_mrt_kd[27];  // (I - K) diagonal (raw index a + 3b + 9c)
static __constant__ float c_mrt_kb[9];   // (I - K) on (xx, yy, zz) = raw 2, 6, 18

constexpr int RAW_XX = 2, RAW_YY = 6, RAW_ZZ = 18;

// tensor position of D3Q27 direction i: (cx+1) + 3 (cy+1) + 9 (cz+1)
template <int I>
constexpr int tpos27() {
    return (Dirs<27>::cx[I] + 1) + 3 * (Dirs<27>::cy[I] + 1) + 9 * (Dirs<27>::cz[I] + 1);
}

// one axis of the raw transform: values at c = -1, 0, +1 -> moments c^0, c^1, c^2
template <int STRIDE>
__device__ __forceinline__ void raw_fwd_axis(float (&t)[27]) {
    static_for<0, 27>([&](auto K_) {
        constexpr int k = decltype(K_)::value;
        if constexpr ((k / STRIDE) % 3 == 0) {
            const float a = t[k], b = t[k + STRIDE], c = t[k + 2 * STRIDE];
            t[k] = (a + c) + b;
            t[k + STRIDE] = c - a;
            t[k + 2 * STRIDE] = c + a;
        }
    });
}

template <int STRIDE>
__device__ __forceinline__ void raw_inv_axis(float (&t)[27]) {
    static_for<0, 27>([&](auto K_) {
        constexpr int k = decltype(K_)::value;
        if constexpr ((k / STRIDE) % 3 == 0) {
            const float m0 = t[k], m1 = t[k + STRIDE], m2 = t[k + 2 * STRIDE];
            t[k] = 0.5f * (m2 - m1);
            t[k + STRIDE] = m0 - m2;
            t[k + 2 * STRIDE] = 0.5f * (m2 + m1);
        }
    });
}

// (c - u + (3 cu) c) for one axis, fp32
template <int C>
__device__ __forceinline__ float guo_axis32(float u, float cu3) {
    if constexpr (C == 1) return (1.0f - u) + cu3;
    else if constexpr (C == -1) return (-1.0f - u) - cu3;
    else return -u;
}

template <int Q, int I, bool XONLY>
__device__ __forceinline__ float guo_F32(float ux, float uy, float uz, float cu,
                                         const KParams& p) {
    using D = Dirs<Q>;
    const float cu3 = 3.0f * cu;
    float t;
    if constexpr (XONLY)
        t = guo_axis32<D::cx[I]>(ux, cu3) * p.ffx;
    else
        t = (guo_axis32<D::cx[I]>(ux, cu3) * p.ffx + guo_axis32<D::cy[I]>(uy, cu3) * p.ffy) +
            guo_axis32<D::cz[I]>(uz, cu3) * p.ffz;
    constexpr float w3 = (float)(3.0 * D::w[I]);
    return w3 * t;
}

template <int Q, int I>
__device__ __forceinline__ constexpr float wtf() {
    constexpr float v = (float)Dirs<Q>::w[I];
    return v;
}

// ------------------------------------------------ D3Q27 MRT in moment space
// Raw moments of the second-order equilibrium feq_i = w_i rho (1 + 3 c.u +
// 4.5 (c.u)^2 - 1.5 u^2) for the product weights of D3Q27 (1D weights 1/6,
// 2/3, 1/6; 1D moments mu_n = <c^n> = 1, 0, 1/3, 0, 1/3 for n = 0..4, as
// c^3 = c and c^4 = c^2 on the lattice).  For raw index r = a + 3b + 9c
// (moment cx^a cy^b cz^c), centred on the weights' own moments:
//   teq_r = drho A + rho (Cx ux + Cy uy + Cz uz + Cxx ux^2 + Cyy uy^2
//           + Czz uz^2 + Cxy ux uy + Cxz ux uz + Cyz uy uz)
// with A = mu_a mu_b mu_c, Cx = 3 mu_{a+1} mu_b mu_c, Cxx = 4.5 mu_{a+2}
// mu_b mu_c - 1.5 A, Cxy = 9 mu_{a+1} mu_{b+1} mu_c (and permutations).
constexpr double raw_mu(int n) { return n == 0 ? 1.0 : (n % 2 ? 0.0 : 1.0 / 3.0); }

struct RawEq {
    double A, Cx, Cy, Cz, Cxx, Cyy, Czz, Cxy, Cxz, Cyz;
};

constexpr RawEq raw_eq(int r) {
    const int a = r % 3, b = (r / 3) % 3, c = r / 9;
    const double A = raw_mu(a) * raw_mu(b) * raw_mu(c);
    return RawEq{A,
                 3.0 * raw_mu(a + 1) * raw_mu(b) * raw_mu(c),
                 3.0 * raw_mu(a) * raw_mu(b + 1) * raw_mu(c),
                 3.0 * raw_mu(a) * raw_mu(b) * raw_mu(c + 1),
                 4.5 * raw_mu(a + 2) * raw_mu(b) * raw_mu(c) - 1.5 * A,
                 4.5 * raw_mu(a) * raw_mu(b + 2) * raw_mu(c) - 1.5 * A,
                 4.5 * raw_mu(a) * raw_mu(b) * raw_mu(c + 2) - 1.5 * A,
                 9.0 * raw_mu(a + 1) * raw_mu(b + 1) * raw_mu(c),
                 9.0 * raw_mu(a + 1) * raw_mu(b) * raw_mu(c + 1),
                 9.0 * raw_mu(a) * raw_mu(b + 1) * raw_mu(c + 1)};
}

template <int R>
__device__ __forceinline__ float raw_teq(float drho, float rho, float ux, float uy, float uz) {
    constexpr RawEq e = raw_eq(R);
    float s = 0.0f;
    bool any = false;
    auto term = [&](double c, float v) {
        if (c != 0.0) {
            s = any ? fmaf((float)c, v, s) : (float)c * v;
            any = true;
        }
    };
    term(e.Cx, ux);
    term(e.Cy, uy);
    term(e.Cz, uz);
    term(e.Cxx, ux * ux);
    term(e.Cyy, uy * uy);
    term(e.Czz, uz * uz);
    term(e.Cxy, ux * uy);
    term(e.Cxz, ux * uz);
    term(e.Cyz, uy * uz);
    float out = any ? rho * s : 0.0f;
    if constexpr (e.A != 0.0) out = fmaf((float)e.A, drho, out);
    return out;
}

// MODEL: 0 SRT, 1 TRT, 2 MRT (dense, fp64 registers), 3 MRT factorised (Q=27),
// 4 SRT with the per-cell rate `om`.
template <int Q, int MODEL, int FORCE>
__device__ __forceinline__ void collide_cell_c32(float (&g)[Q], const KParams& p, double om = 0.0) {
    using D = Dirs<Q>;
    if constexpr (MODEL == 3 && FORCE == 0) {
        // Unforced factorised D3Q27 MRT entirely in raw-moment space:
        //   t = R g,  t' = teq + (I - K)(t - teq),  g' = Rinv t'
        // (R g of the centred populations gives drho = t_0 and j = (t_1,
        // t_3, t_9) directly; teq is analytic, raw_teq).  About 30 % fewer
        // instructions than forming feq per direction and transforming
        // g - feq, on a kernel that runs close to its issue limit.
        static_assert(Q == 27, "factorised MRT is D3Q27 only");
        float t[27];
        static_for<0, 27>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            t[tpos27<i>()] = g[i];
        });
        raw_fwd_axis<1>(t);
        raw_fwd_axis<3>(t);
        raw_fwd_axis<9>(t);
        const float drho = t[0];
        const float rho = 1.0f + drho;
        const float inv = 1.0f / rho;
        const float ux = t[1] * inv, uy = t[3] * inv, uz = t[9] * inv;
        const float ex = raw_teq<RAW_XX>(drho, rho, ux, uy, uz);
        const float ey = raw_teq<RAW_YY>(drho, rho, ux, uy, uz);
        const float ez = raw_teq<RAW_ZZ>(drho, rho, ux, uy, uz);
        const float bx = t[RAW_XX] - ex, by = t[RAW_YY] - ey, bz = t[RAW_ZZ] - ez;
        static_for<0, 27>([&](auto K_) {
            constexpr int k = decltype(K_)::value;
            if constexpr (k != RAW_XX && k != RAW_YY && k != RAW_ZZ) {
                const float teq = raw_teq<k>(drho, rho, ux, uy, uz);
                t[k] = fmaf(c_mrt_kd[k], t[k] - teq, teq);
            }
        });
        t[RAW_XX] = fmaf(c_mrt_kb[0], bx, fmaf(c_mrt_kb[1], by, fmaf(c_mrt_kb[2], bz, ex)));
        t[RAW_YY] = fmaf(c_mrt_kb[3], bx, fmaf(c_mrt_kb[4], by, fmaf(c_mrt_kb[5], bz, ey)));
        t[RAW_ZZ] = fmaf(c_mrt_kb[6], bx, fmaf(c_mrt_kb[7], by, fmaf(c_mrt_kb[8], bz, ez)));
        raw_inv_axis<1>(t);
        raw_inv_axis<3>(t);
        raw_inv_axis<9>(t);
        static_for<0, 27>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            g[i] = t[tpos27<i>()];
        });
        return;
    } else if constexpr (MODEL == 2) {
        // dense tables: widen, run the fp64 restatement, re-centre
        double f[Q];
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            f[i] = (double)g[i] + wt<Q, i>();
        });
        collide_cell<Q, 2, FORCE>(f, p);
        static_for<0, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            g[i] = (float)(f[i] - wt<Q, i>());
        });
        return;
    } else {
        constexpr bool GUO = FORCE == 1 || FORCE == 3;
        constexpr bool XO = FORCE == 3;
        // density deviation and momentum from the pair sums / differences of
        // (i, opp(i)), i < opp(i): drho = g_0 + sum sp, j = sum c_i dm
        float sp[Q], dm[Q];
        float s[3] = {g[0], 0.f, 0.f};
        float mx = 0.f, my = 0.f, mz = 0.f;
        static_for<1, Q>([&](auto I_) {
            constexpr int i = decltype(I_)::value;
            constexpr int j = D::opp[i];
            if constexpr (i < j) {
                sp[i] = g[i] + g[j];
                dm[i] = g[i] - g[j];
                s[i % 3] += sp[i];
                if constexpr (D::cx[i] == 1) mx += dm[i];
                if constexpr (D::cx[i] == -1) mx -= dm[i];
                if constexpr (D::cy[i] == 1) my += dm[i];
                if constexpr (D::cy[i] == -1) my -= dm[i];
                if constexpr (D::cz[i] == 1) mz += dm[i];
                if constexpr (D::cz[i] == -1) mz -= dm[i];
            }
        });
        const float drho = (s[0] + s[1]) + s[2];
        const float rho = 1.0f + drho;
        const float inv = 1.0f / rho;
        float ux = mx * inv;
        float uy = my * inv;
        float uz = mz * inv;
        if constexpr (FORCE != 0) {
            ux = fmaf(p.fsfx, inv, ux);
            uy = fmaf(p.fsfy, inv, uy);
            uz = fmaf(p.fsfz, inv, uz);
        }
        const float usq15 = 1.5f * ((ux * ux + uy * uy) + uz * uz);

        if constexpr (MODEL == 0 || MODEL == 4) {
            const float rem = MODEL == 0 ? p.frem : (float)(1.0 - om);
            const float hw = MODEL == 0 ? p.fhw : (float)(1.0 - 0.5 * om);
            static_for<0, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                const float cu = cu_of<Q, i, float>(ux, uy, uz);
                const float X = fmaf(4.5f * cu, cu, 3.0f * cu) - usq15;
                const float geq = fmaf(wtf<Q, i>() * rho, X, wtf<Q, i>() * drho);
                float v = fmaf(rem, g[i] - geq, geq);
                if constexpr (GUO) v = fmaf(hw, guo_F32<Q, i, XO>(ux, uy, uz, cu, p), v);
                g[i] = v;
            });
        } else if constexpr (MODEL == 1) {
            // TRT on pair sums s = g_i + g_j and differences d = g_i - g_j:
            //   g_i' = g_i + X + Y,  g_j' = g_j + X - Y,
            //   X = P - omega_e (s/2 - g^eq+),  Y = Qd - omega_o (d/2 - g^eq-)
            // with the Guo pair terms P = he_half (F_i + F_j) = he6w (3 cu (c.F) - u.F)
            // and Qd = ho_half (F_i - F_j) = ho6w (c.F), a per-direction constant.
            float uF = 0.f;
            if constexpr (GUO) {
                if constexpr (XO) uF = ux * p.ffx;
                else uF = fmaf(ux, p.ffx, fmaf(uy, p.ffy, uz * p.ffz));
            }
            static_for<0, Q>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                constexpr int j = D::opp[i];
                if constexpr (i == 0) {
                    const float geq0 = fmaf(wtf<Q, 0>() * rho, -usq15, wtf<Q, 0>() * drho);
                    float v = fmaf(-p.fomega_e, g[0] - geq0, g[0]);
                    if constexpr (GUO) v = fmaf(p.fguo_p[0], -uF, v);
                    g[0] = v;
                } else if constexpr (i < j) {
                    const float cu = cu_of<Q, i, float>(ux, uy, uz);
                    const float wr = wtf<Q, i>() * rho;
                    const float ep = fmaf(wr, fmaf(4.5f * cu, cu, -usq15), wtf<Q, i>() * drho);
                    const float em = (3.0f * wr) * cu;
                    float X = p.fomega_e * fmaf(-0.5f, sp[i], ep);
                    float Y = p.fomega_o * fmaf(-0.5f, dm[i], em);
                    if constexpr (GUO) {
                        X = fmaf(p.fguo_p[i], fmaf(3.0f * cu, p.fcF[i], -uF), X);
                        Y = Y + p.fguo_q[i];
                    }
                    g[i] = (g[i] + X) + Y;
                    g[j] = (g[j] + X) - Y;
                }
            });
        } else {
            static_assert(MODEL == 3 && Q == 27, "factorised MRT is D3Q27 only");
            // f' = f + F - Rinv K R (f - feq + F/2) rewritten as
            //   g' = g^eq + F/2 + Rinv (I - K) R e,   e = g - g^eq + F/2,
            // so only ONE 27-value array is live across the transforms: the
            // populations die as e is formed, and g^eq / F are recomputed
            // (cheap ALU) at the end instead of being held in registers
            // (72 -> fewer registers, more resident warps on a latency-bound
            // kernel).  c_mrt_kd / c_mrt_kb hold I - K (set_mrt_fast_f32).
            auto geq_of = [&](auto I_) {
                constexpr int i = decltype(I_)::value;
                const float cu = cu_of<27, i, float>(ux, uy, uz);
                const float X = fmaf(4.5f * cu, cu, 3.0f * cu) - usq15;
                float e = fmaf(wtf<27, i>() * rho, X, wtf<27, i>() * drho);
                if constexpr (GUO) e = fmaf(0.5f, guo_F32<27, i, XO>(ux, uy, uz, cu, p), e);
                return e;    // g^eq (+ F/2)
            };
            float t[27];
            static_for<0, 27>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                float e = g[i] - geq_of(I_);
                if constexpr (GUO) {
                    // e = g - g^eq + F/2 = g - (g^eq + F/2) + F
                    e += guo_F32<27, i, XO>(ux, uy, uz, cu_of<27, i, float>(ux, uy, uz), p);
                }
                t[tpos27<i>()] = e;
            });
            raw_fwd_axis<1>(t);
            raw_fwd_axis<3>(t);
            raw_fwd_axis<9>(t);
            const float bx = t[RAW_XX], by = t[RAW_YY], bz = t[RAW_ZZ];
            static_for<0, 27>([&](auto K_) {
                constexpr int k = decltype(K_)::value;
                if constexpr (k != RAW_XX && k != RAW_YY && k != RAW_ZZ) t[k] *= c_mrt_kd[k];
            });
            t[RAW_XX] = fmaf(c_mrt_kb[0], bx, fmaf(c_mrt_kb[1], by, c_mrt_kb[2] * bz));
            t[RAW_YY] = fmaf(c_mrt_kb[3], bx, fmaf(c_mrt_kb[4], by, c_mrt_kb[5] * bz));
            t[RAW_ZZ] = fmaf(c_mrt_kb[6], bx, fmaf(c_mrt_kb[7], by, c_mrt_kb[8] * bz));
            raw_inv_axis<1>(t);
            raw_inv_axis<3>(t);
            raw_inv_axis<9>(t);
            static_for<0, 27>([&](auto I_) {
                constexpr int i = decltype(I_)::value;
                g[i] = geq_of(I_) + t[tpos27<i>()];
            });
        }
    }
}

}  // namespace lbm
