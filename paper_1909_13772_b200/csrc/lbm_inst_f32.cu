// fp32 storage of (f - w_i), fp32 register arithmetic on the centred
// populations (lbm_collide_f32.cuh); FMA contraction allowed: this variant is
// compared against the fp64 oracle with a relative tolerance, not bitwise.
#include <math.h>

#define LBM_REAL float
#define LBM_UNIT unit_f32
#include "lbm_inst.cuh"

namespace lbm {
LBM_DEFINE_MRT_SETTER(set_mrt_tables_f32)

// K = R Minv diag(S) M Rinv in the tensor raw-moment basis of D3Q27
// (raw index a + 3b + 9c <-> moment cx^a cy^b cz^c).  The factorised kernel
// supports K = diagonal + one 3x3 block on (xx, yy, zz); with Guo forcing the
// G table must equal Minv (I - S/2) M, i.e. R G Rinv = I - K/2 (checked).
cudaError_t set_mrt_fast_f32(int q, const double* tables, cudaStream_t s, int* fast) {
    static DeviceTableCache cache;
    *fast = 0;
    if (q != 27) return cudaSuccess;
    const size_t n = 3 * 27 * 27 + 27;
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    std::lock_guard<std::mutex> lock(cache.mu);
    if (cache.hit(dev, tables, n, fast)) return cudaSuccess;
    const double* M = tables;
    const double* Minv = tables + 27 * 27;
    const double* S = tables + 2 * 27 * 27;
    const double* G = tables + 2 * 27 * 27 + 27;
    using D = Dirs<27>;
    // per-axis transform T1 (rows: power 0,1,2; cols: c = -1,0,1) and inverse
    const double T1[3][3] = {{1, 1, 1}, {-1, 0, 1}, {1, 0, 1}};
    const double T1i[3][3] = {{0, -0.5, 0.5}, {1, 0, -1}, {0, 0.5, 0.5}};  // [c][power]
    // (scratch on the heap of this call: several rank threads may derive at once)
    std::vector<double> scratch(6 * 27 * 27);
    auto R = reinterpret_cast<double(*)[27]>(scratch.data());
    auto Ri = R + 27, A = R + 54, C = R + 81, K = R + 108, H = R + 135;
    for (int r = 0; r < 27; ++r) {
        const int a = r % 3, b = (r / 3) % 3, c = r / 9;
        for (int i = 0; i < 27; ++i) {
            const int x = D::cx[i] + 1, y = D::cy[i] + 1, z = D::cz[i] + 1;
            R[r][i] = T1[a][x] * T1[b][y] * T1[c][z];
            Ri[i][r] = T1i[x][a] * T1i[y][b] * T1i[z][c];
        }
    }
    auto conj = [&](const double* X, bool scale_s, double (*out)[27]) {
        // out = R * Minv * diag(S) * M * Ri (scale_s) or R * X * Ri
        for (int a = 0; a < 27; ++a)
            for (int r = 0; r < 27; ++r) {
                double acc = 0;
                for (int i = 0; i < 27; ++i) acc += (scale_s ? M[a * 27 + i] : X[a * 27 + i]) * Ri[i][r];
                A[a][r] = scale_s ? S[a] * acc : acc;
            }
        if (scale_s) {
            for (int i = 0; i < 27; ++i)
                for (int r = 0; r < 27; ++r) {
                    double acc = 0;
                    for (int a = 0; a < 27; ++a) acc += Minv[i * 27 + a] * A[a][r];
                    C[i][r] = acc;
                }
        } else {
            for (int i = 0; i < 27; ++i)
                for (int r = 0; r < 27; ++r) C[i][r] = A[i][r];
        }
        for (int sg = 0; sg < 27; ++sg)
            for (int r = 0; r < 27; ++r) {
                double acc = 0;
                for (int i = 0; i < 27; ++i) acc += R[sg][i] * C[i][r];
                out[sg][r] = acc;
            }
    };
    conj(nullptr, true, K);
    const int blk[3] = {RAW_XX, RAW_YY, RAW_ZZ};
    auto in_blk = [&](int r) { return r == RAW_XX || r == RAW_YY || r == RAW_ZZ; };
    double kmax = 0;
    for (int a = 0; a < 27; ++a)
        for (int b = 0; b < 27; ++b) kmax = fmax(kmax, fabs(K[a][b]));
    const double tol = 1e-10 * (1.0 + kmax);
    int ok = 1;
    for (int a = 0; a < 27 && ok; ++a)
        for (int b = 0; b < 27; ++b)
            if (a != b && !(in_blk(a) && in_blk(b)) && fabs(K[a][b]) > tol) { ok = 0; break; }
    bool g_zero = true;
    for (int i = 0; i < 27 * 27; ++i) g_zero = g_zero && G[i] == 0.0;
    if (ok && !g_zero) {
        conj(G, false, H);
        for (int a = 0; a < 27 && ok; ++a)
            for (int b = 0; b < 27; ++b)
                if (fabs(H[a][b] - ((a == b ? 1.0 : 0.0) - 0.5 * K[a][b])) > tol) { ok = 0; break; }
    }
    if (ok) {
        // the kernel applies I - K (lbm_collide_f32.cuh, factorised MRT)
        float kd[27], kb[9];
        for (int r = 0; r < 27; ++r) kd[r] = (float)(1.0 - K[r][r]);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                kb[a * 3 + b] = (float)((a == b ? 1.0 : 0.0) - K[blk[a]][blk[b]]);
        cudaError_t e;
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_kd, kd, sizeof(kd), 0, cudaMemcpyHostToDevice, s)) !=
            cudaSuccess)
            return e;
        if ((e = cudaMemcpyToSymbolAsync(c_mrt_kb, kb, sizeof(kb), 0, cudaMemcpyHostToDevice, s)) !=
            cudaSuccess)
            return e;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    }
    cache.store(dev, tables, n, ok);
    *fast = ok;
    return cudaSuccess;
}
}  // namespace lbm
