// Velocity sets, compile-time.
//
// Direction order is the reference's: sorted by (|c|^2, c_z, c_y, c_x), rest
// direction first (lbm/stencil.py:97-111).  Weights are the correctly rounded
// doubles of the exact rationals (stencil.py:36-41, 61).  The storage slot of
// a direction groups directions by c_z (-1, 0, +1) so the populations that
// cross a z-face are one contiguous run per plane (see include/lbm_b200.h).
#pragma once
#include <type_traits>

namespace lbm {

template <int Q> struct Dirs;

template <> struct Dirs<9> {
    static constexpr int q = 9;
    static constexpr int cx[9] = {0, 0, -1, 1, 0, -1, 1, -1, 1};
    static constexpr int cy[9] = {0, -1, 0, 0, 1, -1, -1, 1, 1};
    static constexpr int cz[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    static constexpr int opp[9] = {0, 4, 3, 2, 1, 8, 7, 6, 5};
    static constexpr double w[9] = {4.0 / 9.0, 1.0 / 9.0, 1.0 / 9.0, 1.0 / 9.0, 1.0 / 9.0,
                                    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};
};

template <> struct Dirs<19> {
    static constexpr int q = 19;
    static constexpr int cx[19] = {0, 0, 0, -1, 1, 0, 0, 0, -1, 1, 0, -1, 1, -1, 1, 0, -1, 1, 0};
    static constexpr int cy[19] = {0, 0, -1, 0, 0, 1, 0, -1, 0, 0, 1, -1, -1, 1, 1, -1, 0, 0, 1};
    static constexpr int cz[19] = {0, -1, 0, 0, 0, 0, 1, -1, -1, -1, -1, 0, 0, 0, 0, 1, 1, 1, 1};
    static constexpr int opp[19] = {0, 6, 5, 4, 3, 2, 1, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7};
    static constexpr double w[19] = {
        1.0 / 3.0,  1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
        1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
        1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};
};

template <> struct Dirs<27> {
    static constexpr int q = 27;
    static constexpr int cx[27] = {0, 0, 0, -1, 1, 0, 0, 0, -1, 1, 0, -1, 1, -1,
                                   1, 0, -1, 1, 0, -1, 1, -1, 1, -1, 1, -1, 1};
    static constexpr int cy[27] = {0, 0, -1, 0, 0, 1, 0, -1, 0, 0, 1, -1, -1, 1,
                                   1, -1, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1, 1};
    static constexpr int cz[27] = {0, -1, 0, 0, 0, 0, 1, -1, -1, -1, -1, 0, 0, 0,
                                   0, 1, 1, 1, 1, -1, -1, -1, -1, 1, 1, 1, 1};
    static constexpr int opp[27] = {0, 6, 5, 4, 3, 2, 1, 18, 17, 16, 15, 14, 13, 12,
                                    11, 10, 9, 8, 7, 26, 25, 24, 23, 22, 21, 20, 19};
    static constexpr double w[27] = {
        8.0 / 27.0,  2.0 / 27.0,  2.0 / 27.0,  2.0 / 27.0,  2.0 / 27.0,  2.0 / 27.0,
        2.0 / 27.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,
        1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,  1.0 / 54.0,
        1.0 / 54.0,  1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0,
        1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0};
};

// weight as a compile-time value (no ODR-use of the table in device code)
template <int Q, int I>
__host__ __device__ __forceinline__ constexpr double wt() {
    constexpr double v = Dirs<Q>::w[I];
    return v;
}

// storage slot: directions with smaller c_z first, reference order within
// (host constexpr: device code only uses these in constant expressions)
template <int Q>
constexpr int slot_of(int i) {
    int s = 0;
    for (int j = 0; j < Q; ++j) {
        if (Dirs<Q>::cz[j] < Dirs<Q>::cz[i] || (Dirs<Q>::cz[j] == Dirs<Q>::cz[i] && j < i)) ++s;
    }
    return s;
}

// number of directions with c_z == v
template <int Q>
constexpr int count_cz(int v) {
    int n = 0;
    for (int j = 0; j < Q; ++j) n += (Dirs<Q>::cz[j] == v) ? 1 : 0;
    return n;
}

// compile-time loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

}  // namespace lbm
