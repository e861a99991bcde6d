// winpoly.h -- piecewise-polynomial form of the Kaiser-Bessel window (host side).
//
// For a node at grid coordinate u with c = floor(u), f = u - c in [0, 1), the 2m taps
// l = c - m + 1 + t take the window values phi(f + m - 1 - t), t = 0 .. 2m-1. Each tap is an
// entire function of f (phi(u) = (beta/pi) sum_k (beta^2 (m^2 - u^2))^k / (2k+1)!), so a degree
// kWinDeg polynomial in g = f - 1/2 reproduces it to FP64 roundoff: interpolation at the
// Chebyshev nodes of [-1/2, 1/2] in long double, converted to monomials in g, rounded to
// double (max error <= 4e-16 of the peak phi(0) for m <= 8, checked at plan time). The
// kernels then evaluate 2m Horner polynomials with compile-time coefficient indices, which
// ptxas turns into constant-bank DFMA operands (no loads).
#pragma once

#include <math.h>

namespace sk {

constexpr int kWinDeg = 14;          // polynomial degree per tap
constexpr int kWinNC = kWinDeg + 1;  // coefficients per tap

struct WinPoly {
    double c[16][kWinNC];  // [tap t][power q] of g = f - 1/2
};

inline long double kb_phi_ld(long double u, int m, long double beta) {
    long double s2 = (long double)m * m - u * u;
    if (s2 > 0) {
        long double s = sqrtl(s2);
        return sinhl(beta * s) / (s * 3.14159265358979323846264338327950288L);
    }
    return s2 == 0 ? beta / 3.14159265358979323846264338327950288L : 0.0L;
}

// Returns the max abs error relative to phi(0) over a test grid (or -1 on bad m).
inline double build_winpoly(int m, double sigma, WinPoly* wp) {
    if (m < 1 || m > 8) return -1.0;
    const long double PI = 3.14159265358979323846264338327950288L;
    const long double beta = PI * (2.0L - 1.0L / (long double)sigma);
    const int K = kWinNC;
    for (int t = 0; t < 16; ++t)
        for (int q = 0; q < K; ++q) wp->c[t][q] = 0.0;
    for (int t = 0; t < 2 * m; ++t) {
        // Chebyshev coefficients a_k of p(x), x = 2 g in [-1, 1]
        long double fv[kWinNC], a[kWinNC];
        for (int j = 0; j < K; ++j) {
            long double th = PI * (j + 0.5L) / K;
            long double g = 0.5L * cosl(th);
            fv[j] = kb_phi_ld(g + 0.5L + (long double)(m - 1 - t), m, beta);
        }
        for (int k = 0; k < K; ++k) {
            long double s = 0;
            for (int j = 0; j < K; ++j) s += fv[j] * cosl(PI * k * (j + 0.5L) / K);
            a[k] = s * 2.0L / K;
        }
        a[0] *= 0.5L;
        // monomials in x via T_{k+1} = 2 x T_k - T_{k-1}
        long double Tm1[kWinNC] = {0}, T0[kWinNC] = {0}, T1[kWinNC] = {0}, mono[kWinNC] = {0};
        T0[0] = 1.0L;
        for (int q = 0; q < K; ++q) mono[q] += a[0] * T0[q];
        if (K > 1) {
            T1[1] = 1.0L;
            for (int q = 0; q < K; ++q) mono[q] += a[1] * T1[q];
        }
        for (int q = 0; q < K; ++q) Tm1[q] = T0[q];
        long double cur[kWinNC];
        for (int q = 0; q < K; ++q) cur[q] = T1[q];
        for (int k = 2; k < K; ++k) {
            long double nxt[kWinNC] = {0};
            for (int q = 0; q < K; ++q) {
                if (q > 0) nxt[q] += 2.0L * cur[q - 1];
                nxt[q] -= Tm1[q];
            }
            for (int q = 0; q < K; ++q) mono[q] += a[k] * nxt[q];
            for (int q = 0; q < K; ++q) { Tm1[q] = cur[q]; cur[q] = nxt[q]; }
        }
        // x = 2 g  ->  coefficient of g^q is mono[q] 2^q
        long double p2 = 1.0L;
        for (int q = 0; q < K; ++q) { wp->c[t][q] = (double)(mono[q] * p2); p2 *= 2.0L; }
    }
    // validation against the direct formula in long double
    const long double peak = kb_phi_ld(0.0L, m, beta);
    double worst = 0.0;
    for (int t = 0; t < 2 * m; ++t)
        for (int i = 0; i <= 256; ++i) {
            double f = i / 256.0;
            if (f >= 1.0) f = 1.0 - 1e-16;
            double g = f - 0.5, acc = wp->c[t][K - 1];
            for (int q = K - 2; q >= 0; --q) acc = acc * g + wp->c[t][q];
            long double ex = kb_phi_ld((long double)f + (m - 1 - t), m, beta);
            double e = (double)(fabsl((long double)acc - ex) / peak);
            if (e > worst) worst = e;
        }
    return worst;
}

}  // namespace sk
