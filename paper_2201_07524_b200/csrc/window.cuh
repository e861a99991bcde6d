// window.cuh -- Kaiser-Bessel window of the NFFT (reading Q10 of PAPER.md P:L475-477).
//
// In oversampled-grid units u (one grid cell = 1):
//   phi(u) = sinh(beta * sqrt(m^2 - u^2)) / (pi * sqrt(m^2 - u^2)),  |u| < m
//          = beta / pi                                                |u| = m (limit)
//          = 0                                                        |u| > m (truncated)
// beta = pi (2 - 1/sigma). Its Fourier transform int phi(u) e^{-2 pi i xi u} du is
// I0(m sqrt(beta^2 - (2 pi xi)^2)) (used for the deconvolution in plan.cu).
#pragma once
#include "sk_internal.cuh"

namespace sk {

__device__ __forceinline__ double kb_phi(double u, const Window& w) {
    double s2 = w.m2 - u * u;
    if (s2 > 0.0) {
        double s = sqrt(s2);
        return sinh(w.beta * s) / (s * 3.141592653589793238462643);
    }
    return s2 == 0.0 ? w.beta * w.inv_pi : 0.0;
}

// Tap values of one axis for a node at grid coordinate u: taps l = c - m + 1 + t,
// t = 0 .. 2m-1, c = floor(u); phi_t = phi(u - l). Returns c.
__device__ __forceinline__ int kb_taps(double u, const Window& w, double* phi) {
    double c = floor(u);
    double f = u - c;  // in [0, 1)
    const int W = 2 * w.m;
#pragma unroll 4
    for (int t = 0; t < W; ++t) phi[t] = kb_phi(f + (double)(w.m - 1 - t), w);
    return (int)c;
}

}  // namespace sk
