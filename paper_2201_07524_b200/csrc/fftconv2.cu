// fftconv2.cu -- d = 2: a4 forward FFT, a5 multiply and a6 inverse FFT as three shared-memory
// Stockham kernels pruned to the touched box and the N-band, with the deterministic spread's
// fixed-point -> FP64 conversion fused into the first one.
//
// The fast summation's middle step (Eq. (fastsum); NFFT steps of P:L475-477) is the
// 2-D periodic convolution g -> F^-1 [D . F g] on the sigma N x sigma N grid, with D zero outside
// the band |k| <= N/2. With the box B = [lo0, lo0 + bn0) x [lo1, lo1 + bn1) holding every nonzero
// of g and every grid value the interpolation reads (plan.cu, the a3 box), the three passes are
//   K1 rows (box rows i0):   S[i0][kl]  = sum_{i1 in B1} g[i0][i1] e^{-2 pi i kl i1 / n}, kl <= N/2
//   K2 columns (kl <= N/2):  S[i0][kl] <- sum_{k0 in band} e^{+2 pi i k0 i0 / n} D[k0][kl]
//                                          sum_{j0 in B0} S[j0][kl] e^{-2 pi i k0 j0 / n},  i0 in B0
//   K3 rows (box rows i0):   g[i0][i1]  = Re sum_k F[k] e^{+2 pi i k i1 / n},  F[kl] = S[i0][kl],
//                                          F[n - kl] = conj S[i0][kl] (kl = 1..N/2), 0 elsewhere
// -- the same unnormalised transforms as cuFFT's D2Z / Z2D (every constant lives in D), so the
// result equals D2Z -> multiply_kernel -> Z2D up to rounding. It replaces five cuFFT/multiply
// launches and the deterministic conversion (six kernels) by three: the d = 2 workloads (c2, the
// images) are launch- and latency-bound at ~50 us per fast summation.
//
// Each pass is one length-n radix-2 Stockham FFT per CTA in shared memory (n = sigma N, a power
// of two in [64, 1024]); twiddles e^{-2 pi i k / n}, k < n/2, come from a plan-time table built in
// long double on the host.
#include "sk_internal.cuh"

namespace sk {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
    return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}

// In-place-by-swap Stockham autosort (natural order in and out). Returns the buffer holding the
// result. INV: e^{+2 pi i ...}. Called by all T threads of the CTA; ends with __syncthreads().
template <int NN, int T, bool INV>
__device__ __forceinline__ double2* fft_stockham(double2* x, double2* y, const double2* tw) {
#pragma unroll
    for (int Ns = 1; Ns < NN; Ns <<= 1) {
#pragma unroll
        for (int j = threadIdx.x; j < NN / 2; j += T) {
            const int k = j & (Ns - 1);
            double2 w = tw[k * (NN / (2 * Ns))];
            if (INV) w.y = -w.y;
            const double2 a = x[j];
            const double2 b = cmul(x[j + NN / 2], w);
            const int o = ((j - k) << 1) + k;
            y[o] = make_double2(a.x + b.x, a.y + b.y);
            y[o + Ns] = make_double2(a.x - b.x, a.y - b.y);
        }
        __syncthreads();
        double2* t = x;
        x = y;
        y = t;
    }
    return x;
}

template <int NN, int T>
__device__ __forceinline__ void load_twiddles(double2* tws, const double2* __restrict__ tw) {
    for (int k = threadIdx.x; k < NN / 2; k += T) tws[k] = tw[k];
}

struct FcGeom {
    int n, h;              // grid edge, N / 2
    int lo0, bn0, lo1, bn1;
    long long ld;          // row stride of the spectrum scratch (h + 1)
};

// K1: one box row per CTA. Deterministic mode: X = hi 2^32 + lo read from the fixed-point box
// accumulator (and cleared), value X 2^-S (as grid_fix_convert_kernel); the last CTA clears the
// source vector's bound slot. Atomic mode: the FP64 grid row.
template <int NN, int T>
__global__ void __launch_bounds__(T) fc2_rows_fwd_kernel(const FcGeom g, const GridAcc ga, const double* __restrict__ grid,
                                                         const double2* __restrict__ tw, double2* __restrict__ S,
                                                         unsigned* __restrict__ done, unsigned* __restrict__ slot) {
    __shared__ double2 buf[2][NN];
    __shared__ double2 tws[NN / 2];
    load_twiddles<NN, T>(tws, tw);
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;   // box row
    const int i0 = g.lo0 + r;
    double inv = 1.0;
    bool finite = true;
    if (ga.acc) {
        const unsigned hi = *ga.wmax;
        inv = 1.0 / grid_scale(ga);
        finite = isfinite(__longlong_as_double((long long)(((unsigned long long)hi << 32) | 0xffffffffULL)));
    }
    for (int c = threadIdx.x; c < NN; c += T) {
        const int cb = c - g.lo1;
        double v = 0.0;
        if (cb >= 0 && cb < g.bn1) {
            if (ga.acc) {
                const long long bi = (long long)r * g.bn1 + cb;
                const long long hw = (long long)ga.acc[2 * bi];
                const unsigned long long lw = ga.acc[2 * bi + 1];
                ga.acc[2 * bi] = 0ULL;
                ga.acc[2 * bi + 1] = 0ULL;
                const long long H = hw + (long long)(lw >> 32);
                const double L = (double)(lw & 0xffffffffULL);
                v = finite ? fma((double)H, 4294967296.0, L) * inv : NAN;
            } else {
                v = grid[(long long)i0 * NN + c];
            }
        }
        buf[0][c] = make_double2(v, 0.0);
    }
    __syncthreads();
    const double2* X = fft_stockham<NN, T, false>(buf[0], buf[1], tws);
    for (int k = threadIdx.x; k <= g.h; k += T) S[(long long)i0 * g.ld + k] = X[k];
    if (ga.acc) {   // every CTA has read the slot above; the last one clears it
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(done, 1u) == gridDim.x - 1) {
                *slot = 0u;
                *done = 0u;
            }
        }
    }
}

// K2: one band column kl per CTA: forward along axis 0 over the box rows, x D (zero outside the
// band), inverse, written back for the box rows.
template <int NN, int T>
__global__ void __launch_bounds__(T) fc2_cols_kernel(const FcGeom g, const double* __restrict__ Dk,
                                                     const double2* __restrict__ tw, double2* __restrict__ S) {
    __shared__ double2 buf[2][NN];
    __shared__ double2 tws[NN / 2];
    load_twiddles<NN, T>(tws, tw);
    pdl_trigger();
    pdl_wait();
    const int kl = blockIdx.x;
    for (int i = threadIdx.x; i < NN; i += T) {
        const int ib = i - g.lo0;
        buf[0][i] = (ib >= 0 && ib < g.bn0) ? S[(long long)i * g.ld + kl] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double2* X = fft_stockham<NN, T, false>(buf[0], buf[1], tws);
    double2* Y = X == buf[0] ? buf[1] : buf[0];
    for (int i = threadIdx.x; i < NN; i += T) {
        const int k0 = i <= NN / 2 ? i : i - NN;
        double2 z = make_double2(0.0, 0.0);
        if (k0 >= -g.h && k0 <= g.h) {
            const double D = Dk[(long long)(k0 + g.h) * (g.h + 1) + kl];
            z = make_double2(X[i].x * D, X[i].y * D);
        }
        X[i] = z;
    }
    __syncthreads();
    const double2* R = fft_stockham<NN, T, true>(X, Y, tws);
    for (int ib = threadIdx.x; ib < g.bn0; ib += T) S[(long long)(g.lo0 + ib) * g.ld + kl] = R[g.lo0 + ib];
}

// K3: one box row per CTA: the Hermitian extension of the band half-row, inverse, real part.
template <int NN, int T>
__global__ void __launch_bounds__(T) fc2_rows_inv_kernel(const FcGeom g, const double2* __restrict__ tw,
                                                         const double2* __restrict__ S, double* __restrict__ grid) {
    __shared__ double2 buf[2][NN];
    __shared__ double2 tws[NN / 2];
    load_twiddles<NN, T>(tws, tw);
    pdl_trigger();
    pdl_wait();
    const int i0 = g.lo0 + blockIdx.x;
    const double2* row = S + (long long)i0 * g.ld;
    for (int k = threadIdx.x; k < NN; k += T) {
        double2 z = make_double2(0.0, 0.0);
        if (k <= g.h) z = row[k];
        else if (k >= NN - g.h) { z = row[NN - k]; z.y = -z.y; }
        buf[0][k] = z;
    }
    __syncthreads();
    const double2* R = fft_stockham<NN, T, true>(buf[0], buf[1], tws);
    for (int c = threadIdx.x; c < NN; c += T) grid[(long long)i0 * NN + c] = R[c].x;
}

template <int NN>
int run(const FcGeom& g, const GridAcc& ga, const double* grid_in, const double* Dk, const double2* tw,
        double2* S, double* grid_out, unsigned* done, unsigned* slot, cudaStream_t s) {
    constexpr int T = NN / 2 < 256 ? NN / 2 : 256;
    cudaError_t e = launch_pdl(fc2_rows_fwd_kernel<NN, T>, g.bn0, T, 0, s, g, ga, grid_in, tw, S, done, slot);
    if (e == cudaSuccess) e = launch_pdl(fc2_cols_kernel<NN, T>, g.h + 1, T, 0, s, g, Dk, tw, S);
    if (e == cudaSuccess) e = launch_pdl(fc2_rows_inv_kernel<NN, T>, g.bn0, T, 0, s, g, tw, S, grid_out);
    count_launch(3);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("fftconv2 launch: ") + cudaGetErrorString(e));
    return SK_OK;
}

}  // namespace

bool fftconv2_supported(int d, int n, int N) {
    if (d != 2 || n < 64 || n > 1024 || (n & (n - 1)) || N / 2 >= n / 2) return false;
    return getenv("SK_NO_FFTCONV2") == nullptr;
}

void fftconv2_twiddles(int n, double* out) {   // [n/2] (re, im) of e^{-2 pi i k / n}
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < n / 2; ++k) {
        const long double a = -2.0L * pi * (long double)k / (long double)n;
        out[2 * k] = (double)cosl(a);
        out[2 * k + 1] = (double)sinl(a);
    }
}

int fftconv2_apply(Plan& P, int kernel, const GridAcc& ga, unsigned* slot, cudaStream_t s) {
    FcGeom g;
    g.n = P.n;
    g.h = P.N / 2;
    g.lo0 = P.box_lo[0];
    g.bn0 = P.box_n[0];
    g.lo1 = P.box_lo[1];
    g.bn1 = P.box_n[1];
    g.ld = g.h + 1;
    const double2* tw = reinterpret_cast<const double2*>(P.fc_tw);
    double2* S = reinterpret_cast<double2*>(P.spec);
    unsigned* done = P.deterministic ? P.det_wmax + kWSlots : nullptr;
    switch (P.n) {
        case 64: return run<64>(g, ga, P.grid, P.D[kernel], tw, S, P.grid, done, slot, s);
        case 128: return run<128>(g, ga, P.grid, P.D[kernel], tw, S, P.grid, done, slot, s);
        case 256: return run<256>(g, ga, P.grid, P.D[kernel], tw, S, P.grid, done, slot, s);
        case 512: return run<512>(g, ga, P.grid, P.D[kernel], tw, S, P.grid, done, slot, s);
        case 1024: return run<1024>(g, ga, P.grid, P.D[kernel], tw, S, P.grid, done, slot, s);
        default: return set_error(SK_EINVAL, "fftconv2: unsupported grid edge");
    }
}

}  // namespace sk
