// pruned_fft.cu -- SURVEY §8(f) NEXT-4: the a4-a6 stages (forward FFT, window-deconvolution x
// kernel-coefficient multiply, inverse FFT) for d = 3, computed only where the data are.
//
// The spread writes nothing outside the touched box B (c5: 77^3 of 256^3 cells),
// the multiply keeps only the band |k_a| <= N/2, and the interpolation reads only B. So the
// n^3 transforms of P:L477/L631 reduce to batched 1-D transforms over the rows that can be
// nonzero / are needed, one axis at a time (a multi-dimensional DFT is the product of 1-D DFTs
// along each axis; cuFFT is unnormalised in both directions, like the n^3 D2Z/Z2D it replaces):
//
//   forward  z: D2Z of the nb0 nb1 box rows            -> kz in 0..n/2 (keep 0..h)
//            y: Z2Z of nb0 (h+1) rows, y zero-filled   -> ky (keep |ky| <= h)
//            x: Z2Z of (2h+1)(h+1) rows, x zero-filled -> kx; multiply by D_k, zero outside band
//   inverse  x: Z2Z of the same rows                   -> x (keep the box)
//            y: Z2Z of nb0 (h+1) rows, ky zero-filled  -> y (keep the box)
//            z: Z2D of nb0 nb1 rows, kz > h zero        -> z: the box rows of the grid
// (h = N/2.) Buffers: Ab real [nb0 nb1][n], Zc [nb0 nb1][n/2+1], Yb [nb0][h+1][n],
// Xb [2h+1][h+1][n] (complex). c5: 12 + 12 + 20 + 34 MB instead of two 134 MB passes.
#include <cufft.h>

#include "sk_internal.cuh"

namespace sk {

namespace {

inline int grid_for_p(long long count, int block) {
    long long g = (count + block - 1) / block;
    if (g > 148LL * 32) g = 148LL * 32;
    if (g < 1) g = 1;
    return (int)g;
}

struct PrunedGeom {
    int n, h, hl;              // grid per axis, N/2, n/2 + 1
    int lo0, lo1, lo2;         // box origin
    int nb0, nb1, nb2;         // box extent
};

// grid box rows (full length n in z) -> Ab
__global__ void pack_rows_kernel(PrunedGeom g, const double* __restrict__ grid, double* __restrict__ Ab) {
    const long long total = (long long)g.nb0 * g.nb1 * g.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(e % g.n);
        const long long r = e / g.n;
        const int y = (int)(r % g.nb1), x = (int)(r / g.nb1);
        Ab[e] = grid[((long long)(g.lo0 + x) * g.n + (g.lo1 + y)) * g.n + z];
    }
}

// Zc[(x, y)][kz] -> Yb[x][kz][y_abs] (zero outside the box), kz <= h
__global__ void z_to_y_kernel(PrunedGeom g, const cufftDoubleComplex* __restrict__ Zc,
                              cufftDoubleComplex* __restrict__ Yb) {
    const long long total = (long long)g.nb0 * (g.h + 1) * g.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int ya = (int)(e % g.n);
        const long long r = e / g.n;
        const int kz = (int)(r % (g.h + 1)), x = (int)(r / (g.h + 1));
        const int y = ya - g.lo1;
        cufftDoubleComplex v = make_cuDoubleComplex(0.0, 0.0);
        if (y >= 0 && y < g.nb1) v = Zc[((long long)x * g.nb1 + y) * g.hl + kz];
        Yb[e] = v;
    }
}

// Yb[x][kz][ky_idx] -> Xb[kyb][kz][x_abs] (ky band only; zero outside the box in x)
__global__ void y_to_x_kernel(PrunedGeom g, const cufftDoubleComplex* __restrict__ Yb,
                              cufftDoubleComplex* __restrict__ Xb) {
    const long long total = (long long)(2 * g.h + 1) * (g.h + 1) * g.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int xa = (int)(e % g.n);
        const long long r = e / g.n;
        const int kz = (int)(r % (g.h + 1)), kyb = (int)(r / (g.h + 1));
        const int ky = kyb - g.h, kyi = ky >= 0 ? ky : ky + g.n;
        const int x = xa - g.lo0;
        cufftDoubleComplex v = make_cuDoubleComplex(0.0, 0.0);
        if (x >= 0 && x < g.nb0) v = Yb[((long long)x * (g.h + 1) + kz) * g.n + kyi];
        Xb[e] = v;
    }
}

// Xb[kyb][kz][kx_idx] *= D[(kx + h)(2h+1) + (ky + h)][kz] on the band, 0 elsewhere (a5)
__global__ void band_multiply_kernel(PrunedGeom g, cufftDoubleComplex* __restrict__ Xb,
                                     const double* __restrict__ Dk) {
    const long long total = (long long)(2 * g.h + 1) * (g.h + 1) * g.n;
    const int nb = 2 * g.h + 1;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int kxi = (int)(e % g.n);
        const long long r = e / g.n;
        const int kz = (int)(r % (g.h + 1)), kyb = (int)(r / (g.h + 1));
        const int kx = kxi <= g.n / 2 ? kxi : kxi - g.n;
        cufftDoubleComplex v = Xb[e];
        if (kx >= -g.h && kx <= g.h) {
            const double D = Dk[((long long)(kx + g.h) * nb + kyb) * (g.h + 1) + kz];
            v.x *= D;
            v.y *= D;
        } else {
            v = make_cuDoubleComplex(0.0, 0.0);
        }
        Xb[e] = v;
    }
}

// Xb[kyb][kz][x_abs] -> Yb[x][kz][ky_idx] (ky band, zero elsewhere), x in the box
__global__ void x_to_y_kernel(PrunedGeom g, const cufftDoubleComplex* __restrict__ Xb,
                              cufftDoubleComplex* __restrict__ Yb) {
    const long long total = (long long)g.nb0 * (g.h + 1) * g.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int kyi = (int)(e % g.n);
        const long long r = e / g.n;
        const int kz = (int)(r % (g.h + 1)), x = (int)(r / (g.h + 1));
        const int ky = kyi <= g.n / 2 ? kyi : kyi - g.n;
        cufftDoubleComplex v = make_cuDoubleComplex(0.0, 0.0);
        if (ky >= -g.h && ky <= g.h)
            v = Xb[((long long)(ky + g.h) * (g.h + 1) + kz) * g.n + (g.lo0 + x)];
        Yb[e] = v;
    }
}

// Yb[x][kz][y_abs] -> Zc[(x, y)][kz] (kz <= h, zero above), y in the box
__global__ void y_to_z_kernel(PrunedGeom g, const cufftDoubleComplex* __restrict__ Yb,
                              cufftDoubleComplex* __restrict__ Zc) {
    const long long total = (long long)g.nb0 * g.nb1 * g.hl;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int kz = (int)(e % g.hl);
        const long long r = e / g.hl;
        const int y = (int)(r % g.nb1), x = (int)(r / g.nb1);
        cufftDoubleComplex v = make_cuDoubleComplex(0.0, 0.0);
        if (kz <= g.h) v = Yb[((long long)x * (g.h + 1) + kz) * g.n + (g.lo1 + y)];
        Zc[e] = v;
    }
}

// Ab rows -> grid box rows (full length n in z; the interpolation reads only the box)
__global__ void unpack_rows_kernel(PrunedGeom g, const double* __restrict__ Ab, double* __restrict__ grid) {
    const long long total = (long long)g.nb0 * g.nb1 * g.n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int z = (int)(e % g.n);
        const long long r = e / g.n;
        const int y = (int)(r % g.nb1), x = (int)(r / g.nb1);
        grid[((long long)(g.lo0 + x) * g.n + (g.lo1 + y)) * g.n + z] = Ab[e];
    }
}

PrunedGeom geom_of(const Plan& P) {
    PrunedGeom g;
    g.n = P.n;
    g.h = P.N / 2;
    g.hl = P.n / 2 + 1;
    g.lo0 = P.box_lo[0]; g.lo1 = P.box_lo[1]; g.lo2 = P.box_lo[2];
    g.nb0 = P.box_n[0]; g.nb1 = P.box_n[1]; g.nb2 = P.box_n[2];
    return g;
}

}  // namespace

int pruned_fft_setup(Plan& P, cudaStream_t s) {
    P.pruned = false;
    if (P.d != 3 || getenv("SK_NO_PRUNED_FFT") != nullptr) return SK_OK;
    const long long n = P.n, h = P.N / 2;
    const long long nb0 = P.box_n[0], nb1 = P.box_n[1];
    // only when the box is a real saving (the transforms touch ~ (nb0 nb1 + nb0 h + h^2) rows
    // instead of 3 n^2)
    if (nb0 * nb1 + nb0 * (h + 1) + (2 * h + 1) * (h + 1) >= n * n) return SK_OK;
    P.pr_rows_z = nb0 * nb1;
    P.pr_rows_y = nb0 * (h + 1);
    P.pr_rows_x = (2 * h + 1) * (h + 1);
    SK_TRY(dev_alloc((void**)&P.pr_A, sizeof(double) * P.pr_rows_z * n, s));
    SK_TRY(dev_alloc((void**)&P.pr_Z, sizeof(cufftDoubleComplex) * P.pr_rows_z * (n / 2 + 1), s));
    SK_TRY(dev_alloc((void**)&P.pr_Y, sizeof(cufftDoubleComplex) * P.pr_rows_y * n, s));
    SK_TRY(dev_alloc((void**)&P.pr_X, sizeof(cufftDoubleComplex) * P.pr_rows_x * n, s));
    SK_TRY(fft_acquire(1, (int)n, CUFFT_D2Z, s, &P.pr_fz, P.pr_rows_z));
    SK_TRY(fft_acquire(1, (int)n, CUFFT_Z2D, s, &P.pr_iz, P.pr_rows_z));
    SK_TRY(fft_acquire(1, (int)n, CUFFT_Z2Z, s, &P.pr_y, P.pr_rows_y));
    SK_TRY(fft_acquire(1, (int)n, CUFFT_Z2Z, s, &P.pr_x, P.pr_rows_x));
    P.pruned = true;
    return SK_OK;
}

void pruned_fft_teardown(Plan& P, cudaStream_t s) {
    if (P.pr_fz) fft_release(1, P.n, CUFFT_D2Z, P.pr_fz, P.pr_rows_z);
    if (P.pr_iz) fft_release(1, P.n, CUFFT_Z2D, P.pr_iz, P.pr_rows_z);
    if (P.pr_y) fft_release(1, P.n, CUFFT_Z2Z, P.pr_y, P.pr_rows_y);
    if (P.pr_x) fft_release(1, P.n, CUFFT_Z2Z, P.pr_x, P.pr_rows_x);
    dev_free(P.pr_A, s);
    dev_free(P.pr_Z, s);
    dev_free(P.pr_Y, s);
    dev_free(P.pr_X, s);
    P.pr_A = nullptr; P.pr_Z = nullptr; P.pr_Y = nullptr; P.pr_X = nullptr;
    P.pr_fz = P.pr_iz = P.pr_y = P.pr_x = 0;
    P.pruned = false;
}

#define SK_PR_LAUNCH(kern, total, ...)                                                  \
    do {                                                                                 \
        kern<<<grid_for_p(total, 256), 256, 0, s>>>(__VA_ARGS__);                        \
        count_launch();                                                                  \
        cudaError_t e_ = cudaGetLastError();                                             \
        if (e_ != cudaSuccess) return set_error(SK_ECUDA, std::string(#kern) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// a4 + a5 + a6 on P.grid in place (box rows in, box rows out); kernel selects D_k.
int pruned_fft_apply(Plan& P, int kernel, cudaStream_t s) {
    const PrunedGeom g = geom_of(P);
    const long long n = g.n;
    cufftDoubleComplex* Z = (cufftDoubleComplex*)P.pr_Z;
    cufftDoubleComplex* Y = (cufftDoubleComplex*)P.pr_Y;
    cufftDoubleComplex* X = (cufftDoubleComplex*)P.pr_X;
    prof_begin(ST_FFT_FWD, s);
    SK_PR_LAUNCH(pack_rows_kernel, P.pr_rows_z * n, g, P.grid, P.pr_A);
    SK_CUFFT(cufftExecD2Z(P.pr_fz, P.pr_A, Z));
    count_launch();
    SK_PR_LAUNCH(z_to_y_kernel, P.pr_rows_y * n, g, Z, Y);
    SK_CUFFT(cufftExecZ2Z(P.pr_y, Y, Y, CUFFT_FORWARD));
    count_launch();
    SK_PR_LAUNCH(y_to_x_kernel, P.pr_rows_x * n, g, Y, X);
    SK_CUFFT(cufftExecZ2Z(P.pr_x, X, X, CUFFT_FORWARD));
    count_launch();
    prof_end(ST_FFT_FWD, s);
    prof_begin(ST_MULTIPLY, s);
    SK_PR_LAUNCH(band_multiply_kernel, P.pr_rows_x * n, g, X, P.D[kernel]);
    prof_end(ST_MULTIPLY, s);
    prof_begin(ST_FFT_INV, s);
    SK_CUFFT(cufftExecZ2Z(P.pr_x, X, X, CUFFT_INVERSE));
    count_launch();
    SK_PR_LAUNCH(x_to_y_kernel, P.pr_rows_y * n, g, X, Y);
    SK_CUFFT(cufftExecZ2Z(P.pr_y, Y, Y, CUFFT_INVERSE));
    count_launch();
    SK_PR_LAUNCH(y_to_z_kernel, P.pr_rows_z * (long long)g.hl, g, Y, Z);
    SK_CUFFT(cufftExecZ2D(P.pr_iz, Z, P.pr_A));
    count_launch();
    SK_PR_LAUNCH(unpack_rows_kernel, P.pr_rows_z * n, g, P.pr_A, P.grid);
    prof_end(ST_FFT_INV, s);
    return SK_OK;
}

}  // namespace sk
