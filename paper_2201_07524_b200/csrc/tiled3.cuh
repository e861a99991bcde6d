// tiled3.cuh -- v2 spread / interp for d = 3 on tiles of T^3 = 2^3 grid cells (sm_100a, FP64).
//
// Nodes are sorted by tile (plan.cu); a work item is one tile, or a chunk of at most
// kItemMax nodes of a dense tile. Every node of a tile touches taps inside the tile's
// region of R = T + W - 1 cells per axis (W = 2 m taps per axis), so
//
//   interp: the CTA stages the region of the grid in shared memory (R^3 doubles, one
//           coalesced load per item), lanes = nodes (2 per lane), the per-node window
//           values live in registers (z) and lane-private shared rows (x, y) over the whole
//           region (zeros outside the node's 2m support), and the region loop is
//           warp-uniform: every grid value is a broadcast LDS.128 feeding 4 DFMAs.
//   spread: lanes own 2 region columns (x,y) of R z-values in registers; per chunk of 64
//           nodes the CTA tabulates w*phi_x, phi_y, phi_z in shared memory (lanes = nodes),
//           then loops over the nodes (warp-uniform) with a broadcast phi_z row: per node
//           and lane 2 DMUL + 2R DFMA. The region is flushed once per item with coalesced
//           FP64 atomics (RED) into the global grid (neighbouring regions overlap).
//
// Window values come from the degree-14 tap polynomials of winpoly.h (compile-time indices
// into a __grid_constant__ parameter -> constant-bank operands).
#pragma once
#include "sk_internal.cuh"
#include "winpoly.h"

namespace sk {

struct TileItem {
    int tile;   // tile id (row-major over tiles_per_axis^d)
    int start;  // first node (sorted order)
    int count;  // nodes in this item
    int pad;
};

constexpr int kItemMax = 4096;  // nodes per work item (dense tiles are split)

template <int W>
__device__ __forceinline__ void win_taps(double f, const WinPoly& wp, double (&v)[W]) {
    const double g = f - 0.5;
#pragma unroll
    for (int t = 0; t < W; ++t) {
        double acc = wp.c[t][kWinDeg];
#pragma unroll
        for (int q = kWinDeg - 1; q >= 0; --q) acc = fma(acc, g, wp.c[t][q]);
        v[t] = acc;
    }
}

// Region weights for T = 2: phi[r] = v[r - c] (c in {0,1}), zero outside the support.
template <int W, int RP>
__device__ __forceinline__ void region_weights(const double (&v)[W], int c, double scale, double (&phi)[RP]) {
#pragma unroll
    for (int r = 0; r < RP; ++r) {
        double a = (r < W) ? v[r < W ? r : 0] : 0.0;          // c == 0
        double b = (r >= 1 && r <= W) ? v[(r >= 1 && r <= W) ? r - 1 : 0] : 0.0;  // c == 1
        phi[r] = scale * (c ? b : a);
    }
}

// ------------------------------------------------------------------------------ interp
template <int W>
struct Interp3Cfg {
    static constexpr int T = 2, R = W + T - 1, RZ = (R + 1) & ~1, NT = 128, NW = NT / 32;
    static constexpr int PROW = 2 * R + 1;                 // odd stride: fewer bank conflicts
    static constexpr int SMEM_H = R * R * RZ;              // doubles
    static constexpr int SMEM_P = NT * PROW * 2;           // x and y rows, 2 nodes per lane
    static constexpr size_t SMEM_BYTES = sizeof(double) * (SMEM_H + SMEM_P);
};

template <int W>
__global__ void __launch_bounds__(128)
interp3_v2_kernel(const TileItem* __restrict__ items, int nitems, const double* __restrict__ u,
                  long long count, const double* __restrict__ grid, int n, int tpa,
                  const __grid_constant__ WinPoly wp, double* __restrict__ t_out) {
    using C = Interp3Cfg<W>;
    constexpr int T = C::T, R = C::R, RZ = C::RZ, m = W / 2;
    extern __shared__ __align__(16) double smem[];
    double* H = smem;
    double* PXY = smem + C::SMEM_H;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* px0 = PXY + threadIdx.x * 2 * C::PROW;   // [x0 | y0] rows of node 0
    double* px1 = px0 + C::PROW;                      // [x1 | y1] rows of node 1 (stride PROW)
    const double* uy = u + count;
    const double* uz = u + 2 * count;

    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const TileItem item = items[it];
        const int tz = item.tile % tpa, ty = (item.tile / tpa) % tpa, tx = item.tile / (tpa * tpa);
        const int ox = tx * T, oy = ty * T, oz = tz * T;
        const int gx0 = ox - (m - 1), gy0 = oy - (m - 1), gz0 = oz - (m - 1);
        __syncthreads();
        for (int idx = threadIdx.x; idx < R * R * RZ; idx += C::NT) {
            const int rz = idx % RZ, rest = idx / RZ, ry = rest % R, rx = rest / R;
            H[idx] = rz < R ? __ldg(&grid[((long long)(gx0 + rx) * n + (gy0 + ry)) * n + (gz0 + rz)]) : 0.0;
        }
        __syncthreads();
        for (int base = warp * 64; base < item.count; base += C::NW * 64) {
            const int i0 = base + lane, i1 = base + 32 + lane;
            const bool ok0 = i0 < item.count, ok1 = i1 < item.count;
            const long long j0 = item.start + (ok0 ? i0 : 0), j1 = item.start + (ok1 ? i1 : 0);
            double pz0[RZ], pz1[RZ];
            {
                double v[W];
                double ux0 = u[j0], uy0 = uy[j0], uz0 = uz[j0];
                double ux1 = u[j1], uy1 = uy[j1], uz1 = uz[j1];
                double fx, cx;
                // node 0
                cx = floor(ux0); fx = ux0 - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - ox, ok0 ? 1.0 : 0.0, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) px0[r] = ph[r];
                }
                cx = floor(uy0); fx = uy0 - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - oy, 1.0, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) px0[R + r] = ph[r];
                }
                cx = floor(uz0); fx = uz0 - cx;
                win_taps<W>(fx, wp, v);
                region_weights<W, RZ>(v, (int)cx - oz, 1.0, pz0);
                // node 1
                cx = floor(ux1); fx = ux1 - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - ox, ok1 ? 1.0 : 0.0, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) px1[r] = ph[r];
                }
                cx = floor(uy1); fx = uy1 - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - oy, 1.0, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) px1[R + r] = ph[r];
                }
                cx = floor(uz1); fx = uz1 - cx;
                win_taps<W>(fx, wp, v);
                region_weights<W, RZ>(v, (int)cx - oz, 1.0, pz1);
            }
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 1
            for (int rx = 0; rx < R; ++rx) {
                double sy0 = 0.0, sy1 = 0.0;
#pragma unroll
                for (int ry = 0; ry < R; ++ry) {
                    const double2* h = reinterpret_cast<const double2*>(H + (rx * R + ry) * RZ);
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int k = 0; k < RZ / 2; ++k) {
                        const double2 hv = h[k];
                        s0 = fma(hv.x, pz0[2 * k], s0);
                        s1 = fma(hv.x, pz1[2 * k], s1);
                        s0 = fma(hv.y, pz0[2 * k + 1], s0);
                        s1 = fma(hv.y, pz1[2 * k + 1], s1);
                    }
                    sy0 = fma(px0[R + ry], s0, sy0);
                    sy1 = fma(px1[R + ry], s1, sy1);
                }
                acc0 = fma(px0[rx], sy0, acc0);
                acc1 = fma(px1[rx], sy1, acc1);
            }
            if (ok0) t_out[j0] = acc0;
            if (ok1) t_out[j1] = acc1;
        }
    }
}

// ------------------------------------------------------------------------------ spread
template <int W>
struct Spread3Cfg {
    static constexpr int T = 2, R = W + T - 1, RZ = (R + 1) & ~1;
    static constexpr int NCOL = R * R;
    static constexpr int NT = (((NCOL + 1) / 2) + 31) / 32 * 32;    // 2 columns per lane
    static constexpr int CP = 64;                                   // nodes per chunk
    static constexpr int TXS = R + 1;                                // padded row strides
    static constexpr int SMEM_TAB = CP * (TXS + TXS + RZ);
    static constexpr int SMEM_OUT = NCOL * RZ;
    static constexpr int SMEM = SMEM_TAB > SMEM_OUT ? SMEM_TAB : SMEM_OUT;
    static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM;
};

template <int W>
__global__ void __launch_bounds__(Spread3Cfg<W>::NT)
spread3_v2_kernel(const TileItem* __restrict__ items, int nitems, const double* __restrict__ u,
                  const double* __restrict__ w, long long count, double* __restrict__ grid, int n,
                  int tpa, const __grid_constant__ WinPoly wp) {
    using C = Spread3Cfg<W>;
    constexpr int T = C::T, R = C::R, RZ = C::RZ, m = W / 2, CP = C::CP, NCOL = C::NCOL;
    extern __shared__ __align__(16) double smem[];
    double* TX = smem;                     // [CP][TXS]  w * phi_x
    double* TY = TX + CP * C::TXS;          // [CP][TXS]  phi_y
    double* TZ = TY + CP * C::TXS;          // [CP][RZ]   phi_z (zero padded)
    const int tid = threadIdx.x;
    const int col0 = tid, col1 = tid + C::NT;
    const bool v0 = col0 < NCOL, v1 = col1 < NCOL;
    const int rx0 = v0 ? col0 / R : 0, ry0 = v0 ? col0 % R : 0;
    const int rx1 = v1 ? col1 / R : 0, ry1 = v1 ? col1 % R : 0;
    const double* uy = u + count;
    const double* uz = u + 2 * count;

    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const TileItem item = items[it];
        const int tz = item.tile % tpa, ty = (item.tile / tpa) % tpa, tx = item.tile / (tpa * tpa);
        const int ox = tx * T, oy = ty * T, oz = tz * T;
        double acc0[RZ], acc1[RZ];
#pragma unroll
        for (int r = 0; r < RZ; ++r) { acc0[r] = 0.0; acc1[r] = 0.0; }
        for (int c0 = 0; c0 < item.count; c0 += CP) {
            const int np = min(CP, item.count - c0);
            __syncthreads();
            if (tid < CP) {
                const bool ok = tid < np;
                const long long j = item.start + c0 + (ok ? tid : 0);
                double v[W];
                double cx, fx;
                double ux = u[j], uyy = uy[j], uzz = uz[j], wj = ok ? w[j] : 0.0;
                cx = floor(ux); fx = ux - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - ox, wj, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) TX[tid * C::TXS + r] = ph[r];
                }
                cx = floor(uyy); fx = uyy - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[R];
                    region_weights<W, R>(v, (int)cx - oy, 1.0, ph);
#pragma unroll
                    for (int r = 0; r < R; ++r) TY[tid * C::TXS + r] = ph[r];
                }
                cx = floor(uzz); fx = uzz - cx;
                win_taps<W>(fx, wp, v);
                {
                    double ph[RZ];
                    region_weights<W, RZ>(v, (int)cx - oz, 1.0, ph);
#pragma unroll
                    for (int r = 0; r < RZ; ++r) TZ[tid * RZ + r] = ph[r];
                }
            }
            __syncthreads();
#pragma unroll 2
            for (int p = 0; p < np; ++p) {
                const double a0 = TX[p * C::TXS + rx0] * TY[p * C::TXS + ry0];
                const double a1 = TX[p * C::TXS + rx1] * TY[p * C::TXS + ry1];
                const double2* z = reinterpret_cast<const double2*>(TZ + p * RZ);
#pragma unroll
                for (int k = 0; k < RZ / 2; ++k) {
                    const double2 zv = z[k];
                    acc0[2 * k] = fma(a0, zv.x, acc0[2 * k]);
                    acc0[2 * k + 1] = fma(a0, zv.y, acc0[2 * k + 1]);
                    acc1[2 * k] = fma(a1, zv.x, acc1[2 * k]);
                    acc1[2 * k + 1] = fma(a1, zv.y, acc1[2 * k + 1]);
                }
            }
        }
        // flush: stage the region in shared memory, then coalesced REDs along z rows
        __syncthreads();
        double* OUT = smem;   // [NCOL][RZ]
        if (v0) {
#pragma unroll
            for (int r = 0; r < RZ; ++r) OUT[col0 * RZ + r] = acc0[r];
        }
        if (v1) {
#pragma unroll
            for (int r = 0; r < RZ; ++r) OUT[col1 * RZ + r] = acc1[r];
        }
        __syncthreads();
        const int gx0 = ox - (m - 1), gy0 = oy - (m - 1), gz0 = oz - (m - 1);
        for (int idx = tid; idx < NCOL * R; idx += C::NT) {
            const int rz = idx % R, col = idx / R, ry = col % R, rx = col / R;
            const double val = OUT[col * RZ + rz];
            if (val != 0.0)
                atomicAdd(&grid[((long long)(gx0 + rx) * n + (gy0 + ry)) * n + (gz0 + rz)], val);
        }
    }
}

}  // namespace sk
