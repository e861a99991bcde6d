// tiled3.cuh -- v2 spread / interp for d = 3 on tiles of T^3 = 2^3 grid cells (sm_100a, FP64).
//
// Nodes are sorted by tile (plan.cu); a work item is one tile, or a chunk of at most
// kItemMax nodes of a dense tile. Every node of a tile touches taps inside the tile's
// region of R = T + W - 1 cells per axis (W = 2 m taps per axis), so
//
//   interp: the CTA stages the region of the grid in shared memory (R^3 doubles, one
//           coalesced load per item); lanes = nodes (2 per lane); a node's window values
//           over the whole region (zeros outside its 2m support) live in registers (z) and
//           in lane-private shared rows (x, y); the region loop is warp-uniform, so every
//           grid value is one broadcast LDS.128 feeding 4 DFMAs.
//   spread: lanes own 2 region columns (x,y) of R z-values in registers; per chunk of 64
//           nodes the CTA tabulates w*phi_x, phi_y, phi_z in shared memory (lanes = nodes),
//           then loops over the nodes (warp-uniform) with a broadcast phi_z row: per node
//           and lane 2 DMUL + 2R DFMA. The region is flushed once per item with coalesced
//           FP64 atomics (RED) into the global grid (neighbouring regions overlap).
//
// Window taps: degree-14 polynomials of winpoly.h. The window is even, so tap W-1-t at
// g = f - 1/2 is tap t at -g: with p_t(g) = E_t(g^2) + g O_t(g^2) one pair of taps costs
// 15 DFMA. The W/2 coefficient rows sit in shared memory (broadcast LDS.128).
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
constexpr int kCoefRow = 16;    // [e0..e7 | o0..o6, 0] per tap pair

// Copy the even/odd coefficient rows of taps 0..W/2-1 into shared memory.
template <int W>
__device__ __forceinline__ void load_coefs(const WinPoly& wp, double* csm) {
    for (int i = threadIdx.x; i < (W / 2) * kCoefRow; i += blockDim.x) {
        const int t = i / kCoefRow, k = i % kCoefRow;
        double v = 0.0;
        if (k < 8) v = wp.c[t][2 * k];
        else if (k < 15) v = wp.c[t][2 * (k - 8) + 1];
        csm[i] = v;
    }
}

// row[c + s] = scale * phi(f + m - 1 - s) for s in [0, W), row[r] = 0 for the other r < RP.
// T = 2: c in {0, 1} so exactly one of row[0], row[W] is outside the support.
template <int W, int RP>
__device__ __forceinline__ void taps_to_row(double f, int c, double scale, const double* __restrict__ csm,
                                            double* row) {
    const double g = f - 0.5, g2 = g * g;
    double* base = row + c;
#pragma unroll 2
    for (int t = 0; t < W / 2; ++t) {
        const double2* cr = reinterpret_cast<const double2*>(csm + t * kCoefRow);
        const double2 e01 = cr[0], e23 = cr[1], e45 = cr[2], e67 = cr[3];
        const double2 o01 = cr[4], o23 = cr[5], o45 = cr[6], o67 = cr[7];
        double E = fma(e67.y, g2, e67.x);
        E = fma(E, g2, e45.y);
        E = fma(E, g2, e45.x);
        E = fma(E, g2, e23.y);
        E = fma(E, g2, e23.x);
        E = fma(E, g2, e01.y);
        E = fma(E, g2, e01.x);
        double O = fma(o67.x, g2, o45.y);
        O = fma(O, g2, o45.x);
        O = fma(O, g2, o23.y);
        O = fma(O, g2, o23.x);
        O = fma(O, g2, o01.y);
        O = fma(O, g2, o01.x);
        base[t] = scale * fma(g, O, E);
        base[W - 1 - t] = scale * fma(-g, O, E);
    }
    row[c ? 0 : W] = 0.0;
#pragma unroll
    for (int r = W + 1; r < RP; ++r) row[r] = 0.0;
}

// ------------------------------------------------------------------------------ interp
template <int W>
struct Interp3Cfg {
    static constexpr int T = 2, R = W + T - 1, RZ = (R + 1) & ~1, NT = 128, NW = NT / 32;
    static constexpr int LROW = 4 * RZ + 1;                // per-lane [x0 | y0 | x1 | y1], odd stride
    static constexpr int SMEM_H = R * R * RZ;              // doubles
    static constexpr int SMEM_P = NT * LROW;
    static constexpr int SMEM_C = (W / 2) * kCoefRow;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (SMEM_H + SMEM_P + SMEM_C);
};

template <int W>
__global__ void __launch_bounds__(128, 3)
interp3_v2_kernel(const TileItem* __restrict__ items, int nitems, const double* __restrict__ u,
                  long long count, const double* __restrict__ grid, int n, int tpa,
                  const __grid_constant__ WinPoly wp, double* __restrict__ t_out) {
    using C = Interp3Cfg<W>;
    constexpr int T = C::T, R = C::R, RZ = C::RZ, m = W / 2;
    extern __shared__ __align__(16) double smem[];
    double* H = smem;
    double* csm = smem + C::SMEM_H;
    double* rows = csm + C::SMEM_C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* rx0p = rows + threadIdx.x * C::LROW;   // x-row node 0
    double* ry0p = rx0p + RZ;                      // y-row node 0
    double* rx1p = ry0p + RZ;                      // x-row node 1 (z scratch first)
    double* ry1p = rx1p + RZ;                      // y-row node 1
    const double* uy = u + count;
    const double* uz = u + 2 * count;
    load_coefs<W>(wp, csm);

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
                double c, v;
                v = uz[j0]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oz, 1.0, csm, rx1p);
#pragma unroll
                for (int r = 0; r < RZ; ++r) pz0[r] = rx1p[r];
                v = uz[j1]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oz, 1.0, csm, rx1p);
#pragma unroll
                for (int r = 0; r < RZ; ++r) pz1[r] = rx1p[r];
                v = u[j0]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - ox, ok0 ? 1.0 : 0.0, csm, rx0p);
                v = uy[j0]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oy, 1.0, csm, ry0p);
                v = u[j1]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - ox, ok1 ? 1.0 : 0.0, csm, rx1p);
                v = uy[j1]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oy, 1.0, csm, ry1p);
            }
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 1
            for (int rx = 0; rx < R; ++rx) {
                double sy0 = 0.0, sy1 = 0.0;
#pragma unroll
                for (int ry = 0; ry < R; ++ry) {
                    const double2* h = reinterpret_cast<const double2*>(H + (rx * R + ry) * RZ);
                    double s0 = 0.0, s1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
                    for (int k = 0; k < RZ / 2; ++k) {
                        const double2 hv = h[k];
                        s0 = fma(hv.x, pz0[2 * k], s0);
                        s1 = fma(hv.x, pz1[2 * k], s1);
                        q0 = fma(hv.y, pz0[2 * k + 1], q0);
                        q1 = fma(hv.y, pz1[2 * k + 1], q1);
                    }
                    sy0 = fma(ry0p[ry], s0 + q0, sy0);
                    sy1 = fma(ry1p[ry], s1 + q1, sy1);
                }
                acc0 = fma(rx0p[rx], sy0, acc0);
                acc1 = fma(rx1p[rx], sy1, acc1);
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
    static constexpr int TXS = RZ;                                   // row strides
    static constexpr int SMEM_TAB = CP * (TXS + TXS + RZ);
    static constexpr int SMEM_OUT = NCOL * RZ;
    static constexpr int SMEM_MAIN = SMEM_TAB > SMEM_OUT ? SMEM_TAB : SMEM_OUT;
    static constexpr int SMEM_C = (W / 2) * kCoefRow;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (SMEM_MAIN + SMEM_C);
};

template <int W>
__global__ void __launch_bounds__(Spread3Cfg<W>::NT, 4)
spread3_v2_kernel(const TileItem* __restrict__ items, int nitems, const double* __restrict__ u,
                  const double* __restrict__ w, long long count, const GridAcc ga,
                  int tpa, const __grid_constant__ WinPoly wp) {
    using C = Spread3Cfg<W>;
    const int n = ga.n;
    const double gscale = grid_scale(ga);
    constexpr int T = C::T, R = C::R, RZ = C::RZ, m = W / 2, CP = C::CP, NCOL = C::NCOL;
    extern __shared__ __align__(16) double smem[];
    double* TX = smem;                     // [CP][TXS]  w * phi_x
    double* TY = TX + CP * C::TXS;          // [CP][TXS]  phi_y
    double* TZ = TY + CP * C::TXS;          // [CP][RZ]   phi_z (zero padded)
    double* csm = smem + C::SMEM_MAIN;
    const int tid = threadIdx.x;
    const int col0 = tid, col1 = tid + C::NT;
    const bool v0 = col0 < NCOL, v1 = col1 < NCOL;
    const int rx0 = v0 ? col0 / R : 0, ry0 = v0 ? col0 % R : 0;
    const int rx1 = v1 ? col1 / R : 0, ry1 = v1 ? col1 % R : 0;
    const double* uy = u + count;
    const double* uz = u + 2 * count;
    load_coefs<W>(wp, csm);

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
                const double wj = ok ? w[j] : 0.0;
                double v, c;
                v = u[j]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - ox, wj, csm, TX + tid * C::TXS);
                v = uy[j]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oy, 1.0, csm, TY + tid * C::TXS);
                v = uz[j]; c = floor(v);
                taps_to_row<W, RZ>(v - c, (int)c - oz, 1.0, csm, TZ + tid * RZ);
            }
            __syncthreads();
#pragma unroll 1
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
                grid_add<3>(ga, gscale, gx0 + rx, gy0 + ry, gz0 + rz, val);
        }
    }
}

}  // namespace sk
