// dmma3.cuh -- d = 3 spread / interp on the FP64 tensor cores (mma.sync m8n8k4 .f64 -> DMMA),
// for 2 m_w = W = 12 taps per axis (the d = 3 workloads c3, c5).
//
// All nodes of one grid cell share the same W^3 taps, so per cell the window sums are dense
// contractions over the cell's nodes (P:L475-477 gridding, written as GEMMs):
//
//   interp (NFFT trafo):  E[(tx,ty), j] = sum_tz G[tx,ty,tz] phi_z,j[tz]         (DMMA: M=(tx,ty),
//                         t_j = sum_tx phi_x,j[tx] sum_ty phi_y,j[ty] E[(tx,ty), j]   K=tz, N=nodes)
//   spread (adjoint):     G[tx, (ty,tz)] += sum_j phi_x,j[tx] (w_j phi_y,j[ty] phi_z,j[tz])
//                                                                               (DMMA: M=tx, N=(ty,tz),
//                                                                                K=nodes)
// FP64 DMMA and DFMA share one pipe on B200 (37 TF either way, tools/microbench.cu), but the
// tensor core reuses its operands internally: one A/B register per lane feeds 256 FMAs, so
// shared memory is no longer the limiter (broadcast LDS.128 runs at ~0.5/clk/SM).
//
// Row padding: M = 16 rows per tx (ty padded 12 -> 16) for interp and M = 16 tx rows for
// spread, i.e. 75% of the DMMA work is useful; in exchange the interp epilogue keeps the
// per-node phi_y in registers and the spread needs no per-node product tables.
//
// Fragment layouts (m8n8k4, f64): g = lane/4, q = lane%4
//   A[8x4]: a = A[g][q];  B[4x8]: b = B[q][g];  C[8x8]: c0, c1 = C[g][2q], C[g][2q+1]
#pragma once
#include "sk_internal.cuh"
#include "tiled3.cuh"
#include "winpoly.h"

namespace sk {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Work unit of the interp: up to 32 nodes of one cell.
struct CellBatch {
    int cell;   // packed cell coordinates (cx * n + cy) * n + cz
    int start;  // first node (sorted order)
    int count;  // <= 32
    int pad;
};
// Work unit of the spread: nodes of consecutive cells of one 2^3 super-tile.
struct SpreadItem {
    int stile;      // packed super-tile coordinates (sx * ns + sy) * ns + sz, ns = n / 2
    int seg_begin;  // first segment (CellBatch-like, count <= kSegMax)
    int seg_end;
    int count;      // nodes
};
constexpr int kSegMax = 256;
constexpr int kSpreadItemMax = 2048;

#ifndef SK_WORKLIST_ONLY   // plan.cu only needs the work-list types above

// per-warp node tables: rows of kTabS doubles (kTabS = 20 = 4 mod 16 keeps 8-row x 4-col
// fragment loads conflict-free)
constexpr int kTabS = 20;

// lane writes its node's taps: tab[0..W) = scale * phi(f + m - 1 - t), tab[W..16) = 0
template <int W>
__device__ __forceinline__ void taps_row16(double f, double scale, const double* __restrict__ csm, double* row) {
    const double g = f - 0.5, g2 = g * g;
#pragma unroll
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
        row[t] = scale * fma(g, O, E);
        row[W - 1 - t] = scale * fma(-g, O, E);
    }
#pragma unroll
    for (int t = W; t < 16; ++t) row[t] = 0.0;
}

// ------------------------------------------------------------------------------ interp
struct InterpDCfg {
    static constexpr int W = 12, KS = W / 4, NT = 128, NWARP = NT / 32;
    static constexpr int TAB = 3 * 32 * kTabS;        // TX, TY, TZ per warp
    static constexpr size_t SMEM_BYTES = sizeof(double) * (NWARP * TAB + (W / 2) * kCoefRow);
};

__global__ void __launch_bounds__(128, 3)
interp3_dmma_kernel(const CellBatch* __restrict__ batches, int nbatches, const double* __restrict__ u,
                    long long count, const double* __restrict__ grid, int n,
                    const __grid_constant__ WinPoly wp, double* __restrict__ t_out) {
    using C = InterpDCfg;
    constexpr int W = C::W, KS = C::KS, m = W / 2;
    extern __shared__ __align__(16) double smem[];
    double* csm = smem + C::NWARP * C::TAB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    double* TX = smem + warp * C::TAB;
    double* TY = TX + 32 * kTabS;
    double* TZ = TY + 32 * kTabS;
    load_coefs<W>(wp, csm);
    __syncthreads();
    const double* uy = u + count;
    const double* uz = u + 2 * count;
    const long long n2 = (long long)n * n;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;

    for (int bi = gw; bi < nbatches; bi += nw) {
        const CellBatch B = batches[bi];
        const int cz = B.cell % n, cy = (B.cell / n) % n, cx = B.cell / n / n;
        // node tables (lane = node)
        {
            const bool ok = lane < B.count;
            const long long j = B.start + (ok ? lane : 0);
            const double vx = u[j], vy = uy[j], vz = uz[j];
            taps_row16<W>(vx - floor(vx), ok ? 1.0 : 0.0, csm, TX + lane * kTabS);
            taps_row16<W>(vy - floor(vy), 1.0, csm, TY + lane * kTabS);
            taps_row16<W>(vz - floor(vz), 1.0, csm, TZ + lane * kTabS);
        }
        __syncwarp();
        // B fragments: phi_z of node 8 nt + g at tz = 4 s + q
        double bf[KS][4];
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[s][nt] = TZ[(8 * nt + g) * kTabS + 4 * s + q];
        // phi_y of node 8 nt + 2 q + e at ty = 8 h + g
        double fy[4][2][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int h = 0; h < 2; ++h) fy[nt][e][h] = TY[(8 * nt + 2 * q + e) * kTabS + 8 * h + g];
        double acc[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        const double* Hb = grid + (long long)(cx - m + 1) * n2 + (long long)(cy - m + 1) * n + (cz - m + 1);
#pragma unroll 1
        for (int tx = 0; tx < W; ++tx) {
            double accy[4][2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) accy[nt][0] = accy[nt][1] = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ty = 8 * h + g;
                const bool valid = ty < W;
                const double* row = Hb + (long long)tx * n2 + (long long)(valid ? ty : 0) * n + q;
                double d[4][2];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) d[nt][0] = d[nt][1] = 0.0;
#pragma unroll
                for (int s = 0; s < KS; ++s) {
                    const double a = valid ? __ldg(row + 4 * s) : 0.0;
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma884(d[nt][0], d[nt][1], a, bf[s][nt]);
                }
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) accy[nt][e] = fma(fy[nt][e][h], d[nt][e], accy[nt][e]);
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    acc[nt][e] = fma(TX[(8 * nt + 2 * q + e) * kTabS + tx], accy[nt][e], acc[nt][e]);
        }
        // sum over the 8 rows g held by lanes q, q+4, ..., q+28
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = acc[nt][e];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                acc[nt][e] = v;
            }
        if (g == 0) {
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = 8 * nt + 2 * q + e;
                    if (p < B.count) t_out[B.start + p] = acc[nt][e];
                }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------ spread
struct SpreadDCfg {
    static constexpr int W = 12, S = W + 1, NT = 64, NWARP = NT / 32, NTILE = (W * W) / 8;  // 18
    static constexpr int REG = S * S * S;              // warp-private super-tile region
    static constexpr int TAB = 3 * 32 * kTabS;
    static constexpr int PER_WARP = REG + TAB;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (NWARP * PER_WARP + (W / 2) * kCoefRow);
};

__global__ void __launch_bounds__(64, 3)
spread3_dmma_kernel(const SpreadItem* __restrict__ items, int nitems, const CellBatch* __restrict__ segs,
                    const double* __restrict__ u, const double* __restrict__ w, long long count,
                    double* __restrict__ grid, int n, const __grid_constant__ WinPoly wp) {
    using C = SpreadDCfg;
    constexpr int W = C::W, S = C::S, m = W / 2, NTILE = C::NTILE;
    extern __shared__ __align__(16) double smem[];
    double* csm = smem + C::NWARP * C::PER_WARP;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    double* REGm = smem + warp * C::PER_WARP;
    double* TX = REGm + C::REG;
    double* TY = TX + 32 * kTabS;
    double* TZ = TY + 32 * kTabS;
    load_coefs<W>(wp, csm);
    __syncthreads();
    const double* uy = u + count;
    const double* uz = u + 2 * count;
    const int ns = n / 2;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;

    for (int ii = gw; ii < nitems; ii += nw) {
        const SpreadItem it = items[ii];
        const int sz = it.stile % ns, sy = (it.stile / ns) % ns, sx = it.stile / ns / ns;
        for (int i = lane; i < C::REG; i += 32) REGm[i] = 0.0;
        __syncwarp();
        for (int sg = it.seg_begin; sg < it.seg_end; ++sg) {
            const CellBatch seg = segs[sg];
            const int cz = seg.cell % n, cy = (seg.cell / n) % n, cx = seg.cell / n / n;
            const int ox = cx - 2 * sx, oy = cy - 2 * sy, oz = cz - 2 * sz;   // in {0,1}
            double acc[2][NTILE][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < NTILE; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
            for (int b0 = 0; b0 < seg.count; b0 += 32) {
                const int np = min(32, seg.count - b0);
                {
                    const bool ok = lane < np;
                    const long long j = seg.start + b0 + (ok ? lane : 0);
                    const double vx = u[j], vy = uy[j], vz = uz[j];
                    const double wj = ok ? w[j] : 0.0;
                    taps_row16<W>(vx - floor(vx), ok ? 1.0 : 0.0, csm, TX + lane * kTabS);
                    taps_row16<W>(vy - floor(vy), wj, csm, TY + lane * kTabS);
                    taps_row16<W>(vz - floor(vz), 1.0, csm, TZ + lane * kTabS);
                }
                __syncwarp();
                const int nks = (np + 3) >> 2;
#pragma unroll 1
                for (int s = 0; s < nks; ++s) {
                    const int jr = 4 * s + q;                       // node row of this lane's A/B
                    const double a0 = TX[jr * kTabS + g];           // A[tx = g][k = q]
                    const double a1 = TX[jr * kTabS + 8 + g];       // A[tx = 8 + g][k = q]
                    const double* ty_row = TY + jr * kTabS;
                    const double* tz_row = TZ + jr * kTabS;
#pragma unroll
                    for (int nt = 0; nt < NTILE; ++nt) {
                        const int col = 8 * nt + g;                 // B[k = q][n = g]: (ty, tz) = divmod(col, W)
                        const double b = ty_row[col / W] * tz_row[col % W];
                        dmma884(acc[0][nt][0], acc[0][nt][1], a0, b);
                        dmma884(acc[1][nt][0], acc[1][nt][1], a1, b);
                    }
                }
                __syncwarp();
            }
            // add the cell's W^3 block into the region at offset (ox, oy, oz)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int tx = 8 * mt + g;
                if (tx < W) {
#pragma unroll
                    for (int nt = 0; nt < NTILE; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = 8 * nt + 2 * q + e;
                            const int ty = col / W, tz = col % W;
                            double* r = REGm + ((ox + tx) * S + (oy + ty)) * S + (oz + tz);
                            *r += acc[mt][nt][e];
                        }
                }
            }
            __syncwarp();
        }
        // flush the region: coalesced FP64 atomics along z rows
        const int gx0 = 2 * sx - (m - 1), gy0 = 2 * sy - (m - 1), gz0 = 2 * sz - (m - 1);
        for (int i = lane; i < C::REG; i += 32) {
            const double v = REGm[i];
            if (v != 0.0) {
                const int rz = i % S, rest = i / S, ry = rest % S, rx = rest / S;
                atomicAdd(&grid[((long long)(gx0 + rx) * n + (gy0 + ry)) * n + (gz0 + rz)], v);
            }
        }
        __syncwarp();
    }
}

#endif  // SK_WORKLIST_ONLY

}  // namespace sk
