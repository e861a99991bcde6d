// dmma2.cuh -- d = 2 spread / interp on the FP64 tensor cores (DMMA m8n8k4), W = 2 m_w = 16
// (the d = 2 workloads c2, c4). Per grid cell, all its nodes share the 16 x 16 taps:
//
//   interp:  E[tx, j] = sum_ty G[tx, ty] phi_y,j[ty]        (DMMA: M = tx 16, K = ty 16, N = nodes)
//            t_j = sum_tx phi_x,j[tx] E[tx, j]              (epilogue, 16 DFMA per node)
//   spread:  G[tx, ty] += sum_j (w_j phi_x,j[tx]) phi_y,j[ty]   (DMMA: M = tx, N = ty, K = nodes)
//
// W = 16 tiles the 8 x 8 x 4 DMMA exactly (no padding). The spread accumulates whole
// super-tiles of kSup2 x kSup2 cells in a warp-private shared region and flushes it once
// with coalesced FP64 atomics.
#pragma once
#include "sk_internal.cuh"
#include "dmma3.cuh"
#include "winpoly.h"

namespace sk {

constexpr int kSup2 = 4;  // d = 2 super-tile edge (cells)

#ifndef SK_WORKLIST_ONLY

// ------------------------------------------------------------------------------ interp
struct Interp2Cfg {
    static constexpr int W = 16, KS = W / 4, NT = 128, NWARP = NT / 32;
    static constexpr int TAB = 2 * 32 * kTabS;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (NWARP * TAB + (W / 2) * kCoefRow);
};

__global__ void __launch_bounds__(128, 4)
interp2_dmma_kernel(const CellBatch* __restrict__ batches, int nbatches, const double* __restrict__ u,
                    long long count, const double* __restrict__ grid, int n,
                    const __grid_constant__ WinPoly wp, double* __restrict__ t_out) {
    using C = Interp2Cfg;
    constexpr int W = C::W, KS = C::KS, m = W / 2;
    extern __shared__ __align__(16) double smem[];
    double* csm = smem + C::NWARP * C::TAB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    double* TX = smem + warp * C::TAB;
    double* TY = TX + 32 * kTabS;
    load_coefs<W>(wp, csm);
    __syncthreads();
    const double* uy = u + count;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;

    for (int bi = gw; bi < nbatches; bi += nw) {
        const CellBatch B = batches[bi];
        const int cy = B.cell % n, cx = B.cell / n;
        {
            const bool ok = lane < B.count;
            const long long j = B.start + (ok ? lane : 0);
            const double vx = u[j], vy = uy[j];
            taps_row16<W>(vx - floor(vx), ok ? 1.0 : 0.0, csm, TX + lane * kTabS);
            taps_row16<W>(vy - floor(vy), 1.0, csm, TY + lane * kTabS);
        }
        __syncwarp();
        const double* Hb = grid + (long long)(cx - m + 1) * n + (cy - m + 1);
        double a[2][KS];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int s = 0; s < KS; ++s) a[mt][s] = __ldg(Hb + (long long)(8 * mt + g) * n + 4 * s + q);
        double d[2][4][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            double bf[4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[nt] = TY[(8 * nt + g) * kTabS + 4 * s + q];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                dmma884(d[0][nt][0], d[0][nt][1], a[0][s], bf[nt]);
                dmma884(d[1][nt][0], d[1][nt][1], a[1][s], bf[nt]);
            }
        }
        double acc[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double* tx = TX + (8 * nt + 2 * q + e) * kTabS;
                double v = tx[g] * d[0][nt][e];
                v = fma(tx[8 + g], d[1][nt][e], v);
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
struct Spread2Cfg {
    static constexpr int W = 16, S = W + kSup2 - 1, NT = 128, NWARP = NT / 32;
    static constexpr int REG = S * S;
    static constexpr int TAB = 2 * 32 * kTabS;
    static constexpr int PER_WARP = REG + TAB;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (NWARP * PER_WARP + (W / 2) * kCoefRow);
};

__global__ void __launch_bounds__(128, 4)
spread2_dmma_kernel(const SpreadItem* __restrict__ items, int nitems, const CellBatch* __restrict__ segs,
                    const double* __restrict__ u, const double* __restrict__ w, long long count,
                    double* __restrict__ grid, int n, const __grid_constant__ WinPoly wp) {
    using C = Spread2Cfg;
    constexpr int W = C::W, S = C::S, m = W / 2;
    extern __shared__ __align__(16) double smem[];
    double* csm = smem + C::NWARP * C::PER_WARP;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    double* REGm = smem + warp * C::PER_WARP;
    double* TX = REGm + C::REG;
    double* TY = TX + 32 * kTabS;
    load_coefs<W>(wp, csm);
    __syncthreads();
    const double* uy = u + count;
    const int ns = n / kSup2;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;

    for (int ii = gw; ii < nitems; ii += nw) {
        const SpreadItem it = items[ii];
        const int sy = it.stile % ns, sx = it.stile / ns;
        for (int i = lane; i < C::REG; i += 32) REGm[i] = 0.0;
        __syncwarp();
        for (int sg = it.seg_begin; sg < it.seg_end; ++sg) {
            const CellBatch seg = segs[sg];
            const int cy = seg.cell % n, cx = seg.cell / n;
            const int ox = cx - kSup2 * sx, oy = cy - kSup2 * sy;
            double acc[2][2][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
            for (int b0 = 0; b0 < seg.count; b0 += 32) {
                const int np = min(32, seg.count - b0);
                {
                    const bool ok = lane < np;
                    const long long j = seg.start + b0 + (ok ? lane : 0);
                    const double vx = u[j], vy = uy[j];
                    const double wj = ok ? w[j] : 0.0;
                    taps_row16<W>(vx - floor(vx), wj, csm, TX + lane * kTabS);
                    taps_row16<W>(vy - floor(vy), 1.0, csm, TY + lane * kTabS);
                }
                __syncwarp();
                const int nks = (np + 3) >> 2;
#pragma unroll 2
                for (int s = 0; s < nks; ++s) {
                    const int jr = 4 * s + q;
                    const double a0 = TX[jr * kTabS + g], a1 = TX[jr * kTabS + 8 + g];
                    const double b0v = TY[jr * kTabS + g], b1v = TY[jr * kTabS + 8 + g];
                    dmma884(acc[0][0][0], acc[0][0][1], a0, b0v);
                    dmma884(acc[0][1][0], acc[0][1][1], a0, b1v);
                    dmma884(acc[1][0][0], acc[1][0][1], a1, b0v);
                    dmma884(acc[1][1][0], acc[1][1][1], a1, b1v);
                }
                __syncwarp();
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int tx = 8 * mt + g, ty = 8 * nt + 2 * q + e;
                        REGm[(ox + tx) * S + (oy + ty)] += acc[mt][nt][e];
                    }
            __syncwarp();
        }
        const int gx0 = kSup2 * sx - (m - 1), gy0 = kSup2 * sy - (m - 1);
        for (int i = lane; i < C::REG; i += 32) {
            const double v = REGm[i];
            if (v != 0.0) atomicAdd(&grid[(long long)(gx0 + i / S) * n + (gy0 + i % S)], v);
        }
        __syncwarp();
    }
}

#endif  // SK_WORKLIST_ONLY

}  // namespace sk
