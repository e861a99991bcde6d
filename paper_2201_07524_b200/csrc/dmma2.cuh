// dmma2.cuh -- d = 2 spread / interp on the FP64 tensor cores (DMMA m8n8k4), W = 2 m_w = 16
// (the d = 2 workloads c2, c4). Per grid cell, all its nodes share the 16 x 16 taps:
//
//   interp:  E[tx, j] = sum_ty G[tx, ty] phi_y,j[ty]        (DMMA: M = tx 16, K = ty 16, N = nodes)
//            t_j = sum_tx phi_x,j[tx] E[tx, j]              (epilogue, 16 DFMA per node)
//   spread:  G[tx, ty] += sum_j (w_j phi_x,j[tx]) phi_y,j[ty]   (DMMA: M = tx, N = ty, K = nodes)
//
// W = 16 tiles the 8 x 8 x 4 DMMA exactly (no padding). Window taps come from the per-node
// table precomputed at plan time ([node][2][16] FP64). The spread accumulates whole
// super-tiles of kSup2 x kSup2 cells in a warp-private shared region and flushes it once
// with coalesced FP64 atomics.
#pragma once
#include "sk_internal.cuh"
#include "dmma3.cuh"

namespace sk {

constexpr int kSup2 = 4;  // d = 2 super-tile edge (cells)
constexpr long long kSpread2CtaNodes = 150000;   // node sets at most this large: one spread item per CTA

#ifndef SK_WORKLIST_ONLY

// ------------------------------------------------------------------------------ interp
struct Interp2Cfg {
    static constexpr int W = 16, KS = W / 4, NT = 128, NWARP = NT / 32, TS = 2 * W;
    static constexpr size_t SMEM_BYTES = 0;
};

// One batch (<= 32 nodes of one cell) with NT_ n-tiles of 8 nodes: sparse cells (c2, the
// images: a few nodes per cell) run ceil(count / 8) n-tiles instead of 4.
template <int NT_>
__device__ __forceinline__ void interp2_batch(const CellBatch& B, const double* __restrict__ taps,
                                              const double* __restrict__ grid, int n, int g, int q,
                                              double* __restrict__ t_out, const FusedUpd& fu) {
    using C = Interp2Cfg;
    constexpr int W = C::W, KS = C::KS, m = W / 2, TS = C::TS;
    const int cy = B.cell % n, cx = B.cell / n;
    const double* T0 = taps + (long long)B.start * TS;
    const int last = B.count - 1;
    const double* Hb = grid + (long long)(cx - m + 1) * n + (cy - m + 1) + q;
    double a[2][KS];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int s = 0; s < KS; ++s) a[mt][s] = __ldg(Hb + (long long)(8 * mt + g) * n + 4 * s);
    double d[2][NT_][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT_; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt) {
        const double* ty = T0 + min(8 * nt + g, last) * TS + W;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const double bf = __ldg(ty + 4 * s + q);
            dmma884(d[0][nt][0], d[0][nt][1], a[0][s], bf);
            dmma884(d[1][nt][0], d[1][nt][1], a[1][s], bf);
        }
    }
    double acc[NT_][2];
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double* tx = T0 + min(8 * nt + 2 * q + e, last) * TS;
            double v = __ldg(tx + g) * d[0][nt][e];
            v = fma(__ldg(tx + 8 + g), d[1][nt][e], v);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            acc[nt][e] = v;
        }
    // every lane now holds the sums of its q; lane (g, q) emits node 8 (g/2) + 2 q + g%2, so the
    // results (and the fused division) take one full-warp pass
    double v = acc[0][0];
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
            if (g == 2 * nt + e) v = acc[nt][e];
    const int p = 8 * (g >> 1) + 2 * q + (g & 1);
    if ((g >> 1) < NT_ && p < B.count) emit_t(t_out, fu, B.start + p, v);
}

__global__ void __launch_bounds__(128, 4)
interp2_dmma_kernel(const CellBatch* __restrict__ batches, int nbatches, const double* __restrict__ taps,
                    const double* __restrict__ grid, int n, double* __restrict__ t_out, const FusedUpd fu) {
    using C = Interp2Cfg;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;
    pdl_trigger();
    pdl_wait();   // the grid (and the fused update's p, x) come from the preceding kernels
    for (int bi = gw; bi < nbatches; bi += nw) {
        const CellBatch B = batches[bi];
        const int ntn = (B.count + 7) >> 3;   // warp-uniform
        if (ntn >= 4) interp2_batch<4>(B, taps, grid, n, g, q, t_out, fu);
        else if (ntn == 3) interp2_batch<3>(B, taps, grid, n, g, q, t_out, fu);
        else if (ntn == 2) interp2_batch<2>(B, taps, grid, n, g, q, t_out, fu);
        else interp2_batch<1>(B, taps, grid, n, g, q, t_out, fu);
    }
}

// ------------------------------------------------------------------------------ spread
struct Spread2Cfg {
    static constexpr int W = 16, S = W + kSup2 - 1, NT = 128, NWARP = NT / 32, TS = 2 * W;
    static constexpr int REG = S * S;
    static constexpr size_t SMEM_BYTES = sizeof(double) * (NWARP * REG);
};

template <bool CTA_ITEM>
__global__ void __launch_bounds__(128, 4)
spread2_dmma_kernel(const SpreadItem* __restrict__ items, int nitems, const CellBatch* __restrict__ segs,
                    const double* __restrict__ taps, const double* __restrict__ w, const GridAcc ga) {
    using C = Spread2Cfg;
    const int n = ga.n;
    pdl_trigger();
    pdl_wait();   // w, its bound slot and the cleared accumulator come from the preceding kernels
    const double gscale = grid_scale(ga);
    constexpr int W = C::W, S = C::S, m = W / 2, TS = C::TS;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    double* REGm = smem + warp * C::REG;
    const int ns = n / kSup2;

    // CTA_ITEM (few items: small node sets): one item per CTA, warp w takes segments w, w + 4,
    // ... into its own region and the flush adds the 4 regions in warp order (deterministic):
    // 4 short dependent-load chains per item instead of one long one, which is the critical
    // path at a few nodes per cell (img64 spread 23.5 -> 15.7 us, c2 26 -> 22 us). Otherwise
    // one item per warp (many items: c4, img512 lose 15-35 % in the CTA form).
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;
    for (int ii = CTA_ITEM ? blockIdx.x : gw; ii < nitems; ii += CTA_ITEM ? gridDim.x : nw) {
        const SpreadItem it = items[ii];
        const int sy = it.stile % ns, sx = it.stile / ns;
        for (int i = lane; i < C::REG; i += 32) REGm[i] = 0.0;
        __syncwarp();
        for (int sg = it.seg_begin + (CTA_ITEM ? warp : 0); sg < it.seg_end; sg += CTA_ITEM ? C::NWARP : 1) {
            const CellBatch seg = segs[sg];
            const int cy = seg.cell % n, cx = seg.cell / n;
            const int ox = cx - kSup2 * sx, oy = cy - kSup2 * sy;
            double acc[2][2][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
            const double* T0 = taps + (long long)seg.start * TS;
            const double* w0 = w + seg.start;
            const int nks = (seg.count + 3) >> 2;
#pragma unroll 4
            for (int s = 0; s < nks; ++s) {
                const int jr = 4 * s + q;
                const bool ok = jr < seg.count;
                const double* tr = T0 + (ok ? jr : 0) * TS;
                const double wj = ok ? __ldg(w0 + jr) : 0.0;
                const double a0 = wj * __ldg(tr + g), a1 = wj * __ldg(tr + 8 + g);
                const double b0v = __ldg(tr + W + g), b1v = __ldg(tr + W + 8 + g);
                dmma884(acc[0][0][0], acc[0][0][1], a0, b0v);
                dmma884(acc[0][1][0], acc[0][1][1], a0, b1v);
                dmma884(acc[1][0][0], acc[1][0][1], a1, b0v);
                dmma884(acc[1][1][0], acc[1][1][1], a1, b1v);
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
        if (CTA_ITEM) {
            __syncthreads();
            for (int i = threadIdx.x; i < C::REG; i += C::NT) {
                double v = smem[i];
#pragma unroll
                for (int w = 1; w < C::NWARP; ++w) v += smem[w * C::REG + i];
                if (v != 0.0) grid_add<2>(ga, gscale, gx0 + i / S, gy0 + i % S, 0, v);
            }
            __syncthreads();
        } else {
            __syncwarp();
            for (int i = lane; i < C::REG; i += 32) {
                const double v = REGm[i];
                if (v != 0.0) grid_add<2>(ga, gscale, gx0 + i / S, gy0 + i % S, 0, v);
            }
            __syncwarp();
        }
    }
}

#endif  // SK_WORKLIST_ONLY

}  // namespace sk
