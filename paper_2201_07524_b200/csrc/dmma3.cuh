// dmma3.cuh -- d = 3 spread / interp on the FP64 tensor cores (mma.sync m8n8k4 .f64 -> DMMA),
// for 2 m_w = W = 12 taps per axis (the d = 3 workloads c3, c5); shared helpers for dmma2.cuh.
//
// All nodes of one grid cell share the same W^3 taps, so per cell the window sums are dense
// contractions over the cell's nodes (P:L475-477 gridding, written as GEMMs):
//
//   interp (NFFT trafo):  E[(tx,ty), j] = sum_tz G[tx,ty,tz] phi_z,j[tz]         (DMMA: M=(tx,ty),
//                         t_j = sum_tx phi_x,j[tx] sum_ty phi_y,j[ty] E[(tx,ty), j]   K=tz, N=nodes)
//   spread (adjoint):     G[tx, (ty,tz)] += sum_j (w_j phi_x,j[tx]) (phi_y,j[ty] phi_z,j[tz])
//                                                                               (DMMA: M=tx, N=(ty,tz),
//                                                                                K=nodes)
// FP64 DMMA and DFMA share one pipe on B200 (37 TF either way, tools/microbench.cu), but the
// tensor core reuses its operands internally: one A/B register per lane feeds 256 FMAs, so
// shared memory is no longer the limiter (broadcast LDS.128 runs at ~0.5/clk/SM).
//
// Window taps: the nodes are fixed for the whole solve, so plan.cu tabulates every node's
// d x W window values once (taps_precompute_kernel, [node][axis][W] FP64 in HBM, c5: 52 GB)
// and the kernels load fragments straight from it (L1/L2): no per-apply window evaluation.
//
// DMMA shapes: interp rows are the 144 flattened (tx, ty) pairs (18 m-tiles, K = tz = 12:
// no padding); a lane's row g meets only 3 distinct ty values, so phi_y of its 8 nodes stays
// in registers. Spread rows are tx padded 12 -> 16 (75% useful DMMA work); a lane's 18
// B-operand columns (ty, tz) meet only 3 distinct tz, so each k-step loads 12 phi_y + 3 phi_z
// values and forms the 18 products with one DMUL each.
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
// m16n8k4: A rows g (a0) and g + 8 (a1), one B operand; C rows g (c0, c1) and g + 8 (c2, c3)
__device__ __forceinline__ void dmma1684(double& c0, double& c1, double& c2, double& c3, double a0, double a1,
                                         double b) {
    asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b));
}
#ifndef SK_SPREAD_M16
#define SK_SPREAD_M16 1
#endif

// Work unit of the interp: up to 32 nodes of one cell.
struct CellBatch {
    int cell;   // packed cell coordinates (cx * n + cy) * n + cz  (d = 2: cx * n + cy)
    int start;  // first node (sorted order)
    int count;  // <= 32
    int pad;
};
// Work unit of the spread: nodes of consecutive cells of one super-tile.
struct SpreadItem {
    int stile;      // packed super-tile coordinates, row-major over n / T per axis
    int seg_begin;  // first segment (CellBatch, count <= kSegMax)
    int seg_end;
    int count;      // nodes
};
#ifndef SK_INTERP_NB
#define SK_INTERP_NB 32
#endif
#ifndef SK_TP_SEG_MAX
#define SK_TP_SEG_MAX 32
#endif
constexpr int kInterpBatch3 = SK_INTERP_NB;   // d = 3 interp batch (nodes of one cell per warp pass)
constexpr int kSegMax = 1024;     // d = 2 spread segments (nodes of one cell)
constexpr int kSegTmaPMax = SK_TP_SEG_MAX;   // spread3_tmapad_kernel segments (sparse cells)
#ifndef SK_TP_SEG_DENSE
#define SK_TP_SEG_DENSE 64
#endif
#ifndef SK_SPREAD3_SUNROLL
#define SK_SPREAD3_SUNROLL 0   // 0: per shape (see spread3_tmapad_kernel)
#endif
#ifndef SK_SPREAD3_PRODFIRST
#define SK_SPREAD3_PRODFIRST 0
#endif
constexpr int kSegTmaPDense = SK_TP_SEG_DENSE;   // spread3_tmapad_kernel segments (dense cells)
constexpr int kSegDenseMinMean = 1 << 30;     // mean nodes per occupied cell for the dense shape:
                                              // off since the 28-tile cover (162 registers fit 12
                                              // warps per SM; c5 spread 12.46 -> 12.13 ms (y),
                                              // 15.01 -> 14.91 ms (x)); round 1's 200 gained c5 x/y
#ifndef SK_SPREAD_ITEM_MAX
#define SK_SPREAD_ITEM_MAX 4096
#endif
constexpr int kSpreadItemMax = SK_SPREAD_ITEM_MAX;

#ifndef SK_WORKLIST_ONLY   // plan.cu only needs the work-list types above

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// warp-cooperative L2 prefetch of [p, p + bytes)
__device__ __forceinline__ void prefetch_range(const void* p, long long bytes, int lane) {
    const char* c = reinterpret_cast<const char*>(p);
    for (long long off = (long long)lane * 128; off < bytes; off += 32 * 128) prefetch_l2(c + off);
}

// ------------------------------------------------------------------------------ taps
// out[node][a][t] = phi(f_a + m - 1 - t), f_a = frac(u_a), t < W (even/odd tap polynomials).
// A warp stages its 32 nodes' rows in shared memory and writes them out as one contiguous,
// coalesced block (32 * D * W doubles) instead of 32 scattered row stores.
template <int D, int W>
__global__ void __launch_bounds__(128)
taps_precompute_kernel(const double* __restrict__ u, long long count, const __grid_constant__ WinPoly wp,
                       double* __restrict__ out) {
    constexpr int ROW = D * W;                       // doubles per node
    __shared__ __align__(16) double csm[(W / 2) * kCoefRow];
    __shared__ __align__(16) double stage[4][32 * ROW];   // 128 threads: 4 warps
    load_coefs<W>(wp, csm);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* st = stage[warp];
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long base = (blockIdx.x * (long long)(blockDim.x >> 5) + warp) * 32; base < count;
         base += nwarps * 32) {
        const long long j = base + lane;
        const int nvalid = (int)min(32LL, count - base);
#pragma unroll 1
        for (int a = 0; a < D; ++a) {
            const double uv = j < count ? u[a * count + j] : 0.5;
            const double g = uv - floor(uv) - 0.5, g2 = g * g;
            double v[W];
#pragma unroll
            for (int t = 0; t < W / 2; ++t) {   // tap pair (t, W-1-t): E(g^2) +- g O(g^2)
                const double* cr = csm + t * kCoefRow;
                double E = cr[7], O = cr[14];
#pragma unroll
                for (int i = 6; i >= 0; --i) E = fma(E, g2, cr[i]);
#pragma unroll
                for (int i = 5; i >= 0; --i) O = fma(O, g2, cr[8 + i]);
                v[t] = fma(g, O, E);
                v[W - 1 - t] = fma(-g, O, E);
            }
            double2* o = reinterpret_cast<double2*>(st + lane * ROW + a * W);
#pragma unroll
            for (int t = 0; t < W / 2; ++t) o[t] = make_double2(v[2 * t], v[2 * t + 1]);
        }
        __syncwarp();
        const double2* src = reinterpret_cast<const double2*>(st);
        double2* dst = reinterpret_cast<double2*>(out + base * ROW);
        for (int i = lane; i < nvalid * ROW / 2; i += 32) dst[i] = src[i];
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------ interp
#ifndef SK_INTERP3_MINB
#define SK_INTERP3_MINB 3
#endif
#ifndef SK_INTERP3_KUNROLL
#define SK_INTERP3_KUNROLL 1
#endif
constexpr int kInterpKUnroll = SK_INTERP3_KUNROLL;
#ifndef SK_INTERP3_ORDER
#define SK_INTERP3_ORDER 1   // DMMA issue order within a k-step: 0 = k-slice major, 1 = m-tile major
                             // (c5 interp 13.28 -> 12.86 ms: each m-tile's DFMAs can start while the
                             // next m-tile's DMMAs run)
#endif
#ifndef SK_INTERP3_ACCTY
#define SK_INTERP3_ACCTY 1
#endif
#ifndef SK_INTERP_NT
#define SK_INTERP_NT 128
#endif
struct InterpDCfg {
    static constexpr int W = 12, KS = W / 4, NT = SK_INTERP_NT, NWARP = NT / 32, TS = 3 * W;
    static constexpr int NB = kInterpBatch3, NTN = NB / 8;   // nodes / n-tiles per batch
#ifndef SK_INTERP_PREFETCH
#define SK_INTERP_PREFETCH 1
#endif
#ifndef SK_INTERP_XS
#define SK_INTERP_XS 14
#endif
    static constexpr int XS = SK_INTERP_XS;                   // phi_x row stride (doubles)
    static constexpr int GBLK = W * W * W;                    // the cell's 12^3 grid block
    static constexpr size_t SMEM_BYTES = sizeof(double) * NWARP * (NB * XS + GBLK);   // STAGE
    static constexpr size_t SMEM_BYTES_NOSTAGE = sizeof(double) * NWARP * NB * XS;     // more L1
};

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem_src));
}
#ifndef SK_INTERP_XT_ASYNC
#define SK_INTERP_XT_ASYNC 1   // phi_x staging of the next batch during this batch's epilogue
#endif
#ifndef SK_INTERP_BF_AHEAD
#define SK_INTERP_BF_AHEAD 0   // 1: the next batch's phi_z B fragments loaded during this batch's epilogue (measured slower)
#endif

// One batch (<= 32 nodes of one cell) with NT_ n-tiles of 8 nodes: ragged tail batches of sparse
// cells run ceil(count / 8) n-tiles instead of 4 (c3 x nodes: 29 % fewer DMMAs).
// Hb: the cell's 12^3 block (+ q), row strides sxs (tx) and ry[] (the lane's 3 ty rows).
struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};
// B fragments of a batch: phi_z of node 8 nt + g at tz = 4 s + q
__device__ __forceinline__ void load_bf(double (&bf)[3][4], const double* __restrict__ T0, int last, int g, int q) {
    constexpr int W = 12, TS = 3 * W;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
        const double* tz = T0 + min(8 * nt + g, last) * TS + 2 * W;
#pragma unroll
        for (int s = 0; s < 3; ++s) bf[s][nt] = __ldg(tz + 4 * s + q);
    }
}
// bfio: this batch's B fragments on entry (load_bf); after_kloop may overwrite them with the next
// batch's (they are dead once the k loop is done)
template <int NT_, bool STAGE, typename Hook = NoHook>
__device__ __forceinline__ void interp3_batch(const CellBatch& B, const double* __restrict__ taps,
                                              const double* XT, const double* Hb, long long sxs,
                                              const long long (&ry)[3], int ty1, int txo1, int g, int q,
                                              double* __restrict__ t_out, const FusedUpd& fu,
                                              double (&bf)[3][4], const Hook& after_kloop = Hook()) {
    using C = InterpDCfg;
    constexpr int W = C::W, KS = C::KS, TS = C::TS;
    const double* T0 = taps + (long long)B.start * TS;
    const int last = B.count - 1;
    // per (node, ty) partial sums over tx: phi_y is applied once after the k loop, so each
    // E value costs one DFMA in the loop (24 per k-step at 4 n-tiles)
    double acc3[NT_][2][3];
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc3[nt][e][0] = acc3[nt][e][1] = acc3[nt][e][2] = 0.0;
#pragma unroll kInterpKUnroll
    for (int k = 0; k < W / 2; ++k) {
        // three m-tiles (one period of ty) per step, issued m-tile major (SK_INTERP3_ORDER 1):
        // NT_ independent accumulations separate dependent DMMAs, and the DFMAs of an m-tile
        // can run while the next m-tile's DMMAs issue
        int txr[3];
        txr[0] = 2 * k;
        txr[1] = 2 * k + txo1;
        txr[2] = 2 * k + 1;
        double a[3][KS];
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3) {
            const double* Hrow = Hb + txr[r3] * sxs + ry[r3];
#pragma unroll
            for (int s = 0; s < KS; ++s) a[r3][s] = STAGE ? Hrow[4 * s] : __ldg(Hrow + 4 * s);
        }
        double d[3][NT_][2];
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
            for (int nt = 0; nt < NT_; ++nt) d[r3][nt][0] = d[r3][nt][1] = 0.0;
#if SK_INTERP3_ORDER == 1
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
            for (int s = 0; s < KS; ++s)
#pragma unroll
                for (int nt = 0; nt < NT_; ++nt) dmma884(d[r3][nt][0], d[r3][nt][1], a[r3][s], bf[s][nt]);
#else
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
            for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
                for (int nt = 0; nt < NT_; ++nt) dmma884(d[r3][nt][0], d[r3][nt][1], a[r3][s], bf[s][nt]);
#endif
#pragma unroll
        for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                // phi_x[2k], phi_x[2k+1] of the node in one 16-byte load
                const double2 xx = reinterpret_cast<const double2*>(XT + (8 * nt + 2 * q + e) * C::XS)[k];
                acc3[nt][e][0] = fma(xx.x, d[0][nt][e], acc3[nt][e][0]);
                acc3[nt][e][1] = fma(txo1 ? xx.y : xx.x, d[1][nt][e], acc3[nt][e][1]);
                acc3[nt][e][2] = fma(xx.y, d[2][nt][e], acc3[nt][e][2]);
            }
    }
    after_kloop();   // XT is free from here on (the epilogue reads phi_y from the taps)
    double acc[NT_][2];
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double* tr = T0 + min(8 * nt + 2 * q + e, last) * TS + W;
            acc[nt][e] = fma(__ldg(tr + g), acc3[nt][e][0],
                             fma(__ldg(tr + ty1), acc3[nt][e][1], __ldg(tr + 4 + g) * acc3[nt][e][2]));
        }
    // sum over the 8 rows g held by lanes q, q+4, ..., q+28
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double v = acc[nt][e];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            acc[nt][e] = v;
        }
    // every lane now holds the sums of its q; lane (g, q) emits node 8 (g/2) + 2 q + g%2, so
    // the results (and the fused division) take one full-warp pass
    double v = acc[0][0];
#pragma unroll
    for (int nt = 0; nt < NT_; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e)
            if (g == 2 * nt + e) v = acc[nt][e];
    const int p = 8 * (g >> 1) + 2 * q + (g & 1);
    if ((g >> 1) < NT_ && p < B.count) emit_t(t_out, fu, B.start + p, v);
}

// STAGE: copy each cell's 12^3 grid block to shared memory once and read the A fragments from
// there (pays when cells hold several batches: c5 interp 16.1 -> 14.2 ms); otherwise read them
// through L1 straight from the grid.
template <bool STAGE>
__global__ void __launch_bounds__(SK_INTERP_NT, SK_INTERP3_MINB)
interp3_dmma_kernel(const CellBatch* __restrict__ batches, int nbatches, const double* __restrict__ taps,
                    const double* __restrict__ grid, int n, double* __restrict__ t_out, const FusedUpd fu) {
    using C = InterpDCfg;
    constexpr int W = C::W, m = W / 2, TS = C::TS, NB = C::NB, NTN = C::NTN;
    static_assert(NTN >= 1 && NTN <= 4, "interp3 batches hold 1..4 n-tiles");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const long long n2 = (long long)n * n;
    const int gw = blockIdx.x * C::NWARP + warp, nw = gridDim.x * C::NWARP;
    extern __shared__ __align__(16) double smem[];
    double* XT = smem + warp * (STAGE ? NB * C::XS + C::GBLK : NB * C::XS);   // [node][XS] phi_x rows
    double* GB = XT + NB * C::XS;                          // [tx][ty][tz] grid block of the cell
    int cur_cell = -1;
    // contiguous slice of the cell-sorted batch list per warp: consecutive batches of one
    // cell reuse its 12^3 grid block, and the taps stream sequentially
    const int per = (nbatches + nw - 1) / nw;
    const int b_lo = gw * per, b_hi = min(nbatches, b_lo + per);
    // Rows of the DMMA are the flattened (tx, ty) pairs r = 8 mt + g, mt < 18 (no padding).
    // For lane row g, ty = r % 12 cycles with period 3 in mt through {g, (8+g)%12, 4+g}.
    // Within step k the lane's three rows have tx = 2k (r3 = 0, and r3 = 1 when g < 4) or
    // 2k + 1 (r3 = 2, and r3 = 1 when g >= 4).
    const int ty1 = (8 + g) % W, txo1 = (g >= 4) ? 1 : 0;
    const long long sxs = STAGE ? W * W : n2;
    const long long ry[3] = {STAGE ? g * W : (long long)g * n, STAGE ? ty1 * W : (long long)ty1 * n,
                             STAGE ? (4 + g) * W : (long long)(4 + g) * n};

    pdl_trigger();
    pdl_wait();   // the grid (and the fused update's p, x) come from the preceding kernels
    CellBatch Bnext = b_lo < b_hi ? batches[b_lo] : CellBatch{0, 0, 0, 0};
    double bf[3][4];   // B fragments of the batch about to run (loaded one batch ahead)
#if SK_INTERP_BF_AHEAD
    if (b_lo < b_hi) load_bf(bf, taps + (long long)Bnext.start * TS, Bnext.count - 1, g, q);
#endif
    for (int bi = b_lo; bi < b_hi; ++bi) {
        const CellBatch B = Bnext;   // descriptor loaded one batch ahead
        if (bi + 1 < b_hi) Bnext = batches[bi + 1];
        const int cz = B.cell % n, cy = (B.cell / n) % n, cx = B.cell / n / n;
        const double* T0 = taps + (long long)B.start * TS;
        const int last = B.count - 1;
        // a new cell: copy its 12^3 grid block to shared memory (async, overlapped with the
        // batch's tap loads); the following batches of the cell read it from there
        const bool new_cell = STAGE && B.cell != cur_cell;
        if (new_cell) {
            const double* Gb = grid + (long long)(cx - m + 1) * n2 + (long long)(cy - m + 1) * n + (cz - m + 1);
            for (int i = lane; i < C::GBLK; i += 32) {
                const int r = i / W, c = i % W;
                cp_async8(GB + i, Gb + (long long)(r / W) * n2 + (long long)(r % W) * n + c);
            }
            cur_cell = B.cell;
        }
        if (bi + 1 < b_hi)   // next batch of this warp: stream its taps into L2
            if (SK_INTERP_PREFETCH) prefetch_range(taps + (long long)Bnext.start * TS, (long long)Bnext.count * TS * 8, lane);
#if SK_INTERP_XT_ASYNC
        // phi_x rows of this batch: issued with cp.async during the previous batch's epilogue
        // (first batch: here)
        if (bi == b_lo && lane < NB) {
            const double* src = T0 + min(lane, last) * TS;
#pragma unroll
            for (int i = 0; i < W / 2; ++i) cp_async16(XT + lane * C::XS + 2 * i, src + 2 * i);
        }
        cp_async_wait_all();
#else
        if (lane < NB) {   // stage the batch's phi_x rows (lane = node) in this warp's shared table
            const double2* src = reinterpret_cast<const double2*>(T0 + min(lane, last) * TS);
            double2* dst = reinterpret_cast<double2*>(XT + lane * C::XS);
#pragma unroll
            for (int i = 0; i < W / 2; ++i) dst[i] = __ldg(src + i);
        }
        if (new_cell) cp_async_wait_all();
#endif
        __syncwarp();
        const double* Hb = STAGE ? GB + q
                                 : grid + (long long)(cx - m + 1) * n2 + (long long)(cy - m + 1) * n + (cz - m + 1) + q;
        const int ntn = min(NTN, (B.count + 7) >> 3);   // warp-uniform
        const bool has_next = bi + 1 < b_hi;
        const double* Tn = taps + (long long)Bnext.start * TS;
        const int lastn = Bnext.count - 1;
        auto hook = [&]() {   // the next batch's operands, overlapping this batch's epilogue
#if SK_INTERP_XT_ASYNC
            __syncwarp();
            if (has_next && lane < NB) {   // phi_x rows
                const double* src = Tn + min(lane, lastn) * TS;
#pragma unroll
                for (int i = 0; i < W / 2; ++i) cp_async16(XT + lane * C::XS + 2 * i, src + 2 * i);
            }
#endif
#if SK_INTERP_BF_AHEAD
            if (has_next) load_bf(bf, Tn, lastn, g, q);   // B fragments
#endif
        };
#if !SK_INTERP_BF_AHEAD
        load_bf(bf, T0, last, g, q);
#endif
        if (ntn >= 4 && NTN >= 4) interp3_batch<(NTN >= 4 ? 4 : 1), STAGE>(B, taps, XT, Hb, sxs, ry, ty1, txo1, g, q, t_out, fu, bf, hook);
        else if (ntn == 3 && NTN >= 3) interp3_batch<(NTN >= 3 ? 3 : 1), STAGE>(B, taps, XT, Hb, sxs, ry, ty1, txo1, g, q, t_out, fu, bf, hook);
        else if (ntn == 2 && NTN >= 2) interp3_batch<(NTN >= 2 ? 2 : 1), STAGE>(B, taps, XT, Hb, sxs, ry, ty1, txo1, g, q, t_out, fu, bf, hook);
        else interp3_batch<1, STAGE>(B, taps, XT, Hb, sxs, ry, ty1, txo1, g, q, t_out, fu, bf, hook);
        __syncwarp();   // XT is rewritten by the next batch
    }
}

// ------------------------------------------------------------------------------ spread
// mbarrier / bulk-copy helpers of the TMA-fed spread.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pair_barrier(int pair) { asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory"); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mb)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
}

// ------------------------------------------------------------------------------ spread (TMA, padded)
// The padded DMMA spread (rows tx padded 12 -> 16, one m16n8k4 per n-tile) on a warp pair fed by
// the same TMA double buffer: warp h owns the 9 n-tiles with ty in 6h .. 6h+5, so a lane holds
// 36 accumulators instead of 72 and reads its operands from shared memory, which lets 3 pairs
// share a CTA (12 warps per SM instead of 8).
// Two shapes: 32-node segments on 3 pairs per CTA (12 warps per SM; sparse cells, where the
// per-cell region update dominates) and 64-node segments on 2 pairs (8 warps per SM, half the
// per-segment overhead; dense cells: c5 spread 15.48 -> 15.14 ms). The plan picks per node set.
template <int SEG, int NPAIR_>
struct SpreadTPCfg {
    static constexpr int W = 12, S = W + 1, NPAIR = NPAIR_, NT = 64 * NPAIR, NTH = 9;
    static constexpr int TS = 3 * W;
    static constexpr int REG = S * S * S;
    static constexpr int REGP = REG + 1;
    static constexpr int TBUF = SEG * TS;
    static constexpr int WBUF = SEG + 4;
    static constexpr int PAIR = 4 + REGP + 2 * TBUF + 2 * WBUF;   // 4 mbarrier words (full / empty)
    static constexpr size_t SMEM_BYTES = sizeof(double) * NPAIR * PAIR;
};
#ifndef SK_TP_NPAIR_SPARSE
#define SK_TP_NPAIR_SPARSE 3
#endif
constexpr int kSparsePairs = SK_TP_NPAIR_SPARSE;   // warp pairs per CTA of the 32-node shape
using SpreadTPCfgSparse = SpreadTPCfg<kSegTmaPMax, kSparsePairs>;
using SpreadTPCfgDense = SpreadTPCfg<kSegTmaPDense, 2>;

// ------------------------------------------------------------------------------ 28-tile cover
// A node's 12^3 contributions w phi_x[tx] phi_y[ty] phi_z[tz] tiled by m8n8k4 DMMA tiles instead
// of 12 -> 16 padded rows (36 DMMA.8x8x4 per 4-node k-step, 75 % useful): 1728 = 27 x 64, and
// with each tile's rows and columns products of whole axes the cover needs 28 tiles (96 %):
//   F1 (18): rows tx = g (0..7),                 cols (ty, tz) = flat 8 jn + c      A = w phi_x,  B = phi_y phi_z
//   F2  (6): rows (tx, ty) = (8 + g%4, 2p + g/4), cols tz = c (0..7)                 A = w phi_x phi_y, B = phi_z
//   F3  (2): rows ty = g (0..7),                 cols (tx, tz) = (8 + 2t + c/4, 8 + c%4)  A = phi_y, B = w phi_x phi_z
//   F4  (2): rows as F2 with p = 4, 5,           cols tz = 8 + c (c < 4; c >= 4 zero)
// (F1 tx 0..7 x all (ty, tz): 1152; F2 tx 8..11 x ty 0..11 x tz 0..7: 384; F3 tx 8..11 x ty 0..7 x
// tz 8..11: 128; F4 tx 8..11 x ty 8..11 x tz 8..11: 64.) Warp h of the pair takes 14 tiles:
// h = 0: F1 jn 0..8, F2 p 0..4;  h = 1: F1 jn 9..17, F2 p 5, F3 t 0, 1, F4 p 4, 5 (16 DMULs each).
// acc index: 0..8 F1; h = 0: 9..13 F2 p; h = 1: 9 F2 p5, 10..11 F3, 12..13 F4.
#ifndef SK_SPREAD3_T28
#define SK_SPREAD3_T28 1
#endif
template <int H, int kSU>
__device__ __forceinline__ void spread3_t28_ksteps(double (&acc)[14][2], const double* __restrict__ T0,
                                                   const double* __restrict__ W0, int count, int nks, int g,
                                                   int q) {
    constexpr int W = 12, TS = 3 * W;
    const int z1 = (8 + g) % W;
#pragma unroll kSU
    for (int s = 0; s < nks; ++s) {
        const int jr = 4 * s + q;
        const bool ok = jr < count;
        const double* tr = T0 + (ok ? jr : 0) * TS;
        const double wu = ok ? W0[jr] : 0.0;
        const double wx0 = wu * tr[g];
        const double wx1 = wu * tr[8 + (g & 3)];
        double yv[6];
        {
            const double2* y2 = reinterpret_cast<const double2*>(tr + W + 6 * H);
#pragma unroll
            for (int i = 0; i < 3; ++i) { const double2 v2 = y2[i]; yv[2 * i] = v2.x; yv[2 * i + 1] = v2.y; }
        }
        const double zv[3] = {tr[2 * W + g], tr[2 * W + z1], tr[2 * W + 4 + g]};
#pragma unroll
        for (int j = 0; j < 9; ++j) {   // F1: f = 8 (9H + j) + g -> ty = 6H + 2 (j / 3) + {0, g >= 4, 1}
            const int k3 = j / 3, r3 = j % 3;
            const double yvv = (r3 == 0) ? yv[2 * k3]
                             : ((r3 == 1) ? (g >= 4 ? yv[2 * k3 + 1] : yv[2 * k3]) : yv[2 * k3 + 1]);
            dmma884(acc[j][0], acc[j][1], wx0, yvv * zv[r3]);
        }
        const int gy = g >> 2;
        if constexpr (H == 0) {
#pragma unroll
            for (int p = 0; p < 5; ++p) dmma884(acc[9 + p][0], acc[9 + p][1], wx1 * tr[W + 2 * p + gy], zv[0]);
        } else {
            const double a5 = wx1 * tr[W + 10 + gy], a4 = wx1 * tr[W + 8 + gy];
            dmma884(acc[9][0], acc[9][1], a5, zv[0]);
            const double wz = wu * tr[2 * W + 8 + (g & 3)];
            const double ay = tr[W + g];
            dmma884(acc[10][0], acc[10][1], ay, wz * tr[8 + gy]);
            dmma884(acc[11][0], acc[11][1], ay, wz * tr[10 + gy]);
            const double bz = g < 4 ? zv[1] : 0.0;   // zv[1] = phi_z[8 + g] for g < 4
            dmma884(acc[12][0], acc[12][1], a4, bz);
            dmma884(acc[13][0], acc[13][1], a5, bz);
        }
    }
}
// Adds the 14 tiles' C fragments (c_e = C[g][2q + e]) into the region at rc (the cell's (0,0,0)
// tap; strides S^2, S, 1).
template <int H>
__device__ __forceinline__ void spread3_t28_update(double (&acc)[14][2], double* rc, int g, int q) {
    constexpr int W = 12, S = W + 1;
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int f = 8 * (9 * H + j) + 2 * q + e;
            rc[g * S * S + (f / W) * S + (f % W)] += acc[j][e];
        }
    const int tx1 = 8 + (g & 3), gy = g >> 2;
    if constexpr (H == 0) {
#pragma unroll
        for (int p = 0; p < 5; ++p)
#pragma unroll
            for (int e = 0; e < 2; ++e) rc[tx1 * S * S + (2 * p + gy) * S + 2 * q + e] += acc[9 + p][e];
    } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) rc[tx1 * S * S + (10 + gy) * S + 2 * q + e] += acc[9][e];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 2 * q + e;
                rc[(8 + 2 * t + (c >> 2)) * S * S + g * S + 8 + (c & 3)] += acc[10 + t][e];
            }
        if (q < 2) {
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int e = 0; e < 2; ++e) rc[tx1 * S * S + (8 + 2 * p + gy) * S + 8 + 2 * q + e] += acc[12 + p][e];
        }
    }
}

// The 28-tile spread on a full / empty mbarrier pipeline (non-x-pair segments): the producer
// (lane 0 of the pair's first warp) refills a segment buffer once both warps have released it
// (empty[b], two arrivals) instead of a pair barrier at every segment, so neither warp waits for
// its partner's k-loop; the next segment's descriptor is loaded one segment ahead. The warps meet
// only before each cell's region update (consecutive cells' regions overlap: one barrier per cell
// instead of per segment, c5 x: 56 segments per cell) and around the item flush (which also
// zeroes the region for the next item).
#ifndef SK_SPREAD3_PIPE
#define SK_SPREAD3_PIPE 1
#endif
template <int SEG, int NPAIR_>
__global__ void __launch_bounds__(64 * NPAIR_, 2)
spread3_t28_kernel(const SpreadItem* __restrict__ items, int nitems, const CellBatch* __restrict__ segs,
                   const double* __restrict__ taps, const double* __restrict__ w, const GridAcc ga) {
    using C = SpreadTPCfg<SEG, NPAIR_>;
    constexpr int kSU = SK_SPREAD3_SUNROLL > 0 ? SK_SPREAD3_SUNROLL : (SEG >= 64 ? 4 : 8);
    constexpr int W = C::W, S = C::S, m = W / 2, TS = C::TS;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pair = warp >> 1, half = warp & 1;
    const int g = lane >> 2, q = lane & 3;
    const int plane = half * 32 + lane;
    double* base = smem + pair * C::PAIR;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(base);   // [2]
    unsigned long long* empty = full + 2;                                       // [2]
    double* REGm = base + 4;
    double* TB0 = base + 4 + C::REGP;
    double* WB0 = TB0 + 2 * C::TBUF;
    const int n = ga.n, ns = n / 2;
    pdl_trigger();
    pdl_wait();   // w, its bound slot and the cleared accumulator come from the preceding kernels
    const double gscale = grid_scale(ga);
    const int gp = blockIdx.x * C::NPAIR + pair, np = gridDim.x * C::NPAIR;
    const bool producer = half == 0 && lane == 0;
    if (producer) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], 2);
        mbar_init(&empty[1], 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = plane; i < C::REG; i += 64) REGm[i] = 0.0;
    pair_barrier(pair);
    auto issue = [&](const CellBatch& sq, int b) {
        const long long st = sq.start;
        const long long w0 = st & ~1LL, w1 = (st + sq.count + 1) & ~1LL;
        const unsigned tbytes = (unsigned)sq.count * TS * 8u, wbytes = (unsigned)(w1 - w0) * 8u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[b], tbytes + wbytes);
        tma_load_1d(TB0 + b * C::TBUF, taps + st * TS, tbytes, &full[b]);
        tma_load_1d(WB0 + b * C::WBUF, w + w0, wbytes, &full[b]);
    };
    int t = 0;   // segments of this pair so far (buffer t & 1, its (t >> 1)-th use)
    CellBatch seg_next = gp < nitems ? segs[items[gp].seg_begin] : CellBatch{0, 0, 0, 0};
    if (producer && gp < nitems) issue(seg_next, 0);
    for (int ii = gp; ii < nitems; ii += np) {
        const SpreadItem it = items[ii];
        const int sz = it.stile % ns, sy = (it.stile / ns) % ns, sx = it.stile / ns / ns;
        double acc28[14][2];
        bool fresh = true;
        for (int sg = it.seg_begin; sg < it.seg_end; ++sg, ++t) {
            const int b = t & 1;
            const CellBatch seg = seg_next;
            // the pair's next segment: this item's, or the first of its next item
            const bool more = sg + 1 < it.seg_end;
            const int nxt_item = ii + np;
            if (more) seg_next = segs[sg + 1];
            else if (nxt_item < nitems) seg_next = segs[items[nxt_item].seg_begin];
            if (producer && (more || nxt_item < nitems)) {
                if (t >= 1) mbar_wait(&empty[b ^ 1], (unsigned)((t - 1) >> 1) & 1u);   // both warps released it
                issue(seg_next, b ^ 1);
            }
            mbar_wait(&full[b], (unsigned)(t >> 1) & 1u);
            const double* T0 = TB0 + b * C::TBUF;
            const double* W0 = WB0 + b * C::WBUF + (seg.start & 1LL);
            if (fresh) {
#pragma unroll
                for (int j = 0; j < 14; ++j) acc28[j][0] = acc28[j][1] = 0.0;
                fresh = false;
            }
            const int nks = (seg.count + 3) >> 2;
            if (half == 0) spread3_t28_ksteps<0, kSU>(acc28, T0, W0, seg.count, nks, g, q);
            else spread3_t28_ksteps<1, kSU>(acc28, T0, W0, seg.count, nks, g, q);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[b])) : "memory");
            if (!more || seg_next.cell != seg.cell) {
                // the warps may drift apart by a segment; consecutive cells' regions overlap, so
                // the update of this cell waits until the partner finished the previous one
                pair_barrier(pair);
                const int cz = seg.cell % n, cy = (seg.cell / n) % n, cx = seg.cell / n / n;
                double* rc = REGm + (cx - 2 * sx) * S * S + (cy - 2 * sy) * S + (cz - 2 * sz);
                if (half == 0) spread3_t28_update<0>(acc28, rc, g, q);
                else spread3_t28_update<1>(acc28, rc, g, q);
                fresh = true;
            }
        }
        pair_barrier(pair);
        const int gx0 = 2 * sx - (m - 1), gy0 = 2 * sy - (m - 1), gz0 = 2 * sz - (m - 1);
        for (int i = plane; i < C::REG; i += 64) {   // flush, and zero the region for the next item
            const double v = REGm[i];
            if (v != 0.0) {
                const int rz = i % S, rest = i / S, ry = rest % S, rxx = rest / S;
                grid_add<3>(ga, gscale, gx0 + rxx, gy0 + ry, gz0 + rz, v);
                REGm[i] = 0.0;
            }
        }
        pair_barrier(pair);
    }
}

// XP: segments may hold the nodes of an x-pair of cells (seg.cell is the x-digit-0 cell, its
// seg.pad nodes come first, the rest sit one row lower): 13 of the 16 padded DMMA rows, so a
// sparse pair costs one accumulator flush instead of two at no extra DMMA work.
template <int SEG, int NPAIR_, bool XP>
__global__ void __launch_bounds__(64 * NPAIR_, 2)
spread3_tmapad_kernel(const SpreadItem* __restrict__ items, int nitems, const CellBatch* __restrict__ segs,
                      const double* __restrict__ taps, const double* __restrict__ w, const GridAcc ga) {
    using C = SpreadTPCfg<SEG, NPAIR_>;
    // k-step unroll (measured): 4 for the dense shape (c5 spread 15.17 -> 14.71 ms with 2),
    // 8 for the 32-node shape (c3 0.248 -> 0.243 ms)
    constexpr int kSU = SK_SPREAD3_SUNROLL > 0 ? SK_SPREAD3_SUNROLL : (SEG >= 64 ? 4 : 8);
    constexpr int W = C::W, S = C::S, m = W / 2, NTH = C::NTH, TS = C::TS;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pair = warp >> 1, half = warp & 1;
    const int g = lane >> 2, q = lane & 3;
    const int plane = half * 32 + lane;
    double* base = smem + pair * C::PAIR;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(base);
    double* REGm = base + 2;
    double* TB0 = base + 2 + C::REGP;
    double* WB0 = TB0 + 2 * C::TBUF;
    const int n = ga.n, ns = n / 2;
    pdl_trigger();
    pdl_wait();   // w, its bound slot and the cleared accumulator come from the preceding kernels
    const double gscale = grid_scale(ga);
    const int gp = blockIdx.x * C::NPAIR + pair, np = gridDim.x * C::NPAIR;
    const int z1 = (8 + g) % W;
    const bool producer = half == 0 && lane == 0;

    if (producer) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pair_barrier(pair);
    auto issue = [&](int sg, int b) {
        const CellBatch sq = segs[sg];
        const long long st = sq.start;
        const long long w0 = st & ~1LL, w1 = (st + sq.count + 1) & ~1LL;
        const unsigned tbytes = (unsigned)sq.count * TS * 8u, wbytes = (unsigned)(w1 - w0) * 8u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[b], tbytes + wbytes);
        tma_load_1d(TB0 + b * C::TBUF, taps + st * TS, tbytes, &mbar[b]);
        tma_load_1d(WB0 + b * C::WBUF, w + w0, wbytes, &mbar[b]);
    };
    unsigned uses0 = 0, uses1 = 0;
    int t = 0;
    if (producer && gp < nitems) issue(items[gp].seg_begin, 0);

    for (int ii = gp; ii < nitems; ii += np) {
        const SpreadItem it = items[ii];
        const int sz = it.stile % ns, sy = (it.stile / ns) % ns, sx = it.stile / ns / ns;
        for (int i = plane; i < C::REG; i += 64) REGm[i] = 0.0;
        double acc[NTH][4];   // m16n8k4 C: rows g (0, 1) and 8 + g (2, 3), columns 2q, 2q+1
        bool fresh = true;
#if SK_SPREAD3_T28
        double acc28[14][2];  // 14 m8n8k4 tiles of the 28-tile cover (spread3_t28_ksteps)
        bool fresh28 = true;
#endif
        for (int sg = it.seg_begin; sg < it.seg_end; ++sg, ++t) {
            const int b = t & 1;
            const CellBatch seg = segs[sg];
            int nsg = -1;
            if (sg + 1 < it.seg_end) nsg = sg + 1;
            else if (ii + np < nitems) nsg = items[ii + np].seg_begin;
            pair_barrier(pair);
            if (producer && nsg >= 0) issue(nsg, b ^ 1);
            if (b == 0) { mbar_wait(&mbar[0], uses0 & 1u); ++uses0; }
            else { mbar_wait(&mbar[1], uses1 & 1u); ++uses1; }
            const double* T0 = TB0 + b * C::TBUF;
            const double* W0 = WB0 + b * C::WBUF + (seg.start & 1LL);
            const int cz = seg.cell % n, cy = (seg.cell / n) % n, cx = seg.cell / n / n;
            const int ox = cx - 2 * sx, oy = cy - 2 * sy, oz = cz - 2 * sz;
            if (fresh) {
#pragma unroll
                for (int j = 0; j < NTH; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
                fresh = false;
            }
            const int nks = (seg.count + 3) >> 2;
#if SK_SPREAD3_T28
            if constexpr (!XP) {
                if (fresh28) {
#pragma unroll
                    for (int j = 0; j < 14; ++j) acc28[j][0] = acc28[j][1] = 0.0;
                    fresh28 = false;
                }
                if (half == 0) spread3_t28_ksteps<0, kSU>(acc28, T0, W0, seg.count, nks, g, q);
                else spread3_t28_ksteps<1, kSU>(acc28, T0, W0, seg.count, nks, g, q);
                const bool flush28 = (sg + 1 >= it.seg_end) || (segs[sg + 1].cell != seg.cell);
                if (flush28) {
                    double* rc = REGm + ox * S * S + oy * S + oz;
                    if (half == 0) spread3_t28_update<0>(acc28, rc, g, q);
                    else spread3_t28_update<1>(acc28, rc, g, q);
                    fresh28 = true;
                }
                continue;
            }
#endif
#pragma unroll kSU
            for (int s = 0; s < nks; ++s) {
                const int jr = 4 * s + q;
                const bool ok = jr < seg.count;
                const double* tr = T0 + (ok ? jr : 0) * TS;
                const double wu = ok ? W0[jr] : 0.0;
                double a0, a1;
                if constexpr (XP) {   // A rows are region rows tx + (node in the x-digit-1 cell)
                    const int oxn = jr >= seg.pad ? 1 : 0;
                    a0 = (g - oxn >= 0) ? wu * tr[g - oxn] : 0.0;
                    a1 = (8 + g - oxn < W) ? wu * tr[8 + g - oxn] : 0.0;
                } else {
                    a0 = wu * tr[g];
                    a1 = (8 + g < W) ? wu * tr[8 + g] : 0.0;
                }
                double yv[6];
                {
                    const double2* y2 = reinterpret_cast<const double2*>(tr + W + 6 * half);
#pragma unroll
                    for (int i = 0; i < 3; ++i) { const double2 v2 = y2[i]; yv[2 * i] = v2.x; yv[2 * i + 1] = v2.y; }
                }
                const double zv[3] = {tr[2 * W + g], tr[2 * W + z1], tr[2 * W + 4 + g]};
#if SK_SPREAD3_PRODFIRST
                double bp[NTH];   // the k-step's 9 B products first, then its 9 DMMAs
#pragma unroll
                for (int j = 0; j < NTH; ++j) {
                    const int k3 = j / 3, r3 = j % 3;
                    const double yvv = (r3 == 0) ? yv[2 * k3]
                                     : ((r3 == 1) ? (g >= 4 ? yv[2 * k3 + 1] : yv[2 * k3]) : yv[2 * k3 + 1]);
                    bp[j] = yvv * zv[r3];
                }
#pragma unroll
                for (int j = 0; j < NTH; ++j) dmma1684(acc[j][0], acc[j][1], acc[j][2], acc[j][3], a0, a1, bp[j]);
#else
#pragma unroll
                for (int j = 0; j < NTH; ++j) {
                    const int k3 = j / 3, r3 = j % 3;
                    const double yvv = (r3 == 0) ? yv[2 * k3]
                                     : ((r3 == 1) ? (g >= 4 ? yv[2 * k3 + 1] : yv[2 * k3]) : yv[2 * k3 + 1]);
                    dmma1684(acc[j][0], acc[j][1], acc[j][2], acc[j][3], a0, a1, yvv * zv[r3]);
                }
#endif
            }
            const bool flush_cell = (sg + 1 >= it.seg_end) || (segs[sg + 1].cell != seg.cell);
            if (flush_cell) {
#ifndef SK_TIMING_NO_CELL_UPDATE   // timing-only builds (wrong results): cost of the per-cell update
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const int tx = 8 * mt + g;
                    if (XP ? tx < S : tx < W) {   // XP: seg.cell has ox = 0, rows 0..12
                        double* rx = REGm + (ox + tx) * S * S + oy * S + oz;
#pragma unroll
                        for (int j = 0; j < NTH; ++j)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int col = 8 * (NTH * half + j) + 2 * q + e;
                                rx[(col / W) * S + (col % W)] += acc[j][2 * mt + e];
                            }
                    }
                }
#else
                double sacc = 0.0;   // keep the accumulators live without the shared-memory update
#pragma unroll
                for (int j = 0; j < NTH; ++j) sacc += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
                if (sacc == 1.2345e-300) REGm[plane] = sacc;
#endif
                fresh = true;
            }
        }
        pair_barrier(pair);
        const int gx0 = 2 * sx - (m - 1), gy0 = 2 * sy - (m - 1), gz0 = 2 * sz - (m - 1);
#ifndef SK_TIMING_NO_REGION_FLUSH   // timing-only builds (wrong results): cost of the global flush
        for (int i = plane; i < C::REG; i += 64) {
            const double v = REGm[i];
            if (v != 0.0) {
                const int rz = i % S, rest = i / S, ry = rest % S, rxx = rest / S;
                grid_add<3>(ga, gscale, gx0 + rxx, gy0 + ry, gz0 + rz, v);
            }
        }
#else
        (void)gx0; (void)gy0; (void)gz0;
#endif
        pair_barrier(pair);
    }
}

#endif  // SK_WORKLIST_ONLY

}  // namespace sk
