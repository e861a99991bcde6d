// spread_interp.cuh -- adjoint-NFFT gridding (spread) and NFFT interpolation (interp).
//
//   spread: g[l] += w_j prod_a phi(u_ja - l_a)      over the 2m taps per axis of node j
//   interp: t_j   = sum_l g[l] prod_a phi(u_ja - l_a)
// u = n (x' + 1/2) is the node's grid coordinate; with |x'| <= 1/4 - eps_B/2 and
// n >= 4m no tap wraps around the torus (checked in plan.cu), so indices are direct.
//
// v1 (this file): one thread per node, window values evaluated on the fly; spread
// accumulates with FP64 atomics into the global grid, interp reads it through L1/L2.
#pragma once
#include <atomic>
#include "sk_internal.cuh"
#include "tiled3.cuh"
#include "dmma3.cuh"
#include "dmma2.cuh"
#include "window.cuh"

namespace sk {

// cudaFuncSetAttribute is per device: set the kernel attributes once on every device a
// process launches on (one bit per device ordinal)
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ULL << (dev & 63);
    return !(mask.fetch_or(bit) & bit);
}

template <int D>
__global__ void spread_v1_kernel(const double* __restrict__ u, long long count,
                                 const double* __restrict__ w, Window win, const GridAcc ga) {
    const int W = 2 * win.m;
    const double gscale = grid_scale(ga);
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < count;
         j += (long long)gridDim.x * blockDim.x) {
        double phi[D][kMaxW];
        int base[D];
        for (int a = 0; a < D; ++a) base[a] = kb_taps(u[a * count + j], win, phi[a]) - win.m + 1;
        const double wj = w[j];
        for (int t0 = 0; t0 < W; ++t0) {
            const double w0 = wj * phi[0][t0];
            if (D == 2) {
                for (int t1 = 0; t1 < W; ++t1) grid_add<2>(ga, gscale, base[0] + t0, base[1] + t1, 0, w0 * phi[D - 1][t1]);
            } else {
                for (int t1 = 0; t1 < W; ++t1) {
                    const double w1 = w0 * phi[1][t1];
                    for (int t2 = 0; t2 < W; ++t2)
                        grid_add<3>(ga, gscale, base[0] + t0, base[1] + t1, base[D - 1] + t2, w1 * phi[D - 1][t2]);
                }
            }
        }
    }
}

template <int D>
__global__ void interp_v1_kernel(const double* __restrict__ u, long long count, Window win, int n,
                                 const double* __restrict__ grid, double* __restrict__ t) {
    const int W = 2 * win.m;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < count;
         j += (long long)gridDim.x * blockDim.x) {
        double phi[D][kMaxW];
        int base[D];
        for (int a = 0; a < D; ++a) base[a] = kb_taps(u[a * count + j], win, phi[a]) - win.m + 1;
        double acc = 0.0;
        if (D == 1) {
            for (int t0 = 0; t0 < W; ++t0) acc += phi[0][t0] * __ldg(&grid[base[0] + t0]);
        } else if (D == 2) {
            for (int t0 = 0; t0 < W; ++t0) {
                const double* row = grid + (long long)(base[0] + t0) * n + base[1];
                double s = 0.0;
                for (int t1 = 0; t1 < W; ++t1) s += phi[D - 1][t1] * __ldg(&row[t1]);
                acc += phi[0][t0] * s;
            }
        } else {
            for (int t0 = 0; t0 < W; ++t0) {
                double s1 = 0.0;
                for (int t1 = 0; t1 < W; ++t1) {
                    const double* row = grid + ((long long)(base[0] + t0) * n + (base[1] + t1)) * n + base[D - 1];
                    double s2 = 0.0;
                    for (int t2 = 0; t2 < W; ++t2) s2 += phi[D - 1][t2] * __ldg(&row[t2]);
                    s1 += phi[1][t1] * s2;
                }
                acc += phi[0][t0] * s1;
            }
        }
        t[j] = acc;
    }
}

// d = 1 (c1): one thread per (node, tap) for the spread and one warp per node for the interp,
// so the 2m window evaluations (sqrt + sinh each) of a node run in parallel instead of in one
// thread's dependent sequence (the d = 1 problems are small and latency-bound).
__global__ void spread_d1_kernel(const double* __restrict__ u, long long count, const double* __restrict__ w,
                                 Window win, const GridAcc ga) {
    const int W = 2 * win.m;
    const double gscale = grid_scale(ga);
    const long long total = count * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long j = i / W;
        const int t = (int)(i - j * W);
        const double uj = u[j], c = floor(uj);
        const double phi = kb_phi(uj - c + (double)(win.m - 1 - t), win);
        grid_add<1>(ga, gscale, (int)c - win.m + 1 + t, 0, 0, w[j] * phi);
    }
}

// d = 1 spread privatised per CTA: 256 consecutive sorted nodes (position- or tile-sorted, so
// they cover a short interval) accumulate their 2m taps into a shared-memory window of the grid,
// then the window's nonzero cells are added to the grid once. Deterministic mode keeps the
// fixed-point words in shared memory (integer adds: the totals do not depend on order); a CTA
// whose window exceeds kD1Win cells adds straight to the grid.
constexpr int kD1Nodes = 256, kD1Win = 1024;
__global__ void __launch_bounds__(kD1Nodes) spread_d1_win_kernel(const double* __restrict__ u, long long count,
                                                                 const double* __restrict__ w, Window win,
                                                                 const GridAcc ga, int chunk) {
    __shared__ unsigned long long sacc[2 * kD1Win];   // (hi, lo) per cell, or the FP64 sum in word 0
    __shared__ int wlo_s, whi_s;
    const int W = 2 * win.m;
    const long long j0 = (long long)blockIdx.x * chunk;
    const int cnt = (int)min((long long)chunk, count - j0);
    const double gscale = grid_scale(ga);
    // window [min floor(u) - m + 1, max floor(u) + m] over the chunk
    int c = INT_MAX, cmax = INT_MIN;
    if ((int)threadIdx.x < cnt) { c = (int)floor(u[j0 + threadIdx.x]); cmax = c; }
    const int lo = __reduce_min_sync(0xffffffffu, c), hi = __reduce_max_sync(0xffffffffu, cmax);
    if (threadIdx.x == 0) { wlo_s = INT_MAX; whi_s = INT_MIN; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { atomicMin(&wlo_s, lo); atomicMax(&whi_s, hi); }
    __syncthreads();
    const int wlo = wlo_s - win.m + 1, wn = whi_s + win.m - wlo + 1;
    const bool priv = wn <= kD1Win;
    if (priv) {
        for (int k = threadIdx.x; k < 2 * wn; k += blockDim.x) sacc[k] = 0ULL;
        __syncthreads();
    }
    double* sdbl = reinterpret_cast<double*>(sacc);
    for (int p = threadIdx.x; p < cnt * W; p += blockDim.x) {
        const int jj = p / W, t = p - jj * W;
        const double uj = u[j0 + jj], cj = floor(uj);
        const double v = w[j0 + jj] * kb_phi(uj - cj + (double)(win.m - 1 - t), win);
        const int x = (int)cj - win.m + 1 + t;
        if (!priv) {
            grid_add<1>(ga, gscale, x, 0, 0, v);
        } else if (ga.acc) {
            unsigned long long h, l;
            fixed_words(v, gscale, h, l);
            atomicAdd(&sacc[2 * (x - wlo)], h);
            atomicAdd(&sacc[2 * (x - wlo) + 1], l);
        } else {
            atomicAdd(&sdbl[2 * (x - wlo)], v);
        }
    }
    if (!priv) return;
    __syncthreads();
    for (int k = threadIdx.x; k < wn; k += blockDim.x) {
        const int x = wlo + k;
        if (ga.acc) {
            const unsigned long long h = sacc[2 * k], l = sacc[2 * k + 1];
            if (h | l) {
                const long long i = x - ga.lo[0];
                atomicAdd(&ga.acc[2 * i], h);
                atomicAdd(&ga.acc[2 * i + 1], l);
            }
        } else if (sdbl[2 * k] != 0.0) {
            atomicAdd(&ga.grid[x], sdbl[2 * k]);
        }
    }
}

__global__ void interp_d1_kernel(const double* __restrict__ u, long long count, Window win,
                                 const double* __restrict__ grid, double* __restrict__ t_out, const FusedUpd fu) {
    const int W = 2 * win.m, lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; j < count; j += nw) {
        const double uj = u[j], c = floor(uj);
        double v = 0.0;
        for (int t = lane; t < W; t += 32)
            v += kb_phi(uj - c + (double)(win.m - 1 - t), win) * __ldg(&grid[(long long)c - win.m + 1 + t]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) emit_t(t_out, fu, j, v);
    }
}

inline int v1_grid(long long count) {
    long long g = (count + 127) / 128;
    if (g > 148LL * 32) g = 148LL * 32;
    return (int)(g < 1 ? 1 : g);
}

template <typename K>
inline int persistent_grid(K kernel, int threads, size_t smem, int nitems) {
    static_assert(sizeof(K) > 0, "");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int g = 148 * per_sm;
    return nitems < g ? (nitems < 1 ? 1 : nitems) : g;
}

template <int W>
inline int spread3_launch(Plan& P, const NodeSet& S, const double* w, const GridAcc& ga, cudaStream_t s) {
    using C = Spread3Cfg<W>;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(spread3_v2_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    }
    const int g = persistent_grid(spread3_v2_kernel<W>, C::NT, C::SMEM_BYTES, S.nitems);
    spread3_v2_kernel<W><<<g, C::NT, C::SMEM_BYTES, s>>>((const TileItem*)S.items, S.nitems, S.u, w, S.count,
                                                         ga, P.tiles_per_axis, *(const WinPoly*)P.winpoly);
    return SK_OK;
}

template <int W>
inline int interp3_launch(Plan& P, const NodeSet& S, const double* grid, double* t, cudaStream_t s) {
    using C = Interp3Cfg<W>;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(interp3_v2_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    }
    const int g = persistent_grid(interp3_v2_kernel<W>, C::NT, C::SMEM_BYTES, S.nitems);
    interp3_v2_kernel<W><<<g, C::NT, C::SMEM_BYTES, s>>>((const TileItem*)S.items, S.nitems, S.u, S.count, grid,
                                                          P.n, P.tiles_per_axis, *(const WinPoly*)P.winpoly, t);
    return SK_OK;
}

// Plan time (DMMA path): tabulate the d x 2m window taps of every node, [node][axis][2m].
inline int taps_dispatch(Plan& P, NodeSet& S, cudaStream_t s) {
    if (S.count <= 0) return SK_OK;
    const WinPoly& wp = *(const WinPoly*)P.winpoly;
    long long g = (S.count + 127) / 128;
    if (g > 148LL * 16) g = 148LL * 16;
    if (P.d == 3) taps_precompute_kernel<3, 12><<<(int)g, 128, 0, s>>>(S.u, S.count, wp, S.taps);
    else taps_precompute_kernel<2, 16><<<(int)g, 128, 0, s>>>(S.u, S.count, wp, S.taps);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("taps: ") + cudaGetErrorString(e));
    return SK_OK;
}

inline int spread_dispatch(Plan& P, const NodeSet& S, const double* w, const GridAcc& ga, cudaStream_t s) {
    if (P.dmma && P.d == 2) {
        using C = Spread2Cfg;
        static std::atomic<unsigned long long> attr{0};
        if (first_on_device(attr)) {
            cudaFuncSetAttribute(spread2_dmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
            cudaFuncSetAttribute(spread2_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
        }
        if (S.nsitems > 0) {
            // small sets (c2, images up to 256^2): one item per CTA; larger: one per warp
            // (measured: img512, c4 lose 15-35 % in the CTA form; SK_SPREAD2_CTA_NODES overrides)
            static const long long cta_nodes = getenv("SK_SPREAD2_CTA_NODES") ? atoll(getenv("SK_SPREAD2_CTA_NODES"))
                                                                               : kSpread2CtaNodes;
            const bool cta = S.count <= cta_nodes;
            const auto kern = cta ? spread2_dmma_kernel<true> : spread2_dmma_kernel<false>;
            const int g = persistent_grid(kern, C::NT, C::SMEM_BYTES, cta ? S.nsitems : (S.nsitems + C::NWARP - 1) / C::NWARP);
            const cudaError_t le = launch_pdl(kern, g, C::NT, C::SMEM_BYTES, s, (const SpreadItem*)S.sitems,
                                              S.nsitems, (const CellBatch*)S.segs, S.taps, w, ga);
            count_launch();
            if (le != cudaSuccess) return set_error(SK_ECUDA, std::string("spread2_dmma: ") + cudaGetErrorString(le));
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("spread2_dmma: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.dmma) {   // d = 3, 2 m_w = 12: the padded DMMA spread on TMA-fed warp pairs
        static std::atomic<unsigned long long> attr{0};
        if (first_on_device(attr)) {
            cudaFuncSetAttribute(spread3_tmapad_kernel<kSegTmaPMax, kSparsePairs, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpreadTPCfgSparse::SMEM_BYTES);
            cudaFuncSetAttribute(spread3_tmapad_kernel<kSegTmaPMax, kSparsePairs, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpreadTPCfgSparse::SMEM_BYTES);
            cudaFuncSetAttribute(spread3_tmapad_kernel<kSegTmaPDense, 2, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpreadTPCfgDense::SMEM_BYTES);
            cudaFuncSetAttribute(spread3_t28_kernel<kSegTmaPMax, kSparsePairs>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpreadTPCfgSparse::SMEM_BYTES);
            cudaFuncSetAttribute(spread3_t28_kernel<kSegTmaPDense, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpreadTPCfgDense::SMEM_BYTES);
        }
        const bool pipe = SK_SPREAD3_PIPE && SK_SPREAD3_T28 && P.spread_pipe;
        if (S.nsitems > 0) {
            const auto kern = S.seg_dense ? (pipe ? spread3_t28_kernel<kSegTmaPDense, 2>
                                                  : spread3_tmapad_kernel<kSegTmaPDense, 2, false>)
                              : (S.xpairs ? spread3_tmapad_kernel<kSegTmaPMax, kSparsePairs, true>
                                          : (pipe ? spread3_t28_kernel<kSegTmaPMax, kSparsePairs>
                                                  : spread3_tmapad_kernel<kSegTmaPMax, kSparsePairs, false>));
            const int np = S.seg_dense ? SpreadTPCfgDense::NPAIR : SpreadTPCfgSparse::NPAIR;
            const int nt = S.seg_dense ? SpreadTPCfgDense::NT : SpreadTPCfgSparse::NT;
            const size_t sm = S.seg_dense ? SpreadTPCfgDense::SMEM_BYTES : SpreadTPCfgSparse::SMEM_BYTES;
            const int g = persistent_grid(kern, nt, sm, (S.nsitems + np - 1) / np);
            const cudaError_t le = launch_pdl(kern, g, nt, sm, s, (const SpreadItem*)S.sitems, S.nsitems,
                                              (const CellBatch*)S.segs, S.taps, w, ga);
            count_launch();
            if (le != cudaSuccess) return set_error(SK_ECUDA, std::string("spread3_tmapad: ") + cudaGetErrorString(le));
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("spread3_tmapad: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.tiled && P.d == 3) {
        if (S.nitems > 0) {
            if (P.win.m == 6) spread3_launch<12>(P, S, w, ga, s);
            else spread3_launch<16>(P, S, w, ga, s);
            count_launch();
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("spread3: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.d == 1) {
        static const bool d1_flat = getenv("SK_SPREAD_D1_FLAT") != nullptr;
        if (d1_flat || P.win.m * 2 > kD1Win / 4)
            spread_d1_kernel<<<v1_grid(S.count * 2 * P.win.m), 128, 0, s>>>(S.u, S.count, w, P.win, ga);
        else
        {
            // nodes per CTA: at least ~2 CTAs per SM for small sets, at most kD1Nodes
            const long long chunk = std::max(16LL, std::min((long long)kD1Nodes, S.count / (2 * 148)));
            spread_d1_win_kernel<<<(unsigned)((S.count + chunk - 1) / chunk), kD1Nodes, 0, s>>>(
                S.u, S.count, w, P.win, ga, (int)chunk);
        }
        count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("spread_d1: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    const int g = v1_grid(S.count);
    switch (P.d) {
        case 2: spread_v1_kernel<2><<<g, 128, 0, s>>>(S.u, S.count, w, P.win, ga); break;
        default: spread_v1_kernel<3><<<g, 128, 0, s>>>(S.u, S.count, w, P.win, ga); break;
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("spread: ") + cudaGetErrorString(e));
    return SK_OK;
}

inline int interp_dispatch(Plan& P, const NodeSet& S, const double* grid, double* t, cudaStream_t s,
                           const FusedUpd& fu) {
    if (P.dmma && P.d == 2) {
        using C = Interp2Cfg;
        static std::atomic<unsigned long long> attr{0};
        if (first_on_device(attr)) {
            cudaFuncSetAttribute(interp2_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
        }
        if (S.nbatches > 0) {
            const int g = persistent_grid(interp2_dmma_kernel, C::NT, C::SMEM_BYTES, (S.nbatches + C::NWARP - 1) / C::NWARP);
            const cudaError_t le = launch_pdl(interp2_dmma_kernel, g, C::NT, C::SMEM_BYTES, s,
                                              (const CellBatch*)S.batches, S.nbatches, S.taps, grid, P.n, t, fu);
            count_launch();
            if (le != cudaSuccess) return set_error(SK_ECUDA, std::string("interp2_dmma: ") + cudaGetErrorString(le));
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("interp2_dmma: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.dmma) {
        using C = InterpDCfg;
        static std::atomic<unsigned long long> attr{0};
        if (first_on_device(attr)) {
            cudaFuncSetAttribute(interp3_dmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
            cudaFuncSetAttribute(interp3_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
        }
        if (S.nbatches > 0) {
            // stage grid blocks when cells average >= 1.5 batches (32 nodes each)
            const bool stage = 2LL * S.nbatches >= 3LL * S.ncells;
            const auto kern = stage ? interp3_dmma_kernel<true> : interp3_dmma_kernel<false>;
            const size_t sm = stage ? C::SMEM_BYTES : C::SMEM_BYTES_NOSTAGE;
            const int g = persistent_grid(kern, C::NT, sm, (S.nbatches + C::NWARP - 1) / C::NWARP);
            const cudaError_t le = launch_pdl(kern, g, C::NT, sm, s, (const CellBatch*)S.batches, S.nbatches, S.taps,
                                              grid, P.n, t, fu);
            count_launch();
            if (le != cudaSuccess) return set_error(SK_ECUDA, std::string("interp3_dmma: ") + cudaGetErrorString(le));
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("interp3_dmma: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.tiled && P.d == 3) {
        if (S.nitems > 0) {
            if (P.win.m == 6) interp3_launch<12>(P, S, grid, t, s);
            else interp3_launch<16>(P, S, grid, t, s);
            count_launch();
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("interp3: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    if (P.d == 1) {
        interp_d1_kernel<<<v1_grid(S.count * 32), 128, 0, s>>>(S.u, S.count, P.win, grid, t, fu);
        count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("interp_d1: ") + cudaGetErrorString(e));
        return SK_OK;
    }
    const int g = v1_grid(S.count);
    switch (P.d) {
        case 1: interp_v1_kernel<1><<<g, 128, 0, s>>>(S.u, S.count, P.win, P.n, grid, t); break;
        case 2: interp_v1_kernel<2><<<g, 128, 0, s>>>(S.u, S.count, P.win, P.n, grid, t); break;
        default: interp_v1_kernel<3><<<g, 128, 0, s>>>(S.u, S.count, P.win, P.n, grid, t); break;
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SK_ECUDA, std::string("interp: ") + cudaGetErrorString(e));
    return SK_OK;
}

}  // namespace sk
