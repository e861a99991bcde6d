// kernels.cu -- plan-time and per-apply CUDA kernels of libsk_nfft (sm_100a).
//
// Stages (PAPER.md P:Lx):
//   bbox / scale_key   a0: geometry, torus scaling, tile keys   (reading Q6)
//   sample / band      a1: b_k of the regularised kernel and the multiplier D_k
//   spread             a2: adjoint-NFFT gridding (inner sum of Eq. (fastsum))
//   multiply           a5: spectrum x D_k on the N-band (x b_k, window deconvolution), 0 elsewhere
//   interp             a7: NFFT interpolation at the targets (outer sum of Eq. (fastsum))
//   update             a7: fused marginal-scaling update alpha = p / t (Alg. 2)
//   reductions         a8: deterministic two-pass block reductions
#include <cub/cub.cuh>
#include <math.h>

#include "sk_internal.cuh"
#include "window.cuh"
#include "spread_interp.cuh"

namespace sk {

static inline int grid_for(long long count, int block) {
    long long g = (count + block - 1) / block;
    const long long cap = 148LL * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

#define SK_LAUNCH_CHECK()                                                               \
    do {                                                                                \
        count_launch();                                                                 \
        cudaError_t e_ = cudaGetLastError();                                            \
        if (e_ != cudaSuccess) return set_error(SK_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------------ block reduce helpers
template <int BS>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < BS / 32; ++i) r += sh[i];
    return r;  // valid in thread 0
}
template <int BS>
__device__ __forceinline__ double block_min(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = INFINITY;
    if (threadIdx.x == 0)
        for (int i = 0; i < BS / 32; ++i) r = fmin(r, sh[i]);
    return r;
}
template <int BS>
__device__ __forceinline__ double block_max(double v, double* sh) {
    return -block_min<BS>(-v, sh);
}

// ------------------------------------------------------------------ a0: bbox
constexpr int kRedBlock = 256;

__global__ void bbox_kernel(const double* __restrict__ pts, long long count, int d,
                            double* __restrict__ partial) {
    __shared__ double sh[kRedBlock / 32];
    double mn[kMaxD], mx[kMaxD];
    for (int a = 0; a < kMaxD; ++a) { mn[a] = INFINITY; mx[a] = -INFINITY; }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        for (int a = 0; a < d; ++a) {
            double v = pts[i * d + a];
            mn[a] = fmin(mn[a], v);
            mx[a] = fmax(mx[a], v);
        }
    for (int a = 0; a < d; ++a) {
        double r0 = block_min<kRedBlock>(mn[a], sh);
        if (threadIdx.x == 0) partial[blockIdx.x * 2 * d + a] = r0;
        double r1 = block_max<kRedBlock>(mx[a], sh);
        if (threadIdx.x == 0) partial[blockIdx.x * 2 * d + d + a] = r1;
    }
}

__global__ void bbox_final(const double* __restrict__ partial, int nparts, int d,
                           double* __restrict__ out) {
    __shared__ double sh[kRedBlock / 32];
    for (int a = 0; a < d; ++a) {
        double mn = INFINITY, mx = -INFINITY;
        for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
            mn = fmin(mn, partial[i * 2 * d + a]);
            mx = fmax(mx, partial[i * 2 * d + d + a]);
        }
        double r0 = block_min<kRedBlock>(mn, sh);
        double r1 = block_max<kRedBlock>(mx, sh);
        if (threadIdx.x == 0) {
            // combine with what is already in out (a previous point set)
            out[a] = fmin(out[a], r0);
            out[d + a] = fmax(out[d + a], r1);
        }
    }
}

int launch_bbox(const double* pts, long long count, int d, double* out_minmax, cudaStream_t s) {
    if (count <= 0) return SK_OK;
    int g = grid_for(count, kRedBlock);
    if (g > 1024) g = 1024;
    double* part = nullptr;
    SK_TRY(dev_alloc((void**)&part, sizeof(double) * 2 * d * g, s));
    bbox_kernel<<<g, kRedBlock, 0, s>>>(pts, count, d, part);
    SK_LAUNCH_CHECK();
    bbox_final<<<1, kRedBlock, 0, s>>>(part, g, d, out_minmax);
    SK_LAUNCH_CHECK();
    dev_free(part, s);
    return SK_OK;
}

// ------------------------------------------------------------------ a0: scale + key
struct ScaleParams {
    double centre[kMaxD];
    double rho, n, r2max;
    int d, T, tiles_per_axis;
    int cell_minor;   // 1: key = tile * T^d + cell-within-tile index: nodes sorted by cell
    int xminor;       // cell-within-tile digits with x least significant (d = 3 spread x-pairs)
    int Td;           // T^d
    int fine_shift;   // d = 1 near field: key = floor(u 2^fine_shift) (position order), 0 = off
    int fine_max;     // largest fine key: tiles_per_axis * T * 2^fine_shift - 1
};

// position key of a d = 1 node (the sort key and the near-field range search use this one
// definition, so the binary search below sees exactly the sorted order)
__device__ __forceinline__ int fine_key(double u, int shift, int kmax) {
    const double f = floor(ldexp(u, shift));
    return f < 0.0 ? 0 : (f > (double)kmax ? kmax : (int)f);
}

// x' = rho (x - centre), u = n (x' + 1/2): the one definition both the key and the gather use
// (bit-identical u in both kernels)
__device__ __forceinline__ double scaled_x(const ScaleParams& sp, double x, int a) {
    return sp.rho * (x - sp.centre[a]);
}
__device__ __forceinline__ double grid_u(const ScaleParams& sp, double xs) { return sp.n * (xs + 0.5); }

__global__ void scale_key_kernel(const double* __restrict__ pts, long long count, ScaleParams sp,
                                 int* __restrict__ key, int* __restrict__ idx, int* __restrict__ bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        double r2 = 0.0;
        int k = 0, sub = 0;
        bool ok = true;
        for (int a = 0; a < sp.d; ++a) {
            const double xs = scaled_x(sp, pts[i * sp.d + a], a);
            ok = ok && isfinite(xs);
            r2 += xs * xs;
            const double u = grid_u(sp, xs);
            int c = (int)floor(u);
            int tc = c / sp.T;
            tc = tc < 0 ? 0 : (tc >= sp.tiles_per_axis ? sp.tiles_per_axis - 1 : tc);
            k = k * sp.tiles_per_axis + tc;
            if (sp.xminor) {
                int mul = 1;
                for (int q = 0; q < a; ++q) mul *= sp.T;
                sub += (c - tc * sp.T) * mul;
            } else {
                sub = sub * sp.T + (c - tc * sp.T);
            }
        }
        if (!ok || !(r2 <= sp.r2max)) atomicMin(bad, (int)i);
        key[i] = sp.fine_shift ? fine_key(grid_u(sp, scaled_x(sp, pts[i], 0)), sp.fine_shift, sp.fine_max)
                               : (sp.cell_minor ? k * sp.Td + sub : k);
        idx[i] = (int)i;
    }
}

static ScaleParams scale_params(const Plan& P) {
    ScaleParams sp;
    for (int a = 0; a < kMaxD; ++a) sp.centre[a] = P.centre[a];
    sp.rho = P.rho;
    sp.n = (double)P.n;
    const double R = 0.5 * P.L;
    sp.r2max = R * R * (1.0 + 1e-12);
    sp.d = P.d;
    sp.T = P.tile_cells;
    sp.tiles_per_axis = P.tiles_per_axis;
    sp.cell_minor = (P.dmma || P.near_cell_sort) ? 1 : 0;
    sp.xminor = P.spread_xpairs ? 1 : 0;
    sp.Td = 1;
    for (int a = 0; a < P.d; ++a) sp.Td *= P.tile_cells;
    sp.fine_shift = P.fine_shift;
    sp.fine_max = (int)(((long long)P.tiles_per_axis * P.tile_cells << P.fine_shift) - 1);
    return sp;
}

// fine (position, d = 1) or (tile, cell) keys -> tile index, in place, for tile_offsets
__global__ void key_to_tile_kernel(int* __restrict__ key, long long count, int shift, int T, int tpa, int Td) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x)
        key[k] = shift ? min(tpa - 1, (key[k] >> shift) / T) : key[k] / Td;
}

int launch_key_to_tile(Plan& P, int* key, long long count, cudaStream_t s) {
    if (count <= 0) return SK_OK;
    int Td = 1;
    for (int a = 0; a < P.d; ++a) Td *= P.tile_cells;
    key_to_tile_kernel<<<grid_for(count, 256), 256, 0, s>>>(key, count, P.fine_shift, P.tile_cells,
                                                            P.tiles_per_axis, Td);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

int launch_scale_key(Plan& P, const double* pts, long long count, int* key, int* idx, int* bad,
                     cudaStream_t s) {
    if (count <= 0) return SK_OK;
    const ScaleParams sp = scale_params(P);
    scale_key_kernel<<<grid_for(count, 256), 256, 0, s>>>(pts, count, sp, key, idx, bad);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// sorted SoA grid coordinates: gather the caller's row-major point (d contiguous doubles, one
// or two sectors) and rescale it, instead of gathering d scattered doubles of a scaled copy
// (ncu: the scattered gather moved 15x its useful bytes)
__global__ void gather_coords_kernel(const double* __restrict__ pts, const int* __restrict__ perm,
                                     long long count, ScaleParams sp, double* __restrict__ u_sorted) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        const long long i = perm[k];
        for (int a = 0; a < sp.d; ++a) u_sorted[a * count + k] = grid_u(sp, scaled_x(sp, pts[i * sp.d + a], a));
    }
}

int launch_gather_coords(Plan& P, const double* pts, const int* perm, long long count, double* u_sorted,
                         cudaStream_t s) {
    if (count <= 0) return SK_OK;
    const ScaleParams sp = scale_params(P);
    gather_coords_kernel<<<grid_for(count, 256), 256, 0, s>>>(pts, perm, count, sp, u_sorted);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void tile_offsets_kernel(const int* __restrict__ keys, long long count, int ntiles,
                                    int* __restrict__ start) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= count;
         k += (long long)gridDim.x * blockDim.x) {
        int prev = (k == 0) ? -1 : keys[k - 1];
        int cur = (k == count) ? ntiles : keys[k];
        for (int t = prev + 1; t <= cur; ++t) start[t] = (int)k;
    }
}

int launch_tile_offsets(const int* sorted_keys, long long count, int ntiles, int* tile_start,
                        cudaStream_t s) {
    tile_offsets_kernel<<<grid_for(count + 1, 256), 256, 0, s>>>(sorted_keys, count, ntiles, tile_start);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ permutations / vectors
__global__ void permute_in_kernel(const double* __restrict__ src, const int* __restrict__ perm,
                                  long long count, double* __restrict__ dst, unsigned* __restrict__ slot) {
    unsigned mx = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        const double v = src[perm[k]];
        dst[k] = v;
        mx = max(mx, absmax_hi(v));
    }
    if (slot) note_absmax(slot, mx);
}
__global__ void permute_out_kernel(const double* __restrict__ src, const int* __restrict__ perm,
                                   long long count, double* __restrict__ dst) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x)
        dst[perm[k]] = src[k];
}
unsigned* wslot(Plan& P, int k) { return P.det_wmax ? P.det_wmax + k : nullptr; }

int launch_permute_in(const double* src, const int* perm, long long count, double* dst, cudaStream_t s,
                      unsigned* slot) {
    if (slot) SK_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned), s));
    if (count <= 0) return SK_OK;
    permute_in_kernel<<<grid_for(count, 256), 256, 0, s>>>(src, perm, count, dst, slot);
    SK_LAUNCH_CHECK();
    return SK_OK;
}
int launch_permute_out(const double* src, const int* perm, long long count, double* dst, cudaStream_t s) {
    if (count <= 0) return SK_OK;
    permute_out_kernel<<<grid_for(count, 256), 256, 0, s>>>(src, perm, count, dst);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void fill_kernel(double* p, long long count, double v) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x)
        p[k] = v;
}
// ------------------------------------------------------------------ a3: box pack / unpack
struct BoxParams { long long lo_off; long long stride[kMaxD]; int dims[kMaxD]; int d; };

template <int DIR>
__global__ void box_copy_kernel(double* __restrict__ grid, double* __restrict__ buf, long long total,
                                BoxParams bp) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long rest = i, off = bp.lo_off;
        for (int a = bp.d - 1; a >= 0; --a) {
            off += (rest % bp.dims[a]) * bp.stride[a];
            rest /= bp.dims[a];
        }
        if (DIR == 0) buf[i] = grid[off];
        else grid[off] = buf[i];
    }
}

int launch_box_copy(const Plan& P, double* grid, double* buf, int dir, cudaStream_t s) {
    if (P.box_size <= 0) return SK_OK;
    BoxParams bp;
    bp.d = P.d;
    long long st = 1;
    bp.lo_off = 0;
    for (int a = P.d - 1; a >= 0; --a) {
        bp.stride[a] = st;
        bp.dims[a] = P.box_n[a];
        bp.lo_off += (long long)P.box_lo[a] * st;
        st *= P.n;
    }
    const int g = grid_for(P.box_size, 256);
    if (dir == 0) box_copy_kernel<0><<<g, 256, 0, s>>>(grid, buf, P.box_size, bp);
    else box_copy_kernel<1><<<g, 256, 0, s>>>(grid, buf, P.box_size, bp);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

int launch_fill(double* p, long long count, double v, cudaStream_t s) {
    if (count <= 0) return SK_OK;
    fill_kernel<<<grid_for(count, 256), 256, 0, s>>>(p, count, v);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void scale_vec_kernel(double* p, long long count, const double* __restrict__ sc,
                                 unsigned* __restrict__ slot) {
    const double c = *sc;
    unsigned mx = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        const double v = p[k] * c;
        p[k] = v;
        mx = max(mx, absmax_hi(v));
    }
    if (slot) note_absmax(slot, mx);
}
// slot (deterministic spread): the bound slot of p, re-measured for the scaled vector
int launch_scale_vec(double* p, long long count, const double* scale_dev, cudaStream_t s, unsigned* slot) {
    if (slot) SK_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned), s));
    if (count <= 0) return SK_OK;
    scale_vec_kernel<<<grid_for(count, 256), 256, 0, s>>>(p, count, scale_dev, slot);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void scale_const_kernel(double* p, long long count, double c) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x)
        p[k] *= c;
}
int launch_scale_const(double* p, long long count, double c, cudaStream_t s) {
    if (count <= 0) return SK_OK;
    scale_const_kernel<<<grid_for(count, 256), 256, 0, s>>>(p, count, c);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ a8: reductions
// op 0: sum p_i log x_i;  op 1: sum x_i;  op 2: sum p_i x_i;  op 3: sum log x_i;  op 4: max x_i;
// op 5: min x_i
__global__ void reduce_kernel(const double* __restrict__ p, const double* __restrict__ x,
                              long long count, int op, double* __restrict__ partial) {
    __shared__ double sh[kRedBlock / 32];
    double acc = (op == 4) ? -INFINITY : (op == 5 ? INFINITY : 0.0);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        double xv = x[k];
        switch (op) {
            case 0: acc += p[k] * log(xv); break;
            case 1: acc += xv; break;
            case 2: acc += p[k] * xv; break;
            case 3: acc += log(xv); break;
            case 4: acc = fmax(acc, xv); break;
            default: acc = fmin(acc, xv); break;   // NaN-free inputs; a NaN weight fails the sum check
        }
    }
    double r = (op == 4) ? block_max<kRedBlock>(acc, sh)
                         : (op == 5 ? block_min<kRedBlock>(acc, sh) : block_sum<kRedBlock>(acc, sh));
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

// partial layout [nparts][nvals]; minmask bit v => slot v is a min (else sum); maxmask => max
__global__ void finalize_kernel(const double* __restrict__ partial, int nparts, int nvals,
                                unsigned minmask, unsigned maxmask, double* __restrict__ out) {
    __shared__ double sh[kRedBlock / 32];
    for (int v = 0; v < nvals; ++v) {
        const bool mn = (minmask >> v) & 1u, mx = (maxmask >> v) & 1u;
        double acc = mn ? INFINITY : (mx ? -INFINITY : 0.0);
        for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
            double t = partial[i * nvals + v];
            acc = mn ? fmin(acc, t) : (mx ? fmax(acc, t) : acc + t);
        }
        double r = mn ? block_min<kRedBlock>(acc, sh)
                      : (mx ? block_max<kRedBlock>(acc, sh) : block_sum<kRedBlock>(acc, sh));
        if (threadIdx.x == 0) out[v] = r;
    }
}

constexpr int kRedGrid = kUpdBlocks;  // 4 x 148 SMs

int launch_reduce_sum_log(const double* p, const double* x, long long count, double* out_dev,
                          int op, cudaStream_t s) {
    // out_dev must have room for kRedGrid partials at out_dev + 1 (scratch) -- we use a
    // static-size scratch owned by the caller: out_dev[0] = result, out_dev[1..] scratch.
    double* part = out_dev + 1;
    if (count <= 0) {
        SK_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), s));
        if (op == 4) launch_fill(out_dev, 1, -INFINITY, s);
        if (op == 5) launch_fill(out_dev, 1, INFINITY, s);
        return SK_OK;
    }
    reduce_kernel<<<kRedGrid, kRedBlock, 0, s>>>(p, x, count, op, part);
    SK_LAUNCH_CHECK();
    finalize_kernel<<<1, kRedBlock, 0, s>>>(part, kRedGrid, 1, op == 5 ? 1u : 0u, op == 4 ? 1u : 0u, out_dev);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void rescale_factor_kernel(double* r, int policy, double total) {
    r[0] = policy == 1 ? exp(-r[0] / total) : 1.0 / r[0];
}
int launch_rescale_factor(double* r, int policy, double total, cudaStream_t s) {
    rescale_factor_kernel<<<1, 1, 0, s>>>(r, policy, total);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

int launch_finalize_partials(const double* red, int nparts, int nvals, double* out, cudaStream_t s) {
    // slot 1 (min t) is a min; the others are sums
    finalize_kernel<<<1, kRedBlock, 0, s>>>(red, nparts, nvals, 0x2u, 0u, out);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ a7: fused update
// x_new = p / t; partial slots (kUpdVals per block): [0] sum |x_old t - p| (residual of the
// marginal that this update makes exact, Eq. (Error)), [1] min t, and with
// want_resid == 2 (diagnostics): [2] D_KL(p | x_old t) = sum p log(x_new /
// x_old) (the Lemma at), [3] sum p log x_new (f = 1 - [3]_u - [3]_v after a step).
__global__ void update_kernel(const double* __restrict__ t, const double* __restrict__ p,
                              double* __restrict__ x, long long count, int want_resid, int iter,
                              const int* __restrict__ iter_dev, unsigned long long* __restrict__ bad,
                              int rank, unsigned* __restrict__ xmax, double* __restrict__ partial) {
    __shared__ double sh[kRedBlock / 32];
    double res = 0.0, tmin = INFINITY, kl = 0.0, slog = 0.0;
    unsigned mx = 0;
    if (iter_dev) iter = *iter_dev;   // graph replay: iteration number from the device counter
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x) {
        const double tk = t[k], pk = p[k];
        const double xo = x[k], xn = pk / tk;
        if (want_resid) res += fabs(xo * tk - pk);
        if (want_resid == 2 && pk > 0.0) {
            kl += pk * log(xn / xo);
            slog += pk * log(xn);
        }
        tmin = fmin(tmin, tk);
        if (!(tk > 1e-300) || !isfinite(tk)) record_bad(bad, iter, rank, k);   // SK_ENONPOS (tau_pos = 1e-300)
        x[k] = xn;
        mx = max(mx, absmax_hi(xn));
    }
    if (xmax) note_absmax(xmax, mx);
    const double r0 = block_sum<kRedBlock>(res, sh);
    const double r1 = block_min<kRedBlock>(tmin, sh);
    const double r2 = want_resid == 2 ? block_sum<kRedBlock>(kl, sh) : 0.0;
    const double r3 = want_resid == 2 ? block_sum<kRedBlock>(slog, sh) : 0.0;
    if (threadIdx.x == 0) {
        partial[blockIdx.x * kUpdVals + 0] = r0;
        partial[blockIdx.x * kUpdVals + 1] = r1;
        partial[blockIdx.x * kUpdVals + 2] = r2;
        partial[blockIdx.x * kUpdVals + 3] = r3;
    }
}

int launch_update(Plan& P, int side, const double* t_sorted, const double* p_sorted,
                  double* x_sorted, int want_resid, int iter, const int* iter_dev, cudaStream_t s) {
    long long count = P.side[side].count;  // count == 0 still writes neutral partials
    update_kernel<<<kRedGrid, kRedBlock, 0, s>>>(t_sorted, p_sorted, x_sorted, count, want_resid,
                                                 iter, iter_dev, P.bad64 + side, P.ctx->rank,
                                                 wslot(P, side == 0 ? WSLOT_U : WSLOT_V), P.red);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void increment_kernel(int* p) { p[0] += 1; }

int launch_increment(int* counter_dev, cudaStream_t s) {
    increment_kernel<<<1, 1, 0, s>>>(counter_dev);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ a1: coefficients
struct KernelParams {
    double lam_p, rho2_inv, L, half, tscale;  // tscale = 1 / (1/2 - L)
    int d, M, kernel, kb_deg;
    double kb[32];                          // K_B coefficients in t = (r - L) / (1/2 - L)
    // r = 1 (NEXT-2): K(r) = exp(-lam' r) (c K with c = r / rho), K_I on r <= near_a
    int rpow, ki_n;
    double rho_inv, near_a;
    double ki[16];                          // K_I coefficients in (r / near_a)^2
};

__device__ __forceinline__ double radial(double r, const KernelParams& kp) {
    if (kp.rpow == 1) {
        const double k = exp(-kp.lam_p * r);
        return kp.kernel == 0 ? k : r * kp.rho_inv * k;
    }
    double r2 = r * r;
    double k = exp(-kp.lam_p * r2);
    return kp.kernel == 0 ? k : r2 * kp.rho2_inv * k;
}
__device__ __forceinline__ double ki_poly(double r, const double* c, int nc, double a) {
    const double t2 = (r / a) * (r / a);
    double acc = c[nc - 1];
    for (int i = nc - 2; i >= 0; --i) acc = acc * t2 + c[i];
    return acc;
}
__device__ __forceinline__ double kb_poly(double r, const KernelParams& kp) {
    double t = (r - kp.L) * kp.tscale;
    double acc = kp.kb[kp.kb_deg];
    for (int i = kp.kb_deg - 1; i >= 0; --i) acc = acc * t + kp.kb[i];
    return acc;
}

__global__ void sample_kernel_kernel(KernelParams kp, double* __restrict__ out, long long total) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        long long rest = e;
        double r2 = 0.0;
        for (int a = kp.d - 1; a >= 0; --a) {
            int q = (int)(rest % kp.M);
            rest /= kp.M;
            double xa = (double)q / kp.M - (q >= kp.M / 2 ? 1.0 : 0.0);
            r2 += xa * xa;
        }
        double r = sqrt(r2);
        double v;
        if (kp.rpow == 1 && r <= kp.near_a) v = ki_poly(r, kp.ki, kp.ki_n, kp.near_a);
        else if (r <= kp.L) v = radial(r, kp);
        else if (r <= kp.half) v = kb_poly(r, kp);
        else v = kb_poly(kp.half, kp);
        out[e] = v;
    }
}

int launch_sample_kernel(Plan& P, int kernel, int M, const double* kb_coef, int kb_deg,
                         double* out, cudaStream_t s) {
    KernelParams kp;
    kp.lam_p = P.lambda_p;
    kp.rho2_inv = 1.0 / (P.rho * P.rho);
    kp.L = P.L;
    kp.half = 0.5;
    kp.tscale = 1.0 / (0.5 - P.L);
    kp.d = P.d;
    kp.M = M;
    kp.kernel = kernel;
    kp.kb_deg = kb_deg;
    for (int i = 0; i <= kb_deg && i < 32; ++i) kp.kb[i] = kb_coef[i];
    kp.rpow = P.rpow;
    kp.rho_inv = 1.0 / P.rho;
    kp.near_a = P.near_a;
    kp.ki_n = P.ki_n;
    for (int i = 0; i < 16; ++i) kp.ki[i] = P.ki[kernel][i];
    long long total = 1;
    for (int a = 0; a < P.d; ++a) total *= M;
    sample_kernel_kernel<<<grid_for(total, 256), 256, 0, s>>>(kp, out, total);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

struct BandParams {
    int d, N, M, n, m;
    double beta, inv_Md;
};

__device__ __forceinline__ double kb_phihat(int k, const BandParams& bp) {
    double w = 2.0 * 3.141592653589793238462643 * (double)k / (double)bp.n;
    return cyl_bessel_i0((double)bp.m * sqrt(bp.beta * bp.beta - w * w));
}

// For every k in the full band {-N/2..N/2}^d: b_k = Re B[k] / M^d (B = unnormalised D2Z of
// the samples, half-complex in the last axis); write bk_full; for k_last >= 0 also write
// D_k = w_k b_k / prod_a phihat(k_a)^2 (w_k = prod 1/2 over |k_a| = N/2, reading Q8).
__global__ void band_kernel(BandParams bp, const cufftDoubleComplex* __restrict__ B,
                            double* __restrict__ bk_full, double* __restrict__ Dk) {
    const int nb = bp.N + 1, h = bp.N / 2;
    long long total = 1;
    for (int a = 0; a < bp.d; ++a) total *= nb;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int k[kMaxD];
        long long rest = e;
        for (int a = bp.d - 1; a >= 0; --a) { k[a] = (int)(rest % nb) - h; rest /= nb; }
        // b_k is real and even in each axis: read B at (k_0..k_{d-2}, |k_last|) with
        // conj symmetry folded on the last axis.
        int kl = k[bp.d - 1];
        int sgn_fold = kl < 0 ? -1 : 1;
        long long bidx = 0;
        for (int a = 0; a < bp.d - 1; ++a) {
            int ka = sgn_fold * k[a];
            int ia = ka < 0 ? ka + bp.M : ka;
            bidx = bidx * bp.M + ia;
        }
        bidx = bidx * (bp.M / 2 + 1) + (kl < 0 ? -kl : kl);
        double b = B[bidx].x * bp.inv_Md;
        bk_full[e] = b;
        if (kl >= 0) {
            double wgt = 1.0, ph = 1.0;
            for (int a = 0; a < bp.d; ++a) {
                if (k[a] == h || k[a] == -h) wgt *= 0.5;
                double p = kb_phihat(k[a], bp);
                ph *= p * p;
            }
            long long didx = 0;
            for (int a = 0; a < bp.d - 1; ++a) didx = didx * nb + (k[a] + h);
            didx = didx * (h + 1) + kl;
            Dk[didx] = wgt * b / ph;
        }
    }
}

int launch_band_coeffs(Plan& P, int kernel, int M, const cufftDoubleComplex* B, cudaStream_t s) {
    BandParams bp;
    bp.d = P.d;
    bp.N = P.N;
    bp.M = M;
    bp.n = P.n;
    bp.m = P.win.m;
    bp.beta = P.win.beta;
    double Md = 1.0;
    for (int a = 0; a < P.d; ++a) Md *= M;
    bp.inv_Md = 1.0 / Md;
    long long total = 1;
    for (int a = 0; a < P.d; ++a) total *= (P.N + 1);
    band_kernel<<<grid_for(total, 256), 256, 0, s>>>(bp, B, P.bk[kernel], P.D[kernel]);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// Plan-time accuracy estimate: the part of K~'s Fourier series that the N-band drops, measured
// on the (2N)^d sampling grid: sum |b_k| over the k of that grid with max_a |k_a| > N/2 (the
// +-N/2 modes count half, reading Q8), both Hermitian halves. |K~(x) - K~_N(x)| <= this sum.
__global__ void band_tail_kernel(BandParams bp, const cufftDoubleComplex* __restrict__ B,
                                 double* __restrict__ partial) {
    __shared__ double sh[kRedBlock / 32];
    const int M = bp.M, h = bp.N / 2, Mh = M / 2 + 1;
    long long total = Mh;
    for (int a = 0; a < bp.d - 1; ++a) total *= M;
    double acc = 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        long long rest = e;
        const int kl = (int)(rest % Mh);
        rest /= Mh;
        int kmax = kl;
        double wgt = (kl == h) ? 0.5 : 1.0;
        for (int a = 0; a < bp.d - 1; ++a) {
            int ka = (int)(rest % M);
            rest /= M;
            ka = ka >= M / 2 ? M - ka : ka;   // |k_a|
            kmax = max(kmax, ka);
            if (ka == h) wgt *= 0.5;
        }
        // the band keeps weight wgt of the entries on its faces and all of its interior
        const double drop = kmax > h ? 1.0 : (kmax == h ? 1.0 - wgt : 0.0);
        const double herm = (kl == 0 || kl == M / 2) ? 1.0 : 2.0;
        const cufftDoubleComplex b = B[e];
        acc += drop * herm * sqrt(b.x * b.x + b.y * b.y);
    }
    const double r = block_sum<kRedBlock>(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = r * bp.inv_Md;
}

int launch_band_tail(Plan& P, int M, const cufftDoubleComplex* B, double* out_dev, cudaStream_t s) {
    BandParams bp;
    bp.d = P.d;
    bp.N = P.N;
    bp.M = M;
    bp.n = P.n;
    bp.m = P.win.m;
    bp.beta = P.win.beta;
    double Md = 1.0;
    for (int a = 0; a < P.d; ++a) Md *= M;
    bp.inv_Md = 1.0 / Md;
    double* part = out_dev + 1;
    band_tail_kernel<<<kRedGrid, kRedBlock, 0, s>>>(bp, B, part);
    SK_LAUNCH_CHECK();
    finalize_kernel<<<1, kRedBlock, 0, s>>>(part, kRedGrid, 1, 0u, 0u, out_dev);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ r = 1 near field (NEXT-2)
// t_i += sum over sources j with |x'_i - y'_j| < a of w_j (K - K_I)(|x'_i - y'_j|): the part
// of the Laplace kernel that the inner regularisation K_I removed from the Fourier series
// ("we add a so called nearfield"). One thread per target (sorted order); candidate
// sources come from the source tiles (v1 path CSR) covering the target's cell +- near_cells.
struct NearParams {
    int d, n, T, tpa, R, ki_n, kernel;
    double a, lam_p, rho_inv, inv_n;
    double ki[16];
};

__global__ void nearfield_kernel(NearParams np, const double* __restrict__ ut, long long nt,
                                 const double* __restrict__ us, long long ns,
                                 const int* __restrict__ tile_start, const double* __restrict__ w,
                                 double* __restrict__ t) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nt;
         i += (long long)gridDim.x * blockDim.x) {
        double ui[kMaxD];
        int lo[kMaxD] = {0, 0, 0}, hi[kMaxD] = {0, 0, 0};
        for (int a = 0; a < np.d; ++a) {
            ui[a] = ut[a * nt + i];
            const int c = (int)floor(ui[a]);
            lo[a] = max(0, (c - np.R) / np.T);
            hi[a] = min(np.tpa - 1, (c + np.R + 1) / np.T);
        }
        const double a2 = np.a * np.a;
        double acc = 0.0;
        for (int t0 = lo[0]; t0 <= hi[0]; ++t0)
            for (int t1 = (np.d > 1 ? lo[1] : 0); t1 <= (np.d > 1 ? hi[1] : 0); ++t1)
                for (int t2 = (np.d > 2 ? lo[2] : 0); t2 <= (np.d > 2 ? hi[2] : 0); ++t2) {
                    int tile = t0;
                    if (np.d > 1) tile = tile * np.tpa + t1;
                    if (np.d > 2) tile = tile * np.tpa + t2;
                    for (int j = tile_start[tile]; j < tile_start[tile + 1]; ++j) {
                        double r2 = 0.0;
                        for (int a = 0; a < np.d; ++a) {
                            const double dx = (ui[a] - us[a * ns + j]) * np.inv_n;
                            r2 += dx * dx;
                        }
                        if (r2 < a2) {
                            const double r = sqrt(r2);
                            const double k = exp(-np.lam_p * r);
                            const double kk = np.kernel == 0 ? k : r * np.rho_inv * k;
                            acc += w[j] * (kk - ki_poly(r, np.ki, np.ki_n, np.a));
                        }
                    }
                }
        t[i] += acc;
    }
}

// d = 1 near field on position-sorted nodes (Plan::fine_shift), n-body style: a CTA takes 32
// consecutive targets (one per lane; they span a tiny interval) and the one contiguous source
// range within the radius of them, found by binary search on the same fine keys the sort used.
// Sources are staged in shared memory in blocks of kNearBlk; each of the 8 warps sums its 32
// targets against every 8th source of a block (latency hidden across warps even where the
// source density is high), and the 8 partial sums are added in warp order at the end (the
// result does not depend on scheduling).
// On the line |x - y| = +-(x - y), so exp(-lam' |x - y|) = g_i f_j (x >= y) or 1 / (g_i f_j)
// with g_i = exp(-lam' (x_i - c)), f_j = exp(lam' (y_j - c)) about the chunk's lowest target c:
// one exp per staged source and per target instead of one per pair. The exponents stay below
// lam' x (chunk span + radius), checked against kNearExpMax (else the per-pair exp).
// Per pair: a difference, a compare, a product and the K_I Horner polynomial.
constexpr int kNearBlk = 256, kNearWarps = 8, kNearKI = 8;
constexpr double kNearExpMax = 600.0;

// one warp's share of a staged block: its 32 x kNearTPL targets against sources warp,
// warp + 8, ... (each staged source read once per kNearTPL pairs: shared-memory loads were the
// co-bottleneck with one target per lane). Coordinates are in units of the radius a, so
// t2 = dx^2 = (r / a)^2 feeds the K_I Horner directly; the radius test (t2 < 1) and the side
// test (dx >= 0) read the high words as integers, off the FP64 pipe (t2 >= 0: hi < 0x3ff00000
// <=> t2 < 1). Out-of-radius pairs are masked, not branched. K_I has kNearKI coefficients,
// zero-padded at the top (exact in Horner: fma(0, t2, c) = c). Per pair: 12 FP64 instructions
// (14 for the c K kernel).
constexpr int kNearTPL = 2;
#ifndef SK_NEAR_MINB
#define SK_NEAR_MINB 2
#endif
template <int KERNEL, bool SEP>
__device__ __forceinline__ void near_block(const double2* __restrict__ syw, const double2* __restrict__ sff,
                                           int cnt, int warp, const double* xi, const double* gi,
                                           const double* igi, double lam_a, double r_scale, const double* ki,
                                           double* acc) {
#pragma unroll 2
    for (int k = warp; k < cnt; k += kNearWarps) {
        const double2 yw = syw[k];
        double2 ff;
        if (SEP) ff = sff[k];
#pragma unroll
        for (int e = 0; e < kNearTPL; ++e) {
            const double dx = xi[e] - yw.x;   // (x - y) / a
            const double t2 = dx * dx;
            const int dxh = __double2hiint(dx), t2h = __double2hiint(t2);
            double wk;   // w_j K(r)
            if (SEP) {
                const bool right = dxh >= 0;   // select the factors, then one product
                wk = (right ? gi[e] : igi[e]) * (right ? ff.x : ff.y);
            } else {
                wk = yw.y * exp(-lam_a * fabs(dx));
            }
            if (KERNEL == 1) wk *= fabs(dx) * r_scale;
            double q = ki[kNearKI - 1];
#pragma unroll
            for (int c = kNearKI - 2; c >= 0; --c) q = fma(q, t2, ki[c]);
            const double v = fma(-yw.y, q, wk);
            acc[e] += t2h < 0x3ff00000 ? v : 0.0;
        }
    }
}

template <int KERNEL>
__global__ void __launch_bounds__(kNearWarps * 32, SK_NEAR_MINB) nearfield_d1_kernel(
    NearParams np, const double* __restrict__ ut, long long nt, const double* __restrict__ us, long long ns,
    int shift, int kmax, const double* __restrict__ w, double* __restrict__ t) {
    constexpr int CH = 32 * kNearTPL;   // targets per CTA
    __shared__ double2 syw[kNearBlk], sff[kNearBlk];   // (y_j, w_j), (w_j f_j, w_j / f_j)
    __shared__ double part[kNearWarps][CH];
    __shared__ long long range[2];
    __shared__ double chunk_lo;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i0 = (long long)blockIdx.x * CH;
    const long long ilast = min(nt, i0 + CH) - 1;
    const double ag = np.a * (double)np.n;   // radius in grid units
    if (threadIdx.x == 0) {
        // targets sorted by fine key: the chunk's interval is [u(i0), u(ilast)] to within a key bin
        const double lo = fmin(ut[i0], ut[ilast]) - ldexp(1.0, -shift);
        const double hi = fmax(ut[i0], ut[ilast]) + ldexp(1.0, -shift);
        chunk_lo = lo;
        for (int side = 0; side < 2; ++side) {
            // side 0: first source with key >= key(lo - a); side 1: first with key > key(hi + a)
            const int kb = side == 0 ? fine_key(lo - ag, shift, kmax) : fine_key(hi + ag, shift, kmax);
            long long L = 0, R = ns;
            while (L < R) {
                const long long M = (L + R) >> 1;
                const int km = fine_key(us[M], shift, kmax);
                if (side == 0 ? km < kb : km <= kb) L = M + 1; else R = M;
            }
            range[side] = L;
        }
    }
    __syncthreads();
    const long long j0 = range[0], j1 = range[1];
    const double c = chunk_lo;
    const double lam_n = np.lam_p * np.inv_n;   // lam' per grid unit
    const double to_a = np.inv_n / np.a;        // grid units -> units of the radius
    double xi[kNearTPL], gi[kNearTPL], igi[kNearTPL], acc[kNearTPL];
    bool sep = j1 > j0 && lam_n * fmax(fabs(us[j1 - 1] - c), fabs(us[j0] - c)) < kNearExpMax;
#pragma unroll
    for (int e = 0; e < kNearTPL; ++e) {
        const long long i = i0 + e * 32 + lane;
        const double ui = i < nt ? ut[i] : c;
        sep = sep && lam_n * (ui - c) < kNearExpMax;
        xi[e] = ui * to_a;
        gi[e] = ui;
        acc[e] = 0.0;
    }
    // every exponent lam' |u - c| of this CTA below kNearExpMax (sources sorted: the ends bound it)
    const bool sep_all = __syncthreads_and(sep);
#pragma unroll
    for (int e = 0; e < kNearTPL; ++e) {
        gi[e] = sep_all ? exp(-lam_n * (gi[e] - c)) : 1.0;
        igi[e] = 1.0 / gi[e];
    }
    // K_I coefficients straight from the kernel parameters (constant-bank operands of the DFMAs;
    // Plan::ki is zero beyond ki_n)
    const double* ki = np.ki;
    for (long long jb = j0; jb < j1; jb += kNearBlk) {
        const int cnt = (int)min((long long)kNearBlk, j1 - jb);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
            const double uj = us[jb + k], wj = w[jb + k];
            syw[k] = make_double2(uj * to_a, wj);
            if (sep_all) {
                const double f = exp(lam_n * (uj - c));
                sff[k] = make_double2(wj * f, wj / f);
            }
        }
        __syncthreads();
        // r = a |dx| torus units, r / rho the caller's units (c K kernel)
        if (sep_all) near_block<KERNEL, true>(syw, sff, cnt, warp, xi, gi, igi, np.lam_p * np.a, np.a * np.rho_inv, ki, acc);
        else near_block<KERNEL, false>(syw, sff, cnt, warp, xi, gi, igi, np.lam_p * np.a, np.a * np.rho_inv, ki, acc);
    }
#pragma unroll
    for (int e = 0; e < kNearTPL; ++e) part[warp][e * 32 + lane] = acc[e];
    __syncthreads();
    if (threadIdx.x < CH && i0 + threadIdx.x < nt) {
        double sum = part[0][threadIdx.x];
        for (int q = 1; q < kNearWarps; ++q) sum += part[q][threadIdx.x];
        t[i0 + threadIdx.x] += sum;
    }
}

// d >= 2 near field (r = 1), one CTA per NearItem (<= 64 targets of a run of tiles along the last
// axis, 2 per lane): the source tiles within the radius of the item's tiles form (2 ceil(R / T) + 2)^(d-1) runs that
// are contiguous in sorted order (consecutive tiles along the last axis); the CTA streams their
// concatenation through shared memory in blocks of kNearBlk and each of the 8 warps sums its
// targets against every 8th staged source (partials added in warp order). Per pair in the
// ball: r = sqrt(t2) in units of the radius, exp(-lam' r) (no factoring off the line), the K_I
// Horner in t2; pairs outside the ball are skipped (divergent only near the ball's surface).
constexpr int kNearSegMax = 512;
template <int D, int KERNEL>
__global__ void __launch_bounds__(kNearWarps * 32, 2) nearfield_tiled_kernel(
    NearParams np, const NearItem* __restrict__ items, const double* __restrict__ ut, long long nt,
    const double* __restrict__ us, long long ns, const int* __restrict__ tile_start, const double* __restrict__ w,
    double* __restrict__ t) {
    __shared__ double sy[D][kNearBlk], sw[kNearBlk];
    __shared__ double part[kNearWarps][kNearChunk];
    __shared__ int seg_a[kNearSegMax], seg_pre[kNearSegMax + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const NearItem it = items[blockIdx.x];
    int tc[3] = {0, 0, 0}, te[3] = {0, 0, 0}, lo[3], hi[3];
    for (int a = D - 1, r = it.tile, r2 = it.tile_last; a >= 0; --a) {
        tc[a] = r % np.tpa; r /= np.tpa;
        te[a] = r2 % np.tpa; r2 /= np.tpa;
    }
    for (int a = 0; a < D; ++a) {
        // a target in tiles tc .. te reaches cells [tc T - R, (te + 1) T + R - 1]
        const int lc = tc[a] * np.T - np.R, hc = (te[a] + 1) * np.T + np.R - 1;
        lo[a] = lc <= 0 ? 0 : lc / np.T;
        hi[a] = min(np.tpa - 1, hc / np.T);
    }
    const int n0 = hi[0] - lo[0] + 1, n1 = D > 2 ? hi[1] - lo[1] + 1 : 1;
    const int ncand = n0 * n1;   // <= kNearSegMax (checked at launch)
    // segment k: tiles (lo0 + k / n1, lo1 + k % n1, lo_last .. hi_last), its length, then an
    // exclusive prefix over the lengths (block scans of 256 segments at a time)
    __shared__ int wsum[kNearWarps];
    int carry = 0;
    if (threadIdx.x == 0) seg_pre[0] = 0;
    for (int k0 = 0; k0 < ncand; k0 += kNearWarps * 32) {
        const int k = k0 + threadIdx.x;
        int len = 0;
        if (k < ncand) {
            const int t0 = lo[0] + k / n1, t1 = D > 2 ? lo[1] + k % n1 : 0;
            const int base = D == 2 ? t0 * np.tpa : (t0 * np.tpa + t1) * np.tpa;
            const int a0 = tile_start[base + lo[D - 1]], b0 = tile_start[base + hi[D - 1] + 1];
            seg_a[k] = a0;
            len = b0 - a0;
        }
        int v = len;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        __syncthreads();   // wsum of the previous round consumed
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        int off = carry, all = 0;
        for (int q = 0; q < kNearWarps; ++q) {
            if (q < warp) off += wsum[q];
            all += wsum[q];
        }
        if (k < ncand) seg_pre[k + 1] = off + v;
        carry += all;
    }
    __syncthreads();
    const int total = seg_pre[ncand];
    const double to_a = np.inv_n / np.a;   // grid units -> units of the radius
    double xi[2][D], acc[2] = {0.0, 0.0};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int k = e * 32 + lane;
#pragma unroll
        for (int a = 0; a < D; ++a) xi[e][a] = k < it.count ? ut[a * nt + it.start + k] * to_a : 1e300;
    }
    const double lam_a = np.lam_p * np.a, r_scale = np.a * np.rho_inv;
    const double* ki = np.ki;
    for (int p0 = 0; p0 < total; p0 += kNearBlk) {
        const int cnt = min(kNearBlk, total - p0);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
            const int p = p0 + k;
            int L = 0, R = ncand;   // last segment with seg_pre <= p
            while (R - L > 1) {
                const int M = (L + R) >> 1;
                if (seg_pre[M] <= p) L = M; else R = M;
            }
            const long long j = seg_a[L] + (p - seg_pre[L]);
#pragma unroll
            for (int a = 0; a < D; ++a) sy[a][k] = us[a * ns + j] * to_a;
            sw[k] = w[j];
        }
        __syncthreads();
        for (int k = warp; k < cnt; k += kNearWarps) {
            double yk[D];
#pragma unroll
            for (int a = 0; a < D; ++a) yk[a] = sy[a][k];
            const double wk = sw[k];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double t2 = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const double dx = xi[e][a] - yk[a];
                    t2 = fma(dx, dx, t2);
                }
                if (t2 < 1.0) {
                    const double r = sqrt(t2);   // |x - y| / a
                    double kv = wk * exp(-lam_a * r);
                    if (KERNEL == 1) kv *= r * r_scale;
                    double q = ki[kNearKI - 1];
#pragma unroll
                    for (int c = kNearKI - 2; c >= 0; --c) q = fma(q, t2, ki[c]);
                    acc[e] += fma(-wk, q, kv);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) part[warp][e * 32 + lane] = acc[e];
    __syncthreads();
    if ((int)threadIdx.x < it.count) {
        double sum = part[0][threadIdx.x];
        for (int q = 1; q < kNearWarps; ++q) sum += part[q][threadIdx.x];
        t[it.start + threadIdx.x] += sum;
    }
}

// Near-field sources across ranks (plan.cu, build_near_global): sort keys of gathered grid
// coordinates, the same keys a local side sorts by (d = 1 near field: position keys; otherwise
// the tile index -- the near-field kernels read sources per tile)
__global__ void near_key_kernel(const double* __restrict__ U, long long total, int d, int T, int tpa, int fine_shift,
                                int fine_max, int* __restrict__ key, int* __restrict__ idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int k = 0;
        if (fine_shift) {
            k = fine_key(U[i], fine_shift, fine_max);
        } else {
            for (int a = 0; a < d; ++a) {
                int tc = (int)floor(U[a * total + i]) / T;
                tc = tc < 0 ? 0 : (tc >= tpa ? tpa - 1 : tc);
                k = k * tpa + tc;
            }
        }
        key[i] = k;
        idx[i] = (int)i;
    }
}

int launch_near_keys(Plan& P, const double* U, long long total, int* key, int* idx, cudaStream_t s) {
    if (total <= 0) return SK_OK;
    const int fine_max = (int)(((long long)P.tiles_per_axis * P.tile_cells << P.fine_shift) - 1);
    near_key_kernel<<<grid_for(total, 256), 256, 0, s>>>(U, total, P.d, P.tile_cells, P.tiles_per_axis, P.fine_shift,
                                                          fine_max, key, idx);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

__global__ void gather_rows_kernel(const double* __restrict__ in, long long in_ld, const int* __restrict__ perm,
                                   long long count, int rows, double* __restrict__ out) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < count;
         j += (long long)gridDim.x * blockDim.x) {
        const long long pj = perm[j];
        for (int r = 0; r < rows; ++r) out[r * count + j] = in[r * in_ld + pj];
    }
}

int launch_gather_rows(const double* in, long long in_ld, const int* perm, long long count, int rows, double* out,
                       cudaStream_t s) {
    if (count <= 0) return SK_OK;
    gather_rows_kernel<<<grid_for(count, 256), 256, 0, s>>>(in, in_ld, perm, count, rows, out);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

int launch_nearfield(Plan& P, int src, int dst, int kernel, const double* w_sorted, double* t_sorted,
                     cudaStream_t s) {
    // across ranks the sources are every rank's nodes of the side (build_near_global), weights
    // gathered into their order by the caller
    NodeSet Sg;
    const NodeSet* Sp = &P.side[src];
    if (P.side[src].g_u) {
        Sg.u = P.side[src].g_u;
        Sg.count = P.side[src].g_total;
        Sg.tile_start = P.side[src].g_tile_start;
        Sp = &Sg;
    }
    const NodeSet& S = *Sp;
    const NodeSet& D = P.side[dst];
    if (D.count <= 0 || S.count <= 0) return SK_OK;
    NearParams np;
    np.d = P.d;
    np.n = P.n;
    np.T = P.tile_cells;
    np.tpa = P.tiles_per_axis;
    np.R = P.near_cells;
    np.ki_n = P.ki_n;
    np.kernel = kernel;
    np.a = P.near_a;
    np.lam_p = P.lambda_p;
    np.rho_inv = 1.0 / P.rho;
    np.inv_n = 1.0 / P.n;
    for (int i = 0; i < 16; ++i) np.ki[i] = P.ki[kernel][i];
    if (P.d == 1 && P.fine_shift) {
        const long long blocks = (D.count + 32 * kNearTPL - 1) / (32 * kNearTPL);
        const int kmax = (int)(((long long)P.tiles_per_axis * P.tile_cells << P.fine_shift) - 1);
        if (P.ki_n > kNearKI) return set_error(SK_EINVAL, "near field: more than 8 K_I coefficients");
        const auto kern = kernel == 0 ? nearfield_d1_kernel<0> : nearfield_d1_kernel<1>;
        kern<<<(unsigned)blocks, kNearWarps * 32, 0, s>>>(np, D.u, D.count, S.u, S.count, P.fine_shift, kmax,
                                                          w_sorted, t_sorted);
    } else {
        // d >= 2: the tiled kernel when the item's source runs fit its shared list
        const int span = 2 * ((P.near_cells + P.tile_cells - 1) / P.tile_cells) + 2;
        int runs = 1;
        for (int a = 0; a + 1 < P.d; ++a) runs *= span;
        static const bool v1 = getenv("SK_NEARFIELD_V1") != nullptr;
        if (!v1 && P.d >= 2 && D.n_near > 0 && runs <= kNearSegMax && P.ki_n <= kNearKI) {
            const NearItem* it = (const NearItem*)D.near_items;
            if (P.d == 2)
                (kernel == 0 ? nearfield_tiled_kernel<2, 0> : nearfield_tiled_kernel<2, 1>)
                    <<<D.n_near, kNearWarps * 32, 0, s>>>(np, it, D.u, D.count, S.u, S.count, S.tile_start, w_sorted, t_sorted);
            else
                (kernel == 0 ? nearfield_tiled_kernel<3, 0> : nearfield_tiled_kernel<3, 1>)
                    <<<D.n_near, kNearWarps * 32, 0, s>>>(np, it, D.u, D.count, S.u, S.count, S.tile_start, w_sorted, t_sorted);
        } else {
            nearfield_kernel<<<grid_for(D.count, 128), 128, 0, s>>>(np, D.u, D.count, S.u, S.count, S.tile_start,
                                                                    w_sorted, t_sorted);
        }
    }
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ a5: multiply
struct MulParams {
    int d, n, N;
    long long spec_size;
};

__global__ void multiply_kernel(MulParams mp, cufftDoubleComplex* __restrict__ spec,
                                const double* __restrict__ Dk) {
    const int hl = mp.n / 2 + 1, h = mp.N / 2, nb = mp.N + 1;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mp.spec_size;
         e += (long long)gridDim.x * blockDim.x) {
        int kl = (int)(e % hl);
        long long rest = e / hl;
        bool inband = kl <= h;
        long long didx = 0, mul = 1;
        // non-last axes, from axis d-2 down to 0
        for (int a = mp.d - 2; a >= 0; --a) {
            int ia = (int)(rest % mp.n);
            rest /= mp.n;
            int ka = ia <= mp.n / 2 ? ia : ia - mp.n;
            inband = inband && (ka >= -h && ka <= h);
            didx += (long long)(ka + h) * mul;
            mul *= nb;
        }
        cufftDoubleComplex z = spec[e];
        if (inband) {
            double D = Dk[didx * (h + 1) + kl];
            z.x *= D;
            z.y *= D;
        } else {
            z.x = 0.0;
            z.y = 0.0;
        }
        spec[e] = z;
    }
}

int launch_multiply(Plan& P, int kernel, cudaStream_t s) {
    MulParams mp{P.d, P.n, P.N, P.spec_size};
    multiply_kernel<<<grid_for(P.spec_size, 256), 256, 0, s>>>(mp, P.spec, P.D[kernel]);
    SK_LAUNCH_CHECK();
    return SK_OK;
}

// ------------------------------------------------------------------ a2 / a7: spread, interp
// Deterministic spread (GridAcc): max |w_j| bound of a source vector that no producer recorded
// (fastsum_apply / nfft_spread record theirs in permute_in): the slot must be zero on entry.
__global__ void absmax_kernel(const double* __restrict__ w, long long count, unsigned* __restrict__ slot) {
    unsigned mx = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
         k += (long long)gridDim.x * blockDim.x)
        mx = max(mx, absmax_hi(w[k]));
    note_absmax(slot, mx);
}

// Fixed-point box accumulator -> FP64 grid over the WHOLE grid (zeros outside the box, so no
// separate memset): X = hi 2^32 + lo exactly (carry of lo folded into hi), value = X 2^-S. Each
// accumulator word is cleared after it is read, and the last block to finish clears the source
// vector's bound slot, so the next spread starts from zero without another launch.
__global__ void grid_fix_convert_kernel(const GridAcc ga, int d, long long grid_size, unsigned* __restrict__ done,
                                        unsigned* __restrict__ slot) {
    const unsigned hi = *ga.wmax;
    const double inv = 1.0 / grid_scale(ga);
    const bool finite = isfinite(__longlong_as_double((long long)(((unsigned long long)hi << 32) | 0xffffffffULL)));
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < grid_size;
         gi += (long long)gridDim.x * blockDim.x) {
        long long rest = gi, bi = 0, mul = 1;
        bool in = true;
        for (int a = d - 1; a >= 0; --a) {
            const int c = (int)(rest % ga.n) - ga.lo[a];
            rest /= ga.n;
            in = in && c >= 0 && c < ga.bn[a];
            bi += (long long)c * mul;
            mul *= ga.bn[a];
        }
        double v = 0.0;
        if (in) {
            const long long hw = (long long)ga.acc[2 * bi];
            const unsigned long long lw = ga.acc[2 * bi + 1];
            ga.acc[2 * bi] = 0ULL;
            ga.acc[2 * bi + 1] = 0ULL;
            const long long H = hw + (long long)(lw >> 32);
            const double L = (double)(lw & 0xffffffffULL);
            v = finite ? fma((double)H, 4294967296.0, L) * inv : NAN;
        }
        ga.grid[gi] = v;
    }
    // every block has read the slot above; the last one to arrive clears it for the next producer
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
            *slot = 0u;
            *done = 0u;
        }
    }
}

int launch_spread(Plan& P, int side, const double* w_sorted, double* grid, cudaStream_t s, GridAcc* keep,
                  unsigned** keep_slot) {
    const NodeSet& S = P.side[side];
    if (S.count <= 0 || !P.deterministic) SK_CUDA(cudaMemsetAsync(grid, 0, sizeof(double) * P.grid_size, s));
    if (S.count <= 0) return SK_OK;
    GridAcc ga;
    ga.grid = grid;
    ga.n = P.n;
    ga.phi0d = P.phi0d;
    for (int a = 0; a < P.d; ++a) { ga.lo[a] = P.box_lo[a]; ga.bn[a] = P.box_n[a]; }
    unsigned* slot = nullptr;
    if (P.deterministic) {
        // the bound recorded by the vector's producer; otherwise measure it now
        slot = w_sorted == P.w_sorted ? wslot(P, WSLOT_W)
             : (w_sorted == P.u_s ? wslot(P, WSLOT_U) : (w_sorted == P.v_s ? wslot(P, WSLOT_V) : nullptr));
        if (!slot) {
            slot = wslot(P, WSLOT_TMP);
            SK_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned), s));
            absmax_kernel<<<grid_for(S.count, 256), 256, 0, s>>>(w_sorted, S.count, slot);
            SK_LAUNCH_CHECK();
        }
        ga.acc = P.det_acc;
        ga.wmax = slot;
    }
    SK_TRY(spread_dispatch(P, S, w_sorted, ga, s));
    if (keep) {
        *keep = ga;
        *keep_slot = slot;
        return SK_OK;
    }
    if (P.deterministic) {
        grid_fix_convert_kernel<<<grid_for(P.grid_size, 256), 256, 0, s>>>(ga, P.d, P.grid_size, P.det_wmax + kWSlots,
                                                                           slot);
        SK_LAUNCH_CHECK();
    }
    return SK_OK;
}

int launch_interp(Plan& P, int side, const double* grid, double* t_sorted, cudaStream_t s,
                  const FusedUpd& fu) {
    const NodeSet& S = P.side[side];
    if (S.count <= 0) return SK_OK;
    SK_TRY(interp_dispatch(P, S, grid, t_sorted, s, fu));
    return SK_OK;
}

int launch_taps(Plan& P, int side, cudaStream_t s) {
    return taps_dispatch(P, P.side[side], s);
}

}  // namespace sk
