// plan.cu -- fastsum plan (geometry, binning, kernel coefficients, FFT plans) and one
// fast-summation matvec on sorted data.
#include <cub/cub.cuh>
#include <math.h>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "sk_internal.cuh"
#include "tiled3.cuh"
#define SK_WORKLIST_ONLY
#include "dmma3.cuh"
#include "dmma2.cuh"
#undef SK_WORKLIST_ONLY
#include "winpoly.h"

namespace sk {

// ---------------------------------------------------------------- two-point Taylor K_B (host)
// Derivatives K^{(k)}(L), k < p, of the radial profile of
//   kernel 0: f(r) = exp(-a r^2)                 via physicists' Hermite polynomials
//             f^{(k)}(r) = (-sqrt(a))^k H_k(sqrt(a) r) exp(-a r^2)
//   kernel 1: g(r) = (r^2 / rho^2) f(r)          via Leibniz' rule
static void radial_derivs(double a, double rho, int kernel, double r, int p, double* out) {
    std::vector<double> f(p + 2), H(p + 2);
    const double sa = sqrt(a), z = sa * r, e = exp(-a * r * r);
    H[0] = 1.0;
    H[1] = 2.0 * z;
    for (int k = 1; k + 1 < p; ++k) H[k + 1] = 2.0 * z * H[k] - 2.0 * k * H[k - 1];
    double sak = 1.0;
    for (int k = 0; k < p; ++k) {
        f[k] = ((k & 1) ? -1.0 : 1.0) * sak * H[k] * e;
        sak *= sa;
    }
    for (int k = 0; k < p; ++k) {
        if (kernel == 0) {
            out[k] = f[k];
        } else {
            double v = r * r * f[k];
            if (k >= 1) v += 2.0 * k * r * f[k - 1];
            if (k >= 2) v += (double)k * (k - 1) * f[k - 2];
            out[k] = v / (rho * rho);
        }
    }
}

// r = 1 (NEXT-2): f(r) = P0(r) exp(-a r), P0 = 1 (kernel 0) or r / rho (kernel 1);
// f^{(k)} = P_k exp(-a r) with P_{k+1} = P_k' - a P_k (P_k of degree <= 1).
static void radial_derivs_r1(double a, double rho, int kernel, double r, int p, double* out) {
    double c0 = kernel == 0 ? 1.0 : 0.0, c1 = kernel == 0 ? 0.0 : 1.0 / rho;   // P = c0 + c1 r
    const double e = exp(-a * r);
    for (int k = 0; k < p; ++k) {
        out[k] = (c0 + c1 * r) * e;
        const double n0 = c1 - a * c0, n1 = -a * c1;
        c0 = n0;
        c1 = n1;
    }
}

static void radial_derivs_any(int rpow, double a, double rho, int kernel, double r, int p, double* out) {
    if (rpow == 1) radial_derivs_r1(a, rho, kernel, r, p, out);
    else radial_derivs(a, rho, kernel, r, p, out);
}

// Inner regularisation for r = 1 (NEXT-2): K_I(r) = sum_{i<p} c_i (r/a)^{2i} with
// K_I^{(k)}(a) = K^{(k)}(a), k < p (even, so smooth at 0). Dense p x p solve with partial
// pivoting on the host.
static int ki_coefficients(double lam_p, double rho, int kernel, double a, int p, std::vector<double>& c) {
    std::vector<double> dK(p), A(p * p, 0.0), rhs(p);
    radial_derivs_r1(lam_p, rho, kernel, a, p, dK.data());
    for (int k = 0; k < p; ++k) {
        for (int i = 0; i < p; ++i) {
            const int e = 2 * i;
            if (e < k) continue;
            double f = 1.0;
            for (int q = e - k + 1; q <= e; ++q) f *= q;   // e! / (e - k)!
            A[k * p + i] = f / pow(a, k);
        }
        rhs[k] = dK[k];
    }
    for (int col = 0; col < p; ++col) {
        int piv = col;
        for (int r = col + 1; r < p; ++r)
            if (fabs(A[r * p + col]) > fabs(A[piv * p + col])) piv = r;
        if (A[piv * p + col] == 0.0) return set_error(SK_EINVAL, "inner regularisation system is singular");
        if (piv != col) {
            for (int i = 0; i < p; ++i) std::swap(A[col * p + i], A[piv * p + i]);
            std::swap(rhs[col], rhs[piv]);
        }
        for (int r = col + 1; r < p; ++r) {
            const double f = A[r * p + col] / A[col * p + col];
            for (int i = col; i < p; ++i) A[r * p + i] -= f * A[col * p + i];
            rhs[r] -= f * rhs[col];
        }
    }
    c.assign(p, 0.0);
    for (int r = p - 1; r >= 0; --r) {
        double v = rhs[r];
        for (int i = r + 1; i < p; ++i) v -= A[r * p + i] * c[i];
        c[r] = v / A[r * p + r];
    }
    return SK_OK;
}

static double binom(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

// Coefficients c_0..c_{2p-2} of K_B(r) = sum_i c_i t^i, t = (r - L)/(1/2 - L), with
// K_B^{(k)}(L) = K^{(k)}(L) (k < p) and K_B^{(k)}(1/2) = 0 (1 <= k < p), Eq. (intpol_cond_3/4)
// (P:L489-496). Construction: s = dK_B/dt is the two-point Taylor interpolant of order
// r = p - 1 at t = 0 (data F^{(k+1)}(0)) and t = 1 (zeros):
//   s(t) = (1-t)^r sum_{k<r} sum_{j<r-k} C(r-1+j, j) s^{(k)}(0)/k! t^{k+j},
// and K_B(t) = F(0) + int_0^t s.
static void kb_coefficients(int rpow, double lam_p, double rho, int kernel, double L, int p,
                            std::vector<double>& c) {
    const double D = 0.5 - L;
    std::vector<double> dK(p);
    radial_derivs_any(rpow, lam_p, rho, kernel, L, p, dK.data());
    std::vector<double> F(p);
    double Dk = 1.0;
    for (int k = 0; k < p; ++k) { F[k] = dK[k] * Dk; Dk *= D; }
    const int r = p - 1;
    // inner polynomial P(t) = sum_{k<r} sum_{j<r-k} C(r-1+j,j) F^{(k+1)}(0)/k! t^{k+j}
    std::vector<double> Pc(std::max(r, 1), 0.0);
    double kf = 1.0;
    for (int k = 0; k < r; ++k) {
        if (k > 0) kf *= k;
        for (int j = 0; j < r - k; ++j) Pc[k + j] += binom(r - 1 + j, j) * F[k + 1] / kf;
    }
    // (1-t)^r
    std::vector<double> Q(r + 1);
    for (int i = 0; i <= r; ++i) Q[i] = binom(r, i) * ((i & 1) ? -1.0 : 1.0);
    std::vector<double> s(Pc.size() + Q.size() - 1, 0.0);
    for (size_t i = 0; i < Pc.size(); ++i)
        for (size_t j = 0; j < Q.size(); ++j) s[i + j] += Pc[i] * Q[j];
    c.assign(s.size() + 1, 0.0);
    c[0] = F[0];
    for (size_t i = 0; i < s.size(); ++i) c[i + 1] = s[i] / (double)(i + 1);
}

// ---------------------------------------------------------------- cuFFT plan pool
// cufftPlanMany / cufftDestroy allocate and free work areas (device-synchronising) and cost
// milliseconds; a plan takes its FFT handles from this pool and returns them when destroyed,
// so back-to-back plans of one size (every bench step, every solve) reuse them. A handle is
// owned by one plan at a time, so distinct live plans never share one.
struct FftKey {
    int device, d, n, type;
    long long batch;
    bool operator<(const FftKey& o) const {
        return std::tie(device, d, n, type, batch) < std::tie(o.device, o.d, o.n, o.type, o.batch);
    }
};
static std::mutex g_fft_mu;
static std::multimap<FftKey, cufftHandle> g_fft_pool;

// d-dimensional n^d transform; batch > 1: `batch` contiguous transforms (rank d, default
// strides) -- the 1-D batched transforms of the pruned FFT use d = 1.
int fft_acquire(int d, int n, cufftType type, cudaStream_t s, cufftHandle* out, long long batch) {
    int dev = 0;
    cudaGetDevice(&dev);
    const FftKey k{dev, d, n, (int)type, batch};
    {
        std::lock_guard<std::mutex> g(g_fft_mu);
        auto it = g_fft_pool.find(k);
        if (it != g_fft_pool.end()) {
            *out = it->second;
            g_fft_pool.erase(it);
            SK_CUFFT(cufftSetStream(*out, s));
            return SK_OK;
        }
    }
    int dims[3] = {n, n, n};
    SK_CUFFT(cufftPlanMany(out, d, dims, nullptr, 1, 0, nullptr, 1, 0, type, (int)batch));
    SK_CUFFT(cufftSetStream(*out, s));
    return SK_OK;
}

void fft_release(int d, int n, cufftType type, cufftHandle h, long long batch) {
    if (!h) return;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_fft_mu);
    g_fft_pool.emplace(FftKey{dev, d, n, (int)type, batch}, h);
}

void fft_pool_release() {
    std::lock_guard<std::mutex> g(g_fft_mu);
    for (auto& kv : g_fft_pool) cufftDestroy(kv.second);
    g_fft_pool.clear();
}

// ---------------------------------------------------------------- pinned scalar buffers
// Every plan needs 64 pinned doubles for its host-read scalars; cudaMallocHost costs ~ms, so
// freed buffers are pooled (plans are created per solve).
static std::mutex g_pin_mu;
static std::vector<double*> g_pin_pool;

static int pinned_acquire(double** out) {
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        if (!g_pin_pool.empty()) {
            *out = g_pin_pool.back();
            g_pin_pool.pop_back();
            return SK_OK;
        }
    }
    if (cudaMallocHost((void**)out, sizeof(double) * 64) != cudaSuccess)
        return set_error(SK_ENOMEM, "cudaMallocHost");
    return SK_OK;
}

static void pinned_release(double* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_pin_mu);
    g_pin_pool.push_back(p);
}

// ---------------------------------------------------------------- plan
// All plan memory goes through the caching allocator, ordered on the plan's stream.
static thread_local cudaStream_t tls_stream = nullptr;
static int alloc(void** p, size_t bytes) { return dev_alloc(p, bytes, tls_stream); }
static void sk_free(void* p) { dev_free(p, tls_stream); }

static int choose_tile(int d, int n, bool tiled) {
    int T = tiled ? 2 : (d == 1 ? 16 : (d == 2 ? 8 : 4));
    while (T > 1 && n % T) T >>= 1;
    return T;
}

// r = 1, d >= 2 near-field work list: every non-empty tile's targets in chunks of
// <= kNearChunk, so a CTA's targets share one tile and one neighbourhood of source tiles.
static int build_near_items(Plan& P, NodeSet& S, cudaStream_t s) {
    std::vector<int> ts(S.ntiles + 1);
    SK_CUDA(cudaMemcpyAsync(ts.data(), S.tile_start, sizeof(int) * (S.ntiles + 1), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    // sparse tiles (a few targets each, e.g. d = 3 with 2^3-cell tiles) are merged along the
    // last axis while they share the row and the item stays <= kNearChunk targets
    std::vector<NearItem> items;
    const int tpa = P.tiles_per_axis;
    for (int t = 0; t < S.ntiles; ++t) {
        const int cnt = ts[t + 1] - ts[t];
        if (cnt <= 0) continue;
        NearItem* last = items.empty() ? nullptr : &items.back();
        if (last && last->tile_last / tpa == t / tpa && last->start + last->count == ts[t] &&
            last->count + cnt <= kNearChunk) {
            last->count += cnt;
            last->tile_last = t;
            continue;
        }
        for (int c = ts[t]; c < ts[t + 1]; c += kNearChunk)
            items.push_back(NearItem{t, c, std::min(kNearChunk, ts[t + 1] - c), t});
    }
    S.n_near = (int)items.size();
    SK_TRY(alloc(&S.near_items, sizeof(NearItem) * std::max<size_t>(items.size(), 1)));
    if (!items.empty())
        SK_CUDA(cudaMemcpyAsync(S.near_items, items.data(), sizeof(NearItem) * items.size(), cudaMemcpyHostToDevice, s));
    SK_CUDA(cudaStreamSynchronize(s));
    return SK_OK;
}

// Work list of the tiled kernels: one item per non-empty tile, dense tiles split into
// balanced chunks of <= kItemMax nodes; sorted by size (largest first) so the static
// round-robin over CTAs balances.
static int build_items(Plan& P, NodeSet& S, cudaStream_t s) {
    std::vector<int> ts(S.ntiles + 1);
    SK_CUDA(cudaMemcpyAsync(ts.data(), S.tile_start, sizeof(int) * (S.ntiles + 1), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    std::vector<TileItem> items;
    for (int t = 0; t < S.ntiles; ++t) {
        const int cnt = ts[t + 1] - ts[t];
        if (cnt <= 0) continue;
        const int nch = (cnt + kItemMax - 1) / kItemMax;
        const int per = (cnt + nch - 1) / nch;
        for (int c = 0; c < cnt; c += per) items.push_back(TileItem{t, ts[t] + c, std::min(per, cnt - c), 0});
    }
    std::stable_sort(items.begin(), items.end(),
                     [](const TileItem& a, const TileItem& b) { return a.count > b.count; });
    S.nitems = (int)items.size();
    if (S.nitems == 0) return SK_OK;
    SK_TRY(alloc(&S.items, sizeof(TileItem) * items.size()));
    SK_CUDA(cudaMemcpyAsync(S.items, items.data(), sizeof(TileItem) * items.size(), cudaMemcpyHostToDevice, s));
    SK_CUDA(cudaStreamSynchronize(s));
    (void)P;
    return SK_OK;
}

// DMMA path: nodes are sorted by key = (super-tile << log2 Td) | cell bits. Run-length encode
// the keys (one run per non-empty cell) and build, on the device,
//   batches: <= 32 nodes of one cell (interp work unit of a warp),
//   segs:    <= seg_max nodes of one cell (spread),
//   sitems:  consecutive segs of one super-tile, <= item_max nodes (spread work unit of a
//            warp, flushed once with coalesced atomics), sorted by size (stable) for balance.
struct CellGeom { int d, n, tpa, T, Td, xminor, xpairs; };

__device__ __forceinline__ int cell_of_key(int key, const CellGeom g) {
    const int tile = key / g.Td;
    int sub = key % g.Td, rest = tile, tc[3], cc[3];
    for (int a = g.d - 1; a >= 0; --a) { tc[a] = rest % g.tpa; rest /= g.tpa; }
    if (g.xminor)   // x least significant (scale_key_kernel's xminor order)
        for (int a = 0; a < g.d; ++a) { cc[a] = g.T * tc[a] + sub % g.T; sub /= g.T; }
    else
        for (int a = g.d - 1; a >= 0; --a) { cc[a] = g.T * tc[a] + sub % g.T; sub /= g.T; }
    int cell = 0;
    for (int a = 0; a < g.d; ++a) cell = cell * g.n + cc[a];
    return cell;
}

// Spread segments group the runs (cells) of a tile: with xpairs, the two cells of an x-pair
// (same y, z; x digits 0 and 1, adjacent keys) form one group whose nodes are contiguous, the
// x-digit-0 cell's nodes first; otherwise a group is one cell. Returns the run after the group.
__device__ __forceinline__ int spread_group(const int* __restrict__ keys, const int* __restrict__ cnts,
                                            int q, int nruns, int tile, const CellGeom g, int& count,
                                            int& countA, int& key0) {
    count = cnts[q];
    countA = count;
    key0 = keys[q];
    if (!g.xpairs) return q + 1;
    const int dx = (keys[q] % g.Td) % g.T;
    if (dx != 0) {            // a lone x-digit-1 cell: all its nodes sit at x offset 1
        countA = 0;
        key0 = keys[q] - dx;
        return q + 1;
    }
    if (q + 1 < nruns && keys[q + 1] / g.Td == tile && keys[q + 1] == keys[q] + 1) {
        count += cnts[q + 1];
        return q + 2;
    }
    return q + 1;
}

// per run: interp batches; per tile-head run: number of segs / items of its tile (greedy
// fill in run order, exactly the sequential rule)
__global__ void cell_counts_kernel(const int* __restrict__ keys, const int* __restrict__ cnts, int nruns,
                                   CellGeom g, int seg_max, int item_max, int bmax, int* __restrict__ nb,
                                   int* __restrict__ nseg, int* __restrict__ nitem) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    nb[r] = (cnts[r] + bmax - 1) / bmax;
    const int tile = keys[r] / g.Td;
    int ns = 0, ni = 0;
    if (r == 0 || keys[r - 1] / g.Td != tile) {
        int fill = 0;
        for (int q = r; q < nruns && keys[q] / g.Td == tile;) {
            int cnt, cntA, key0;
            q = spread_group(keys, cnts, q, nruns, tile, g, cnt, cntA, key0);
            for (int b = 0; b < cnt; b += seg_max) {
                const int c = min(seg_max, cnt - b);
                if (ni == 0 || fill + c > item_max) { ++ni; fill = 0; }
                fill += c;
                ++ns;
            }
        }
    }
    nseg[r] = ns;
    nitem[r] = ni;
}

__global__ void cell_write_kernel(const int* __restrict__ keys, const int* __restrict__ cnts,
                                  const int* __restrict__ rstart, int nruns, CellGeom g, int seg_max,
                                  int item_max, int bmax, const int* __restrict__ nb_off, const int* __restrict__ seg_off,
                                  const int* __restrict__ item_off, CellBatch* __restrict__ batches,
                                  CellBatch* __restrict__ segs, SpreadItem* __restrict__ items,
                                  int* __restrict__ item_cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int cell = cell_of_key(keys[r], g), cnt = cnts[r], st = rstart[r];
    int o = nb_off[r];
    for (int b = 0; b < cnt; b += bmax) batches[o++] = CellBatch{cell, st + b, min(bmax, cnt - b), 0};
    const int tile = keys[r] / g.Td;
    if (!(r == 0 || keys[r - 1] / g.Td != tile)) return;
    int so = seg_off[r], io = item_off[r] - 1, fill = 0;
    bool first = true;
    for (int q = r; q < nruns && keys[q] / g.Td == tile;) {
        const int q0 = q;
        int cnt, cntA, key0;
        q = spread_group(keys, cnts, q, nruns, tile, g, cnt, cntA, key0);
        const int cq = cell_of_key(key0, g);
        for (int b = 0; b < cnt; b += seg_max) {
            const int c = min(seg_max, cnt - b);
            if (first || fill + c > item_max) {
                if (!first) { items[io].count = fill; item_cnt[io] = fill; }
                ++io;
                items[io] = SpreadItem{tile, so, so, 0};
                fill = 0;
                first = false;
            }
            // pad = nodes of this piece in the x-digit-0 cell (the first ones)
            segs[so++] = CellBatch{cq, rstart[q0] + b, c, g.xpairs ? min(max(cntA - b, 0), c) : c};
            items[io].seg_end = so;
            fill += c;
        }
    }
    if (!first) { items[io].count = fill; item_cnt[io] = fill; }
}

__global__ void iota_kernel(int* __restrict__ o, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = i;
}

__global__ void gather_items_kernel(const SpreadItem* __restrict__ in, const int* __restrict__ order, int n,
                                    SpreadItem* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[order[i]];
}

#ifndef SK_SPREAD_ITEM_MIN
#define SK_SPREAD_ITEM_MIN 64   // small sets: more, smaller spread items (c2 spread 23.0 -> 20.6 us; 32 is worse)
#endif
static int build_cell_lists(Plan& P, NodeSet& S, cudaStream_t s) {
    const long long count = S.count;
    const int d = P.d, n = P.n, tpa = P.tiles_per_axis, T = P.tile_cells;
    int Td = 1;
    for (int a = 0; a < d; ++a) Td *= T;
    // x-pair spread segments pay where cells are sparse (few nodes per cell, so the per-segment
    // region update dominates): decided per side once the cells are counted (below)
    CellGeom g{d, n, tpa, T, Td, P.spread_xpairs ? 1 : 0, 0};
    // spread work-unit size: enough items to keep ~4 per resident warp busy (148 SMs x 8
    // warps), at most kSpreadItemMax nodes (one region flush per item)
    // (the floor is a runtime knob for measurements: SK_SPREAD_ITEM_MIN overrides the default)
    static const long long item_min_env = getenv("SK_SPREAD_ITEM_MIN") ? atoll(getenv("SK_SPREAD_ITEM_MIN")) : 0;
    // deterministic flushes cost twice the atomics: a larger floor for small sets (measured, DESIGN.md
    // §6: img512 spread 44 -> 34 us at 128 nodes, c2 26.9 -> 27.6 us; c3 / c4 / c5 items are larger)
    const long long item_min = item_min_env > 0 ? item_min_env
                                                : (P.deterministic ? 2LL * SK_SPREAD_ITEM_MIN : (long long)SK_SPREAD_ITEM_MIN);
    const int item_max = (int)std::max(item_min, std::min((long long)kSpreadItemMax, count / 4736));

    // run-length encode the sorted keys; 7 int arrays of nruns (<= count) entries
    int* buf = nullptr;
    SK_TRY(alloc((void**)&buf, sizeof(int) * (7 * count + 16)));
    int *keys = buf, *cnts = keys + count, *rstart = cnts + count, *nb = rstart + count,
        *nseg = nb + count, *nitem = nseg + count, *scratch = nitem + count, *small = scratch + count;
    size_t tb = 0, tb2 = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb, S.cell_key, keys, cnts, small, (int)count, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnts, rstart, (int)count, s);
    tb = std::max(tb, tb2);
    void* tmp = nullptr;
    SK_TRY(alloc(&tmp, tb));
    SK_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, tb, S.cell_key, keys, cnts, small, (int)count, s));
    count_launch(2);
    int nruns = 0;
    SK_CUDA(cudaMemcpyAsync(&nruns, small, sizeof(int), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    const int thr = 256, blk = (nruns + thr - 1) / thr;
    S.xpairs = P.spread_xpairs && (long long)kXPairMaxDensity * nruns > count;
    // dense cells: longer TMA segments on fewer warp pairs (SK_SEG_DENSE_MIN overrides the mean
    // nodes-per-cell threshold; 0 = always, a large value = never)
    {
        const char* ev = getenv("SK_SEG_DENSE_MIN");
        const long long thr = ev ? atoll(ev) : (long long)kSegDenseMinMean;
        S.seg_dense = P.spread_tmapad && P.d == 3 && !S.xpairs && count >= thr * (long long)nruns;
    }
    const int seg_max = std::min(P.spread_tmapad ? (S.seg_dense ? kSegTmaPDense : kSegTmaPMax)
                                 : kSegMax,
                                 item_max);
    g.xpairs = S.xpairs ? 1 : 0;
    SK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnts, rstart, nruns, s));
    const int bmax = d == 3 ? kInterpBatch3 : 32;   // interp batch: nodes of one cell per warp pass
    cell_counts_kernel<<<blk, thr, 0, s>>>(keys, cnts, nruns, g, seg_max, item_max, bmax, nb, nseg, nitem);
    SK_CUDA(cudaGetLastError());
    // totals = last exclusive prefix + last count (in-place scans)
    int last[3];
    SK_CUDA(cudaMemcpyAsync(small + 4, nb + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    SK_CUDA(cudaMemcpyAsync(small + 5, nseg + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    SK_CUDA(cudaMemcpyAsync(small + 6, nitem + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    SK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nb, nb, nruns, s));
    SK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nseg, nseg, nruns, s));
    SK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nitem, nitem, nruns, s));
    count_launch(5);
    SK_CUDA(cudaMemcpyAsync(small + 7, nb + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    SK_CUDA(cudaMemcpyAsync(small + 8, nseg + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    SK_CUDA(cudaMemcpyAsync(small + 9, nitem + nruns - 1, sizeof(int), cudaMemcpyDeviceToDevice, s));
    int h[10];
    SK_CUDA(cudaMemcpyAsync(h, small, sizeof(int) * 10, cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    last[0] = h[4] + h[7]; last[1] = h[5] + h[8]; last[2] = h[6] + h[9];
    S.nbatches = last[0];
    S.ncells = nruns;
    S.nsegs = last[1];
    S.nsitems = last[2];
    SK_TRY(alloc(&S.batches, sizeof(CellBatch) * std::max(S.nbatches, 1)));
    SK_TRY(alloc(&S.segs, sizeof(CellBatch) * std::max(S.nsegs, 1)));
    SK_TRY(alloc(&S.sitems, sizeof(SpreadItem) * std::max(S.nsitems, 1)));
    SpreadItem* items_unsorted = nullptr;
    SK_TRY(alloc((void**)&items_unsorted, sizeof(SpreadItem) * std::max(S.nsitems, 1)));
    // item counts and identity order in the (now free) cnts-sized scratch arrays
    int *icnt = scratch, *icnt_sorted = nullptr, *ord = nullptr, *ord_sorted = nullptr;
    SK_TRY(alloc((void**)&icnt_sorted, sizeof(int) * 3 * std::max(S.nsitems, 1)));
    ord = icnt_sorted + std::max(S.nsitems, 1);
    ord_sorted = ord + std::max(S.nsitems, 1);
    cell_write_kernel<<<blk, thr, 0, s>>>(keys, cnts, rstart, nruns, g, seg_max, item_max, bmax, nb, nseg, nitem,
                                          (CellBatch*)S.batches, (CellBatch*)S.segs, items_unsorted, icnt);
    SK_CUDA(cudaGetLastError());
    count_launch(2);
    // stable sort of the items by node count, largest first (static round-robin balance)
    const int ni = S.nsitems;
    if (ni > 0) {
        size_t tb3 = 0;
        SK_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb3, icnt, icnt_sorted, ord, ord_sorted, ni, 0,
                                                          32, s));
        void* tmp3 = nullptr;
        SK_TRY(alloc(&tmp3, tb3));
        iota_kernel<<<(ni + 255) / 256, 256, 0, s>>>(ord, ni);
        SK_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp3, tb3, icnt, icnt_sorted, ord, ord_sorted, ni, 0,
                                                          32, s));
        gather_items_kernel<<<(ni + 255) / 256, 256, 0, s>>>(items_unsorted, ord_sorted, ni,
                                                             (SpreadItem*)S.sitems);
        SK_CUDA(cudaGetLastError());
        count_launch(4);
        sk_free(tmp3);
    }
    sk_free(icnt_sorted);
    sk_free(items_unsorted);
    sk_free(tmp);
    sk_free(buf);
    return SK_OK;
}

static int plan_side(Plan& P, int sidx, const double* pts, long long count, cudaStream_t s) {
    NodeSet& S = P.side[sidx];
    S.count = count;
    S.ntiles = 1;
    for (int a = 0; a < P.d; ++a) S.ntiles *= P.tiles_per_axis;
    SK_TRY(alloc((void**)&S.tile_start, sizeof(int) * (S.ntiles + 1)));
    if (count == 0) {
        SK_CUDA(cudaMemsetAsync(S.tile_start, 0, sizeof(int) * (S.ntiles + 1), s));
        return SK_OK;
    }
    int *key_in = nullptr, *idx_in = nullptr, *bad = nullptr;
    SK_TRY(alloc((void**)&key_in, sizeof(int) * count));
    SK_TRY(alloc((void**)&idx_in, sizeof(int) * count));
    SK_TRY(alloc((void**)&bad, sizeof(int)));
    SK_TRY(alloc((void**)&S.cell_key, sizeof(int) * count));
    SK_TRY(alloc((void**)&S.perm, sizeof(int) * count));
    SK_TRY(alloc((void**)&S.u, sizeof(double) * P.d * count));
    const int big = 0x7fffffff;
    SK_CUDA(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    plan_trace("side: alloc", s);
    SK_TRY(launch_scale_key(P, pts, count, key_in, idx_in, bad, s));
    plan_trace("side: scale_key", s);
    int hbad = 0;
    SK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    if (hbad != big) {
        sk_free(key_in); sk_free(idx_in); sk_free(bad);
        return set_error(SK_EGEOMETRY, "node " + std::to_string(hbad) + " of side " + std::to_string(sidx) +
                                           " is non-finite or outside the ball |x'| <= 1/4 - eps_B/2");
    }
    long long Td = 1;
    for (int a = 0; a < P.d; ++a) Td *= P.tile_cells;
    const long long nkeys = P.fine_shift ? ((long long)S.ntiles * P.tile_cells << P.fine_shift)
                                         : ((P.dmma || P.near_cell_sort) ? (long long)S.ntiles * Td : S.ntiles);
    int end_bit = 1;
    while ((1LL << end_bit) < nkeys) ++end_bit;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key_in, S.cell_key, idx_in, S.perm, (int)count, 0,
                                    end_bit, s);
    void* tmp = nullptr;
    SK_TRY(alloc(&tmp, tmp_bytes));
    SK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key_in, S.cell_key, idx_in, S.perm, (int)count,
                                            0, end_bit, s));
    count_launch(4);
    plan_trace("side: sort", s);
    SK_TRY(launch_gather_coords(P, pts, S.perm, count, S.u, s));
    plan_trace("side: gather", s);
    if (P.dmma) {
        SK_TRY(build_cell_lists(P, S, s));
        plan_trace("side: cell lists", s);
        SK_TRY(alloc((void**)&S.taps, sizeof(double) * count * P.d * 2 * P.win.m));
        SK_TRY(launch_taps(P, sidx, s));
        plan_trace("side: taps", s);
        if (P.rpow == 1) {   // the near field's tile CSR (keys are tile * T^d + cell; scratch now)
            SK_TRY(launch_key_to_tile(P, S.cell_key, count, s));
            SK_TRY(launch_tile_offsets(S.cell_key, count, S.ntiles, S.tile_start, s));
            SK_TRY(build_near_items(P, S, s));
        }
    } else {
        if (P.fine_shift || P.near_cell_sort) SK_TRY(launch_key_to_tile(P, S.cell_key, count, s));
        SK_TRY(launch_tile_offsets(S.cell_key, count, S.ntiles, S.tile_start, s));
        SK_CUDA(cudaStreamSynchronize(s));
        if (P.tiled) SK_TRY(build_items(P, S, s));
        if (P.rpow == 1 && P.d >= 2) SK_TRY(build_near_items(P, S, s));
    }
    sk_free(tmp);
    sk_free(key_in);
    sk_free(idx_in);
    sk_free(bad);
    return SK_OK;
}

// r = 1 across ranks (world > 1, an emulated world, or a one-rank NCCL communicator): the near
// field of a target needs every source within the radius, wherever it lives. Each side's sorted
// grid coordinates are all-gathered (rank-major concatenation), sorted by the key a local side
// uses, and kept with the sorted -> concatenation map; each fast summation all-gathers the source
// weights into the same order (apply_sorted). The far field is unchanged (grid all-reduce).
static int build_near_global(Plan& P, NodeSet& S, cudaStream_t s) {
    Ctx* C = P.ctx;
    SK_TRY(gather_counts(C, S.count, S.g_counts));
    long long total = 0;
    for (int r = 0; r < C->world; ++r) total += S.g_counts[r];
    S.g_total = total;
    const int d = P.d;
    SK_TRY(alloc((void**)&S.g_u, sizeof(double) * std::max(1LL, d * total)));
    SK_TRY(alloc((void**)&S.g_tile_start, sizeof(int) * (S.ntiles + 1)));
    SK_TRY(alloc((void**)&S.g_perm, sizeof(int) * std::max(1LL, total)));
    SK_TRY(alloc((void**)&S.g_wcat, sizeof(double) * std::max(1LL, total)));
    SK_TRY(alloc((void**)&S.g_w, sizeof(double) * std::max(1LL, total)));
    double* ucat = nullptr;
    int *key_in = nullptr, *idx_in = nullptr, *key_out = nullptr;
    SK_TRY(alloc((void**)&ucat, sizeof(double) * std::max(1LL, d * total)));
    SK_TRY(alloc((void**)&key_in, sizeof(int) * 3 * std::max(1LL, total)));
    idx_in = key_in + std::max(1LL, total);
    key_out = idx_in + std::max(1LL, total);
    int st = SK_OK;
    for (int a = 0; a < d && !st; ++a) st = allgather_concat(C, S.u + a * S.count, S.count, S.g_counts, ucat + a * total);
    if (!st) st = launch_near_keys(P, ucat, total, key_in, idx_in, s);
    if (!st && total > 0) {
        const long long nkeys = P.fine_shift ? ((long long)S.ntiles * P.tile_cells << P.fine_shift) : S.ntiles;
        int end_bit = 1;
        while ((1LL << end_bit) < nkeys) ++end_bit;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key_in, key_out, idx_in, S.g_perm, (int)total, 0, end_bit, s);
        void* tmp = nullptr;
        st = alloc(&tmp, tb);
        if (!st && cub::DeviceRadixSort::SortPairs(tmp, tb, key_in, key_out, idx_in, S.g_perm, (int)total, 0, end_bit,
                                                   s) != cudaSuccess)
            st = set_error(SK_ECUDA, "near-field sort across ranks");
        count_launch(4);
        sk_free(tmp);
        if (!st) st = launch_gather_rows(ucat, total, S.g_perm, total, d, S.g_u, s);
        if (!st && P.fine_shift) st = launch_key_to_tile(P, key_out, total, s);
    }
    if (!st) st = launch_tile_offsets(key_out, total, S.ntiles, S.g_tile_start, s);
    if (!st && cudaStreamSynchronize(s) != cudaSuccess) st = set_error(SK_ECUDA, "near-field gather sync");
    sk_free(ucat);
    sk_free(key_in);
    return st;
}

static int plan_coefficients(Plan& P, cudaStream_t s) {
    const int M = 2 * P.N;  // sampling grid of K~_per (reading Q9)
    long long Md = 1, Bsz = 1;
    for (int a = 0; a < P.d; ++a) Md *= M;
    for (int a = 0; a < P.d - 1; ++a) Bsz *= M;
    Bsz *= (M / 2 + 1);
    double* samp = nullptr;
    cufftDoubleComplex* B = nullptr;
    SK_TRY(alloc((void**)&samp, sizeof(double) * Md));
    SK_TRY(alloc((void**)&B, sizeof(cufftDoubleComplex) * Bsz));
    double* tail = nullptr;   // [kernel][1 + kUpdBlocks]: band-tail estimate + partial scratch
    SK_TRY(alloc((void**)&tail, sizeof(double) * 2 * (1 + kUpdBlocks)));
    cufftHandle h = 0;
    SK_TRY(fft_acquire(P.d, M, CUFFT_D2Z, s, &h));
    for (int kernel = 0; kernel < 2; ++kernel) {
        std::vector<double> c;
        kb_coefficients(P.rpow, P.lambda_p, P.rho, kernel, P.L, P.p_smooth, c);
        if (P.rpow == 1) {
            std::vector<double> ci;
            SK_TRY(ki_coefficients(P.lambda_p, P.rho, kernel, P.near_a, P.p_smooth, ci));
            for (int i = 0; i < (int)ci.size(); ++i) P.ki[kernel][i] = ci[i];
            P.ki_n = (int)ci.size();
        }
        SK_TRY(launch_sample_kernel(P, kernel, M, c.data(), (int)c.size() - 1, samp, s));
        SK_CUFFT(cufftExecD2Z(h, samp, B));
        count_launch();
        SK_TRY(launch_band_coeffs(P, kernel, M, B, s));
        SK_TRY(launch_band_tail(P, M, B, tail + kernel * (1 + kUpdBlocks), s));
    }
    SK_CUDA(cudaMemcpyAsync(&P.acc_tail[0], tail, sizeof(double), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaMemcpyAsync(&P.acc_tail[1], tail + 1 + kUpdBlocks, sizeof(double), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    sk_free(tail);
    fft_release(P.d, M, CUFFT_D2Z, h);
    sk_free(samp);
    sk_free(B);
    return SK_OK;
}

int build_plan(Ctx* ctx, Plan** out, int d, const double* x, long long n, const double* y,
               long long m, double lambda, int N, double sigma, int m_w, double eps_B, int p,
               int rpow, int near_cells) {
    if (d < 1 || d > 3) return set_error(SK_EINVAL, "d must be 1, 2 or 3");
    if (rpow != 1 && rpow != 2) return set_error(SK_EINVAL, "r must be 1 or 2");
    if (rpow == 1 && (near_cells < 1 || p > 8))
        return set_error(SK_EINVAL, "r = 1 needs near_cells >= 1 and p_smooth <= 8 (K_I monomial system)");
    if (N < 2 || (N & 1)) return set_error(SK_EINVAL, "N must be even and >= 2");
    if (!(lambda > 0.0) || !isfinite(lambda)) return set_error(SK_EINVAL, "lambda must be > 0");
    if (m_w < 2 || m_w > 8) return set_error(SK_EINVAL, "m_w must be in [2, 8]");
    if (!(eps_B > 0.0 && eps_B < 0.25)) return set_error(SK_EINVAL, "eps_B must be in (0, 1/4)");
    if (p < 1 || p > 15) return set_error(SK_EINVAL, "p_smooth must be in [1, 15]");
    if (n < 0 || m < 0) return set_error(SK_EINVAL, "negative node count");
    if ((n > 0 && !x) || (m > 0 && !y)) return set_error(SK_EINVAL, "NULL node array");
    if (n > 0x7ffffffeLL || m > 0x7ffffffeLL) return set_error(SK_EINVAL, "local node count exceeds 2^31-2");
    const double nd = sigma * N;
    const int ng = (int)llround(nd);
    if (!(sigma >= 1.0) || fabs(nd - ng) > 1e-9 || (ng & 1))
        return set_error(SK_EINVAL, "sigma*N must be an even integer");
    if (ng < 4 * m_w) return set_error(SK_EINVAL, "sigma*N must be >= 4*m_w (no tap wraps the torus)");
    {   // cell indices and sort keys are int: the grid must have < 2^31 cells
        long long cells = 1;
        for (int a = 0; a < d; ++a) cells *= ng;
        if (cells > 0x7fffffffLL) return set_error(SK_EINVAL, "(sigma N)^d must be < 2^31 grid cells");
    }

    cudaStream_t s = ctx->stream;
    tls_stream = s;
    Plan* P = new Plan();
    P->ctx = ctx;
    P->d = d;
    P->N = N;
    P->n = ng;
    P->sigma = sigma;
    P->win.m = m_w;
    P->win.beta = 3.141592653589793238462643 * (2.0 - 1.0 / sigma);
    P->win.m2 = (double)m_w * m_w;
    P->win.inv_pi = 1.0 / 3.141592653589793238462643;
    P->lambda = lambda;
    P->eps_B = eps_B;
    P->p_smooth = p;
    P->L = 0.5 - eps_B;
    P->rpow = rpow;
    P->near_cells = rpow == 1 ? near_cells : 0;
    P->near_a = rpow == 1 ? (double)near_cells / ng : 0.0;
    if (rpow == 1 && !(P->near_a < P->L)) {
        delete P;
        return set_error(SK_EINVAL, "near-field radius near_cells / (sigma N) must be < 1/2 - eps_B");
    }
    P->grid_size = 1;
    for (int a = 0; a < d; ++a) P->grid_size *= ng;
    P->spec_size = 1;
    for (int a = 0; a < d - 1; ++a) P->spec_size *= ng;
    P->spec_size *= (ng / 2 + 1);
    P->band_size = 1;
    for (int a = 0; a < d - 1; ++a) P->band_size *= (N + 1);
    P->band_size *= (N / 2 + 1);
    {
        WinPoly* wp = new WinPoly();
        const double err = build_winpoly(m_w, sigma, wp);
        P->winpoly = wp;
        // r = 1 takes the same spread / interp (its near field walks the tile CSR, built for it
        // on the DMMA path too); SK_R1_V1=1 keeps r = 1 on the plain v1 kernels
        const bool fast = rpow == 2 || getenv("SK_R1_V1") == nullptr;
        P->tiled = (d == 3) && (m_w == 6 || m_w == 8) && err >= 0.0 && err <= 1e-14 && fast &&
                   getenv("SK_FORCE_V1") == nullptr;
        P->dmma = ((P->tiled && m_w == 6) || (d == 2 && m_w == 8 && err >= 0.0 && err <= 1e-14)) &&
                  fast && getenv("SK_NO_DMMA") == nullptr && getenv("SK_FORCE_V1") == nullptr;
        if (P->dmma && d == 2) P->tiled = false;
        // d = 3 spread: the DMMA spread on TMA-fed warp pairs. x-pair segments for sparse sets
        // (16-row padded tiles) are opt-in (SK_XPAIRS=1): the 28-tile cover without them is faster
        // on c3 (924 -> 945 it/s, tools/ab_env.sh)
        P->spread_tmapad = P->dmma && d == 3;
        P->spread_pipe = getenv("SK_SPREAD3_NOPIPE") == nullptr;
        P->spread_xpairs = P->dmma && d == 3 && getenv("SK_XPAIRS") != nullptr;
    }
    {   // phi(0)^d bounds one node's spread contribution |w| prod_a phi (deterministic mode)
        const double bm = P->win.beta * m_w;
        P->phi0d = pow(sinh(bm) / (3.141592653589793238462643 * m_w), d);
        const char* det = getenv("SK_DETERMINISTIC");
        P->deterministic = det ? atoi(det) != 0 : kDeterministicDefault;
    }
    P->tile_cells = P->dmma ? (d == 3 ? 2 : kSup2) : choose_tile(d, ng, P->tiled);
    P->tiles_per_axis = ng / P->tile_cells;
    if (d == 1 && rpow == 1 && !P->dmma && getenv("SK_NEARFIELD_V1") == nullptr) {
        // position sort for the d = 1 near field: fine keys below 2^30
        int shift = 0;
        while (((long long)ng << (shift + 1)) <= (1LL << 30)) ++shift;
        P->fine_shift = shift;
    }
    P->near_cell_sort = d >= 2 && rpow == 1 && !P->dmma && getenv("SK_NEARFIELD_V1") == nullptr;

    auto fail = [&](int code) { destroy_plan(P); return code; };

    plan_trace("start", s);
    // ---- a0: geometry (bbox over x u y on all ranks), reading Q6
    double* mm = nullptr;
    if (alloc((void**)&mm, sizeof(double) * 2 * kMaxD)) return fail(SK_ENOMEM);
    {
        double init[2 * kMaxD];
        for (int a = 0; a < d; ++a) { init[a] = INFINITY; init[d + a] = -INFINITY; }
        if (cudaMemcpyAsync(mm, init, sizeof(double) * 2 * d, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return fail(set_error(SK_ECUDA, "bbox init"));
        int st = launch_bbox(x, n, d, mm, s);
        if (!st) st = launch_bbox(y, m, d, mm, s);
        if (!st) st = allreduce_minmax(ctx, mm, mm + d, d);
        if (st) { sk_free(mm); return fail(st); }
        double h[2 * kMaxD];
        cudaMemcpyAsync(h, mm, sizeof(double) * 2 * d, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) { sk_free(mm); return fail(set_error(SK_ECUDA, "bbox sync")); }
        sk_free(mm);
        double diag2 = 0.0;
        bool any = true;
        for (int a = 0; a < d; ++a) {
            if (!isfinite(h[a]) || !isfinite(h[d + a])) any = false;
            P->centre[a] = 0.5 * (h[a] + h[d + a]);
            diag2 += (h[d + a] - h[a]) * (h[d + a] - h[a]);
        }
        if (!any) {
            // no nodes at all, or a NaN/Inf coordinate
            return fail(set_error(SK_EGEOMETRY, "empty node sets or non-finite coordinates"));
        }
        const double diag = sqrt(diag2);
        // diag = 0 (every atom at one point, reading Q6b): the limit diag -> 0 of rho = L / diag
        // sends lambda' to 0, where the kernel is constant and its Fourier series exact; taken
        // at lambda' = kLampDegenerate
        P->rho = diag > 0.0 ? P->L / diag
                            : (rpow == 2 ? sqrt(lambda / kLampDegenerate) : lambda / kLampDegenerate);
        // exp(-lam |x - y|^r) = exp(-lam' |x' - y'|^r) with x' = rho (x - centre)
        P->lambda_p = rpow == 2 ? lambda / (P->rho * P->rho) : lambda / P->rho;
        // touched grid box: cells floor(u) - m + 1 .. floor(u) + m of every node, u = n(rho(x -
        // centre) + 1/2) over the global bbox, one cell of margin against rounding
        P->box_size = 1;
        for (int a = 0; a < d; ++a) {
            const double ulo = ng * (P->rho * (h[a] - P->centre[a]) + 0.5);
            const double uhi = ng * (P->rho * (h[d + a] - P->centre[a]) + 0.5);
            const int lo = std::max(0, (int)floor(ulo) - m_w);
            const int hi = std::min(ng - 1, (int)floor(uhi) + m_w + 1);
            P->box_lo[a] = lo;
            P->box_n[a] = hi - lo + 1;
            P->box_size *= P->box_n[a];
        }
    }
    // global counts
    {
        double cnt[2] = {(double)n, (double)m};
        double* dc = nullptr;
        if (alloc((void**)&dc, sizeof(cnt))) return fail(SK_ENOMEM);
        cudaMemcpyAsync(dc, cnt, sizeof(cnt), cudaMemcpyHostToDevice, s);
        int st = allreduce_sum(ctx, dc, 2);
        cudaMemcpyAsync(cnt, dc, sizeof(cnt), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        sk_free(dc);
        if (st) return fail(st);
        P->side[0].total = (long long)llround(cnt[0]);
        P->side[1].total = (long long)llround(cnt[1]);
    }
    plan_trace("bbox + counts", s);
    // ---- a0: scale, bin, sort (both sides)
    int st = plan_side(*P, 0, x, n, s);
    if (!st) st = plan_side(*P, 1, y, m, s);
    if (st && st != SK_EGEOMETRY) return fail(st);
    if (ctx->world > 1 || ctx->nccl_comm) {
        // a node outside the ball (or NaN) on any rank fails the plan on every rank; a rank
        // returning alone would leave the others blocked in their next collective
        const std::string local_msg = st ? sk_last_error() : "";
        double flag = st ? 1.0 : 0.0;
        double* df = nullptr;
        int st2 = alloc((void**)&df, sizeof(double));
        if (!st2) st2 = cudaMemcpyAsync(df, &flag, sizeof(double), cudaMemcpyHostToDevice, s) ? SK_ECUDA : SK_OK;
        if (!st2) st2 = allreduce_sum(ctx, df, 1);
        if (!st2) st2 = cudaMemcpyAsync(&flag, df, sizeof(double), cudaMemcpyDeviceToHost, s) ? SK_ECUDA : SK_OK;
        if (!st2) st2 = cudaStreamSynchronize(s) ? SK_ECUDA : SK_OK;
        sk_free(df);
        if (st2) return fail(st2);
        if (flag > 0.0)
            return fail(set_error(SK_EGEOMETRY, st ? local_msg : "a node of another rank is non-finite or outside "
                                                                  "the ball |x'| <= 1/4 - eps_B/2"));
    } else if (st) {
        return fail(st);
    }
    if (rpow == 1 && (ctx->world > 1 || ctx->nccl_comm)) {   // every rank reaches this point together
        st = build_near_global(*P, P->side[0], s);
        if (!st) st = build_near_global(*P, P->side[1], s);
        if (st) return fail(st);
    }
    // ---- a1: coefficients
    if ((st = alloc((void**)&P->D[0], sizeof(double) * P->band_size))) return fail(st);
    if ((st = alloc((void**)&P->D[1], sizeof(double) * P->band_size))) return fail(st);
    long long full = 1;
    for (int a = 0; a < d; ++a) full *= (N + 1);
    if ((st = alloc((void**)&P->bk[0], sizeof(double) * full))) return fail(st);
    if ((st = alloc((void**)&P->bk[1], sizeof(double) * full))) return fail(st);
    if ((st = plan_coefficients(*P, s))) return fail(st);
    plan_trace("coefficients", s);
    // ---- grid, spectrum, FFT plans
    if ((st = alloc((void**)&P->grid, sizeof(double) * P->grid_size))) return fail(st);
    if ((st = alloc((void**)&P->spec, sizeof(cufftDoubleComplex) * P->spec_size))) return fail(st);
    {
        if ((st = fft_acquire(d, ng, CUFFT_D2Z, s, &P->fwd))) return fail(st);
        if ((st = fft_acquire(d, ng, CUFFT_Z2D, s, &P->inv))) return fail(st);
    }
    if ((st = pruned_fft_setup(*P, s))) return fail(st);
    plan_trace("fft plans", s);
    // ---- scratch
    P->max_count = std::max(n, m);
    long long mc = std::max(P->max_count, 1LL);
    // spread weights (w_sorted, u_s, v_s) carry 2 doubles of slack: the TMA spread copies
    // 16-byte aligned ranges that may extend one element past either end
    if ((st = alloc((void**)&P->w_sorted, sizeof(double) * (mc + 2)))) return fail(st);
    if ((st = alloc((void**)&P->t_sorted, sizeof(double) * mc))) return fail(st);
    if ((st = alloc((void**)&P->a_s, sizeof(double) * std::max(n, 1LL)))) return fail(st);
    if ((st = alloc((void**)&P->u_s, sizeof(double) * (std::max(n, 1LL) + 2)))) return fail(st);
    if ((st = alloc((void**)&P->b_s, sizeof(double) * std::max(m, 1LL)))) return fail(st);
    if ((st = alloc((void**)&P->v_s, sizeof(double) * (std::max(m, 1LL) + 2)))) return fail(st);
    if (P->deterministic) {   // [2 box] accumulator, then 4 bound slots + the conversion's counter, all zero
        const size_t words = 2 * std::max(P->box_size, 1LL) + 4;
        if ((st = alloc((void**)&P->det_acc, sizeof(unsigned long long) * words))) return fail(st);
        if (cudaMemsetAsync(P->det_acc, 0, sizeof(unsigned long long) * words, s) != cudaSuccess)
            return fail(set_error(SK_ECUDA, "memset det_acc"));
        P->det_wmax = reinterpret_cast<unsigned*>(P->det_acc + 2 * std::max(P->box_size, 1LL));
    }
    P->box_exchange = ctx->world > 1 || ctx->nccl_comm || getenv("SK_FORCE_BOX_EXCHANGE") != nullptr;
    if (P->box_exchange && (st = alloc((void**)&P->box_buf, sizeof(double) * std::max(P->box_size, 1LL))))
        return fail(st);
    P->fftconv2 = !P->box_exchange && !P->pruned && fftconv2_supported(d, P->n, P->N);
    if (P->fftconv2) {
        std::vector<double> tw((size_t)P->n);
        fftconv2_twiddles(P->n, tw.data());
        if ((st = alloc((void**)&P->fc_tw, sizeof(double) * P->n))) return fail(st);
        if (cudaMemcpyAsync(P->fc_tw, tw.data(), sizeof(double) * P->n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fail(set_error(SK_ECUDA, "fftconv2 twiddles"));
    }
    if ((st = alloc((void**)&P->red, sizeof(double) * 4096))) return fail(st);
    if ((st = alloc((void**)&P->red_out, sizeof(double) * 8192))) return fail(st);
    if ((st = alloc((void**)&P->flag, sizeof(int) * 16))) return fail(st);
    P->bad64 = reinterpret_cast<unsigned long long*>(P->flag + 8);
    if ((st = pinned_acquire(&P->host_red))) return fail(st);
    plan_trace("scratch", s);
    *out = P;
    return SK_OK;
}

void plan_set_stream(Plan& P, cudaStream_t s) {
    for (cufftHandle h : {P.fwd, P.inv, P.pr_fz, P.pr_iz, P.pr_y, P.pr_x})
        if (h) cufftSetStream(h, s);
}

int destroy_plan(Plan* P) {
    if (!P) return SK_OK;
    tls_stream = P->ctx->stream;
    for (int sidx = 0; sidx < 2; ++sidx) {
        NodeSet& S = P->side[sidx];
        sk_free(S.u); sk_free(S.perm); sk_free(S.cell_key); sk_free(S.tile_start); sk_free(S.items);
        sk_free(S.near_items);
        sk_free(S.g_u); sk_free(S.g_tile_start); sk_free(S.g_perm); sk_free(S.g_wcat); sk_free(S.g_w);
        sk_free(S.batches); sk_free(S.segs); sk_free(S.sitems); sk_free(S.taps);
    }
    sk_free(P->grid); sk_free(P->spec);
    for (int k = 0; k < 2; ++k) { sk_free(P->D[k]); sk_free(P->bk[k]); }
    fft_release(P->d, P->n, CUFFT_D2Z, P->fwd);
    fft_release(P->d, P->n, CUFFT_Z2D, P->inv);
    pruned_fft_teardown(*P, P->ctx->stream);
    if (P->cap_stream) cudaStreamDestroy(P->cap_stream);
    sk_free(P->w_sorted); sk_free(P->t_sorted);
    sk_free(P->a_s); sk_free(P->b_s); sk_free(P->u_s); sk_free(P->v_s);
    sk_free(P->red); sk_free(P->red_out); sk_free(P->flag); sk_free(P->box_buf); sk_free(P->det_acc);
    sk_free(P->fc_tw);
    pinned_release(P->host_red);
    delete (WinPoly*)P->winpoly;
    delete P;
    return SK_OK;
}

// One fast summation on sorted data: transpose 0: sources y (side 1) -> targets x (side 0).
int apply_sorted(Plan& P, int transpose, int kernel, const double* w_sorted, double* t_sorted,
                 const FusedUpd* fu) {
    cudaStream_t s = P.ctx->stream;
    const int src = transpose ? 0 : 1, dst = transpose ? 1 : 0;
    prof_begin(ST_SPREAD, s);
    GridAcc ga;
    unsigned* slot = nullptr;
    if (P.fftconv2) SK_TRY(launch_spread(P, src, w_sorted, P.grid, s, &ga, &slot));   // conversion in K1
    else SK_TRY(launch_spread(P, src, w_sorted, P.grid, s));   // writes every grid cell
    prof_end(ST_SPREAD, s);
    if (P.box_exchange) {
        // a3: sum the partial grids of all ranks over the touched box only (pack, NCCL
        // all-reduce, unpack; with one rank and SK_FORCE_BOX_EXCHANGE the grid is cleared
        // in between, which checks that the box holds every nonzero)
        prof_begin(ST_ALLREDUCE, s);
        SK_TRY(launch_box_copy(P, P.grid, P.box_buf, 0, s));
        SK_TRY(allreduce_sum(P.ctx, P.box_buf, P.box_size));
        if (P.ctx->world == 1) SK_CUDA(cudaMemsetAsync(P.grid, 0, sizeof(double) * P.grid_size, s));
        SK_TRY(launch_box_copy(P, P.grid, P.box_buf, 1, s));
        prof_end(ST_ALLREDUCE, s);
    }
    if (P.fftconv2) {
        prof_begin(ST_FFT_FWD, s);
        SK_TRY(fftconv2_apply(P, kernel, ga, slot, s));
        prof_end(ST_FFT_FWD, s);
    } else if (P.pruned) {
        SK_TRY(pruned_fft_apply(P, kernel, s));
    } else {
        prof_begin(ST_FFT_FWD, s);
        SK_CUFFT(cufftExecD2Z(P.fwd, P.grid, P.spec));
        count_launch();
        prof_end(ST_FFT_FWD, s);
        prof_begin(ST_MULTIPLY, s);
        SK_TRY(launch_multiply(P, kernel, s));
        prof_end(ST_MULTIPLY, s);
        prof_begin(ST_FFT_INV, s);
        SK_CUFFT(cufftExecZ2D(P.inv, P.spec, P.grid));
        count_launch();
        prof_end(ST_FFT_INV, s);
    }
    auto nearfield = [&]() -> int {   // r = 1: the near-field correction, its own profiled stage
        prof_begin(ST_NEARFIELD, s);
        const double* wn = w_sorted;
        const NodeSet& Ssrc = P.side[src];
        if (Ssrc.g_u) {   // across ranks: every rank's source weights, in the gathered sources' order
            SK_TRY(allgather_concat(P.ctx, w_sorted, Ssrc.count, Ssrc.g_counts, Ssrc.g_wcat));
            SK_TRY(launch_gather_rows(Ssrc.g_wcat, Ssrc.g_total, Ssrc.g_perm, Ssrc.g_total, 1, Ssrc.g_w, s));
            wn = Ssrc.g_w;
        }
        SK_TRY(launch_nearfield(P, src, dst, kernel, wn, t_sorted, s));
        prof_end(ST_NEARFIELD, s);
        return SK_OK;
    };
    prof_begin(ST_INTERP, s);
    if (fu && fu->x) {
        // the caller wants x = p / t: fused into the DMMA (or d = 1) interpolation when it can be
        if ((P.dmma || P.d == 1) && P.rpow == 2) {
            SK_TRY(launch_interp(P, dst, P.grid, t_sorted, s, *fu));
            prof_end(ST_INTERP, s);
        } else {
            SK_TRY(launch_interp(P, dst, P.grid, t_sorted, s));
            prof_end(ST_INTERP, s);
            if (P.rpow == 1) SK_TRY(nearfield());
            SK_TRY(launch_update(P, dst, t_sorted, fu->p, fu->x, 0, fu->iter, fu->iter_dev, s));
        }
    } else {
        SK_TRY(launch_interp(P, dst, P.grid, t_sorted, s));
        prof_end(ST_INTERP, s);
        if (P.rpow == 1) SK_TRY(nearfield());
    }
    return SK_OK;
}

}  // namespace sk
