// sk_internal.cuh -- internal types of libsk_nfft (B200 / sm_100a).
// Product code: shares nothing with oracle/ (see DESIGN.md "Boundary").
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>
#include <string>

#include "../../include/sinkhorn_nfft.h"

namespace sk {

constexpr int kMaxD = 3;
constexpr int kMaxRanks = 64;        // r = 1 across ranks: per-rank node counts kept on the host
constexpr int kMaxW = 16;            // 2 * m_w taps per axis, m_w <= 8
constexpr int kXPairMaxDensity = 96; // x-pair spread segments when nodes per cell < this
constexpr double kLampDegenerate = 1e-16;   // lambda' of a zero-diameter geometry (reading Q6b)
constexpr bool kDeterministicDefault = true;    // spread mode when SK_DETERMINISTIC is unset

// Thread-local error message + status helpers (api.cu).
int set_error(int code, const std::string& msg);
#define SK_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return ::sk::set_error(SK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define SK_CUFFT(call)                                                                 \
    do {                                                                               \
        cufftResult r_ = (call);                                                       \
        if (r_ != CUFFT_SUCCESS)                                                       \
            return ::sk::set_error(SK_ECUFFT, std::string(#call) + ": cufft error " + std::to_string((int)r_)); \
    } while (0)
#define SK_TRY(call)                                                                   \
    do { int s_ = (call); if (s_ != SK_OK) return s_; } while (0)

void count_launch(long long k = 1);

// Programmatic dependent launch (sm_90+) on the per-apply kernel chain (spread -> FFT stages ->
// interp): a kernel launched with launch_pdl may be scheduled while its predecessor in the stream
// still runs; it must call pdl_wait() before touching memory the predecessor writes or reads, and
// triggers its own successor's launch with pdl_trigger(). Kernels launched without the attribute
// see both as no-ops. SK_NO_PDL=1 launches plainly (A/B).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef SK_PDL_EARLY
#define SK_PDL_EARLY 0   // 1: trigger at kernel start (measured slower on c2 / images: the waiting
                         // successor CTAs take SM slots); 0: implicit trigger at block exit
#endif
__device__ __forceinline__ void pdl_trigger() {
    if (SK_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// Caching device allocator (api.cu): stream-ordered reuse of freed blocks.
int dev_alloc(void** out, size_t bytes, cudaStream_t s);
void dev_free(void* p, cudaStream_t s);
void dev_cache_release();

// Kaiser-Bessel window parameters in oversampled-grid units (reading Q10).
struct Window {
    int m;            // cutoff: support |u| < m, 2m taps per axis
    double beta;      // pi (2 - 1/sigma)
    double m2;        // m*m
    double inv_pi;    // 1/pi
};

// One node set (x or y) of the local rank, sorted by tile key.
struct NodeSet {
    long long count = 0;      // local nodes
    long long total = 0;      // nodes over all ranks
    double* u = nullptr;      // [d][count] grid coordinates n*(x'_a + 1/2), sorted order (SoA)
    int* perm = nullptr;      // [count] sorted position -> caller index
    int* cell_key = nullptr;  // [count] sort key (scratch after plan)
    // tile decomposition (bins) for the tiled spread/gather kernels
    int* tile_start = nullptr;   // [ntiles + 1] CSR offsets into the sorted order
    int ntiles = 0;
    void* items = nullptr;       // TileItem[nitems] work list of the tiled kernels (size-sorted)
    int nitems = 0;
    // DMMA path (d = 3, W = 12): per-cell work lists
    void* batches = nullptr;     // CellBatch[nbatches]: <= 32 nodes of one cell (interp)
    int nbatches = 0;
    int ncells = 0;              // non-empty cells
    bool xpairs = false;         // spread segments span x-pairs of cells (sparse cells, d = 3)
    bool seg_dense = false;      // 64-node spread segments on 2 warp pairs (dense cells, d = 3)
    void* segs = nullptr;        // CellBatch[nsegs]: <= kSegMax nodes of one cell (spread)
    int nsegs = 0;
    void* sitems = nullptr;      // SpreadItem[nsitems]: segments of one 2^3 super-tile (spread)
    int nsitems = 0;
    double* taps = nullptr;      // [count][d][2 m_w] window taps of every node (sorted order)
    // r = 1, d >= 2: near-field work list, <= kNearChunk consecutive targets of one tile row each
    void* near_items = nullptr;  // NearItem[n_near]
    int n_near = 0;
    // r = 1 across ranks: every rank's nodes of this side as near-field sources (plan.cu,
    // build_near_global): gathered grid coordinates sorted like a local side, the sorted ->
    // concatenated (rank-major, each rank's sorted order) map, and per-apply weight buffers
    long long g_total = 0;
    double* g_u = nullptr;         // [d][g_total]
    int* g_tile_start = nullptr;   // [ntiles + 1]
    int* g_perm = nullptr;         // [g_total] position in the concatenation
    double* g_wcat = nullptr;      // [g_total] all-gathered weights (concatenation)
    double* g_w = nullptr;         // [g_total] weights in g_u's order
    long long g_counts[kMaxRanks] = {};   // nodes per rank
};
// consecutive targets of tiles tile .. tile_last of one row along the last axis
struct NearItem { int tile, start, count, tile_last; };
constexpr int kNearChunk = 64;

struct Ctx {
    int device = 0;
    int rank = 0;
    int world = 1;
    cudaStream_t stream = nullptr;
    void* nccl_comm = nullptr;    // ncclComm_t when world > 1 (or the one-rank NCCL path)
    bool emulated = false;        // SK_EMULATE_WORLD test hook: `world` identical ranks, no NCCL
};

struct Plan {
    Ctx* ctx = nullptr;
    int d = 0;
    int N = 0;                // bandwidth per axis
    int n = 0;                // oversampled grid per axis (sigma N)
    double sigma = 2.0;
    Window win{};
    double lambda = 0, lambda_p = 0, rho = 1, L = 0, eps_B = 0;
    int rpow = 2;             // cost |x - y|^r, r in {1, 2}
    // r = 1 (NEXT-2): inner regularisation K_I on |x'| <= near_a (torus units) and the
    // near-field correction sum over |x'_i - y'_j| < near_a of w_j (K - K_I)
    int near_cells = 0;
    double near_a = 0.0;
    double ki[2][16] = {};    // K_I coefficients in (r / near_a)^2, kernels 0 and 1
    // d = 1 with a near field: nodes sorted by position (key = floor(u 2^fine_shift)), not only by
    // tile, so a chunk of consecutive targets has one contiguous source range (0 = tile sort)
    int fine_shift = 0;
    // d >= 2 with a near field: nodes sorted by (tile, cell within the tile), so the 64 targets
    // of a near-field item (and each warp's 32) sit in a few adjacent cells
    bool near_cell_sort = false;
    int ki_n = 0;
    int p_smooth = 8;
    double centre[kMaxD] = {0, 0, 0};
    // plan-time accuracy report (fastsum_plan_info): sum of |b_k| that the N-band drops, measured
    // on the (2N)^d sampling grid, per kernel (bounds |K~ - K~_N| pointwise)
    double acc_tail[2] = {0.0, 0.0};
    long long grid_size = 0;  // n^d
    long long spec_size = 0;  // n^{d-1} (n/2 + 1)
    long long band_size = 0;  // (N+1)^{d-1} (N/2 + 1)
    NodeSet side[2];          // 0 = x (targets of K v), 1 = y (sources of K v)
    double* grid = nullptr;             // [n^d] real
    cufftDoubleComplex* spec = nullptr; // [spec_size]
    double* D[2] = {nullptr, nullptr};  // multiplier tables (kernel 0, 1) over the half band
    double* bk[2] = {nullptr, nullptr}; // b_k on the full band (N+1)^d (diagnostics)
    cufftHandle fwd = 0, inv = 0;
    cudaStream_t cap_stream = nullptr;  // private stream for CUDA-graph capture of iterations
    // NEXT-4 pruned FFT (d = 3, pruned_fft.cu): batched 1-D transforms over box rows / band rows
    bool pruned = false;
    long long pr_rows_z = 0, pr_rows_y = 0, pr_rows_x = 0;
    double* pr_A = nullptr;
    void *pr_Z = nullptr, *pr_Y = nullptr, *pr_X = nullptr;   // cufftDoubleComplex buffers
    cufftHandle pr_fz = 0, pr_iz = 0, pr_y = 0, pr_x = 0;
    // d = 2 shared-memory FFT convolution (fftconv2.cu): replaces D2Z / multiply / Z2D and the
    // deterministic conversion; twiddle table [n/2] complex
    bool fftconv2 = false;
    double* fc_tw = nullptr;
    // scratch
    double* w_sorted = nullptr;   // [max count]
    double* t_sorted = nullptr;   // [max count]
    double* red = nullptr;        // block partials
    double* red_out = nullptr;    // reduced scalars (device)
    double* host_red = nullptr;   // pinned host mirror
    int* flag = nullptr;          // [4] graph iteration counter; 8-byte aligned [8..11]: bad64
    unsigned long long* bad64 = nullptr;   // [side] first non-positive denominator, packed
                                           // (iteration << 40 | rank << 32 | sorted index), atomicMin
    // Sinkhorn state in sorted order
    double* a_s = nullptr; double* b_s = nullptr; double* u_s = nullptr; double* v_s = nullptr;
    long long max_count = 0;
    // a3 exchange: the grid cells any node's window can touch form one box (same on all
    // ranks, from the global bbox); only the box is all-reduced (c5: 77^3 of 256^3 cells)
    int box_lo[kMaxD] = {0, 0, 0};
    int box_n[kMaxD] = {1, 1, 1};
    long long box_size = 0;
    double* box_buf = nullptr;   // packed box (world > 1, or SK_FORCE_BOX_EXCHANGE)
    bool box_exchange = false;
    int tile_cells = 0;       // tile edge in grid cells (per axis)
    int tiles_per_axis = 0;
    bool tiled = false;       // v2 tiled spread/interp usable (d = 3, 2 m_w in {12, 16})
    bool dmma = false;        // FP64 tensor-core spread/interp (d = 3, 2 m_w = 12)
    bool spread_tmapad = false;  // d = 3 spread: the padded DMMA spread on TMA-fed warp pairs
    bool spread_pipe = true;     // its full / empty mbarrier pipeline (SK_SPREAD3_NOPIPE=1: pair barriers)
    // deterministic spread (GridAcc): fixed-point box accumulator [box_size][2] + 1 word max |w|
    bool deterministic = false;
    unsigned long long* det_acc = nullptr;   // [2 box_size] accumulator, then 8 uint: 4 bound slots,
    unsigned* det_wmax = nullptr;            // the conversion's block counter (zeroed at plan time)
    double phi0d = 1.0;          // phi(0)^d: the largest product of d window taps
    bool spread_xpairs = false;  // d = 3 padded spread: x-minor keys; sides with sparse cells group
                                 // x-pairs of cells into one segment (13 of 16 rows)
    void* winpoly = nullptr;  // host WinPoly (window tap polynomials)
};

// Spread output (a2). Default: FP64 atomics straight into the grid (the order of the adds, hence
// the last bits, varies from run to run). Deterministic mode (acc != nullptr): every spread
// contribution v is rounded once to an integer multiple of 2^-S, X = rint(v 2^S), and added as
// two 64-bit integer words X = hi 2^32 + lo (hi signed, lo in [0, 2^32)) into a fixed-point
// accumulator over the touched box; integer addition is associative, so the sum does not depend
// on the order and the grid is bit-identical from run to run. S = 61 - ilogb(B phi(0)^d) with
// B >= max_j |w_j| (B from the high 32 bits of max |w|, at most 2x above it): one node contributes
// < 2^62 and a cell sum of <= 2^31 nodes stays < 2^93 (hi < 2^61, the lo sum of <= 2^31
// contributions < 2^63); the rounding is <= 2^-62 of the largest single-node contribution.
// The kernel that produces a spread's source vector (the permutation into sorted order, the
// fused Sinkhorn update) records B (note_absmax) in the vector's bound slot; grid_fix_convert
// writes the grid back as FP64, clears the accumulator and the slot.
struct GridAcc {
    double* grid = nullptr;                 // [n^d] FP64 (atomic mode; conversion target)
    unsigned long long* acc = nullptr;      // deterministic: [box cells][2] (hi, lo)
    const unsigned int* wmax = nullptr;     // deterministic: high 32 bits of max_j |w_j| (device)
    double phi0d = 1.0;                     // phi(0)^d, the largest product of d taps
    int n = 0;                              // grid edge
    int lo[3] = {0, 0, 0};                  // box origin and extent per axis
    int bn[3] = {1, 1, 1};
};
// bound slots of the deterministic spread's source vectors (Plan::det_wmax[k])
enum { WSLOT_W = 0, WSLOT_U = 1, WSLOT_V = 2, WSLOT_TMP = 3, kWSlots = 4 };
#ifdef __CUDACC__
// high 32 bits of |x| (monotone in |x| for doubles; NaN sorts above every number)
__device__ __forceinline__ unsigned absmax_hi(double x) {
    return (unsigned)((unsigned long long)__double_as_longlong(fabs(x)) >> 32);
}
// max of the converged lanes' values into a bound slot (one atomic per warp)
__device__ __forceinline__ void note_absmax(unsigned* slot, unsigned hi) {
    const unsigned mask = __activemask();
    const unsigned mx = __reduce_max_sync(mask, hi);
    if ((int)(threadIdx.x & 31) == __ffs(mask) - 1 && mx) atomicMax(slot, mx);
}
// 2^S of the deterministic mode (1 in atomic mode, for all-zero or non-finite weights)
__device__ __forceinline__ double grid_scale(const GridAcc& g) {
    if (!g.acc) return 1.0;
    const unsigned hi = *g.wmax;
    const double c = __longlong_as_double((long long)(((unsigned long long)hi << 32) | 0xffffffffULL)) * g.phi0d;
    return (hi != 0 && isfinite(c)) ? ldexp(1.0, 61 - ilogb(c)) : 1.0;
}
// v 2^S as the two words (hi, lo) of the fixed-point accumulator: X = hi 2^32 + lo
__device__ __forceinline__ void fixed_words(double v, double scale, unsigned long long& hi, unsigned long long& lo) {
    const double X = v * scale;                              // exact (power of 2)
    const double h = floor(X * 2.3283064365386963e-10);      // X / 2^32, exact
    const double l = rint(X - h * 4294967296.0);             // low part in [0, 2^32], exact before rint
    hi = (unsigned long long)(long long)h;
    lo = (unsigned long long)l;
}
template <int D>
__device__ __forceinline__ void grid_add(const GridAcc& g, double scale, int x, int y, int z, double v) {
    if (!g.acc) {
        long long i = x;
        if (D >= 2) i = i * g.n + y;
        if (D >= 3) i = i * g.n + z;
        atomicAdd(&g.grid[i], v);
        return;
    }
    long long i = x - g.lo[0];
    if (D >= 2) i = i * g.bn[1] + (y - g.lo[1]);
    if (D >= 3) i = i * g.bn[2] + (z - g.lo[2]);
    unsigned long long h, l;
    fixed_words(v, scale, h, l);
    atomicAdd(&g.acc[2 * i], h);
    atomicAdd(&g.acc[2 * i + 1], l);
}
#endif

// SK_ENONPOS event record: one 64-bit word per side, the minimum over events of
// (iteration << 40 | rank << 32 | sorted index), so the reported (iteration, rank, index) is one
// event -- the earliest iteration, then the lowest rank and index -- and a min all-reduce over
// ranks keeps that property.
constexpr unsigned long long kNoBad = ~0ULL;
#ifdef __CUDACC__
// (out of line: the failure path stays out of the interpolation epilogue's schedule)
static __device__ __noinline__ void record_bad(unsigned long long* bad, int iter, int rank, long long idx) {
    const unsigned long long v = ((unsigned long long)(unsigned)iter << 40) |
                                 ((unsigned long long)(rank & 0xff) << 32) | (unsigned long long)(idx & 0xffffffffLL);
    atomicMin(bad, v);
}
#endif

// Optional u/v update fused into the interpolation epilogue (a7): with x != nullptr the
// interpolation writes x[i] = p[i] / t_i instead of t_i and flags t_i <= 1e-300 (SK_ENONPOS,
// record_bad). Used when no residual or trace is wanted.
struct FusedUpd {
    const double* p = nullptr;
    double* x = nullptr;
    unsigned long long* bad = nullptr;   // packed first non-positive t (record_bad)
    const int* iter_dev = nullptr;       // graph replay: iteration number on the device
    unsigned* xmax = nullptr;            // deterministic spread: bound slot of x (note_absmax)
    int iter = 0;
    int rank = 0;
};
#ifdef __CUDACC__
__device__ __forceinline__ void emit_t(double* __restrict__ t_out, const FusedUpd& fu, long long idx, double t) {
    if (fu.x) {
        if (!(t > 1e-300) || !isfinite(t)) record_bad(fu.bad, fu.iter_dev ? *fu.iter_dev : fu.iter, fu.rank, idx);
        const double x = fu.p[idx] / t;
        fu.x[idx] = x;
        if (fu.xmax) note_absmax(fu.xmax, absmax_hi(x));
    } else {
        t_out[idx] = t;
    }
}
#endif

// ---- kernels.cu launchers ----
int launch_bbox(const double* pts, long long count, int d, double* out_minmax /*device [2*d]*/,
                cudaStream_t s);
int launch_scale_key(Plan& P, const double* pts, long long count, int* key, int* idx, int* bad,
                     cudaStream_t s);
int launch_gather_coords(Plan& P, const double* pts, const int* perm, long long count, double* u_sorted,
                         cudaStream_t s);   // rescales the caller's points in sorted order
int launch_tile_offsets(const int* sorted_keys, long long count, int ntiles, int* tile_start,
                        cudaStream_t s);
// keep != nullptr: the deterministic conversion is left to the caller (fftconv2_apply), which
// gets the accumulator descriptor and the source vector's bound slot
int launch_spread(Plan& P, int side, const double* w_sorted, double* grid, cudaStream_t s,
                  GridAcc* keep = nullptr, unsigned** keep_slot = nullptr);
bool fftconv2_supported(int d, int n, int N);
void fftconv2_twiddles(int n, double* out);
int fftconv2_apply(Plan& P, int kernel, const GridAcc& ga, unsigned* slot, cudaStream_t s);
int launch_taps(Plan& P, int side, cudaStream_t s);
int launch_interp(Plan& P, int side, const double* grid, double* t_sorted, cudaStream_t s,
                  const FusedUpd& fu = FusedUpd());   // fu.x only on the DMMA interps (P.dmma)
int launch_multiply(Plan& P, int kernel, cudaStream_t s);
// slot (deterministic spread): cleared, then max |dst| recorded in it (note_absmax)
int launch_permute_in(const double* src, const int* perm, long long count, double* dst, cudaStream_t s,
                      unsigned* slot = nullptr);
unsigned* wslot(Plan& P, int k);   // Plan::det_wmax + k, nullptr in atomic mode
int launch_permute_out(const double* src, const int* perm, long long count, double* dst, cudaStream_t s);
int launch_sample_kernel(Plan& P, int kernel, int M, const double* kb_coef, int kb_deg,
                         double* out, cudaStream_t s);
int launch_band_coeffs(Plan& P, int kernel, int M, const cufftDoubleComplex* B, cudaStream_t s);
// out_dev[0] = sum of the |b_k| outside the N-band (out_dev[1..kUpdBlocks] scratch)
int launch_band_tail(Plan& P, int M, const cufftDoubleComplex* B, double* out_dev, cudaStream_t s);
// Sinkhorn fused update: x_s <- p_s / t (t = interpolated), partial sums into red
int launch_update(Plan& P, int side, const double* t_sorted, const double* p_sorted,
                  double* x_sorted, int want_resid, int iter, const int* iter_dev, cudaStream_t s);
int launch_increment(int* counter_dev, cudaStream_t s);   // counter_dev[0] += 1 (graph iteration counter)
int launch_fill(double* p, long long count, double v, cudaStream_t s);
constexpr int kUpdVals = 4;     // update_kernel partials per block (residual, min t, KL, sum p log x)
constexpr int kUpdBlocks = 592; // update / reduction grid (4 x 148 SMs)
// a3: grid box <-> packed buffer (dir 0: pack grid -> buf, 1: unpack buf -> grid)
int launch_box_copy(const Plan& P, double* grid, double* buf, int dir, cudaStream_t s);
int launch_scale_vec(double* p, long long count, const double* scale_dev, cudaStream_t s,
                     unsigned* slot = nullptr);
int launch_scale_const(double* p, long long count, double c, cudaStream_t s);
int launch_reduce_sum_log(const double* p, const double* x, long long count, double* out_dev,
                          int op, cudaStream_t s);
int launch_rescale_factor(double* r, int policy, double total, cudaStream_t s);
int launch_finalize_partials(const double* red, int nparts, int nvals, double* out, cudaStream_t s);

// ---- plan.cu ----
int build_plan(Ctx* ctx, Plan** out, int d, const double* x, long long n, const double* y,
               long long m, double lambda, int N, double sigma, int m_w, double eps_B, int p,
               int rpow, int near_cells);
int launch_key_to_tile(Plan& P, int* key, long long count, cudaStream_t s);
int launch_near_keys(Plan& P, const double* U, long long total, int* key, int* idx, cudaStream_t s);
int launch_gather_rows(const double* in, long long in_ld, const int* perm, long long count, int rows, double* out,
                       cudaStream_t s);   // out[r][j] = in[r * in_ld + perm[j]]
int launch_nearfield(Plan& P, int src, int dst, int kernel, const double* w_sorted, double* t_sorted,
                     cudaStream_t s);
int destroy_plan(Plan* P);
void plan_set_stream(Plan& P, cudaStream_t s);   // cufftSetStream on all of the plan's handles
void fft_pool_release();   // destroy the pooled cuFFT handles (sk_release_cache)
// ---- pruned_fft.cu (NEXT-4) ----
int pruned_fft_setup(Plan& P, cudaStream_t s);      // sets P.pruned when the box pays
void pruned_fft_teardown(Plan& P, cudaStream_t s);
int pruned_fft_apply(Plan& P, int kernel, cudaStream_t s);   // a4 + a5 + a6 on P.grid in place
int fft_acquire(int d, int n, cufftType type, cudaStream_t s, cufftHandle* out, long long batch = 1);
void fft_release(int d, int n, cufftType type, cufftHandle h, long long batch = 1);
int apply_sorted(Plan& P, int transpose, int kernel, const double* w_sorted, double* t_sorted,
                 const FusedUpd* fu = nullptr);   // fu: update fused into a7 where supported

// ---- stage profiling (api.cu): CUDA-event pairs around each stage when enabled ----
enum Stage { ST_SPREAD = 0, ST_ALLREDUCE, ST_FFT_FWD, ST_MULTIPLY, ST_FFT_INV, ST_INTERP, ST_UPDATE, ST_PLAN, ST_NEARFIELD, ST_COUNT };
// host wall-clock trace of the plan phases (SK_PLAN_TRACE=1), printed to stderr
void plan_trace(const char* phase, cudaStream_t s);
void prof_begin(int stage, cudaStream_t s);
void prof_end(int stage, cudaStream_t s);
void prof_harvest();

// ---- comm (api.cu) ----
int allreduce_sum(Ctx* c, double* buf, long long count);           // in-place, device
// every rank's `count` local doubles, concatenated in rank order into out (counts[r] per rank);
// emulated world: world copies of the local buffer; one rank: a copy
int allgather_concat(Ctx* c, const double* local, long long count, const long long* counts, double* out);
// per-rank counts of a local quantity (host), via a sum all-reduce of one slot per rank
int gather_counts(Ctx* c, long long local, long long* counts);
int allreduce_minmax(Ctx* c, double* mins, double* maxs, int count); // in-place, device

}  // namespace sk

struct sk_ctx { sk::Ctx c; };
struct sk_plan { sk::Plan* p; };
