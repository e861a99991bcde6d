/*
 * sinkhorn_nfft.h -- C-ABI of the B200-native NFFT fast-summation Sinkhorn library
 * (libsk_nfft.so). Hot path of arXiv 2201.07524, Alg. 2.
 *
 * P:Lx refers to /root/reference/PAPER.md line x. Readings of the paper (Q1..Q15)
 * are listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   - Pointers are DEVICE pointers (CUDA global memory of the context's device) unless
 *     marked "host". Arrays are FP64, C-contiguous; point sets are row-major [count][d].
 *   - The caller owns every array and keeps it alive for the duration of the call.
 *     fastsum_plan copies what it needs (x, y may be freed afterwards).
 *   - Return value: SK_OK (0) or one of the SK_E* codes below; the message of the last
 *     failure on the calling thread is returned by sk_last_error(). On error no output
 *     array is guaranteed to be written.
 *   - Work is enqueued on the context's CUDA stream (sinkhorn_init). fastsum_apply,
 *     nfft_spread and nfft_interp are asynchronous; calls returning host scalars
 *     (sinkhorn_run, sinkhorn_divergence, sinkhorn_solve) synchronise that stream.
 *   - SPMD multi-GPU: every rank calls every entry point with its local shard of the
 *     points/weights (contiguous index ranges); world_size > 1 uses NCCL (loaded at
 *     run time) for the grid all-reduce and scalar reductions.
 *   - A plan serves one stream at a time; distinct plans are independent.
 */
#ifndef SINKHORN_NFFT_H
#define SINKHORN_NFFT_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SK_OK = 0,
    SK_EINVAL = 1,          /* bad argument: d not in {1,2,3}, N odd or < 2, sigma*N not an even
                               integer, sigma*N < 4*m_w, (sigma*N)^d >= 2^31, m_w not in [2,8],
                               lambda <= 0, eps_B not in (0,1/4), p_smooth < 1, count < 0, NULL
                               pointer, weights a / b not all > 0 or not summing to 1 +- 1e-12
                               over all ranks (sinkhorn_run, sinkhorn_solve) ... */
    SK_EGEOMETRY = 2,       /* a node is NaN/Inf or falls outside the ball |x'| <= 1/4 - eps_B/2
                               after scaling ("we assume that |x_j| <= L/2") */
    SK_ENONPOS = 3,         /* a fast-summation denominator t_i <= 1e-300 (or non-finite) in an
                               update alpha_i = p_i / t_i (Alg. 2); run info holds the
                               first (iteration, caller-order index) */
    SK_ENOTCONVERGED = 4,   /* tol > 0 and the residual (Eq. (Error)) is still > tol after
                               `iters` iterations; outputs are valid */
    SK_ECUDA = 5,
    SK_ECUFFT = 6,
    SK_ENCCL = 7,
    SK_ENOMEM = 8
};

typedef struct sk_ctx*  sk_ctx_t;   /* owns: NCCL communicator (world > 1); borrows: the stream */
typedef struct sk_plan* sk_plan_t;  /* owns: sorted node copies, permutations, grid, spectrum,
                                       multiplier tables, cuFFT plans, scratch */

typedef struct {
    int       iters_done;        /* full iterations completed (1 iteration = u- then v-update) */
    double    residual;          /* ||pi 1 - a||_1 + ||pi^T 1 - b||_1 (Eq. (Error)) of the
                                    iterate entering the last iteration's u-update, i.e. after the
                                    previous v-update (the second term is 0 there);
                                    global over ranks */
    int       bad_iter;          /* SK_ENONPOS: iteration (0-based) of the first non-positive
                                    denominator over all ranks; -1 otherwise */
    long long bad_index;         /* SK_ENONPOS: its caller-order index, local to rank bad_rank
                                    (-1 on the other ranks) */
    double    kappa_log10_est;   /* log10( ||v||_1 / min_i (K v)_i ) at the last u-update: the
                                    conditioning that amplifies the absolute fast-summation error
                                    (DESIGN.md "Conditioning"); global over ranks */
    double    seconds;           /* device time of the iteration loop (CUDA events) */
    double    kappa_u_log10_est; /* log10( ||u||_1 / min_j (K^T u)_j ) at the last v-update */
    int       bad_side;          /* SK_ENONPOS: 0 = u-update (K v), 1 = v-update (K^T u); -1 otherwise */
    int       bad_rank;          /* SK_ENONPOS: rank holding the node; -1 otherwise. (bad_iter,
                                    bad_side, bad_rank, bad_index) describe one event: the earliest
                                    iteration, u before v, then the lowest rank and sorted index */
} sk_run_info;

/* Create a context on `device` (the current CUDA device is switched to it). rank/world_size
 * describe the SPMD job; nccl_unique_id: 128-byte ncclUniqueId (host) from
 * sk_nccl_unique_id() on rank 0, broadcast by the caller; required when world_size > 1. With
 * world_size == 1 it may be NULL (no communicator) or an id, which creates a one-rank NCCL
 * communicator: every collective (bbox min/max, box exchange, scalar sums) then runs through
 * NCCL as the identity, i.e. the multi-rank NCCL code path on one GPU.
 * cuda_stream: cudaStream_t to enqueue on (NULL = legacy default stream).
 * Test hook: with world_size == 1 and the environment variable SK_EMULATE_WORLD=k (k >= 2) the
 * context behaves as k ranks holding identical shards (every sum over ranks is k times the
 * local one, min/max are unchanged, no NCCL), which exercises every multi-rank code path
 * (global counts, box exchange, scalar all-reduces) on one GPU. */
int sinkhorn_init(sk_ctx_t* ctx, int device, int rank, int world_size,
                  const void* nccl_unique_id, void* cuda_stream);
int sinkhorn_finalize(sk_ctx_t ctx);
/* Rank 0: write a fresh ncclUniqueId (128 bytes, host) into out. Loads NCCL. */
int sk_nccl_unique_id(void* out);

/* Plan the fast summation of Eq. (fastsum) for the node sets x (targets of K v)
 * and y (sources of K v):
 *   geometry (reading Q6 of P:L479-486): centre = midpoint of bbox(x u y) over all ranks,
 *     rho = L / diag(bbox), L = 1/2 - eps_B, x' = rho (x - centre) lies in |x'| <= L/2,
 *     lambda' = lambda / rho^2 (so exp(-lambda |x-y|^2) = exp(-lambda' |x'-y'|^2));
 *   regularised kernel K~ with two-point Taylor K_B of order p_smooth on
 *     (L, 1/2], its Fourier coefficients b_k on the centred N-band (reading Q9)
 *     for K = exp(-lambda c) and for c K (divergence kernel, reading Q1);
 *   Kaiser-Bessel window, oversampled grid n = sigma*N per axis, 2*m_w taps per axis.
 * x: [n_local][d], y: [m_local][d] (device, caller order). Counts may be 0 on some ranks. */
int fastsum_plan(sk_ctx_t ctx, sk_plan_t* plan, int d,
                 const double* x, long long n_local, const double* y, long long m_local,
                 double lambda, int N, double sigma, int m_w, double eps_B, int p_smooth);

/* Extended plan: the cost |x - y|^r for r in {1, 2}.
 * r = 2 is fastsum_plan. r = 1 is the Laplace kernel exp(-lambda |x - y|) (P:L456-470 with
 * r = 1): lambda' = lambda / rho; the kernel is also regularised at 0 by
 *   K_I(r) = sum_{i < p_smooth} c_i (r / a)^{2i} on r <= a = near_cells / (sigma N) (torus
 *   units), K_I^{(k)}(a) = K^{(k)}(a) for k < p_smooth (even, so smooth at 0),
 * the Fourier series is built from K_I | K | K_B, and every fast summation adds the near field
 *   t_i += sum over |x'_i - y'_j| < a of w_j (K - K_I)(|x'_i - y'_j|)
 * (direct sum over the source tiles around each target). The divergence kernel c K uses
 * c = |x - y| in original units. r = 1 runs the same spread / interp kernels as r = 2.
 * Across ranks (world_size > 1) the near field of a target needs every source within the radius,
 * wherever it lives: the plan all-gathers each side's scaled coordinates once (ncclBroadcast per
 * rank, rank-major) and every r = 1 fast summation all-gathers the source weights; the far field
 * stays the grid all-reduce. Memory: every rank holds all nodes' coordinates for the near field.
 * Errors: SK_EINVAL for r not in {1, 2}, near_cells < 1, p_smooth > 8 (r = 1; the monomial K_I system is ill-conditioned beyond),
 * a >= 1/2 - eps_B, or r = 1 with more than 64 ranks; SK_ENCCL if libnccl lacks ncclBroadcast;
 * otherwise as fastsum_plan. */
typedef struct {
    double lambda;
    int    r;             /* 1 or 2 */
    int    N;
    double sigma;
    int    m_w;
    double eps_B;
    int    p_smooth;
    int    near_cells;    /* r = 1: near-field radius in oversampled-grid cells */
} sk_plan_opts;
int fastsum_plan_ex(sk_ctx_t ctx, sk_plan_t* plan, int d, const double* x, long long n_local,
                    const double* y, long long m_local, const sk_plan_opts* opts);
int fastsum_plan_destroy(sk_plan_t plan);

/* One fast-summation matvec (Eq. (matexp)/(matexpt)):
 *   transpose = 0: t_i = sum_j w_j K(x_i, y_j)   (w: [m_local], t: [n_local])
 *   transpose = 1: t_j = sum_i w_i K(x_i, y_j)   (w: [n_local], t: [m_local])
 *   kernel 0: K = exp(-lambda |x-y|^2);  kernel 1: K = |x-y|^2 exp(-lambda |x-y|^2).
 * Sums run over all ranks' sources; t covers the local targets. Caller order. Async. */
int fastsum_apply(sk_plan_t plan, int transpose, int kernel, const double* w, double* t);

/* Alg. 2 for `iters` iterations (u-update then v-update, reading Q2/Q3):
 *   u <- a / (K v), v <- b / (K^T u)   (each K product = one fast summation)
 * u, v: in = starting values (all-ones for a cold start), out = final scalings,
 * caller order. tol > 0 stops early once the residual <= tol (checked every iteration);
 * tol == 0 runs exactly `iters` (< 2^24). a and b are checked first: every entry > 0 and each
 * summing to 1 +- 1e-12 over all ranks, else SK_EINVAL. SK_ENONPOS: some t_i <= 1e-300 (or
 * non-finite) in an update; all ranks return it, info describes the first event. rescale_policy (Eq. (scale), reading Q4):
 * 0 none, 1 v <- v / geomean(v), 2 v <- v / max(v) before every u-update. info: host,
 * may be NULL. Synchronises the stream. */
int sinkhorn_run(sk_plan_t plan, const double* a, const double* b, int iters, double tol,
                 int rescale_policy, double* u, double* v, sk_run_info* info);

/* (sinkhorn_run with tol == 0, no profiling and iters > 2 captures one iteration as a CUDA
 * graph on a plan-private stream and replays it iters-1 times on the context stream.) */

/* sinkhorn_run plus per-iteration convergence diagnostics (Sec. 3.3
 * P:L312-424). trace: HOST array of 6 * iters doubles, iteration k (0-based) at trace[6k..]:
 *   [0] ||pi 1 - p||_1 of the iterate before the u-update (row part of Eq. (Error) P:L333;
 *       its column part is 0 there), [1] D_KL(p | pi 1) at that iterate (Lemma
 *       f decreases by exactly this), [2] sum_i p_i log alpha_i after the update,
 *   [3..5] the same for the v-update: ||pi^T 1 - p~||_1, D_KL(p~ | pi^T 1), sum_j p~_j log alpha~_j.
 * After any half-step the objective (Eq. (objfunc), unnormalised k) is
 * f = 1 - sum p log alpha - sum p~ log alpha~. Entries of iterations not run (tol stop) are NaN.
 * Sums over all ranks. Costs two extra log() per node and half-step. */
int sinkhorn_run_trace(sk_plan_t plan, const double* a, const double* b, int iters, double tol,
                       int rescale_policy, double* u, double* v, sk_run_info* info, double* trace);

/* Divergences at (u, v) (reading Q1):
 *   s_dual = 1/lambda + (1/lambda) (sum a log u + sum b log v) - (1/lambda) sum_j (K^T u)_j v_j
 *            (Eq. (14) P:L211 / Alg. 2 result line P:L732; 2 fast summations incl. K^T u)
 *   s_cost = sum_i u_i ((c K) v)_i = sum_ij pi_ij c_ij (Def 3.1)
 * s_dual, s_cost: host. Global over ranks. Synchronises the stream. */
int sinkhorn_divergence(sk_plan_t plan, const double* a, const double* b, const double* u,
                        const double* v, double* s_dual, double* s_cost);

/* End-to-end solve: plan + Alg. 2 (cold start) + divergences + destroy. inputs_on_host != 0:
 * x, y, a, b are HOST arrays (copied to the device inside the call); else device arrays.
 * s_dual, s_cost, info: host. */
int sinkhorn_solve(sk_ctx_t ctx, int d, const double* x, long long n_local, const double* y,
                   long long m_local, const double* a, const double* b, double lambda, int N,
                   double sigma, int m_w, double eps_B, int p_smooth, int iters,
                   int inputs_on_host, double* s_dual, double* s_cost, sk_run_info* info);

/* ---- stage entry points (the NFFT building blocks of P:L473-477; used by parity tests) ----
 * side 0 = the x nodes, side 1 = the y nodes. Grid: real [n]^d, row-major (axis 0 slowest),
 * grid index l <-> torus position l/n - 1/2 of the scaled node x' (reading Q6).
 * nfft_spread: g[l] = sum_j w_j prod_a phi(n (x'_ja + 1/2) - l_a)   (adjoint-NFFT gridding)
 * nfft_interp: t_j = sum_l g[l] prod_a phi(n (x'_ja + 1/2) - l_a)   (NFFT interpolation)
 * phi = Kaiser-Bessel window in grid units (reading Q10). Local nodes only, no all-reduce.
 * w, t: caller order. Async. */
int nfft_spread(sk_plan_t plan, int side, const double* w, double* grid);
int nfft_interp(sk_plan_t plan, int side, const double* grid, double* t);

/* Plan-time quantities (host outputs):
 * fastsum_plan_info: out[0..2] centre, out[3] rho, out[4] lambda', out[5] L, out[6] n = sigma N,
 *   out[7] band length per axis (N+1), out[8] d, out[9] total nodes x (all ranks),
 *   out[10] total nodes y (all ranks), out[11..13] first grid index of the exchange box per
 *   axis, out[14..16] its extent per axis (the cells any node window touches; only this box
 *   is all-reduced across ranks), out[17] box cells; accuracy report of the plan:
 *   out[18], out[19] sum of |b_k| of K~ (kernel 0, 1) outside the N-band, measured on the (2N)^d
 *   sampling grid (a pointwise bound on the Fourier truncation |K~ - K~_N|, absolute: kernel 0
 *   has K(0) = 1); out[20] K(L) = exp(-lambda' L^r) (the regularisation K_B of P:L481-502 is
 *   inert when this is negligible); out[21] exp(-pi^2 (N/2)^2 / lambda') (r = 2: the first
 *   dropped Gaussian coefficient ratio; NaN for r = 1). out must hold 22 doubles.
 * fastsum_coefficients: b (host, (N+1)^d, index prod over axes of (k_a + N/2), row-major):
 *   the Fourier coefficients b_k of K~_per (kernel 0 or 1) on k in {-N/2..N/2}^d. */
int fastsum_plan_info(sk_plan_t plan, double* out);
int fastsum_coefficients(sk_plan_t plan, int kernel, double* b);

/* Number of CUDA kernels this library launched in the calling process (for the bench's
 * gpu_launches count; cuFFT and NCCL internal kernels are counted per call as 1). */
long long sk_launch_count(void);

/* Stage profiling with CUDA events on the context stream (off by default). sk_profile(1)
 * starts recording an event pair around every stage of every fast summation; sk_profile_read
 * writes out[2k] = number of timed launches and out[2k+1] = their total device milliseconds
 * for stage k = 0 spread, 1 grid all-reduce, 2 forward FFT, 3 multiply, 4 inverse FFT,
 * 5 interp, 6 update, 7 plan (sinkhorn_solve's fastsum_plan), 8 near field (r = 1;
 * nstages <= 9 entries are written); reset != 0 clears the totals. While profiling, sinkhorn_run launches every kernel
 * eagerly (no CUDA-graph replay of iterations). */
void sk_profile(int on);
int sk_profile_read(double* out, int nstages, int reset);

/* Device memory of destroyed plans is cached by the library and reused (best fit, ordered on
 * the allocating stream with events); this returns every cached block to the driver. Call it
 * after fastsum_plan_destroy when the memory is needed elsewhere. The cuFFT handles of
 * destroyed plans are pooled the same way and destroyed here too. */
void sk_release_cache(void);

const char* sk_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SINKHORN_NFFT_H */
