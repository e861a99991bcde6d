// api.cu -- C-ABI entry points of libsk_nfft (declared in include/sinkhorn_nfft.h).
//
// Alg. 2 on top of the fast summation of plan.cu; NCCL (loaded at run
// time with dlopen) for the grid all-reduce and scalar reductions when world_size > 1.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sk_internal.cuh"

namespace sk {

// ---------------------------------------------------------------- errors, launch counter
static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
void count_launch(long long k) { g_launches += k; }
bool pdl_enabled() {
    static const bool on = getenv("SK_NO_PDL") == nullptr;
    return on;
}

// ---------------------------------------------------------------- caching device allocator
// Plans allocate tens of GB (c5: sorted nodes, 52 GB of window taps, grids); cudaMalloc /
// cudaFree of such blocks costs tens of ms and synchronises the device. Freed blocks are kept
// per process and reused best-fit (size in [req, 2 req)); a block freed on stream A carries
// an event that a later user on stream B waits for, so reuse is stream-ordered. On OOM the
// cache is released and the allocation retried.
struct CachedBlock {
    void* p;
    size_t bytes;
    cudaEvent_t ready;
    int device;
};
static std::mutex g_alloc_mu;
static std::multimap<size_t, CachedBlock> g_cache;
static std::map<void*, std::pair<size_t, int>> g_live;   // ptr -> (bytes, device)

static size_t round_bytes(size_t b) {
    const size_t g = b >= (1u << 20) ? (2u << 20) : 512;
    return (b + g - 1) / g * g;
}

void dev_cache_release() {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    for (auto& kv : g_cache) {
        cudaEventSynchronize(kv.second.ready);
        cudaEventDestroy(kv.second.ready);
        cudaFree(kv.second.p);
    }
    g_cache.clear();
}

int dev_alloc(void** out, size_t bytes, cudaStream_t s) {
    *out = nullptr;
    if (bytes == 0) return SK_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t want = round_bytes(bytes);
    {
        std::lock_guard<std::mutex> lk(g_alloc_mu);
        for (auto it = g_cache.lower_bound(want); it != g_cache.end() && it->first < 2 * want; ++it) {
            if (it->second.device != dev) continue;
            CachedBlock blk = it->second;
            g_cache.erase(it);
            cudaStreamWaitEvent(s, blk.ready, 0);
            cudaEventDestroy(blk.ready);
            g_live[blk.p] = {blk.bytes, dev};
            *out = blk.p;
            return SK_OK;
        }
    }
    cudaError_t e = cudaMalloc(out, want);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        dev_cache_release();
        e = cudaMalloc(out, want);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return set_error(e == cudaErrorMemoryAllocation ? SK_ENOMEM : SK_ECUDA,
                         std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_live[*out] = {want, dev};
    return SK_OK;
}

void dev_free(void* p, cudaStream_t s) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) return;
    CachedBlock blk{p, it->second.first, nullptr, it->second.second};
    g_live.erase(it);
    cudaEventCreateWithFlags(&blk.ready, cudaEventDisableTiming);
    cudaEventRecord(blk.ready, s);
    g_cache.emplace(blk.bytes, blk);
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    bool loaded = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;

static int nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.loaded) return SK_OK;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return set_error(SK_ENCCL, std::string("dlopen libnccl.so.2: ") + dlerror());
    g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.errStr = (decltype(g_nccl.errStr))dlsym(h, "ncclGetErrorString");
    g_nccl.broadcast = (decltype(g_nccl.broadcast))dlsym(h, "ncclBroadcast");
    g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
    g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.commDestroy)
        return set_error(SK_ENCCL, "libnccl is missing a required symbol");
    g_nccl.loaded = true;
    return SK_OK;
}

#define SK_NCCL(call)                                                                  \
    do {                                                                               \
        ncclResult_t r_ = (call);                                                      \
        if (r_ != ncclSuccess)                                                         \
            return set_error(SK_ENCCL, std::string(#call) + ": " +                      \
                                           (g_nccl.errStr ? g_nccl.errStr(r_) : "nccl error")); \
    } while (0)

// Emulated world (SK_EMULATE_WORLD=k on a one-process context): k ranks that hold identical
// shards, so a sum over ranks is k times the local value and min/max are the local ones.
// A one-rank NCCL communicator (world_size 1 with an ncclUniqueId) runs every collective
// through NCCL as the identity.
int allreduce_sum(Ctx* c, double* buf, long long count) {
    if (count <= 0) return SK_OK;
    if (c->emulated) return launch_scale_const(buf, count, (double)c->world, c->stream);
    if (!c->nccl_comm) return SK_OK;   // one rank, no communicator
    SK_NCCL(g_nccl.allReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm,
                             c->stream));
    count_launch();
    return SK_OK;
}

int allgather_concat(Ctx* c, const double* local, long long count, const long long* counts, double* out) {
    if (c->emulated || !c->nccl_comm) {   // identical shards (emulated) or one rank
        const int copies = c->emulated ? c->world : 1;
        for (int r = 0; r < copies; ++r)
            if (count > 0)
                SK_CUDA(cudaMemcpyAsync(out + (long long)r * count, local, sizeof(double) * count,
                                        cudaMemcpyDeviceToDevice, c->stream));
        return SK_OK;
    }
    if (!g_nccl.broadcast || !g_nccl.groupStart || !g_nccl.groupEnd)
        return set_error(SK_ENCCL, "libnccl lacks ncclBroadcast / ncclGroupStart / ncclGroupEnd");
    long long off = 0;
    SK_NCCL(g_nccl.groupStart());
    for (int r = 0; r < c->world; ++r) {
        if (counts[r] > 0)
            SK_NCCL(g_nccl.broadcast(r == c->rank ? (const void*)local : (const void*)(out + off), out + off,
                                     (size_t)counts[r], ncclFloat64, r, (ncclComm_t)c->nccl_comm, c->stream));
        off += counts[r];
    }
    SK_NCCL(g_nccl.groupEnd());
    count_launch();
    return SK_OK;
}

int gather_counts(Ctx* c, long long local, long long* counts) {
    if (c->world > kMaxRanks) return set_error(SK_EINVAL, "r = 1 across ranks: at most 64 ranks");
    if (c->emulated || !c->nccl_comm) {
        for (int r = 0; r < c->world; ++r) counts[r] = local;
        return SK_OK;
    }
    std::vector<double> h((size_t)c->world, 0.0);
    h[(size_t)c->rank] = (double)local;
    double* d = nullptr;
    SK_TRY(dev_alloc((void**)&d, sizeof(double) * c->world, c->stream));
    int st = SK_OK;
    if (cudaMemcpyAsync(d, h.data(), sizeof(double) * c->world, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        st = set_error(SK_ECUDA, "gather_counts copy");
    if (!st) st = allreduce_sum(c, d, c->world);
    if (!st && (cudaMemcpyAsync(h.data(), d, sizeof(double) * c->world, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaStreamSynchronize(c->stream) != cudaSuccess))
        st = set_error(SK_ECUDA, "gather_counts copy back");
    dev_free(d, c->stream);
    for (int r = 0; r < c->world && !st; ++r) counts[r] = (long long)llround(h[(size_t)r]);
    return st;
}

int allreduce_minmax(Ctx* c, double* mins, double* maxs, int count) {
    if (count <= 0 || c->emulated || !c->nccl_comm) return SK_OK;
    SK_NCCL(g_nccl.allReduce(mins, mins, (size_t)count, ncclFloat64, ncclMin, (ncclComm_t)c->nccl_comm,
                             c->stream));
    SK_NCCL(g_nccl.allReduce(maxs, maxs, (size_t)count, ncclFloat64, ncclMax, (ncclComm_t)c->nccl_comm,
                             c->stream));
    count_launch(2);
    return SK_OK;
}

// ---------------------------------------------------------------- stage profiling
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> ev[ST_COUNT][2];
    int used[ST_COUNT] = {0};
    double total_ms[ST_COUNT] = {0};
    long long count[ST_COUNT] = {0};
};
static Prof g_prof;

void prof_begin(int st, cudaStream_t s) {
    if (!g_prof.on) return;
    int i = g_prof.used[st];
    if ((int)g_prof.ev[st][0].size() <= i) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        g_prof.ev[st][0].push_back(a);
        g_prof.ev[st][1].push_back(b);
    }
    cudaEventRecord(g_prof.ev[st][0][i], s);
}
void prof_end(int st, cudaStream_t s) {
    if (!g_prof.on) return;
    cudaEventRecord(g_prof.ev[st][1][g_prof.used[st]], s);
    g_prof.used[st]++;
}
void prof_harvest() {
    for (int st = 0; st < ST_COUNT; ++st) {
        for (int i = 0; i < g_prof.used[st]; ++i) {
            float ms = 0.f;
            cudaEventSynchronize(g_prof.ev[st][1][i]);
            if (cudaEventElapsedTime(&ms, g_prof.ev[st][0][i], g_prof.ev[st][1][i]) == cudaSuccess) {
                g_prof.total_ms[st] += ms;
                g_prof.count[st] += 1;
            }
        }
        g_prof.used[st] = 0;
    }
}

void plan_trace(const char* phase, cudaStream_t s) {
    static const bool on = getenv("SK_PLAN_TRACE") != nullptr;
    if (!on) return;
    static auto t0 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[plan] %-28s %9.2f ms\n", phase, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
}

// reduction output slots inside Plan::red_out (each slot: result + partial scratch)
constexpr int kSlot = 608;
static inline double* slot(Plan& P, int k) { return P.red_out + k * kSlot; }

}  // namespace sk

using namespace sk;

// reduction slot ids
enum { SL_UPD = 0, SL_A = 1, SL_B = 2, SL_C = 3, SL_D = 4, SL_E = 5, SL_SCALARS = 6 };

extern "C" {

const char* sk_last_error(void) { return g_err.c_str(); }

void sk_release_cache(void) {
    fft_pool_release();
    dev_cache_release();
}

void sk_profile(int on) {
    if (!on) prof_harvest();
    g_prof.on = on != 0;
}

// out[2*k] = launches timed, out[2*k+1] = total ms, for stage k in {spread, allreduce,
// fft_fwd, multiply, fft_inv, interp, update, plan}; reset != 0 clears the accumulators.
int sk_profile_read(double* out, int nstages, int reset) {
    prof_harvest();
    for (int st = 0; st < ST_COUNT && st < nstages; ++st) {
        out[2 * st] = (double)g_prof.count[st];
        out[2 * st + 1] = g_prof.total_ms[st];
        if (reset) { g_prof.count[st] = 0; g_prof.total_ms[st] = 0.0; }
    }
    return SK_OK;
}
long long sk_launch_count(void) { return g_launches.load(); }

int sk_nccl_unique_id(void* out) {
    if (!out) return set_error(SK_EINVAL, "NULL out");
    SK_TRY(nccl_load());
    ncclUniqueId id;
    SK_NCCL(g_nccl.getUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return SK_OK;
}

int sinkhorn_init(sk_ctx_t* ctx, int device, int rank, int world_size, const void* nccl_unique_id,
                  void* cuda_stream) {
    if (!ctx) return set_error(SK_EINVAL, "NULL ctx");
    if (world_size < 1 || rank < 0 || rank >= world_size) return set_error(SK_EINVAL, "bad rank/world_size");
    if (world_size > 1 && !nccl_unique_id) return set_error(SK_EINVAL, "world_size > 1 needs an ncclUniqueId");
    SK_CUDA(cudaSetDevice(device));
    sk_ctx* c = new sk_ctx();
    c->c.device = device;
    c->c.rank = rank;
    c->c.world = world_size;
    c->c.stream = (cudaStream_t)cuda_stream;
    if (world_size == 1 && !nccl_unique_id) {
        const char* ew = getenv("SK_EMULATE_WORLD");
        if (ew && atoi(ew) > 1) {   // test hook, see allreduce_sum
            c->c.world = atoi(ew);
            c->c.emulated = true;
        }
    }
    if (nccl_unique_id) {   // world_size > 1, or the one-rank NCCL path
        int st = nccl_load();
        if (st) { delete c; return st; }
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof(id));
        ncclComm_t comm;
        ncclResult_t r = g_nccl.commInitRank(&comm, world_size, id, rank);
        if (r != ncclSuccess) {
            delete c;
            return set_error(SK_ENCCL, std::string("ncclCommInitRank: ") + (g_nccl.errStr ? g_nccl.errStr(r) : ""));
        }
        c->c.nccl_comm = comm;
    }
    *ctx = c;
    return SK_OK;
}

int sinkhorn_finalize(sk_ctx_t ctx) {
    if (!ctx) return SK_OK;
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.nccl_comm) g_nccl.commDestroy((ncclComm_t)ctx->c.nccl_comm);
    delete ctx;
    return SK_OK;
}

int fastsum_plan(sk_ctx_t ctx, sk_plan_t* plan, int d, const double* x, long long n_local,
                 const double* y, long long m_local, double lambda, int N, double sigma, int m_w,
                 double eps_B, int p_smooth) {
    if (!ctx || !plan) return set_error(SK_EINVAL, "NULL ctx/plan");
    SK_CUDA(cudaSetDevice(ctx->c.device));
    Plan* P = nullptr;
    SK_TRY(build_plan(&ctx->c, &P, d, x, n_local, y, m_local, lambda, N, sigma, m_w, eps_B, p_smooth, 2, 0));
    sk_plan* h = new sk_plan();
    h->p = P;
    *plan = h;
    return SK_OK;
}

int fastsum_plan_ex(sk_ctx_t ctx, sk_plan_t* plan, int d, const double* x, long long n_local,
                    const double* y, long long m_local, const sk_plan_opts* o) {
    if (!ctx || !plan || !o) return set_error(SK_EINVAL, "NULL ctx/plan/opts");
    SK_CUDA(cudaSetDevice(ctx->c.device));
    Plan* P = nullptr;
    SK_TRY(build_plan(&ctx->c, &P, d, x, n_local, y, m_local, o->lambda, o->N, o->sigma, o->m_w, o->eps_B,
                      o->p_smooth, o->r, o->near_cells));
    sk_plan* h = new sk_plan();
    h->p = P;
    *plan = h;
    return SK_OK;
}

int fastsum_plan_destroy(sk_plan_t plan) {
    if (!plan) return SK_OK;
    destroy_plan(plan->p);
    delete plan;
    return SK_OK;
}

int fastsum_apply(sk_plan_t plan, int transpose, int kernel, const double* w, double* t) {
    if (!plan) return set_error(SK_EINVAL, "NULL plan");
    if (kernel != 0 && kernel != 1) return set_error(SK_EINVAL, "kernel must be 0 or 1");
    Plan& P = *plan->p;
    cudaStream_t s = P.ctx->stream;
    const NodeSet& src = P.side[transpose ? 0 : 1];
    const NodeSet& dst = P.side[transpose ? 1 : 0];
    if ((src.count > 0 && !w) || (dst.count > 0 && !t)) return set_error(SK_EINVAL, "NULL w/t");
    SK_TRY(launch_permute_in(w, src.perm, src.count, P.w_sorted, s, wslot(P, WSLOT_W)));
    SK_TRY(apply_sorted(P, transpose, kernel, P.w_sorted, P.t_sorted));
    SK_TRY(launch_permute_out(P.t_sorted, dst.perm, dst.count, t, s));
    return SK_OK;
}

int nfft_spread(sk_plan_t plan, int side, const double* w, double* grid) {
    if (!plan || (side != 0 && side != 1) || !grid) return set_error(SK_EINVAL, "bad args");
    Plan& P = *plan->p;
    cudaStream_t s = P.ctx->stream;
    const NodeSet& S = P.side[side];
    SK_TRY(launch_permute_in(w, S.perm, S.count, P.w_sorted, s, wslot(P, WSLOT_W)));
    SK_TRY(launch_spread(P, side, P.w_sorted, grid, s));   // writes every grid cell
    return SK_OK;
}

int nfft_interp(sk_plan_t plan, int side, const double* grid, double* t) {
    if (!plan || (side != 0 && side != 1) || !grid) return set_error(SK_EINVAL, "bad args");
    Plan& P = *plan->p;
    cudaStream_t s = P.ctx->stream;
    const NodeSet& S = P.side[side];
    SK_TRY(launch_interp(P, side, grid, P.t_sorted, s));
    SK_TRY(launch_permute_out(P.t_sorted, S.perm, S.count, t, s));
    return SK_OK;
}

int fastsum_plan_info(sk_plan_t plan, double* out) {
    if (!plan || !out) return set_error(SK_EINVAL, "bad args");
    Plan& P = *plan->p;
    for (int a = 0; a < 3; ++a) out[a] = a < P.d ? P.centre[a] : 0.0;
    out[3] = P.rho;
    out[4] = P.lambda_p;
    out[5] = P.L;
    out[6] = P.n;
    out[7] = P.N + 1;
    out[8] = P.d;
    out[9] = (double)P.side[0].total;
    out[10] = (double)P.side[1].total;
    for (int a = 0; a < 3; ++a) {
        out[11 + a] = a < P.d ? P.box_lo[a] : 0.0;
        out[14 + a] = a < P.d ? P.box_n[a] : 1.0;
    }
    out[17] = (double)P.box_size;
    // accuracy report: the band's dropped Fourier mass per kernel (pointwise bound on the
    // truncation of K~), K at the regularisation radius L (K_B is inert when tiny) and, for
    // r = 2, the Gaussian's first dropped 1-D coefficient ratio exp(-pi^2 (N/2)^2 / lambda')
    out[18] = P.acc_tail[0];
    out[19] = P.acc_tail[1];
    out[20] = P.rpow == 2 ? exp(-P.lambda_p * P.L * P.L) : exp(-P.lambda_p * P.L);
    const double pi = 3.141592653589793238462643;
    out[21] = P.rpow == 2 ? exp(-pi * pi * (P.N / 2.0) * (P.N / 2.0) / P.lambda_p) : NAN;
    return SK_OK;
}

int fastsum_coefficients(sk_plan_t plan, int kernel, double* b) {
    if (!plan || !b || (kernel != 0 && kernel != 1)) return set_error(SK_EINVAL, "bad args");
    Plan& P = *plan->p;
    long long full = 1;
    for (int a = 0; a < P.d; ++a) full *= (P.N + 1);
    SK_CUDA(cudaMemcpyAsync(b, P.bk[kernel], sizeof(double) * full, cudaMemcpyDeviceToHost, P.ctx->stream));
    SK_CUDA(cudaStreamSynchronize(P.ctx->stream));
    return SK_OK;
}

// Sum of the 3-slot update partials -> slot(SL_UPD)[0..2] (resid sum, min t, 0).
static int finalize_update(Plan& P, double* out) {
    return launch_finalize_partials(P.red, kUpdBlocks, kUpdVals, out, P.ctx->stream);
}

// Weight check of the boundary: a, b > 0 and each sums to 1 +- kWeightTol over all
// ranks (the measures of Alg. 2 are probability vectors). a_s, b_s hold the sorted copies.
constexpr double kWeightTol = 1e-12;
static int check_weights(Plan& P) {
    Ctx* C = P.ctx;
    cudaStream_t s = C->stream;
    double* r = slot(P, SL_SCALARS);   // [0] sum a, [1] sum b, [2] min a, [3] min b (+ scratch)
    SK_TRY(launch_reduce_sum_log(nullptr, P.a_s, P.side[0].count, slot(P, SL_A), 1, s));
    SK_TRY(launch_reduce_sum_log(nullptr, P.b_s, P.side[1].count, slot(P, SL_B), 1, s));
    SK_TRY(launch_reduce_sum_log(nullptr, P.a_s, P.side[0].count, slot(P, SL_C), 5, s));
    SK_TRY(launch_reduce_sum_log(nullptr, P.b_s, P.side[1].count, slot(P, SL_D), 5, s));
    for (int k = 0; k < 4; ++k)
        SK_CUDA(cudaMemcpyAsync(r + k, slot(P, SL_A + k), sizeof(double), cudaMemcpyDeviceToDevice, s));
    SK_TRY(allreduce_sum(C, r, 2));
    SK_TRY(allreduce_minmax(C, r + 2, r + 600, 2));
    SK_CUDA(cudaMemcpyAsync(P.host_red, r, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    const double* h = P.host_red;
    if (!(h[2] > 0.0) || !(h[3] > 0.0))
        return set_error(SK_EINVAL, "weights must be > 0 (min a = " + std::to_string(h[2]) +
                                        ", min b = " + std::to_string(h[3]) + ")");
    if (!(fabs(h[0] - 1.0) <= kWeightTol) || !(fabs(h[1] - 1.0) <= kWeightTol)) {
        char msg[160];
        snprintf(msg, sizeof(msg), "weights must sum to 1 +- 1e-12 over all ranks (sum a - 1 = %.3e, sum b - 1 = %.3e)",
                 h[0] - 1.0, h[1] - 1.0);
        return set_error(SK_EINVAL, msg);
    }
    return SK_OK;
}

// Min over ranks of the two packed SK_ENONPOS words (uint64; ncclUint64 ncclMin).
static int allreduce_bad(Ctx* c, unsigned long long* bad) {
    if (c->emulated || !c->nccl_comm) return SK_OK;
    SK_NCCL(g_nccl.allReduce(bad, bad, 2, ncclUint64, ncclMin, (ncclComm_t)c->nccl_comm, c->stream));
    count_launch();
    return SK_OK;
}

// Alg. 2. trace (host, may be NULL): per iteration kTraceVals doubles, see
// sinkhorn_run_trace in include/sinkhorn_nfft.h.
constexpr int kTraceVals = 6;
static int run_impl(sk_plan_t plan, const double* a, const double* b, int iters, double tol,
                    int rescale_policy, double* u, double* v, sk_run_info* info, double* trace) {
    if (!plan) return set_error(SK_EINVAL, "NULL plan");
    Plan& P = *plan->p;
    Ctx* C = P.ctx;
    cudaStream_t s = C->stream;
    const NodeSet& X = P.side[0];
    const NodeSet& Y = P.side[1];
    if (iters < 0 || tol < 0 || rescale_policy < 0 || rescale_policy > 2)
        return set_error(SK_EINVAL, "bad iters/tol/rescale_policy");
    if (iters >= (1 << 24)) return set_error(SK_EINVAL, "iters must be < 2^24");
    if ((X.count > 0 && (!a || !u)) || (Y.count > 0 && (!b || !v))) return set_error(SK_EINVAL, "NULL a/b/u/v");
    SK_TRY(launch_permute_in(a, X.perm, X.count, P.a_s, s));
    SK_TRY(launch_permute_in(b, Y.perm, Y.count, P.b_s, s));
    SK_TRY(check_weights(P));
    // u is rewritten (and its bound recorded) before it is first spread; v is spread first
    SK_TRY(launch_permute_in(u, X.perm, X.count, P.u_s, s));
    if (wslot(P, WSLOT_U)) SK_CUDA(cudaMemsetAsync(wslot(P, WSLOT_U), 0, sizeof(unsigned), s));
    SK_TRY(launch_permute_in(v, Y.perm, Y.count, P.v_s, s, wslot(P, WSLOT_V)));
    const unsigned long long nobad[2] = {kNoBad, kNoBad};
    SK_CUDA(cudaMemcpyAsync(P.bad64, nobad, sizeof(nobad), cudaMemcpyHostToDevice, s));
    // resources released on every exit path
    struct Scoped {
        cudaStream_t s;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        double* trace_dev = nullptr;
        cudaGraphExec_t exec = nullptr;
        ~Scoped() {
            if (exec) cudaGraphExecDestroy(exec);
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
            dev_free(trace_dev, s);
        }
    } R{s};
    if (trace && iters > 0) SK_TRY(dev_alloc((void**)&R.trace_dev, sizeof(double) * kTraceVals * iters, s));
    double* const trace_dev = R.trace_dev;
    // per half-step (residual, KL, sum p log x) from the finalized update slot
    auto record = [&](int it, int half) -> int {
        double* r = slot(P, SL_C);
        SK_TRY(finalize_update(P, r));
        double* dst = trace_dev + (long long)it * kTraceVals + 3 * half;
        SK_CUDA(cudaMemcpyAsync(dst, r, sizeof(double), cudaMemcpyDeviceToDevice, s));
        SK_CUDA(cudaMemcpyAsync(dst + 1, r + 2, 2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
        return SK_OK;
    };
    SK_CUDA(cudaEventCreate(&R.e0));
    SK_CUDA(cudaEventCreate(&R.e1));
    SK_CUDA(cudaEventRecord(R.e0, s));
    double resid = NAN, kappa = NAN, kappa_u = NAN;
    int done = 0;
    // one iteration of Alg. 2; it < 0: inside a CUDA graph, the iteration number for error
    // reports comes from the device counter P.flag[4]
    auto body = [&](int it, bool last) -> int {
        const int* iter_dev = it < 0 ? P.flag + 4 : nullptr;
        if (rescale_policy != 0) {
            // Eq. (scale): v <- c v, c = 1/geomean(v) or 1/max(v) (reading Q4)
            double* r = slot(P, SL_E);
            SK_TRY(launch_reduce_sum_log(nullptr, P.v_s, Y.count, r, rescale_policy == 1 ? 3 : 4, s));
            if (rescale_policy == 1) SK_TRY(allreduce_sum(C, r, 1));
            else SK_TRY(allreduce_minmax(C, r + 600, r, 1));
            SK_TRY(launch_rescale_factor(r, rescale_policy, (double)Y.total, s));
            SK_TRY(launch_scale_vec(P.v_s, Y.count, r, s, wslot(P, WSLOT_V)));
        }
        if (last) SK_TRY(launch_reduce_sum_log(nullptr, P.v_s, Y.count, slot(P, SL_D), 1, s));
        // odd Delta: t = K v, u = a / t   (Eq. (even_F_sink)). Without a residual or
        // trace to reduce, the division is fused into the interpolation epilogue (no t round
        // trip through HBM, one kernel fewer); otherwise the update kernel also reduces.
        const int want_u = trace_dev ? 2 : ((tol > 0 || last) ? 1 : 0);
        FusedUpd fu_u;
        fu_u.p = P.a_s; fu_u.x = P.u_s; fu_u.bad = P.bad64; fu_u.iter_dev = iter_dev; fu_u.iter = it;
        fu_u.rank = C->rank;
        fu_u.xmax = wslot(P, WSLOT_U);
        SK_TRY(apply_sorted(P, 0, 0, P.v_s, P.t_sorted, want_u ? nullptr : &fu_u));
        if (want_u) {
            prof_begin(ST_UPDATE, s);
            SK_TRY(launch_update(P, 0, P.t_sorted, P.a_s, P.u_s, want_u, it, iter_dev, s));
            prof_end(ST_UPDATE, s);
        }
        if (tol > 0 || last) SK_TRY(finalize_update(P, slot(P, SL_UPD)));
        if (trace_dev) SK_TRY(record(it, 0));
        // even Delta: t~ = K^T u, v = b / t~   (Eq. (odd_F_sink)); the last one also
        // reduces min t~ and ||u||_1 for the u-side conditioning estimate
        if (last) SK_TRY(launch_reduce_sum_log(nullptr, P.u_s, X.count, slot(P, SL_A), 1, s));
        const int want_v = trace_dev ? 2 : (last ? 1 : 0);
        FusedUpd fu_v;
        fu_v.p = P.b_s; fu_v.x = P.v_s; fu_v.bad = P.bad64 + 1; fu_v.iter_dev = iter_dev; fu_v.iter = it;
        fu_v.rank = C->rank;
        fu_v.xmax = wslot(P, WSLOT_V);
        SK_TRY(apply_sorted(P, 1, 0, P.u_s, P.t_sorted, want_v ? nullptr : &fu_v));
        if (want_v) {
            prof_begin(ST_UPDATE, s);
            SK_TRY(launch_update(P, 1, P.t_sorted, P.b_s, P.v_s, want_v, it, iter_dev, s));
            prof_end(ST_UPDATE, s);
        }
        if (last) SK_TRY(finalize_update(P, slot(P, SL_B)));
        if (trace_dev) SK_TRY(record(it, 1));
        return SK_OK;
    };
    int it0 = 0;
    // Fixed-count runs replay iterations 0 .. iters-2 as one CUDA graph (cuFFT, NCCL and the
    // kernels of an iteration captured once): launch-bound small workloads lose the per-kernel
    // CPU launch cost. Off under the stage profiler, tracing, tol > 0 or SK_NO_GRAPH.
    static const bool no_graph = getenv("SK_NO_GRAPH") != nullptr;
    if (!trace_dev && tol == 0 && !g_prof.on && iters > 2 && !no_graph) {
        int zero = 0;
        SK_CUDA(cudaMemcpyAsync(P.flag + 4, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
        cudaGraph_t graph = nullptr;
        const long long l0 = g_launches.load();
        // capture on the plan's private stream (the caller's may be the legacy default stream,
        // which cannot be captured); the graph is then launched on the caller's stream
        if (!P.cap_stream) SK_CUDA(cudaStreamCreateWithFlags(&P.cap_stream, cudaStreamNonBlocking));
        const cudaStream_t user = s;
        auto use_stream = [&](cudaStream_t t) {
            s = t;
            C->stream = t;
            plan_set_stream(P, t);   // every cuFFT handle of the plan (full and pruned)
        };
        use_stream(P.cap_stream);
        cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) { use_stream(user); return set_error(SK_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce)); }
        int st = body(-1, false);
        if (!st) st = launch_increment(P.flag + 4, s);
        ce = cudaStreamEndCapture(s, &graph);
        use_stream(user);
        if (st) { if (graph) cudaGraphDestroy(graph); return st; }
        if (ce != cudaSuccess) return set_error(SK_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        const long long per_iter = g_launches.load() - l0;
        ce = cudaGraphInstantiate(&R.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return set_error(SK_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
        for (int it = 0; it < iters - 1; ++it) {
            ce = cudaGraphLaunch(R.exec, s);
            if (ce != cudaSuccess) return set_error(SK_ECUDA, std::string("graph launch: ") + cudaGetErrorString(ce));
        }
        count_launch(per_iter * (iters - 2));   // the capture counted one iteration's kernels
        it0 = iters - 1;
        done = iters - 1;
    }
    for (int it = it0; it < iters; ++it) {
        const bool last = (it == iters - 1);
        SK_TRY(body(it, last));
        done = it + 1;
        if (tol > 0 || last) {
            double* r = slot(P, SL_UPD);
            // residual: sum over ranks; min t: min over ranks; ||v||_1: sum over ranks
            SK_TRY(allreduce_sum(C, r, 1));
            SK_TRY(allreduce_minmax(C, r + 1, r + 600, 1));
            if (last) {
                SK_TRY(allreduce_sum(C, slot(P, SL_D), 1));
                SK_TRY(allreduce_sum(C, slot(P, SL_A), 1));
                SK_TRY(allreduce_minmax(C, slot(P, SL_B) + 1, slot(P, SL_B) + 600, 1));
                SK_CUDA(cudaMemcpyAsync(P.host_red + 2, slot(P, SL_D), sizeof(double), cudaMemcpyDeviceToHost, s));
                SK_CUDA(cudaMemcpyAsync(P.host_red + 3, slot(P, SL_A), sizeof(double), cudaMemcpyDeviceToHost, s));
                SK_CUDA(cudaMemcpyAsync(P.host_red + 4, slot(P, SL_B) + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
            }
            SK_CUDA(cudaMemcpyAsync(P.host_red, r, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
            SK_CUDA(cudaStreamSynchronize(s));
            resid = P.host_red[0];
            if (last) {
                kappa = log10(P.host_red[2] / P.host_red[1]);     // ||v||_1 / min (K v)
                kappa_u = log10(P.host_red[3] / P.host_red[4]);   // ||u||_1 / min (K^T u)
            }
            if (tol > 0 && resid <= tol) break;
        }
    }
    SK_CUDA(cudaEventRecord(R.e1, s));
    if (trace_dev) {
        // every trace entry is a sum over nodes: one all-reduce over ranks
        SK_TRY(allreduce_sum(C, trace_dev, (long long)kTraceVals * iters));
        for (int i = 0; i < kTraceVals * iters; ++i) trace[i] = NAN;
        SK_CUDA(cudaMemcpyAsync(trace, trace_dev, sizeof(double) * kTraceVals * done, cudaMemcpyDeviceToHost, s));
    }
    SK_TRY(launch_permute_out(P.u_s, X.perm, X.count, u, s));
    SK_TRY(launch_permute_out(P.v_s, Y.perm, Y.count, v, s));
    // SK_ENONPOS decided on the global (min over ranks) event words, so every rank agrees
    SK_TRY(allreduce_bad(C, P.bad64));
    unsigned long long hbad[2];
    SK_CUDA(cudaMemcpyAsync(hbad, P.bad64, sizeof(hbad), cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, R.e0, R.e1);
    if (info) {
        info->iters_done = done;
        info->residual = resid;
        info->kappa_log10_est = kappa;
        info->kappa_u_log10_est = kappa_u;
        info->seconds = ms * 1e-3;
        info->bad_iter = -1;
        info->bad_index = -1;
        info->bad_side = -1;
        info->bad_rank = -1;
    }
    if (hbad[0] != kNoBad || hbad[1] != kNoBad) {
        // the earlier iteration wins; within one iteration the u-update (side 0) comes first
        const int it0b = (int)(hbad[0] >> 40), it1b = (int)(hbad[1] >> 40);
        const int side = (hbad[0] != kNoBad && (hbad[1] == kNoBad || it0b <= it1b)) ? 0 : 1;
        const unsigned long long w = hbad[side];
        const int brank = (int)((w >> 32) & 0xff), sidx = (int)(w & 0xffffffffULL);
        int hperm = -1;
        if (brank == C->rank || C->emulated)
            SK_CUDA(cudaMemcpy(&hperm, P.side[side].perm + sidx, sizeof(int), cudaMemcpyDeviceToHost));
        if (info) {
            info->bad_iter = (int)(w >> 40);
            info->bad_index = hperm;
            info->bad_side = side;
            info->bad_rank = brank;
        }
        return set_error(SK_ENONPOS, "non-positive fast-summation denominator in iteration " +
                                         std::to_string((int)(w >> 40)) + " on side " + std::to_string(side) +
                                         " at caller index " + std::to_string(hperm) + " of rank " +
                                         std::to_string(brank));
    }
    if (tol > 0 && !(resid <= tol)) return set_error(SK_ENOTCONVERGED, "residual above tol");
    return SK_OK;
}

int sinkhorn_run(sk_plan_t plan, const double* a, const double* b, int iters, double tol,
                 int rescale_policy, double* u, double* v, sk_run_info* info) {
    return run_impl(plan, a, b, iters, tol, rescale_policy, u, v, info, nullptr);
}

int sinkhorn_run_trace(sk_plan_t plan, const double* a, const double* b, int iters, double tol,
                       int rescale_policy, double* u, double* v, sk_run_info* info, double* trace) {
    if (!trace) return set_error(SK_EINVAL, "NULL trace");
    return run_impl(plan, a, b, iters, tol, rescale_policy, u, v, info, trace);
}

int sinkhorn_divergence(sk_plan_t plan, const double* a, const double* b, const double* u,
                        const double* v, double* s_dual, double* s_cost) {
    if (!plan || !s_dual || !s_cost) return set_error(SK_EINVAL, "NULL plan/outputs");
    Plan& P = *plan->p;
    Ctx* C = P.ctx;
    cudaStream_t s = C->stream;
    const NodeSet& X = P.side[0];
    const NodeSet& Y = P.side[1];
    if ((X.count > 0 && (!a || !u)) || (Y.count > 0 && (!b || !v))) return set_error(SK_EINVAL, "NULL a/b/u/v");
    SK_TRY(launch_permute_in(a, X.perm, X.count, P.a_s, s));
    SK_TRY(launch_permute_in(b, Y.perm, Y.count, P.b_s, s));
    SK_TRY(launch_permute_in(u, X.perm, X.count, P.u_s, s, wslot(P, WSLOT_U)));
    SK_TRY(launch_permute_in(v, Y.perm, Y.count, P.v_s, s, wslot(P, WSLOT_V)));
    double* sc = slot(P, SL_SCALARS);
    // S1 = sum a log u, S2 = sum b log v
    SK_TRY(launch_reduce_sum_log(P.a_s, P.u_s, X.count, slot(P, SL_A), 0, s));
    SK_TRY(launch_reduce_sum_log(P.b_s, P.v_s, Y.count, slot(P, SL_B), 0, s));
    // S3 = sum_j (K^T u)_j v_j
    SK_TRY(apply_sorted(P, 1, 0, P.u_s, P.t_sorted));
    SK_TRY(launch_reduce_sum_log(P.t_sorted, P.v_s, Y.count, slot(P, SL_C), 2, s));
    // S4 = sum_i u_i ((c K) v)_i
    SK_TRY(apply_sorted(P, 0, 1, P.v_s, P.t_sorted));
    SK_TRY(launch_reduce_sum_log(P.t_sorted, P.u_s, X.count, slot(P, SL_D), 2, s));
    for (int k = 0; k < 4; ++k)
        SK_CUDA(cudaMemcpyAsync(sc + k, slot(P, SL_A + k), sizeof(double), cudaMemcpyDeviceToDevice, s));
    SK_TRY(allreduce_sum(C, sc, 4));
    SK_CUDA(cudaMemcpyAsync(P.host_red, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    SK_CUDA(cudaStreamSynchronize(s));
    const double S1 = P.host_red[0], S2 = P.host_red[1], S3 = P.host_red[2], S4 = P.host_red[3];
    // Eq. (14): d = 1/lam + (1/lam) sum p log alpha + (1/lam) sum p~ log alpha~ - (1/lam) sum alpha k alpha~
    *s_dual = (1.0 + S1 + S2 - S3) / P.lambda;
    *s_cost = S4;
    return SK_OK;
}

int sinkhorn_solve(sk_ctx_t ctx, int d, const double* x, long long n_local, const double* y,
                   long long m_local, const double* a, const double* b, double lambda, int N,
                   double sigma, int m_w, double eps_B, int p_smooth, int iters, int inputs_on_host,
                   double* s_dual, double* s_cost, sk_run_info* info) {
    if (!ctx || !s_dual || !s_cost) return set_error(SK_EINVAL, "NULL ctx/outputs");
    if (d < 1 || d > 3 || n_local < 0 || m_local < 0) return set_error(SK_EINVAL, "bad d/counts");
    cudaStream_t s = ctx->c.stream;
    SK_CUDA(cudaSetDevice(ctx->c.device));
    const double *dx = x, *dy = y, *da = a, *db = b;
    double* buf = nullptr;
    const long long nn = n_local, mm = m_local;
    // device work buffers: [x | y | a | b | u | v]
    const size_t tot = (size_t)(nn * d + mm * d + nn + mm + nn + mm);
    SK_TRY(dev_alloc((void**)&buf, sizeof(double) * (tot ? tot : 1), s));
    double* px = buf;
    double* py = px + nn * d;
    double* pa = py + mm * d;
    double* pb = pa + nn;
    double* pu = pb + mm;
    double* pv = pu + nn;
    // host inputs: the nodes go first on the context stream (the plan needs them); the
    // weights, needed only from sinkhorn_run on, travel on a side stream behind the plan
    static thread_local cudaStream_t copy_stream = nullptr;
    cudaEvent_t weights_ready = nullptr;
    if (inputs_on_host) {
        if (nn) SK_CUDA(cudaMemcpyAsync(px, x, sizeof(double) * nn * d, cudaMemcpyHostToDevice, s));
        if (mm) SK_CUDA(cudaMemcpyAsync(py, y, sizeof(double) * mm * d, cudaMemcpyHostToDevice, s));
        if (!copy_stream) SK_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        SK_CUDA(cudaEventCreateWithFlags(&weights_ready, cudaEventDisableTiming));
        SK_CUDA(cudaEventRecord(weights_ready, s));            // buf is ordered on s
        SK_CUDA(cudaStreamWaitEvent(copy_stream, weights_ready, 0));
        if (nn) SK_CUDA(cudaMemcpyAsync(pa, a, sizeof(double) * nn, cudaMemcpyHostToDevice, copy_stream));
        if (mm) SK_CUDA(cudaMemcpyAsync(pb, b, sizeof(double) * mm, cudaMemcpyHostToDevice, copy_stream));
        SK_CUDA(cudaEventRecord(weights_ready, copy_stream));
        dx = px; dy = py; da = pa; db = pb;
    }
    SK_TRY(launch_fill(pu, nn, 1.0, s));
    SK_TRY(launch_fill(pv, mm, 1.0, s));
    sk_plan_t plan = nullptr;
    prof_begin(ST_PLAN, s);
    int st = fastsum_plan(ctx, &plan, d, dx, nn, dy, mm, lambda, N, sigma, m_w, eps_B, p_smooth);
    prof_end(ST_PLAN, s);
    if (weights_ready) {
        cudaStreamWaitEvent(s, weights_ready, 0);
        cudaEventDestroy(weights_ready);
    }
    if (!st) st = sinkhorn_run(plan, da, db, iters, 0.0, 0, pu, pv, info);
    if (!st) st = sinkhorn_divergence(plan, da, db, pu, pv, s_dual, s_cost);
    fastsum_plan_destroy(plan);
    dev_free(buf, s);
    cudaStreamSynchronize(s);
    return st;
}

}  // extern "C"
