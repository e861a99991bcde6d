// microbench.cu -- FP64 throughput probes on B200 (sm_100a) that set the roofline of the
// FP64-bound spread/interp kernels:
//   dfma   : FP64 FMA (vector pipe), 8 independent chains per thread
//   dmma   : FP64 tensor-core MMA mma.sync m8n8k4 and m16n8k4/k8/k16 (.f64)
//   atoms  : shared-memory FP64 atomicAdd, distinct addresses per lane
//   redg   : global FP64 atomicAdd (RED) to scattered addresses in a 16 MB grid
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double c0 = threadIdx.x, c1 = c0 + 1, c2 = c0 + 2, c3 = c0 + 3, c4 = c0 + 4, c5 = c0 + 5, c6 = c0 + 6, c7 = c0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            c0 = fma(c0, a, b); c1 = fma(c1, a, b); c2 = fma(c2, a, b); c3 = fma(c3, a, b);
            c4 = fma(c4, a, b); c5 = fma(c5, a, b); c6 = fma(c6, a, b); c7 = fma(c7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

__global__ void dmma884_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma1684_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
        }
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
    double a[8], b[4];
    for (int k = 0; k < 8; ++k) a[k] = (threadIdx.x + k) * 1e-3;
    for (int k = 0; k < 4; ++k) b[k] = 1.0 - (threadIdx.x + k) * 1e-4;
    double c[2][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    double s = 0;
    for (int k = 0; k < 2; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void atoms_kernel(double* out, int iters) {
    __shared__ double sh[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int base = (threadIdx.x * 33) & 4095;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) atomicAdd(&sh[(base + k * 128 + i) & 4095], 1.0);
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sh[threadIdx.x];
}

__global__ void lds_bcast_kernel(double* out, int iters) {
    __shared__ double sh[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i * 1e-3;
    __syncthreads();
    double acc = 0, acc2 = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            double2 v = *reinterpret_cast<const double2*>(&sh[((i * 16 + k) * 2) & 1023]);
            acc = fma(acc, v.x, 1e-9);
            acc2 = fma(acc2, v.y, 1e-9);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + acc2;
}

__global__ void redg_kernel(double* grid, long long gsize, int iters) {
    unsigned long long h = (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
    for (int i = 0; i < iters; ++i) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        long long base = (h >> 20) % (gsize - 64);
        atomicAdd(&grid[base + (threadIdx.x & 31)], 1.0);
    }
}

// half the warps DFMA, half DMMA: are the FP64 vector and tensor pipes additive?
__global__ void mixed_kernel(double* out, int iters) {
    const int warp = threadIdx.x >> 5;
    if (warp & 1) {
        double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
        double c[4][2] = {};
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
        double s = 0;
        for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {
        double c0 = threadIdx.x, c1 = c0 + 1, c2 = c0 + 2, c3 = c0 + 3, c4 = c0 + 4, c5 = c0 + 5, c6 = c0 + 6, c7 = c0 + 7;
        const double a = 0.999999, b = 1e-7;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // 32 DFMA per thread = 1024 FMA per warp ~ 4 DMMA
                c0 = fma(c0, a, b); c1 = fma(c1, a, b); c2 = fma(c2, a, b); c3 = fma(c3, a, b);
                c4 = fma(c4, a, b); c5 = fma(c5, a, b); c6 = fma(c6, a, b); c7 = fma(c7, a, b);
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
    }
}

// LDS.128 broadcast throughput with 8 independent FMA chains per thread
__global__ void lds_tp_kernel(double* out, int iters) {
    __shared__ __align__(16) double sh[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i * 1e-3;
    __syncthreads();
    double a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            double2 v = *reinterpret_cast<const double2*>(&sh[((i * 16 + k) * 2) & 1023]);
            a[(2 * k) & 7] = fma(a[(2 * k) & 7], v.x, 1e-9);
            a[(2 * k + 1) & 7] = fma(a[(2 * k + 1) & 7], v.y, 1e-9);
        }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the spread3 inner-loop mix: per k-step 18 products (DMUL) feeding 36 DMMAs into 36
// independent accumulators (72 doubles/lane), 2 warps x 2 CTAs per SMSP-quad like the kernel
template <bool WITH_DMUL>
__global__ void __launch_bounds__(128, 2) spreadmix_kernel(double* out, int iters) {
    double acc[2][18][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double y = 1.0 + threadIdx.x * 1e-6, z = 1.0 - threadIdx.x * 1e-6, a0 = 1e-3, a1 = 2e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 18; ++j) {
            const double b = WITH_DMUL ? y * (z + j) : y + j;
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[0][j][0]), "+d"(acc[0][j][1]) : "d"(a0), "d"(b));
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[1][j][0]), "+d"(acc[1][j][1]) : "d"(a1), "d"(b));
        }
        y *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) s += acc[i][j][0] + acc[i][j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the 28-tile spread3 mix (dmma3.cuh spread3_t28_ksteps): per warp and k-step 14 DMMA.8x8x4 into
// 14 accumulators fed by 16 DMUL products; useful work 1728 of 1792 issued FMAs per node
template <int MINB>
__global__ void __launch_bounds__(192, MINB) t28mix_kernel(double* out, int iters) {
    double acc[14][2];
#pragma unroll
    for (int j = 0; j < 14; ++j) acc[j][0] = acc[j][1] = 0.0;
    double y = 1.0 + threadIdx.x * 1e-6, z = 1.0 - threadIdx.x * 1e-6, w = 1e-3;
    for (int it = 0; it < iters; ++it) {
        const double a0 = w * y, a1 = w * z;
#pragma unroll
        for (int j = 0; j < 14; ++j) {
            const double b = j < 9 ? y * (z + j) : (z + j);
            const double a = j < 9 ? a0 : a1 * (y + j);
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
        }
        y *= 0.9999999;
        z *= 1.0000001;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 14; ++j) s += acc[j][0] + acc[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// operand-order variants of the spread mix: ORDER 0 = (a0,b_j),(a1,b_j) pairs; 1 = all a0 then
// all a1 (A reused, B changes every DMMA); 2 = b_j varies but computed without DMUL chains
template <int ORDER>
__global__ void __launch_bounds__(128, 2) spreadorder_kernel(double* out, int iters) {
    double acc[2][18][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double y = 1.0 + threadIdx.x * 1e-6, a0 = 1e-3, a1 = 2e-3;
    double b[18];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 18; ++j) b[j] = y + j;
        if (ORDER == 1) {
#pragma unroll
            for (int j = 0; j < 18; ++j)
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[0][j][0]), "+d"(acc[0][j][1]) : "d"(a0), "d"(b[j]));
#pragma unroll
            for (int j = 0; j < 18; ++j)
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[1][j][0]), "+d"(acc[1][j][1]) : "d"(a1), "d"(b[j]));
        } else {
#pragma unroll
            for (int j = 0; j < 18; ++j) {
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[0][j][0]), "+d"(acc[0][j][1]) : "d"(a0), "d"(b[j]));
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[1][j][0]), "+d"(acc[1][j][1]) : "d"(a1), "d"(b[j]));
            }
        }
        y *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) s += acc[i][j][0] + acc[i][j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// accumulator-count sweep: NACC independent m8n8k4 accumulators per lane, same A/B
template <int NACC>
__global__ void __launch_bounds__(128, 2) accsweep_kernel(double* out, int iters) {
    double acc[NACC][2];
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j][0] = acc[j][1] = 0.0;
    double a = 1e-3 + threadIdx.x * 1e-9, b = 1.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 36 / NACC; ++r)
#pragma unroll
            for (int j = 0; j < NACC; ++j)
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
        b *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += acc[j][0] + acc[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// hybrid spread mix: rows tx 0..7 on DMMA (one m-tile), rows 8..11 on DFMA with per-lane
// accumulators (lane (g,q) owns columns 8j+g of node slot q): no padded tensor-core rows.
// NT n-tiles (18 = all (ty,tz) columns, 9 = half of them per warp).
template <int NT>
__global__ void __launch_bounds__(128, NT == 18 ? 2 : 4) hybrid_kernel(double* out, int iters) {
    double acc[NT][2], acc2[4][NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) acc2[r][j] = 0.0;
    }
    double y = 1.0 + threadIdx.x * 1e-6, z = 1.0 - threadIdx.x * 1e-6, a0 = 1e-3, w = 0.5;
    for (int it = 0; it < iters; ++it) {
        double xr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) xr[r] = w * (y + r);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const double b = y * (z + j);
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a0), "d"(b));
#pragma unroll
            for (int r = 0; r < 4; ++r) acc2[r][j] = fma(xr[r], b, acc2[r][j]);
        }
        y *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        s += acc[j][0] + acc[j][1];
#pragma unroll
        for (int r = 0; r < 4; ++r) s += acc2[r][j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the spread mix with m16n8k4: one DMMA covers both m-tiles (rows g, 8+g) with one B operand
template <bool WITH_DMUL>
__global__ void __launch_bounds__(128, 2) spreadmix16_kernel(double* out, int iters) {
    double acc[18][4];
#pragma unroll
    for (int j = 0; j < 18; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    double y = 1.0 + threadIdx.x * 1e-6, z = 1.0 - threadIdx.x * 1e-6, a0 = 1e-3, a1 = 2e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 18; ++j) {
            const double b = WITH_DMUL ? y * (z + j) : y;
            asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3]) : "d"(a0), "d"(a1), "d"(b));
        }
        y *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 18; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// spread mix with the 18 products grouped in one asm block ahead of the 36 DMMAs: does grouping
// the FP64 vector ops (fewer DMMA <-> DMUL transitions on the shared pipe) lower their cost?
__global__ void __launch_bounds__(128, 2) spreadmix_grouped_kernel(double* out, int iters) {
    double acc[2][18][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double y = 1.0 + threadIdx.x * 1e-6, a0 = 1e-3, a1 = 2e-3;
    double zz[18];
#pragma unroll
    for (int j = 0; j < 18; ++j) zz[j] = 1.0 - threadIdx.x * 1e-6 + j;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        // 18 products as a dependent chain (b_j = b_{j-1} c + z_j, one DFMA each) so that the
        // token below depends on all of them
        double b[18];
        b[0] = fma(y, zz[17], zz[0]);
#pragma unroll
        for (int j = 1; j < 18; ++j) b[j] = fma(b[j - 1], y, zz[j]);
        // token: every DMMA waits for the last product, so ptxas cannot interleave the DMULs
        // with the DMMAs (one DMMA <-> FP64-vector transition per k-step instead of 36)
        double tok;
        asm volatile("sub.f64 %0, %1, %1;" : "=d"(tok) : "d"(b[17]));
        const double a0t = a0 + tok, a1t = a1 + tok;
#pragma unroll
        for (int j = 0; j < 18; ++j) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[0][j][0]), "+d"(acc[0][j][1]) : "d"(a0t), "d"(b[j]));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[1][j][0]), "+d"(acc[1][j][1]) : "d"(a1t), "d"(b[j]));
        }
        y *= 0.9999999;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 18; ++j) s += acc[i][j][0] + acc[i][j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, clk);
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    double* out; CK(cudaMalloc(&out, sizeof(double) * blocks * threads));
    {
        int iters = 4096;
        float ms = timeit([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
        double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        printf("dfma: %.2f TFLOP/s  (%.1f FMA/clk/SM at %d MHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), clk / 1000);
    }
    {
        int iters = 4096;
        float ms = timeit([&] { dmma884_kernel<<<blocks, threads>>>(out, iters); });
        double fl = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32);
        printf("dmma m8n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { dmma1684_kernel<<<blocks, threads>>>(out, iters); });
        fl = 2.0 * 512 * 4 * (double)iters * blocks * (threads / 32);
        printf("dmma m16n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { dmma16816_kernel<<<blocks, threads>>>(out, iters); });
        fl = 2.0 * 2048 * 2 * (double)iters * blocks * (threads / 32);
        printf("dmma m16n8k16: %.2f TFLOP/s\n", fl / ms / 1e9);
    }
    {
        int iters = 2048;
        float ms = timeit([&] { atoms_kernel<<<blocks, threads>>>(out, iters); });
        double ops = 8.0 * iters * blocks * threads;
        printf("smem f64 atomicAdd: %.1f Gop/s (%.2f per clk per SM)\n", ops / ms / 1e6, ops / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
        ms = timeit([&] { lds_bcast_kernel<<<blocks, threads>>>(out, iters); });
        ops = 16.0 * iters * blocks * threads;
        printf("LDS.128 broadcast + 2 DFMA: %.1f G lane-loads/s (%.2f warp-LDS per clk per SM)\n", ops / ms / 1e6, ops / 32 / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
    }
    {
        int iters = 4096;
        float ms = timeit([&] { mixed_kernel<<<blocks, threads>>>(out, iters); });
        // per pair of warps: DMMA warp 4*256 FMA, DFMA warp 32*32 FMA per iteration
        double fl = 2.0 * 1024 * (double)iters * blocks * (threads / 32);
        printf("mixed DFMA+DMMA: %.2f TFLOP/s (additive pipes would give ~2x dfma)\n", fl / ms / 1e9);
        ms = timeit([&] { lds_tp_kernel<<<blocks, threads>>>(out, iters); });
        double ops = 16.0 * iters * blocks * (threads / 32);
        printf("LDS.128 broadcast, 8 chains: %.2f warp-LDS per clk per SM, %.2f TFLOP/s\n",
               ops / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3), ops * 32 * 4 / ms / 1e9);
    }
    {
        int iters = 2048;
        const int g2 = p.multiProcessorCount * 2;
        float ms = timeit([&] { spreadmix_kernel<true><<<g2, 128>>>(out, iters); });
        double fl = 2.0 * 256 * 36 * (double)iters * g2 * 4;
        printf("spread mix (36 DMMA + 18 DMUL, 8 warps/SM): %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { spreadmix_kernel<false><<<g2, 128>>>(out, iters); });
        printf("spread mix without DMUL (36 DMMA, 8 warps/SM): %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { spreadmix_kernel<true><<<g2 * 2, 128>>>(out, iters); });
        printf("spread mix, 16 warps/SM: %.2f TFLOP/s\n", 2 * fl / ms / 1e9);
        ms = timeit([&] { spreadorder_kernel<0><<<g2, 128>>>(out, iters); });
        printf("spread order 0 (pairs, b precomputed): %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { spreadorder_kernel<1><<<g2, 128>>>(out, iters); });
        printf("spread order 1 (A-major): %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { accsweep_kernel<4><<<g2, 128>>>(out, iters); });
        printf("36 DMMA/iter, 4 accumulators, 8 warps/SM: %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { accsweep_kernel<12><<<g2, 128>>>(out, iters); });
        printf("36 DMMA/iter, 12 accumulators, 8 warps/SM: %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { accsweep_kernel<36><<<g2, 128>>>(out, iters); });
        printf("36 DMMA/iter, 36 accumulators, 8 warps/SM: %.2f TFLOP/s\n", fl / ms / 1e9);
        ms = timeit([&] { accsweep_kernel<4><<<g2 * 4, 128>>>(out, iters); });
        printf("36 DMMA/iter, 4 accumulators, 32 warps/SM: %.2f TFLOP/s\n", 4 * fl / ms / 1e9);
        // useful = 12 of 16 DMMA rows in the spread mixes above
        ms = timeit([&] { spreadmix_kernel<true><<<g2, 128>>>(out, iters); });
        printf("spread mix (36 DMMA + 18 DMUL), USEFUL rate: %.2f TFLOP/s\n", 0.75 * fl / ms / 1e9);
        ms = timeit([&] { spreadmix16_kernel<true><<<g2, 128>>>(out, iters); });
        printf("spread mix m16n8k4 (18 DMMA16 + 18 DMUL, 8 warps/SM): %.2f TFLOP/s issued, USEFUL %.2f\n", fl / ms / 1e9, 0.75 * fl / ms / 1e9);
        ms = timeit([&] { spreadmix16_kernel<false><<<g2, 128>>>(out, iters); });
        printf("spread mix m16n8k4 without DMUL: %.2f TFLOP/s issued\n", fl / ms / 1e9);
        ms = timeit([&] { spreadmix_grouped_kernel<<<g2, 128>>>(out, iters); });
        printf("spread mix, 18 DMUL grouped in one asm block: %.2f TFLOP/s issued, USEFUL %.2f\n", fl / ms / 1e9, 0.75 * fl / ms / 1e9);
        {   // 28-tile cover: 14 DMMA + 16 DMUL per warp and k-step, 12 warps/SM (2 CTAs x 6 warps)
            const double fl28 = 2.0 * 256 * 14 * (double)iters * g2 * 6;
            ms = timeit([&] { t28mix_kernel<2><<<g2, 192>>>(out, iters); });
            printf("t28 mix (14 DMMA + 16 DMUL, 12 warps/SM): %.2f TFLOP/s issued, USEFUL %.2f\n", fl28 / ms / 1e9,
                   fl28 * 1728.0 / 1792.0 / ms / 1e9);
        }
        double flu = 2.0 * 12 * 8 * 18 * 4 * (double)iters * g2 * 4;
        ms = timeit([&] { hybrid_kernel<18><<<g2, 128>>>(out, iters); });
        printf("hybrid 18 DMMA + 72 DFMA + 22 DMUL, 8 warps/SM, USEFUL: %.2f TFLOP/s\n", flu / ms / 1e9);
        ms = timeit([&] { hybrid_kernel<9><<<g2 * 2, 128>>>(out, iters); });
        printf("hybrid half (9 DMMA + 36 DFMA + 13 DMUL), 16 warps/SM, USEFUL: %.2f TFLOP/s\n", flu / ms / 1e9);
        ms = timeit([&] { hybrid_kernel<9><<<g2, 128>>>(out, iters); });
        printf("hybrid half, 8 warps/SM, USEFUL: %.2f TFLOP/s\n", flu / 2 / ms / 1e9);
    }
    {
        long long gs = 1 << 21;
        double* g; CK(cudaMalloc(&g, sizeof(double) * gs));
        cudaMemset(g, 0, sizeof(double) * gs);
        int iters = 256;
        float ms = timeit([&] { redg_kernel<<<blocks, threads>>>(g, gs, iters); });
        double ops = (double)iters * blocks * threads;
        printf("global f64 RED (16 MB grid, 32 contiguous per warp): %.1f Gop/s\n", ops / ms / 1e6);
        cudaFree(g);
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
