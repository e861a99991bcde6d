// interp_mix.cu -- microbenchmark of the interp3 k-step instruction mix on the shared FP64 pipe:
// 36 DMMA m8n8k4 (3 m-tiles x 4 n-tiles x 3 k-slices, fresh accumulators per step) followed by
// 24 DFMAs that consume the step's DMMA results, as in interp3_dmma_kernel.
//   MODE 0: DFMAs consume this step's d (the kernel's dependency structure)
//   MODE 1: DFMAs consume the previous step's d (software-pipelined, 2x accumulator registers)
//   MODE 2: 36 DMMA only, accumulators carried across steps (no vector ops: the DMMA ceiling)
//   MODE 3: MODE 0 with the 24 DFMAs replaced by 8 (one per n-tile/e pair)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/interp_mix tools/interp_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(128, MODE == 1 ? 2 : 3) mix_kernel(double* out, int iters) {
    const int t = threadIdx.x;
    double a[3][3], b[3][4];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) a[i][j] = 1e-3 * (i + 1) + 1e-6 * (j + t);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) b[i][j] = 1e-3 * (j + 1) - 1e-7 * (i + t);
    double acc[4][2][3];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[i][e][0] = acc[i][e][1] = acc[i][e][2] = 0.0;
    double dp[3][4][2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dp[r][nt][0] = dp[r][nt][1] = 0.0;
    double x0 = 0.5 + 1e-7 * t, x1 = 0.25 - 1e-7 * t;
    __shared__ double sa[8 * 9 * 32];
    for (int i = t; i < 8 * 9 * 32; i += blockDim.x) sa[i] = 1e-3 + 1e-6 * i;
    __syncthreads();
    const int lane = t & 31;
    for (int it = 0; it < iters; ++it) {
        // A fragments from shared memory, as in the kernel (keeps the DMMAs loop-variant)
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s) a[r][s] = sa[((it & 7) * 9 + r * 3 + s) * 32 + lane];
        double d[3][4][2];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
                if (MODE == 2) { d[r][nt][0] = dp[r][nt][0]; d[r][nt][1] = dp[r][nt][1]; }
                else d[r][nt][0] = d[r][nt][1] = 0.0;
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma884(d[r][nt][0], d[r][nt][1], a[r][s], b[s][nt]);
        if (MODE == 0 || MODE == 3) {
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (MODE == 0) {
                        acc[nt][e][0] = fma(x0, d[0][nt][e], acc[nt][e][0]);
                        acc[nt][e][1] = fma(x1, d[1][nt][e], acc[nt][e][1]);
                        acc[nt][e][2] = fma(x1, d[2][nt][e], acc[nt][e][2]);
                    } else {
                        acc[nt][e][0] = fma(x0, d[0][nt][e], acc[nt][e][0]);
                    }
                }
        } else if (MODE == 1) {
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    acc[nt][e][0] = fma(x0, dp[0][nt][e], acc[nt][e][0]);
                    acc[nt][e][1] = fma(x1, dp[1][nt][e], acc[nt][e][1]);
                    acc[nt][e][2] = fma(x1, dp[2][nt][e], acc[nt][e][2]);
                }
        }
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) { dp[r][nt][0] = d[r][nt][0]; dp[r][nt][1] = d[r][nt][1]; }
        x0 += 1e-9;
        x1 -= 1e-9;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e) s += acc[i][e][0] + acc[i][e][1] + acc[i][e][2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) s += dp[r][nt][0] + dp[r][nt][1];
    out[blockIdx.x * blockDim.x + t] = s;
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 4 * 128);
    const int iters = 20000;
    for (int cps : {2, 3}) {
        const int grid = sms * cps;
        const double fl = 2.0 * 256 * 36 * (double)iters * grid * 4;
        float ms0 = timeit([&] { mix_kernel<0><<<grid, 128>>>(out, iters); });
        float ms1 = timeit([&] { mix_kernel<1><<<grid, 128>>>(out, iters); });
        float ms2 = timeit([&] { mix_kernel<2><<<grid, 128>>>(out, iters); });
        float ms3 = timeit([&] { mix_kernel<3><<<grid, 128>>>(out, iters); });
        printf("%d warps/SM: 36 DMMA + 24 dependent DFMA: %.2f TF | DFMAs on previous step: %.2f TF | "
               "DMMA only: %.2f TF | 36 DMMA + 8 DFMA: %.2f TF (DMMA flops)\n",
               4 * cps, fl / ms0 / 1e9, fl / ms1 / 1e9, fl / ms2 / 1e9, fl / ms3 / 1e9);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
