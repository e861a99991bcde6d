// tma_rank_probe.cu -- which tensor-copy ranks / boxes work on this B200 (diagnostic for the
// interpolation's TMA block staging): rank R in {1,2,3}, box edge B, FP64, map passed as a
// __grid_constant__ kernel parameter.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct alignas(64) Tmap { unsigned char b[128]; };
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int R>
__global__ void k(const __grid_constant__ Tmap tm, int c0, int c1, int c2, double* out, int elems) {
    extern __shared__ __align__(1024) double sm[];
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(sm + 16384);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(elems * 8) : "memory");
        if (R == 1)
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                         ::"r"(su32(sm)), "l"(&tm), "r"(c0), "r"(su32(mb)) : "memory");
        else if (R == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(sm)), "l"(&tm), "r"(c0), "r"(c1), "r"(su32(mb)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(sm)), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(mb)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(mb)) : "memory");
    for (int i = threadIdx.x; i < elems; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int R = atoi(argv[1]), B = atoi(argv[2]), c = argc > 3 ? atoi(argv[3]) : 0;
    const int n = 64;
    std::vector<double> h((size_t)n * n * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *g, *o;
    cudaMalloc(&g, h.size() * 8);
    cudaMalloc(&o, 16384 * 8);
    cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    Tmap tm;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
    if (R == 1) dims[0] = (cuuint64_t)n * n * n;
    const cuuint64_t str[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
    const cuuint32_t bd[3] = {(cuuint32_t)B, (cuuint32_t)B, (cuuint32_t)B}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled((CUtensorMap*)&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, R, g, dims, str, bd, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int elems = B;
    for (int a = 1; a < R; ++a) elems *= B;
    const size_t smb = 16384 * 8 + 64;
    cudaError_t e;
    if (R == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb); k<1><<<1, 128, smb>>>(tm, c, c, c, o, elems); }
    else if (R == 2) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb); k<2><<<1, 128, smb>>>(tm, c, c, c, o, elems); }
    else { cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb); k<3><<<1, 128, smb>>>(tm, c, c, c, o, elems); }
    e = cudaDeviceSynchronize();
    std::vector<double> ho(elems);
    cudaMemcpy(ho.data(), o, elems * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < elems; ++i) {
        int z = i % B, y = (i / B) % B, x = i / B / B;
        size_t gi = R == 1 ? (size_t)(c + i) : R == 2 ? (size_t)(c + y) * n + (c + z) : ((size_t)(c + x) * n + (c + y)) * n + (c + z);
        if (R == 2) gi = (size_t)(c + i / B) * n + (c + i % B);
        bad += ho[i] != h[gi];
    }
    printf("rank %d box %d corner %d: encode %d, %s, mismatches %d\n", R, B, c, (int)r, cudaGetErrorString(e), bad);
    return 0;
}
