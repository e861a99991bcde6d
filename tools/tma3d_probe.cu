// tma3d_probe.cu -- isolated check of the 3-D tensor copy (cp.async.bulk.tensor.3d, UTMALDG) the
// interpolation stages its 12^3 grid blocks with: one warp loads a box of an n^3 FP64 grid at a
// given corner into shared memory on an mbarrier and writes it back; compared on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma3d_probe tools/tma3d_probe.cu && ./tma3d_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct alignas(64) Tmap { unsigned char b[128]; };

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE, int NOTILE>
__global__ void probe(const __grid_constant__ Tmap tm, const Tmap* gtm, int c0, int c1, int c2, double* out, int box) {
    extern __shared__ __align__(128) double sm[];
    unsigned long long& mb = *reinterpret_cast<unsigned long long*>(sm + box * box * box);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mb)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const void* map = MODE == 0 ? (const void*)&tm : (const void*)gtm;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb)), "r"(box * box * box * 8) : "memory");
        if (NOTILE)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(sm)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&mb)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(sm)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&mb)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&mb)) : "memory");
    for (int i = threadIdx.x; i < box * box * box; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int n = 64, box = 12;
    std::vector<double> h((size_t)n * n * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *g, *o;
    cudaMalloc(&g, h.size() * 8);
    cudaMalloc(&o, box * box * box * 8);
    cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    Tmap tm;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
    const cuuint64_t str[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
    const cuuint32_t bd[3] = {(cuuint32_t)box, (cuuint32_t)box, (cuuint32_t)box}, es[3] = {1, 1, 1};
    const int var = argc > 2 ? atoi(argv[2]) : 0;   // bit 0: no .tile, bit 1: no L2 promotion, bit 2: UINT64
    CUresult r = fn((CUtensorMap*)&tm, (var & 4) ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g,
                    dims, str, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    (var & 2) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (entry query %d) map[0..15] =", (int)r, (int)q);
    for (int i = 0; i < 16; ++i) printf(" %02x", tm.b[i]);
    printf("\n");
    if (var & 8) {   // direct driver call (linked -lcuda)
        r = cuTensorMapEncodeTiled((CUtensorMap*)&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, bd, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("direct encode %d\n", (int)r);
    }
    Tmap* gtm;
    cudaMalloc(&gtm, sizeof(Tmap));
    cudaMemcpy(gtm, &tm, sizeof(Tmap), cudaMemcpyHostToDevice);
    const int c0 = 5, c1 = 7, c2 = 9;   // (z, y, x) corner
    const int mode0 = argc > 1 ? atoi(argv[1]) : 0;
    for (int mode = mode0; mode < mode0 + 1; ++mode) {
        cudaMemset(o, 0, box * box * box * 8);
        const size_t smb = box * box * box * 8 + 16;
        if (mode == 0 && !(var & 1)) probe<0, 0><<<1, 128, smb>>>(tm, gtm, c0, c1, c2, o, box);
        else if (mode == 0) probe<0, 1><<<1, 128, smb>>>(tm, gtm, c0, c1, c2, o, box);
        else if (!(var & 1)) probe<1, 0><<<1, 128, smb>>>(tm, gtm, c0, c1, c2, o, box);
        else probe<1, 1><<<1, 128, smb>>>(tm, gtm, c0, c1, c2, o, box);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(box * box * box);
        cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int x = 0; x < box; ++x)
            for (int y = 0; y < box; ++y)
                for (int z = 0; z < box; ++z)
                    bad += ho[(x * box + y) * box + z] != h[((size_t)(c2 + x) * n + (c1 + y)) * n + (c0 + z)];
        printf("var %d mode %d (%s): %s, mismatches %d\n", var, mode, mode ? "map in global" : "grid_constant param",
               cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
