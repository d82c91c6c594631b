// Probe: TMA 2-D tile load from a tensor map held in (a) global memory, (b) a
// __grid_constant__ kernel parameter; mbarrier completion.  Not product code.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <dlfcn.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const CUtensorMap* gmap, const __grid_constant__ CUtensorMap pmap, float* out, int col, int row) {
    __shared__ __align__(128) float buf[16 * 16];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
        if (MODE == 2 || MODE >= 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (MODE == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
        } else {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(16 * 16 * 4) : "memory");
        }
        const void* m = (MODE == 3 || MODE == 5) ? (const void*)&pmap : (const void*)gmap;
        if (MODE == 1 || MODE == 2 || MODE == 3)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(su(buf)), "l"(m), "r"(col), "r"(row), "r"(su(&bar)) : "memory");
        if (MODE == 8)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(su(buf)), "l"(m), "r"(col), "r"(row), "r"(su(&bar)) : "memory");
        if (MODE == 4 || MODE == 5)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(su(buf)), "l"(m), "r"(col), "r"(row), "r"(su(&bar)) : "memory");
    }
    if (MODE == 6) {
        __syncthreads();
    } else {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(su(&bar)), "r"(0) : "memory");
    }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int CX = argc > 2 ? atoi(argv[2]) : -2, CY = argc > 3 ? atoi(argv[3]) : 3;
    const int W = 40, Hh = 40, P = 40;
    float* src; cudaMalloc(&src, P * Hh * 4);
    float h[P * Hh]; for (int i = 0; i < P * Hh; ++i) h[i] = (float)i;
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m; memset(&m, 0, sizeof(m));
    cuuint64_t dims[2] = {W, Hh}; cuuint64_t str[1] = {P * 4}; cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    if (mode >= 10) {
        void* h = dlopen("libcuda.so.1", RTLD_NOW);
        auto enc2 = (PFN_cuTensorMapEncodeTiled_v12000)dlsym(h, "cuTensorMapEncodeTiled");
        CUtensorMap m2; memset(&m2, 0, sizeof(m2));
        CUresult r2 = enc2(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("dlsym encode %d same=%d fn %p vs %p\n", (int)r2, memcmp(&m, &m2, sizeof(m)) == 0, fn, (void*)enc2);
        const unsigned* w = (const unsigned*)&m; const unsigned* w2 = (const unsigned*)&m2;
        for (int i = 0; i < 32; ++i) printf("%08x%s", w[i], i % 8 == 7 ? "\n" : " ");
        for (int i = 0; i < 32; ++i) printf("%08x%s", w2[i], i % 8 == 7 ? "\n" : " ");
        m = m2;
        mode -= 10;
    }
    CUtensorMap* g; cudaMalloc(&g, sizeof(m)); cudaMemcpy(g, &m, sizeof(m), cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 256 * 4);
    float o[256];
#define RUN(M) { cudaMemset(out, 0, 1024); probe<M><<<1, 128>>>(g, m, out, CX, CY); cudaError_t e = cudaDeviceSynchronize(); \
    cudaMemcpy(o, out, 1024, cudaMemcpyDeviceToHost); printf("mode %d: %s  o[0]=%g o[2]=%g o[17]=%g\n", M, cudaGetErrorString(e), o[0], o[2], o[17]); if (e) return 1; }
    if (mode == 7) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
        cudaMemset(out, 0, 1024);
        cudaError_t e0 = cudaLaunchKernelEx(&cfg, probe<1>, (const CUtensorMap*)g, m, out, -2, 3);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(o, out, 1024, cudaMemcpyDeviceToHost);
        printf("mode 7 (cluster launch): %s %s o[0]=%g o[2]=%g o[17]=%g\n", cudaGetErrorString(e0), cudaGetErrorString(e), o[0], o[2], o[17]);
        return 0;
    }
    switch (mode) { case 8: RUN(8) break; case 0: RUN(0) break; case 1: RUN(1) break; case 2: RUN(2) break; case 3: RUN(3) break;
                    case 4: RUN(4) break; case 5: RUN(5) break; }
    return 0;
}
