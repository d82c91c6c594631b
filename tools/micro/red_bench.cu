// Microbenchmark: bilinear splat of N random particles into a W x W grid
// with scalar REDs vs 16-byte vector REDs (red.global.add.v4.f32).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void splat_scalar(float* g, int W, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    unsigned h = hash(i); int r = h % (W - 1), c = (h >> 12) % (W - 1); float a = 1.f, fu = 0.3f, fv = 0.6f;
    float* q = g + (size_t)r * W + c;
    atomicAdd(q, a * (1 - fu) * (1 - fv)); atomicAdd(q + W, a * fu * (1 - fv)); atomicAdd(q + 1, a * (1 - fu) * fv); atomicAdd(q + W + 1, a * fu * fv);
}
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red2(float* p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void row_pair(float* row, int c, float v0, float v1) {
    const int s = c & 3; float* b = row + (c - s);
    if (s == 0) red4(b, v0, v1, 0.f, 0.f);
    else if (s == 1) red4(b, 0.f, v0, v1, 0.f);
    else if (s == 2) red2(b + 2, v0, v1);
    else { red2(b + 2, 0.f, v0); red2(b + 4, v1, 0.f); }
}
__global__ void splat_vec(float* g, int W, int n) {   // W multiple of 4
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    unsigned h = hash(i); int r = h % (W - 1), c = (h >> 12) % (W - 5); float a = 1.f, fu = 0.3f, fv = 0.6f;
    row_pair(g + (size_t)r * W, c, a * (1 - fu) * (1 - fv), a * (1 - fu) * fv);
    row_pair(g + (size_t)(r + 1) * W, c, a * fu * (1 - fv), a * fu * fv);
}
__global__ void splat_quad(float4* g, int W, int n) {   // one v4 RED per particle at its corner cell
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    unsigned h = hash(i); int r = h % (W - 1), c = (h >> 12) % (W - 1); float a = 1.f, fu = 0.3f, fv = 0.6f;
    red4((float*)(g + (size_t)r * W + c), a * (1 - fu) * (1 - fv), a * fu * (1 - fv), a * (1 - fu) * fv, a * fu * fv);
}
int main() {
    const int W = 1040, n = 860000; float* g; cudaMalloc(&g, sizeof(float) * W * W * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = 0; v < 3; ++v) {
        float best = 1e9;
        for (int rep = 0; rep < 20; ++rep) {
            cudaEventRecord(e0);
            cudaMemsetAsync(g, 0, sizeof(float) * W * W * (v == 2 ? 4 : 1));
            if (v == 0) splat_scalar<<<(n + 255) / 256, 256>>>(g, W, n);
            else if (v == 1) splat_vec<<<(n + 255) / 256, 256>>>(g, W, n);
            else splat_quad<<<(n + 255) / 256, 256>>>((float4*)g, W, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 2 && ms < best) best = ms;
        }
        printf("%s: %.1f us for %d particles\n", v == 0 ? "scalar red x4" : v == 1 ? "vector red v4/v2" : "quad v4 x1 (memset incl)", best * 1e3, n);
    }
    return cudaGetLastError() != cudaSuccess;
}
