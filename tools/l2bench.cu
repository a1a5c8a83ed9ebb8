// Microbenchmark: random 256-B row gathers from an L2-resident table (the
// gspmm access pattern without the sparse bookkeeping).  Prints GB/s for
// several unroll depths / occupancies.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/l2bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld8(float *r, const float *p) {
    unsigned u[8];
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p));
    for (int k = 0; k < 8; k++) r[k] = __uint_as_float(u[k]);
}

template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) gather(const float *X, const int *idx, int64_t n, float *out) {
    // 8 lanes per 256-B row, 4 rows per warp instruction
    const int lane = threadIdx.x & 31, g = lane >> 3, sub = lane & 7;
    const int64_t warps = (int64_t)gridDim.x * 8;
    const int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t base = w * 4 * U; base < n; base += warps * 4 * U) {
        float x[U][8];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t e = base + u * 4 + g;
            const int c = e < n ? __ldg(idx + e) : 0;
            ld8(x[u], X + (int64_t)c * 64 + sub * 8);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int k = 0; k < 8; k++) acc[k] += x[u][k];
    }
    float s = 0;
    for (int k = 0; k < 8; k++) s += acc[k];
    if (s == 12345.f) out[0] = s;
}

template <int U, int MINB>
void run(const float *X, const int *idx, int64_t n, float *out, int blocks_per_sm) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    int grid = 148 * blocks_per_sm;
    for (int r = 0; r < 3; r++) gather<U, MINB><<<grid, 256>>>(X, idx, n, out);
    cudaEventRecord(a);
    const int R = 10;
    for (int r = 0; r < R; r++) gather<U, MINB><<<grid, 256>>>(X, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= R;
    printf("U=%d minB=%d blocks/SM=%d: %.3f ms  %.1f GB/s (rows) \n", U, MINB, blocks_per_sm, ms, n * 256.0 / ms / 1e6);
}

int main(int argc, char **argv) {
    const int64_t V = argc > 1 ? atoll(argv[1]) : 232965;   // rows of 64 floats
    const int64_t n = 114615892;
    std::vector<int> h(n);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < n; i++) h[i] = (int)(rng() % V);
    float *X, *out; int *idx;
    cudaMalloc(&X, V * 64 * 4); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    cudaMemset(X, 0, V * 64 * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    printf("table %.1f MB, %ld gathers\n", V * 256 / 1e6, (long)n);
    run<2, 4>(X, idx, n, out, 8);
    run<4, 4>(X, idx, n, out, 8);
    run<4, 3>(X, idx, n, out, 6);
    run<8, 3>(X, idx, n, out, 6);
    run<8, 2>(X, idx, n, out, 4);
    run<16, 2>(X, idx, n, out, 4);
    run<4, 8>(X, idx, n, out, 8);
    run<8, 4>(X, idx, n, out, 8);
    return 0;
}
