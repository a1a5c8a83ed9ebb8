// Random 32-byte row reads from a DRAM-sized array (the weighted-reverse alpha
// gather).  One lane per row; reports time and effective bytes/row from HBM
// throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/randbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__global__ void rd(const float *A, const int *idx, int64_t n, float *out) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    float acc = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float *p = A + (int64_t)idx[i] * 8;
        unsigned u[8];
        if (MODE == 0) {
            asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p));
        } else if (MODE == 1) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p), "l"(pol));
        } else if (MODE == 2) {
            asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]) : "l"(p));
            asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p + 4));
        } else if (MODE == 3) {
            asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(u[0]) : "l"(p));
            for (int k = 1; k < 8; k++) u[k] = 0;
        } else if (MODE == 4) {
            asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p));
        } else {
            asm volatile("ld.global.nc.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]) : "l"(p));
        }
        for (int k = 0; k < 8; k++) acc += __uint_as_float(u[k]);
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int MODE>
void run(const float *A, const int *idx, int64_t n, float *out, const char *name) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < 2; r++) rd<MODE><<<148 * 8, 256>>>(A, idx, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) rd<MODE><<<148 * 8, 256>>>(A, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-40s %.3f ms  %.2f G rows/s  (x32B = %.0f GB/s)\n", name, ms, n / ms / 1e6, n * 32.0 / ms / 1e6);
}

int main() {
    const int64_t rows = 114615892LL * 1;   // alpha rows (E), 32 B each = 3.67 GB
    const int64_t n = 114615892LL;
    std::vector<int> h(n);
    std::mt19937_64 rng(7);
    for (int64_t i = 0; i < n; i++) h[i] = (int)(rng() % rows);
    float *A, *out; int *idx;
    cudaMalloc(&A, rows * 32); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    cudaMemset(A, 0, rows * 32);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    run<0>(A, idx, n, out, "nc.v8");
    run<1>(A, idx, n, out, "nc.no_alloc.evict_first_policy.v8");
    run<2>(A, idx, n, out, "nc.v4 x2");
    run<3>(A, idx, n, out, "nc.b32 (4B of the row)");
    run<4>(A, idx, n, out, "cs.v8");
    run<5>(A, idx, n, out, "nc.L2::evict_first.v8");
    return 0;
}
