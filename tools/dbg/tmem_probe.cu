// TMEM semantics probe: each warp stores lane*1000 + col into its lane quarter /
// column half, reads back, reports mismatches.
#include <cstdio>
#include <cstdint>
__global__ void k(int *bad, int mode) {
    __shared__ uint32_t s_tmem;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(&s_tmem);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa), "r"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t base = s_tmem;
    uint32_t t = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
#pragma unroll 1
    for (int c = 0; c < 128; c += 8) {
        float v[8];
        for (int i = 0; i < 8; i++) v[i] = (float)(warp * 100000 + lane * 1000 + c + i);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(t + c),
                     "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]) : "memory");
        if (mode == 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    int nb = 0;
    for (int c = 0; c < 128; c += 8) {
        float v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "r"(t + c) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; i++) if (v[i] != (float)(warp * 100000 + lane * 1000 + c + i)) { if (nb < 3 && blockIdx.x == 0) printf("w%d l%d c%d got %f\n", warp, lane, c + i, v[i]); nb++; }
    }
    atomicAdd(bad, nb);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(256) : "memory");
    }
}
int main() {
    int *bad; cudaMallocManaged(&bad, 4);
    for (int mode = 0; mode < 2; mode++) {
        *bad = 0;
        k<<<296, 256>>>(bad, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: err=%s bad=%d\n", mode, cudaGetErrorString(e), *bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
