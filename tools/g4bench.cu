// Microbenchmark: TMA gather4 (UTMALDG.2D.GATHER4) of random 256-B rows into a
// per-warp shared-memory ring vs the LDG.256 register path (tools/l2bench.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/g4bench.cu -o tools/g4bench
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void g4(float *dst, const CUtensorMap *tm, int c0, int r0, int r1, int r2, int r3, uint64_t *b) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                   "r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}

template <int NS, int G4>   // NS ring slots per warp, G4 gather4 per slot (slot = 4*G4 rows)
__global__ void __launch_bounds__(256) tma_gather(const __grid_constant__ CUtensorMap tm, const int *idx, int64_t n, float *out) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bars[8][NS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *ring = smem + warp * NS * G4 * 256;
    constexpr int ROWS = 4 * G4;
    const int64_t warps = (int64_t)gridDim.x * 8, w = (int64_t)blockIdx.x * 8 + warp;
    const int64_t chunk = (n + warps - 1) / warps;
    const int64_t b0 = w * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
    if (lane == 0) for (int s = 0; s < NS; s++) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t nslots = b0 < b1 ? (b1 - b0 + ROWS - 1) / ROWS : 0;
    // indices: each lane holds idx for one edge of a 32-edge window; the window for
    // slots [8k, 8k+8) (G4 = 1) is loaded one window ahead, rows fetched via shfl
    constexpr int SPW = 32 / ROWS;   // slots per 32-edge window
    auto load_win = [&](int64_t wi) { int64_t e = b0 + wi * 32 + lane; return e < b1 ? idx[e] : 0; };
    int cur = load_win(0), nxt = load_win(1);
    int64_t curw = 0;
    auto issue = [&](int64_t t) {     // all lanes call (shfl); lane 0 issues
        const int64_t wi = t / SPW;
        while (curw < wi) { cur = nxt; nxt = load_win(curw + 2); curw++; }
        const int s = (int)(t % NS);
        const int base = (int)(t % SPW) * ROWS;
        int r[ROWS];
        for (int k = 0; k < ROWS; k++) r[k] = __shfl_sync(0xffffffffu, cur, base + k);
        if (lane == 0) {
            mbar_expect(&bars[warp][s], ROWS * 256);
            for (int q = 0; q < G4; q++)
                g4(ring + s * ROWS * 64 + q * 256, &tm, 0, r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3], &bars[warp][s]);
        }
    };
    for (int64_t t = 0; t < NS - 1 && t < nslots; t++) issue(t);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t t = 0; t < nslots; t++) {
        if (t + NS - 1 < nslots) issue(t + NS - 1);
        const int s = (int)(t % NS);
        mbar_wait(&bars[warp][s], (unsigned)((t / NS) & 1));
        const float *src = ring + s * ROWS * 64;
        for (int k = lane * 8; k < ROWS * 64; k += 256) {
            float4 a = *reinterpret_cast<const float4 *>(src + k), b = *reinterpret_cast<const float4 *>(src + k + 4);
            acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w; acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
        }
        __syncwarp();
    }
    float sum = 0; for (int k = 0; k < 8; k++) sum += acc[k];
    if (sum == 1234.5f) out[0] = sum;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NS, int G4>
void run(const CUtensorMap &tm, const int *idx, int64_t n, float *out, int cps) {
    const size_t smem = (size_t)8 * NS * G4 * 1024;
    cudaFuncSetAttribute(tma_gather<NS, G4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < 2; r++) tma_gather<NS, G4><<<148 * cps, 256, smem>>>(tm, idx, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) tma_gather<NS, G4><<<148 * cps, 256, smem>>>(tm, idx, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    cudaError_t e = cudaGetLastError();
    printf("NS=%d G4=%d ctas/SM=%d smem=%zuKB: %.3f ms %.1f GB/s %s\n", NS, G4, cps, smem >> 10, ms, n * 256.0 / ms / 1e6, cudaGetErrorString(e));
}

int main(int argc, char **argv) {
    const int64_t V = 232965, n = 114615892;
    std::vector<int> h(n);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < n; i++) h[i] = (int)(rng() % V);
    float *X, *out; int *idx;
    cudaMalloc(&X, V * 64 * 4); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
    cudaMemset(X, 0, V * 64 * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)V}, strides[1] = {64 * 4};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    run<4, 1>(tm, idx, n, out, 4);
    run<8, 1>(tm, idx, n, out, 3);
    run<8, 1>(tm, idx, n, out, 2);
    run<4, 2>(tm, idx, n, out, 3);
    run<6, 1>(tm, idx, n, out, 4);
    run<12, 1>(tm, idx, n, out, 2);
    return 0;
}
