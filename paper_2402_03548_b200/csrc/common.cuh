// sm_100a kernels of the GraphPy sparse hot path (arxiv 2402.03548): shared
// device primitives (internal).  Kernels: spmm.cu, sddmm.cu, softmax.cu, gat.cu.
//
// All three families are sparse gather-reduces (no dense contraction), so they
// run on the LSU / L2 path, not on tensor cores.  Common
// structure:
//   * rows come from a degree-ordered schedule built at graph create (rows by
//     descending degree, LPT order): the first n_heavy rows (degree > kHeavyThreshold = 2048)
//     get a whole CTA (8 warps split the row's edge list, deterministic smem
//     combine), the rest one warp each (8 rows per CTA);
//   * a warp walks its edge list in 32-edge tiles: one coalesced load of 32
//     column ids (+ the per-edge scale / edge-ID-indirected weight row), staged
//     in shared memory so that each lane group fetches (col, weight) pairs with
//     one 128-bit LDS per two edges;
//   * feature rows are gathered by groups of LPE lanes, G = 32/LPE edges per
//     warp instruction, with 256-bit (LDG.E.256, sm_100) or 128-bit loads and
//     an L2 evict_last policy (the gathered table is the reused operand);
//     index / edge-value streams use L1::no_allocate + L2 evict_first so they
//     do not push the table out of L2;
//   * fp32 accumulation: plain sums over <= 128-edge chunks folded into a
//     Kahan-compensated running sum (error independent of row length).
// No atomics; every output element is written exactly once per call.
#pragma once
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace gsp {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kHMax = 16;        // weighted modes stage w rows of <= kHMax heads in smem
constexpr int kFoldTiles = 4;    // 32-edge tiles summed plainly before a Kahan fold

template <int VEC>
struct Vec {
    float v[VEC];
};

// ------------------------------------------------------- memory primitives
struct Pol {
    uint64_t keep, stream;
};
__device__ __forceinline__ Pol make_pol() {
    Pol p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.stream));
    return p;
}

// gathered feature rows: read-only path, L2 evict_last
template <int VEC>
__device__ __forceinline__ void ld_keep(Vec<VEC> &r, const float *p, uint64_t pol) {
    if constexpr (VEC == 8) {
        unsigned u0, u1, u2, u3, u4, u5, u6, u7;
        asm volatile("ld.global.nc.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3), "=r"(u4), "=r"(u5), "=r"(u6), "=r"(u7)
                     : "l"(p), "l"(pol));
        r.v[0] = __uint_as_float(u0); r.v[1] = __uint_as_float(u1);
        r.v[2] = __uint_as_float(u2); r.v[3] = __uint_as_float(u3);
        r.v[4] = __uint_as_float(u4); r.v[5] = __uint_as_float(u5);
        r.v[6] = __uint_as_float(u6); r.v[7] = __uint_as_float(u7);
    } else if constexpr (VEC == 4) {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                     : "l"(p), "l"(pol));
    } else {
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.v[0]) : "l"(p), "l"(pol));
    }
}
// streamed once: no L1 allocation, L2 evict_first
__device__ __forceinline__ int ld_stream_i32(const int32_t *p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
// one 32-byte edge-value row (H = 8) in a single 256-bit request: one L2 sector
__device__ __forceinline__ void ld_stream_v8(float *d, const float *p, uint64_t pol) {
    unsigned u0, u1, u2, u3, u4, u5, u6, u7;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3), "=r"(u4), "=r"(u5), "=r"(u6), "=r"(u7)
                 : "l"(p), "l"(pol));
    d[0] = __uint_as_float(u0); d[1] = __uint_as_float(u1); d[2] = __uint_as_float(u2); d[3] = __uint_as_float(u3);
    d[4] = __uint_as_float(u4); d[5] = __uint_as_float(u5); d[6] = __uint_as_float(u6); d[7] = __uint_as_float(u7);
}

__device__ __forceinline__ float ld_stream_f32(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// one streamed 16-byte vector (edge-value rows of H = 4k heads)
__device__ __forceinline__ float4 ld_stream_f4(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}

// bulk L2 prefetch of the 16-B-aligned span covering [p, p + bytes) (a hint:
// streamed edge arrays reach L2 tiles ahead of their register loads).  The span
// may round past the array end by < 16 B: device allocations are >= 256-B granular.
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    const uintptr_t s = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s), "r"((uint32_t)(e - s)) : "memory");
}

// async global -> shared copies (LDGSTS): edge-value rows land in smem without
// occupying registers; src_size 0 zero-fills (padding lanes)
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc, int src_size) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async4(void *sdst, const void *gsrc, int src_size) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gsrc), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// plain (coherent) loads of data the caller may alias with the output (softmax in place)
__device__ __forceinline__ float4 ld_f4(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_f32(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream_f32(float *p, float v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream_f4(float *p, float4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}

// Packed fp32 pair FMA (FFMA2, sm_100): a[0:2] = w * x[0:2] + a[0:2], each lane
// an IEEE round-to-nearest fma exactly like FFMA -- half the issue slots of the
// gather-reduce and dot-product inner loops (DESIGN.md §6 "FFMA2").
__device__ __forceinline__ void fma2(float &a0, float &a1, float w0, float w1, float x0, float x1) {
    const float2 r = __ffma2_rn(make_float2(w0, w1), make_float2(x0, x1), make_float2(a0, a1));
    a0 = r.x;
    a1 = r.y;
}

template <int VEC>
__device__ __forceinline__ void vzero(Vec<VEC> &r) {
#pragma unroll
    for (int k = 0; k < VEC; k++) r.v[k] = 0.f;
}
// store the first `lim` (<= VEC) elements; vector stores when lim == VEC
template <int VEC>
__device__ __forceinline__ void vstore(float *p, const Vec<VEC> &r, int64_t lim) {
    if constexpr (VEC >= 4) {
        if (lim >= VEC) {
#pragma unroll
            for (int k = 0; k < VEC; k += 4)
                *reinterpret_cast<float4 *>(p + k) = make_float4(r.v[k], r.v[k + 1], r.v[k + 2], r.v[k + 3]);
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < VEC; k++)
        if (k < lim) p[k] = r.v[k];
}

// Row and edge range of this warp.  Heavy rows: the whole CTA, contiguous
// 32-aligned slices per warp.  Returns false if the warp has no row.
__device__ __forceinline__ bool warp_task(const int32_t *task, int64_t nrows, int64_t n_heavy, int warp,
                                          int64_t &row, int64_t &b, int64_t &e, bool &heavy) {
    heavy = (int64_t)blockIdx.x < n_heavy;
    const int64_t idx = heavy ? (int64_t)blockIdx.x : n_heavy + ((int64_t)blockIdx.x - n_heavy) * kWarps + warp;
    if (idx >= nrows) return false;
    const int4 t = __ldg(reinterpret_cast<const int4 *>(task) + idx);   // {row, degree, b lo, b hi}
    row = t.x;
    const int64_t rb = (int64_t)(((uint64_t)(uint32_t)t.w << 32) | (uint32_t)t.z), deg = t.y;
    if (heavy) {
        const int64_t re = rb + deg;
        const int64_t per = (((deg + kWarps - 1) / kWarps) + 31) & ~int64_t(31);
        b = min(re, rb + per * warp);
        e = min(re, b + per);
    } else {
        b = rb;
        e = rb + deg;
    }
    return true;
}

// exp(x) for x <= 0 via ex2.approx: relative error ~2^-22 + |x| 2^-24 (x is a
// logit difference, |x| <~ 100), far inside the 2e-5 absolute bound on alpha.
__device__ __forceinline__ float fast_exp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}

inline bool aligned(const void *p, unsigned bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }
inline int pow2ceil(int64_t x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline dim3 row_grid(int64_t nrows, int64_t n_heavy, int64_t slabs) {
    return dim3((unsigned)(n_heavy + ceil_div(nrows - n_heavy, kWarps)), (unsigned)slabs, 1);
}

}  // namespace
}  // namespace gsp
