// sm_100a kernels of the GraphPy sparse hot path (arxiv 2402.03548).
//
// All three families are sparse gather-reduces (no dense contraction), so they
// run on the LSU / L2 path, not on tensor cores.  Common
// structure:
//   * rows come from a degree-ordered schedule built at graph create (rows by
//     descending degree, LPT order): the first n_heavy rows (degree > 1024)
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
__device__ __forceinline__ bool warp_task(const int64_t *off, const int32_t *order, int64_t nrows,
                                          int64_t n_heavy, int warp, int64_t &row, int64_t &b,
                                          int64_t &e, bool &heavy) {
    heavy = (int64_t)blockIdx.x < n_heavy;
    if (heavy) {
        row = order[blockIdx.x];
        const int64_t rb = off[row], re = off[row + 1];
        const int64_t deg = re - rb;
        const int64_t per = (((deg + kWarps - 1) / kWarps) + 31) & ~int64_t(31);
        b = min(re, rb + per * warp);
        e = min(re, b + per);
        return true;
    }
    const int64_t idx = n_heavy + ((int64_t)blockIdx.x - n_heavy) * kWarps + warp;
    if (idx >= nrows) return false;
    row = order[idx];
    b = off[row];
    e = off[row + 1];
    return true;
}

// ============================================================ gSpMM family
// MODE kSpmmScaled      : out[r] = rs(r) * sum_j cs(col_j) * X[col_j]          (gSpMMv + norm)
// MODE kSpmmWeightedFwd : out[r, h-block] = sum_j w[j, h] * X[col_j, h-block]   (gSpMMve)
// MODE kSpmmWeightedRev : out[r, h-block] = sum_k w[eid_k, h] * X[col_k, ...]   (gSpMMve^T via eid)
template <int VEC, int LPE, int CPL, int MODE, bool HAS_CS, int UOVR = 0, int MINB = 0>
__global__ void __launch_bounds__(kThreads, (MINB ? MINB : (VEC * CPL <= 8 ? 3 : 2))) spmm_kernel(const SpmmArgs a) {
    constexpr int G = 32 / LPE;           // edge groups per warp
    constexpr int PER = LPE;              // edges per group per 32-edge tile
    constexpr int UB = 32 / (VEC * CPL);  // loads in flight per lane: ~32 floats
    constexpr int U0 = UOVR ? UOVR : (UB < 2 ? 2 : (UB > 4 ? 4 : UB));
    constexpr int U = U0 > PER ? PER : U0;
    constexpr int SW = VEC * LPE * CPL;   // feature slab handled by this CTA
    constexpr bool W = MODE == kSpmmWeightedFwd || MODE == kSpmmWeightedRev;
    constexpr bool MM = MODE == kSpmmMin || MODE == kSpmmMax;   // min / max reductions (NEXT-3)
    constexpr float ID = MODE == kSpmmMin ? INFINITY : (MODE == kSpmmMax ? -INFINITY : 0.f);
    auto comb = [](float x, float y) {
        if constexpr (MODE == kSpmmMin) return fminf(x, y);
        else if constexpr (MODE == kSpmmMax) return fmaxf(x, y);
        else return x + y;
    };
    constexpr int RED = kWarps * SW;
    constexpr int WS = W ? 2 * kWarps * 32 * kHMax : 0;   // double-buffered weight rows
    __shared__ __align__(16) int2 s_pair[kWarps][32];
    __shared__ __align__(16) float s_raw[RED > WS ? RED : WS];   // weights during the walk, then heavy combine
    // Kahan compensation of narrow lanes lives in smem (touched once per fold):
    // the registers go to gathers in flight
    constexpr bool CMP_SMEM = VEC * CPL <= 8 && !MM;
    __shared__ __align__(16) float s_cmp[CMP_SMEM ? kWarps : 1][CMP_SMEM ? 32 : 1][CMP_SMEM ? VEC * CPL : 1];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, sub = lane % LPE;
    const int64_t f0 = (int64_t)blockIdx.y * SW;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    float rs = 1.f;   // row scale, fetched up front (its latency hides under the row's gathers)
    if constexpr (MODE == kSpmmScaled)
        if (a.row_scale) rs = __ldg(a.row_scale + row);

    // lane constants: feature chunk q covers [f, f + VEC) of head hq
    const char *xl[CPL];
    bool fv[CPL];
    int hq[CPL];
#pragma unroll
    for (int q = 0; q < CPL; q++) {
        const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
        fv[q] = f < a.F;
        xl[q] = reinterpret_cast<const char *>(a.X + (fv[q] ? f : 0));
        hq[q] = W ? (int)((fv[q] ? f : 0) / a.Fh) : 0;
    }
    const uint32_t ldxb = (uint32_t)(a.ldx * 4);
    const int H = W ? (int)a.H : 0;
    const bool w16 = W && (H % 4 == 0) && (a.ldw % 4 == 0) && (reinterpret_cast<uintptr_t>(a.w) & 15u) == 0;
    // H = 8 rows (32 B, one sector): one 256-bit register load per lane, one tile ahead
    const bool w8 = W && H == 8 && a.ldw == 8 && (reinterpret_cast<uintptr_t>(a.w) & 31u) == 0;

    // Summation: <= kFoldTiles*32/G terms per
    // lane summed plainly into `tile`, then folded into a Kahan-compensated
    // running sum (acc, cmp): error O((128/G) u) relative to sum|terms|,
    // independent of the row length.
    constexpr int NT = VEC >= 4 ? 1 : 2;   // independent tile accumulators (ILP for narrow lanes)
    Vec<VEC> acc[CPL], cmp_r[CMP_SMEM ? 1 : CPL], tile[NT][CPL];
    auto cmp_ref = [&](int q, int t) -> float & {
        if constexpr (CMP_SMEM) return s_cmp[warp][lane][q * VEC + t];
        else return cmp_r[q].v[t];
    };
#pragma unroll
    for (int q = 0; q < CPL; q++) {
#pragma unroll
        for (int t = 0; t < VEC; t++) cmp_ref(q, t) = 0.f;
#pragma unroll
        for (int t = 0; t < VEC; t++) {
            acc[q].v[t] = ID;
#pragma unroll
            for (int k = 0; k < NT; k++) tile[k][q].v[t] = ID;
        }
    }
    int ntile = 0;

    // Index pipeline: column ids (and rev edge ids) are
    // loaded two tiles ahead, the dependent per-edge scale one tile ahead, and
    // weight rows are copied global -> smem asynchronously one tile ahead
    // (double buffer), so a tile's gathers never wait on its own index trips.
    const int slot = (lane % G) * PER + lane / G;   // group-contiguous layout
    auto load_idx = [&](int64_t tb, int &c, int &ev) {
        c = 0;
        ev = 0;
        if (tb + lane < e) {
            c = ld_stream_i32(a.col + tb + lane, pol.stream);
            if constexpr (MODE == kSpmmWeightedFwd) ev = (int)(tb + lane);
            else if constexpr (MODE == kSpmmWeightedRev) ev = ld_stream_i32(a.eid + tb + lane, pol.stream);
        }
    };
    auto load_scale = [&](int64_t tb, int c) -> float {
        if constexpr (MODE == kSpmmScaled) {
            if (tb + lane < e) {
                if constexpr (!HAS_CS) return 1.f;
                // per-edge scales: one coalesced stream instead of a gather per edge
                return a.edge_scale ? ld_stream_f32(a.edge_scale + tb + lane, pol.stream) : __ldg(a.col_scale + c);
            }
        }
        return 0.f;
    };
    auto load_w8 = [&](int64_t tb, int ev, float *d) {
        if constexpr (W) {
            if (tb + lane < e) ld_stream_v8(d, a.w + (int64_t)ev * 8, pol.stream);
            else {
#pragma unroll
                for (int t = 0; t < 8; t++) d[t] = 0.f;
            }
        }
    };
    auto issue_w = [&](int64_t tb, int ev, int buf) {
        if constexpr (W) {
            if (w8) return;
            float *dst = s_raw + (buf * kWarps + warp) * 32 * kHMax + slot * H;
            const bool valid = tb + lane < e;
            const float *src = a.w + (int64_t)(valid ? ev : 0) * a.ldw;
            if (w16) {
                for (int t = 0; t < H; t += 4) cp_async16(dst + t, src + t, valid ? 16 : 0);
            } else {
                for (int t = 0; t < H; t++) cp_async4(dst + t, src + t, valid ? 4 : 0);
            }
            cp_async_commit();
        }
    };
    int c1, e1, c2, e2;
    load_idx(b, c1, e1);
    load_idx(b + 32, c2, e2);
    float wv1 = load_scale(b, c1);
    float w8a[W ? 8 : 1];
    if (w8) load_w8(b, e1, w8a);
    else issue_w(b, e1, 0);
    int buf = 0;

    for (int64_t base = b; base < e; base += 32) {
        const int n = (int)(e - base < 32 ? e - base : 32);
        s_pair[warp][slot] = make_int2(c1, __float_as_int(wv1));
        // ---- advance the pipeline before this tile's gathers
        int c3, e3;
        load_idx(base + 64, c3, e3);
        const float wv2 = load_scale(base + 32, c2);
        float w8b[W ? 8 : 1];
        if constexpr (W) {
            if (w8) {
                float *dst = s_raw + (buf * kWarps + warp) * 32 * kHMax + slot * 8;
                reinterpret_cast<float4 *>(dst)[0] = make_float4(w8a[0], w8a[1], w8a[2], w8a[3]);
                reinterpret_cast<float4 *>(dst)[1] = make_float4(w8a[4], w8a[5], w8a[6], w8a[7]);
                load_w8(base + 32, e2, w8b);
            } else {
                issue_w(base + 32, e2, buf ^ 1);
                cp_async_wait<1>();   // this tile's weight rows have landed
            }
        }
        const float *s_w = s_raw + (buf * kWarps + warp) * 32 * kHMax;
        __syncwarp();
        const int2 *gp = &s_pair[warp][g * PER];
        const float *gw = s_w + g * PER * H;

        auto body = [&](int i, bool full, int m) {
            Vec<VEC> x[U][CPL];
            float wt[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                const int4 pp = *reinterpret_cast<const int4 *>(gp + i + u);
                const int cc[2] = {pp.x, pp.z};
                const float ww[2] = {__int_as_float(pp.y), __int_as_float(pp.w)};
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const bool ok = full || (i + u + k < m);
#pragma unroll
                    for (int q = 0; q < CPL; q++) {
                        if (ok && fv[q]) {
                            ld_keep(x[u + k][q],
                                    reinterpret_cast<const float *>(xl[q] + (uint64_t)(uint32_t)cc[k] * ldxb),
                                    pol.keep);
                        } else {
#pragma unroll
                            for (int t = 0; t < VEC; t++) x[u + k][q].v[t] = ID;   // identity of the reduction
                        }
                        if constexpr (W) wt[u + k][q] = gw[(i + u + k) * H + hq[q]];
                        else wt[u + k][q] = ww[k];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < CPL; q++)
#pragma unroll
                    for (int t = 0; t < VEC; t++)
                        if constexpr (MM) tile[u % NT][q].v[t] = comb(tile[u % NT][q].v[t], x[u][q].v[t]);
                        else tile[u % NT][q].v[t] = fmaf(wt[u][q], x[u][q].v[t], tile[u % NT][q].v[t]);
        };
        if (n == 32) {
#pragma unroll 1
            for (int i = 0; i < PER; i += U) body(i, true, PER);
        } else {
            const int m = n > g ? (n - g + G - 1) / G : 0;
#pragma unroll 1
            for (int i = 0; i < m; i += U) body(i, false, m);
        }
        __syncwarp();
        c1 = c2; e1 = e2; c2 = c3; e2 = e3; wv1 = wv2;
        buf ^= 1;
        if constexpr (W) {
#pragma unroll
            for (int t = 0; t < 8; t++) w8a[t] = w8b[t];
        }
        if (++ntile == kFoldTiles || base + 32 >= e) {
            ntile = 0;
#pragma unroll
            for (int q = 0; q < CPL; q++)
#pragma unroll
                for (int t = 0; t < VEC; t++) {
                    if constexpr (MM) {
                        float y = tile[0][q].v[t];
                        if constexpr (NT == 2) y = comb(y, tile[1][q].v[t]);
                        acc[q].v[t] = comb(acc[q].v[t], y);
                    } else {
                        float y = tile[0][q].v[t];
                        if constexpr (NT == 2) y += tile[1][q].v[t];
                        y -= cmp_ref(q, t);
                        const float sum = acc[q].v[t] + y;
                        cmp_ref(q, t) = (sum - acc[q].v[t]) - y;
                        acc[q].v[t] = sum;
                    }
#pragma unroll
                    for (int k = 0; k < NT; k++) tile[k][q].v[t] = ID;
                }
        }
    }
    if constexpr (W) cp_async_wait<0>();   // no copy may outlive the loop (smem is reused)
    // compensated totals, then the G edge groups of the warp (xor tree)
#pragma unroll
    for (int q = 0; q < CPL; q++)
#pragma unroll
        for (int t = 0; t < VEC; t++) {
            float v = acc[q].v[t] - cmp_ref(q, t);
#pragma unroll
            for (int o = LPE; o < 32; o <<= 1) v = comb(v, __shfl_xor_sync(kFull, v, o));
            acc[q].v[t] = v;
        }

    if (!heavy) {
        if (g == 0) {
#pragma unroll
            for (int q = 0; q < CPL; q++) {
                const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
                if (f < a.F) {
                    Vec<VEC> r;
#pragma unroll
                    for (int t = 0; t < VEC; t++) r.v[t] = (MM && b == e) ? 0.f : rs * acc[q].v[t];   // empty row -> 0
                    vstore(a.out + row * a.ldo + f, r, a.F - f);
                }
            }
        }
        return;
    }
    // heavy row: deterministic cross-warp combine in warp order
    float *red = s_raw;
    if constexpr (W) cp_async_wait<0>();
    __syncthreads();   // every warp is done with its s_w slices (aliased by red)
    if (g == 0) {
#pragma unroll
        for (int q = 0; q < CPL; q++)
#pragma unroll
            for (int t = 0; t < VEC; t++) red[warp * SW + (sub + q * LPE) * VEC + t] = acc[q].v[t];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < SW; t += kThreads) {
        const int64_t f = f0 + t;
        if (f < a.F) {
            float v = ID;
#pragma unroll
            for (int w = 0; w < kWarps; w++) v = comb(v, red[w * SW + t]);
            a.out[row * a.ldo + f] = rs * v;
        }
    }
}

// ================================================================ gSDDMMvv
// out[j, h] = <X[row_base + v, head h], Y[col_j, head h]>; CPH = Fh / VEC lanes per head.
template <int VEC, int LPE, int CPL, int CPH, int UOVR = 0, int MINB = 0>
__global__ void __launch_bounds__(kThreads, (MINB ? MINB : (VEC * CPL <= 8 ? 3 : 2))) sddmm_kernel(const SddmmArgs a) {
    constexpr int G = 32 / LPE;
    constexpr int PER = LPE;
    constexpr int UB = 32 / (VEC * CPL);
    constexpr int U0 = UOVR ? UOVR : (UB < 2 ? 2 : (UB > 4 ? 4 : UB));
    constexpr int U = U0 > PER ? PER : U0;
    constexpr int SW = VEC * LPE * CPL;
    __shared__ __align__(16) int s_col[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, sub = lane % LPE;
    const int64_t F = a.H * a.Fh;
    const int64_t f0 = (int64_t)blockIdx.y * SW;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    if (b >= e) return;
    const Pol pol = make_pol();

    const char *yl[CPL];
    bool fv[CPL], wr[CPL];
    int hq[CPL];
    Vec<VEC> xv[CPL];
    // the row's features are fetched once and reused for every edge
    const float *xr = a.X + (a.row_base + row) * a.ldx;
#pragma unroll
    for (int q = 0; q < CPL; q++) {
        const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
        fv[q] = f < F;
        yl[q] = reinterpret_cast<const char *>(a.Y + (fv[q] ? f : 0));
        hq[q] = (int)((fv[q] ? f : 0) / a.Fh);
        wr[q] = fv[q] && (sub % CPH) == 0;
        if (fv[q]) ld_keep(xv[q], xr + f, pol.stream);
        else vzero(xv[q]);
    }
    const uint32_t ldyb = (uint32_t)(a.ldy * 4);

    // column ids are loaded two tiles ahead of their gathers (index pipeline)
    auto load_col = [&](int64_t tb) { return tb + lane < e ? ld_stream_i32(a.col + tb + lane, pol.stream) : 0; };
    int c1 = load_col(b), c2 = load_col(b + 32);
    for (int64_t base = b; base < e; base += 32) {
        const int n = (int)(e - base < 32 ? e - base : 32);
        s_col[warp][(lane % G) * PER + lane / G] = c1;
        c1 = c2;
        c2 = load_col(base + 64);
        __syncwarp();
        const int *gp = &s_col[warp][g * PER];
        float *ob = a.out + (base + g) * a.ldo;   // group g's i-th edge is tile edge g + G*i

        auto body = [&](int i, bool full, int m) {
            Vec<VEC> y[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                const int2 cc = *reinterpret_cast<const int2 *>(gp + i + u);
                const int c2[2] = {cc.x, cc.y};
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const bool ok = full || (i + u + k < m);
#pragma unroll
                    for (int q = 0; q < CPL; q++) {
                        if (ok && fv[q])
                            ld_keep(y[u + k][q],
                                    reinterpret_cast<const float *>(yl[q] + (uint64_t)(uint32_t)c2[k] * ldyb),
                                    pol.keep);
                        else vzero(y[u + k][q]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const bool ok = full || (i + u < m);
#pragma unroll
                for (int q = 0; q < CPL; q++) {
                    float p = 0.f;
#pragma unroll
                    for (int t = 0; t < VEC; t++) p = fmaf(xv[q].v[t], y[u][q].v[t], p);
#pragma unroll
                    for (int o = 1; o < CPH; o <<= 1) p += __shfl_xor_sync(kFull, p, o);
                    if (ok && wr[q]) st_stream_f32(ob + (int64_t)(G * (i + u)) * a.ldo + hq[q], p, pol.stream);
                }
            }
        };
        if (n == 32) {
#pragma unroll 1
            for (int i = 0; i < PER; i += U) body(i, true, PER);
        } else {
            const int m = n > g ? (n - g + G - 1) / G : 0;
            // all lanes run the same trip count (the xor-shuffles need the full warp)
            const int mmax = (n + G - 1) / G;
#pragma unroll 1
            for (int i = 0; i < mmax; i += U) body(i, false, m);
        }
        __syncwarp();
    }
}

// generic gSDDMM for head shapes the vector path does not cover: one thread
// per (edge, head), sequential dot over Fh.
__global__ void __launch_bounds__(kThreads) sddmm_generic_kernel(const SddmmArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const float *xr = a.X + (a.row_base + row) * a.ldx;
    const int64_t tot = (e - b) * a.H;
    for (int64_t t = lane; t < tot; t += 32) {
        const int64_t j = b + t / a.H, h = t % a.H;
        const float *yr = a.Y + (int64_t)__ldg(a.col + j) * a.ldy + h * a.Fh;
        float p = 0.f;
        for (int64_t f = 0; f < a.Fh; f++) p = fmaf(__ldg(xr + h * a.Fh + f), __ldg(yr + f), p);
        a.out[j * a.ldo + h] = p;
    }
}

// ============================================================ edge softmax
__device__ __forceinline__ void online_push(float &m, float &s, float x) {
    if (x > m) {
        s = s * expf(m - x) + 1.f;
        m = x;
    } else {
        s += expf(x - m);
    }
}

// exp(x) for x <= 0 via ex2.approx: relative error ~2^-22 + |x| 2^-24 (x is a
// logit difference, |x| <~ 100), far inside the 2e-5 absolute bound on alpha.
__device__ __forceinline__ float fast_exp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}

// Fast path: e, out contiguous [E, H] (ld == H) with H | 32*VEC, so every lane
// always sees the same VEC heads; HPL = H / VEC lanes per head period.  Pass 1
// keeps a running (max, sum) per head, updated once per batch of UNR values
// (one rescale per batch); pass 2 re-reads the row block (L2-resident: pass 1
// loads use evict_last) and streams alpha = exp(x - m) * (1/s) out.
template <int VEC>
__global__ void __launch_bounds__(kThreads) softmax_kernel(const SoftmaxArgs a) {
    constexpr int UNR = 4;
    constexpr int STEP = 32 * VEC;
    __shared__ float sm_m[kWarps][32];
    __shared__ float sm_s[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = (int)a.H;
    const int HPL = H / VEC > 0 ? H / VEC : 1;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();

    float m[VEC], s[VEC];
#pragma unroll
    for (int t = 0; t < VEC; t++) { m[t] = -INFINITY; s[t] = 0.f; }
    const int64_t lo = b * H, hi = e * H;
    for (int64_t i0 = lo + (int64_t)lane * VEC; i0 < hi; i0 += STEP * UNR) {
        float x[UNR][VEC];
#pragma unroll
        for (int k = 0; k < UNR; k++) {
            const int64_t i = i0 + (int64_t)k * STEP;
            if (i < hi) {
                if constexpr (VEC == 4) {
                    const float4 v = ld_f4(a.e + i, pol.keep);
                    x[k][0] = v.x; x[k][1] = v.y; x[k][2] = v.z; x[k][3] = v.w;
                } else {
                    x[k][0] = ld_f32(a.e + i, pol.keep);
                }
            } else {
#pragma unroll
                for (int t = 0; t < VEC; t++) x[k][t] = -INFINITY;
            }
        }
#pragma unroll
        for (int t = 0; t < VEC; t++) {
            float mb = x[0][t];
#pragma unroll
            for (int k = 1; k < UNR; k++) mb = fmaxf(mb, x[k][t]);
            const float mn = fmaxf(m[t], mb);            // finite: x[0] is always in range
            float acc = (m[t] == -INFINITY) ? 0.f : s[t] * fast_exp(m[t] - mn);
#pragma unroll
            for (int k = 0; k < UNR; k++) acc += fast_exp(x[k][t] - mn);   // exp(-inf) = 0 for padding
            m[t] = mn;
            s[t] = acc;
        }
    }
#pragma unroll
    for (int t = 0; t < VEC; t++)
        for (int o = HPL; o < 32; o <<= 1) {
            const float mo = __shfl_xor_sync(kFull, m[t], o);
            const float so = __shfl_xor_sync(kFull, s[t], o);
            const float mn = fmaxf(m[t], mo);
            if (mn != -INFINITY) {
                s[t] = ((m[t] == -INFINITY) ? 0.f : s[t] * fast_exp(m[t] - mn)) +
                       ((mo == -INFINITY) ? 0.f : so * fast_exp(mo - mn));
                m[t] = mn;
            }
        }
    if (heavy) {
        // lanes 0..HPL-1 hold heads lane*VEC + t; combine across warps in order
        if (lane < HPL) {
#pragma unroll
            for (int t = 0; t < VEC; t++) {
                sm_m[warp][lane * VEC + t] = m[t];
                sm_s[warp][lane * VEC + t] = s[t];
            }
        }
        __syncthreads();
        const int hl = lane % HPL;
#pragma unroll
        for (int t = 0; t < VEC; t++) {
            float mm = -INFINITY, ss = 0.f;
            for (int w = 0; w < kWarps; w++) {
                const float mo = sm_m[w][hl * VEC + t], so = sm_s[w][hl * VEC + t];
                const float mn = fmaxf(mm, mo);
                if (mn == -INFINITY) continue;
                ss = ((mm == -INFINITY) ? 0.f : ss * fast_exp(mm - mn)) + ((mo == -INFINITY) ? 0.f : so * fast_exp(mo - mn));
                mm = mn;
            }
            m[t] = mm;
            s[t] = ss;
        }
    }
    float rinv[VEC];
#pragma unroll
    for (int t = 0; t < VEC; t++) rinv[t] = 1.0f / s[t];
    for (int64_t i0 = lo + (int64_t)lane * VEC; i0 < hi; i0 += STEP * UNR) {
        float x[UNR][VEC];
#pragma unroll
        for (int k = 0; k < UNR; k++) {
            const int64_t i = i0 + (int64_t)k * STEP;
            if (i < hi) {
                if constexpr (VEC == 4) {
                    const float4 v = ld_f4(a.e + i, pol.stream);
                    x[k][0] = v.x; x[k][1] = v.y; x[k][2] = v.z; x[k][3] = v.w;
                } else {
                    x[k][0] = ld_f32(a.e + i, pol.stream);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < UNR; k++) {
            const int64_t i = i0 + (int64_t)k * STEP;
            if (i < hi) {
                if constexpr (VEC == 4) {
                    st_stream_f4(a.out + i, make_float4(fast_exp(x[k][0] - m[0]) * rinv[0], fast_exp(x[k][1] - m[1]) * rinv[1],
                                                        fast_exp(x[k][2] - m[2]) * rinv[2], fast_exp(x[k][3] - m[3]) * rinv[3]),
                                 pol.stream);
                } else {
                    st_stream_f32(a.out + i, fast_exp(x[k][0] - m[0]) * rinv[0], pol.stream);
                }
            }
        }
    }
}

// Generic edge softmax (any H, any ld): one warp per row, lanes over heads.
__global__ void __launch_bounds__(kThreads) softmax_generic_kernel(const SoftmaxArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    for (int64_t h = lane; h < a.H; h += 32) {
        float m = -INFINITY, s = 0.f;
        for (int64_t j = b; j < e; j++) online_push(m, s, a.e[j * a.lde + h]);
        for (int64_t j = b; j < e; j++) {
            const float x = a.e[j * a.lde + h];
            a.out[j * a.ldo + h] = expf(x - m) / s;
        }
    }
}

// ===================================================== fused GAT forward
// NEXT-2 ("18 kernels in each layer"; a fused forward is
// legal only if it still materialises the state tensor alpha).  One pass per
// destination row v: for each in-edge j = (u -> v) and head h (one lane per
// head, Fh = 8 features per lane):
//   s = <X[v,h], Y[u,h]>          -> written to alpha (raw) ;
//   online softmax (m, S) and acc = sum exp(s - m) Vt[u,h]   (flash-style);
// then out[v,h] = acc / S and the row's raw scores are re-read (L2-hot) and
// overwritten with alpha = exp(s - m) / S.  Y and Vt may be the same table
// (one gather serves both).  Heavy rows: CTA split + deterministic merge.
template <int LPE, bool SAME>
__global__ void __launch_bounds__(kThreads, 2) gat_fused_kernel(const GatArgs a) {
    constexpr int VEC = 8;
    constexpr int G = 32 / LPE;
    constexpr int PER = LPE;
    constexpr int U = SAME ? (PER >= 8 ? 8 : PER) : (PER >= 4 ? 4 : PER);   // edges in flight per lane
    __shared__ __align__(16) int s_col[kWarps][32];
    // running Kahan state (acc, accc) per lane lives in smem: touched once per
    // tile (fold) and on the rare max increase (rescale), keeping registers for
    // the gathers in flight.  Reused for the heavy-row cross-warp merge.
    __shared__ __align__(16) float s_run[kWarps][32][2 * VEC];
    __shared__ float sm_ms[kWarps][LPE][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, h = lane % LPE;   // head of this lane
    const int H = LPE;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();

    Vec<VEC> xv;
    ld_keep(xv, a.X + (a.row_base + row) * a.ldx + h * VEC, pol.stream);
    const char *yl = reinterpret_cast<const char *>(a.Y + h * VEC);
    const char *vl = reinterpret_cast<const char *>(a.Vt + h * VEC);
    const uint32_t ldyb = (uint32_t)(a.ldy * 4), ldvb = (uint32_t)(a.ldv * 4);

    // (m, S + Sc compensation) in registers; acc / accc in smem; tile sums in registers
    float m = -INFINITY, S = 0.f, Sc = 0.f, St = 0.f;
    float *run = s_run[warp][lane];
#pragma unroll
    for (int t = 0; t < 2 * VEC; t++) run[t] = 0.f;
    Vec<VEC> acct;
    vzero(acct);
    int ntile = 0;

    auto load_col = [&](int64_t tb) { return tb + lane < e ? ld_stream_i32(a.col + tb + lane, pol.stream) : 0; };
    int c1 = load_col(b), c2 = load_col(b + 32);
    for (int64_t base = b; base < e; base += 32) {
        const int n = (int)(e - base < 32 ? e - base : 32);
        s_col[warp][(lane % G) * PER + lane / G] = c1;
        c1 = c2;
        c2 = load_col(base + 64);
        __syncwarp();
        const int *gp = &s_col[warp][g * PER];
        float *ab = a.alpha + (base + g) * H + h;   // group g's i-th edge is tile edge g + G*i
        const int mcount = n == 32 ? PER : (n > g ? (n - g + G - 1) / G : 0);
        auto body = [&](int i, auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            Vec<VEC> y[U], vv[SAME ? 1 : U];
            int cc[U];
            if constexpr (U % 4 == 0) {
#pragma unroll
                for (int u = 0; u < U; u += 4) {
                    const int4 c4 = *reinterpret_cast<const int4 *>(gp + i + u);
                    cc[u] = c4.x; cc[u + 1] = c4.y; cc[u + 2] = c4.z; cc[u + 3] = c4.w;
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; u++) cc[u] = gp[i + u];
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (FULL || i + u < mcount) {
                    ld_keep(y[u], reinterpret_cast<const float *>(yl + (uint64_t)(uint32_t)cc[u] * ldyb), pol.keep);
                    if constexpr (!SAME)
                        ld_keep(vv[u], reinterpret_cast<const float *>(vl + (uint64_t)(uint32_t)cc[u] * ldvb), pol.keep);
                } else {
                    vzero(y[u]);
                    if constexpr (!SAME) vzero(vv[u]);
                }
            }
            // scores of the batch, at most one rescale per batch, then the weights
            float sc[U];
            float mb = -INFINITY;
#pragma unroll
            for (int u = 0; u < U; u++) {
                float s0 = 0.f, s1 = 0.f;   // two chains: shorter dependency
#pragma unroll
                for (int t = 0; t < VEC; t += 2) {
                    s0 = fmaf(xv.v[t], y[u].v[t], s0);
                    s1 = fmaf(xv.v[t + 1], y[u].v[t + 1], s1);
                }
                sc[u] = s0 + s1;
                if (FULL || i + u < mcount) {
                    ab[(int64_t)(G * (i + u)) * H] = sc[u];   // raw score (default L2 policy), re-read below
                    mb = fmaxf(mb, sc[u]);
                } else {
                    sc[u] = -INFINITY;
                }
            }
            // lazy rescale: the reference m moves only when a score exceeds it by
            // more than 8 (exp(s - m) <= e^8 keeps every sum finite); the result
            // exp(s - m) / sum exp(s - m) does not depend on the reference, and the
            // (warp-divergent) branch is taken about once per row.
            if (mb > m + 8.f) {
                const float r = fast_exp(m - mb);   // 0 when m = -inf
                S *= r; Sc *= r; St *= r;
#pragma unroll
                for (int t = 0; t < VEC; t++) {
                    run[t] *= r;
                    run[VEC + t] *= r;
                    acct.v[t] *= r;
                }
                m = mb;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const float pu = fast_exp(sc[u] - m);   // 0 for padding (-inf)
                const Vec<VEC> &val = SAME ? y[u] : vv[SAME ? 0 : u];
                St += pu;
#pragma unroll
                for (int t = 0; t < VEC; t++) acct.v[t] = fmaf(pu, val.v[t], acct.v[t]);
            }
        };
        if (n == 32) {
#pragma unroll 1
            for (int i = 0; i < PER; i += U) body(i, std::true_type{});
        } else {
#pragma unroll 1
            for (int i = 0; i < mcount; i += U) body(i, std::false_type{});
        }
        __syncwarp();
        if (++ntile == kFoldTiles || base + 32 >= e) {   // Kahan fold of the tile sums
            ntile = 0;
            float y2 = St - Sc, t2 = S + y2;
            Sc = (t2 - S) - y2; S = t2; St = 0.f;
#pragma unroll
            for (int t = 0; t < VEC; t++) {
                const float ac = run[t], cc = run[VEC + t];
                y2 = acct.v[t] - cc;
                t2 = ac + y2;
                run[VEC + t] = (t2 - ac) - y2;
                run[t] = t2;
                acct.v[t] = 0.f;
            }
        }
    }
    S -= Sc;
    Vec<VEC> acc;
#pragma unroll
    for (int t = 0; t < VEC; t++) acc.v[t] = run[t] - run[VEC + t];
    // merge the G edge groups (same head h): online-softmax merge
    auto merge = [&](float mo, float So, const Vec<VEC> &ao) {
        const float mn = fmaxf(m, mo);
        if (mn == -INFINITY) return;
        const float r1 = m == -INFINITY ? 0.f : fast_exp(m - mn), r2 = mo == -INFINITY ? 0.f : fast_exp(mo - mn);
        S = S * r1 + So * r2;
#pragma unroll
        for (int t = 0; t < VEC; t++) acc.v[t] = acc.v[t] * r1 + ao.v[t] * r2;
        m = mn;
    };
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1) {
        Vec<VEC> ao;
        const float mo = __shfl_xor_sync(kFull, m, o), So = __shfl_xor_sync(kFull, S, o);
#pragma unroll
        for (int t = 0; t < VEC; t++) ao.v[t] = __shfl_xor_sync(kFull, acc.v[t], o);
        merge(mo, So, ao);
    }
    if (heavy) {
        // every warp of the CTA holds (m, S, acc) of its slice per head: merge in warp order
        __syncthreads();   // s_run is reused for the cross-warp state
        if (g == 0) {
            sm_ms[warp][h][0] = m;
            sm_ms[warp][h][1] = S;
#pragma unroll
            for (int t = 0; t < VEC; t++) s_run[warp][h][t] = acc.v[t];
        }
        __syncthreads();
        m = -INFINITY;
        S = 0.f;
        vzero(acc);
        for (int w = 0; w < kWarps; w++) {
            Vec<VEC> ao;
#pragma unroll
            for (int t = 0; t < VEC; t++) ao.v[t] = s_run[w][h][t];
            merge(sm_ms[w][h][0], sm_ms[w][h][1], ao);
        }
    }
    const float rS = S > 0.f ? 1.0f / S : 0.f;
    if (g == 0 && (!heavy || warp == 0)) {
        Vec<VEC> r;
#pragma unroll
        for (int t = 0; t < VEC; t++) r.v[t] = acc.v[t] * rS;
        vstore(a.out + row * a.ldo + h * VEC, r, VEC);
    }
    // normalise this warp's slice of raw scores in place: element i has head i % H
    __syncwarp();
    const int64_t lo = b * H, hi = e * H;
    if (H % 4 == 0) {
        float mh[4], rh[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int hh = (lane * 4 + t) % H;
            mh[t] = __shfl_sync(kFull, m, hh);
            rh[t] = __shfl_sync(kFull, rS, hh);
        }
        constexpr int NU = 8;   // loads in flight per lane (the row block is L2-hot)
        for (int64_t i0 = lo + (int64_t)lane * 4; i0 < hi; i0 += 128 * NU) {
            float4 v[NU];
#pragma unroll
            for (int k = 0; k < NU; k++)
                if (i0 + 128 * k < hi) v[k] = ld_f4(a.alpha + i0 + 128 * k, pol.stream);
#pragma unroll
            for (int k = 0; k < NU; k++)
                if (i0 + 128 * k < hi)
                    st_stream_f4(a.alpha + i0 + 128 * k,
                                 make_float4(fast_exp(v[k].x - mh[0]) * rh[0], fast_exp(v[k].y - mh[1]) * rh[1],
                                             fast_exp(v[k].z - mh[2]) * rh[2], fast_exp(v[k].w - mh[3]) * rh[3]),
                                 pol.stream);
        }
    } else {
        const int hh = lane % H;
        const float mh = __shfl_sync(kFull, m, hh), rh = __shfl_sync(kFull, rS, hh);
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const float v = ld_f32(a.alpha + i, pol.stream);
            st_stream_f32(a.alpha + i, fast_exp(v - mh) * rh, pol.stream);
        }
    }
}

// ========================================================= NEXT-3 kernels
// gSpMMe / gSpMMeid: out[r,h] = RED over the row's edges of w[eid, h] (sum in
// fp64: few values per edge, any row length).  One warp per row; H | 32 maps
// lane -> (edge offset lane / H, head lane % H), else lanes loop over heads.
__global__ void __launch_bounds__(kThreads) spmm_e_kernel(const SpmmEArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t idx = (int64_t)blockIdx.x * kWarps + warp;
    if (idx >= a.nrows) return;
    const int64_t row = a.order[idx], b = a.off[row], e = a.off[row + 1];
    const int H = (int)a.H;
    auto red = [&](double x, double y) {
        return a.red == 1 ? (y < x ? y : x) : (a.red == 2 ? (y > x ? y : x) : x + y);
    };
    const double id = a.red == 1 ? INFINITY : (a.red == 2 ? -INFINITY : 0.0);
    if (H <= 32 && (32 % H) == 0) {
        const int eo = lane / H, h = lane % H, step = 32 / H;
        double acc = id;
        for (int64_t j = b + eo; j < e; j += step) {
            const int64_t ei = a.eid ? (int64_t)__ldg(a.eid + j) : j;
            acc = red(acc, (double)__ldg(a.w + ei * a.ldw + h));
        }
        for (int o = H; o < 32; o <<= 1) acc = red(acc, __shfl_xor_sync(kFull, acc, o));
        if (eo == 0) a.out[row * a.ldo + h] = b == e ? 0.f : (float)acc;
    } else {
        for (int h = lane; h < H; h += 32) {
            double acc = id;
            for (int64_t j = b; j < e; j++) {
                const int64_t ei = a.eid ? (int64_t)__ldg(a.eid + j) : j;
                acc = red(acc, (double)__ldg(a.w + ei * a.ldw + h));
            }
            a.out[row * a.ldo + h] = b == e ? 0.f : (float)acc;
        }
    }
}

// gSDDMMve: out[j,h] = w[j,h] OP X[side ? col_j : row_base + row, h]; out may be w (in place).
__global__ void __launch_bounds__(kThreads) sddmm_ve_kernel(const SddmmVeArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t idx = (int64_t)blockIdx.x * kWarps + warp;
    if (idx >= a.nrows) return;
    const int64_t row = a.order[idx], b = a.off[row], e = a.off[row + 1];
    const int64_t H = a.H;
    const int64_t tot = (e - b) * H;
    for (int64_t t = lane; t < tot; t += 32) {
        const int64_t j = b + t / H, h = t % H;
        const int64_t vx = a.side_src ? (int64_t)__ldg(a.col + j) : a.row_base + row;
        const float x = __ldg(a.X + vx * a.ldx + h), wv = a.w[j * a.ldw + h];
        float r;
        switch (a.op) {
            case 0: r = wv + x; break;
            case 1: r = wv - x; break;
            case 2: r = wv * x; break;
            default: r = wv / x; break;
        }
        a.out[j * a.ldo + h] = r;
    }
}

// ==================================================== edge softmax backward
// ds[j,h] = alpha[j,h] * (dalpha[j,h] - <alpha[row,h], dalpha[row,h]>)   (NEXT-1)
// Fast path: contiguous [E, H], H % 4 == 0, H | 32 (lane owns heads (4 lane + t) mod H).
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(const SoftmaxBwdArgs a) {
    __shared__ float sm_d[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = (int)a.H, HPL = H / 4;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int64_t lo = b * H, hi = e * H;
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int NU = 4;   // loads in flight per lane
    for (int64_t i0 = lo + (int64_t)lane * 4; i0 < hi; i0 += 128 * NU) {
        float4 x[NU], y[NU];
#pragma unroll
        for (int k = 0; k < NU; k++)
            if (i0 + 128 * k < hi) {
                x[k] = ld_f4(a.alpha + i0 + 128 * k, pol.keep);
                y[k] = ld_f4(a.dalpha + i0 + 128 * k, pol.keep);
            }
#pragma unroll
        for (int k = 0; k < NU; k++)
            if (i0 + 128 * k < hi) {
                d[0] = fmaf(x[k].x, y[k].x, d[0]); d[1] = fmaf(x[k].y, y[k].y, d[1]);
                d[2] = fmaf(x[k].z, y[k].z, d[2]); d[3] = fmaf(x[k].w, y[k].w, d[3]);
            }
    }
#pragma unroll
    for (int t = 0; t < 4; t++)
        for (int o = HPL; o < 32; o <<= 1) d[t] += __shfl_xor_sync(kFull, d[t], o);
    if (heavy) {
        if (lane < HPL)
#pragma unroll
            for (int t = 0; t < 4; t++) sm_d[warp][lane * 4 + t] = d[t];
        __syncthreads();
        const int hl = lane % HPL;
#pragma unroll
        for (int t = 0; t < 4; t++) {
            float acc = 0.f;
            for (int w = 0; w < kWarps; w++) acc += sm_d[w][hl * 4 + t];
            d[t] = acc;
        }
    }
    for (int64_t i0 = lo + (int64_t)lane * 4; i0 < hi; i0 += 128 * NU) {
        float4 x[NU], y[NU];
#pragma unroll
        for (int k = 0; k < NU; k++)
            if (i0 + 128 * k < hi) {
                x[k] = ld_f4(a.alpha + i0 + 128 * k, pol.stream);
                y[k] = ld_f4(a.dalpha + i0 + 128 * k, pol.stream);
            }
#pragma unroll
        for (int k = 0; k < NU; k++)
            if (i0 + 128 * k < hi)
                st_stream_f4(a.out + i0 + 128 * k,
                             make_float4(x[k].x * (y[k].x - d[0]), x[k].y * (y[k].y - d[1]), x[k].z * (y[k].z - d[2]),
                                         x[k].w * (y[k].w - d[3])),
                             pol.stream);
    }
}

// generic (any H, any ld): one warp per row, lanes over heads
__global__ void __launch_bounds__(kThreads) softmax_bwd_generic_kernel(const SoftmaxBwdArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    for (int64_t h = lane; h < a.H; h += 32) {
        float d = 0.f;
        for (int64_t j = b; j < e; j++) d = fmaf(a.alpha[j * a.lda + h], a.dalpha[j * a.ldd + h], d);
        for (int64_t j = b; j < e; j++) {
            const float x = a.alpha[j * a.lda + h], y = a.dalpha[j * a.ldd + h];
            a.out[j * a.ldo + h] = x * (y - d);
        }
    }
}

__global__ void gather_scale_kernel(const int32_t *col, int64_t nnz, const float *scale, float *out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = scale[col[j]];
}

__global__ void degree_scales_kernel(const int64_t *deg, int64_t n, float *inv, float *rsq) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = deg[i] < 1 ? 1.0 : (double)deg[i];   // clamp d^ = max(d, 1)
        inv[i] = (float)(1.0 / d);
        rsq[i] = (float)(1.0 / sqrt(d));
    }
}

// ---------------------------------------------------------------- dispatch
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

template <int VEC, int LPE, int CPL, int UOVR = 0, int MINB = 0>
cudaError_t spmm_go_v(const SpmmArgs &a, int mode, int64_t slabs, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, slabs);
    if (mode == kSpmmScaled) {
        if (a.col_scale || a.edge_scale) spmm_kernel<VEC, LPE, CPL, kSpmmScaled, true, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
        else spmm_kernel<VEC, LPE, CPL, kSpmmScaled, false, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
    } else if (mode == kSpmmWeightedFwd) {
        spmm_kernel<VEC, LPE, CPL, kSpmmWeightedFwd, false, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
    } else if (mode == kSpmmWeightedRev) {
        spmm_kernel<VEC, LPE, CPL, kSpmmWeightedRev, false, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
    } else if (mode == kSpmmMin) {
        spmm_kernel<VEC, LPE, CPL, kSpmmMin, false, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
    } else {
        spmm_kernel<VEC, LPE, CPL, kSpmmMax, false, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// tuning knob for the hot shape (VEC 8, LPE 8: F = 64): GSP_TUNE_SPMM selects
// (U, min blocks/SM); read once.  0 = default.
int tune_spmm() {
    static int v = [] {
        const char *e = getenv("GSP_TUNE_SPMM");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <int VEC, int LPE, int CPL>
cudaError_t spmm_go(const SpmmArgs &a, int mode, int64_t slabs, cudaStream_t s) {
    if constexpr (VEC == 8 && LPE == 8 && CPL == 1) {
        switch (tune_spmm()) {
            case 0:   // measured best on B200 (Reddit-shaped F = 64, tools/opbench.py)
                return spmm_go_v<VEC, LPE, CPL, 8, 2>(a, mode, slabs, s);
            case 5: return spmm_go_v<VEC, LPE, CPL>(a, mode, slabs, s);
            case 6: return spmm_go_v<VEC, LPE, CPL, 4, 2>(a, mode, slabs, s);
            case 1: return spmm_go_v<VEC, LPE, CPL, 8, 2>(a, mode, slabs, s);
            case 2: return spmm_go_v<VEC, LPE, CPL, 4, 4>(a, mode, slabs, s);
            case 3: return spmm_go_v<VEC, LPE, CPL, 2, 4>(a, mode, slabs, s);
            case 4: return spmm_go_v<VEC, LPE, CPL, 8, 3>(a, mode, slabs, s);
            default: break;
        }
    }
    return spmm_go_v<VEC, LPE, CPL>(a, mode, slabs, s);
}

template <int VEC, int MAXCPL>
cudaError_t spmm_dispatch(const SpmmArgs &a, int mode, cudaStream_t s) {
    const int64_t nch = ceil_div(a.F, VEC);
    if (nch <= 16) {
        const int lpe = pow2ceil(nch < 2 ? 2 : nch);
        if (lpe == 2) return spmm_go<VEC, 2, 1>(a, mode, 1, s);
        if (lpe == 4) return spmm_go<VEC, 4, 1>(a, mode, 1, s);
        if (lpe == 8) return spmm_go<VEC, 8, 1>(a, mode, 1, s);
        return spmm_go<VEC, 16, 1>(a, mode, 1, s);
    }
    // wide rows: balanced feature slabs of <= 32*MAXCPL chunks (VEC*CPL <= 16
    // floats of state per lane and chunk keeps the kernel spill-free)
    const int64_t slabs = ceil_div(nch, 32 * MAXCPL);
    const int64_t cpl = ceil_div(nch, 32 * slabs);
    switch (cpl) {
        case 1: return spmm_go<VEC, 32, 1>(a, mode, slabs, s);
        case 2: return spmm_go<VEC, 32, (MAXCPL >= 2 ? 2 : MAXCPL)>(a, mode, slabs, s);
        case 3: return spmm_go<VEC, 32, (MAXCPL >= 3 ? 3 : MAXCPL)>(a, mode, slabs, s);
        case 4: return spmm_go<VEC, 32, (MAXCPL >= 4 ? 4 : MAXCPL)>(a, mode, slabs, s);
        case 5: return spmm_go<VEC, 32, (MAXCPL >= 5 ? 5 : MAXCPL)>(a, mode, slabs, s);
        case 6: return spmm_go<VEC, 32, (MAXCPL >= 6 ? 6 : MAXCPL)>(a, mode, slabs, s);
        case 7: return spmm_go<VEC, 32, (MAXCPL >= 7 ? 7 : MAXCPL)>(a, mode, slabs, s);
        default: return spmm_go<VEC, 32, MAXCPL>(a, mode, slabs, s);
    }
}

int tune_sddmm() {
    static int v = [] {
        const char *e = getenv("GSP_TUNE_SDDMM");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <int VEC, int LPE, int CPL>
cudaError_t sddmm_go_cph(const SddmmArgs &a, int cph, int64_t slabs, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, slabs);
    if constexpr (VEC == 8 && LPE == 8 && CPL == 1) {
        if (cph == 1) {
            switch (tune_sddmm()) {
                case 0:   // measured best on B200 (Reddit-shaped H = 8 x 8, tools/opbench.py)
                case 2: sddmm_kernel<VEC, LPE, CPL, 1, 4, 4><<<grid, kThreads, 0, s>>>(a); return cudaGetLastError();
                case 1: sddmm_kernel<VEC, LPE, CPL, 1, 8, 2><<<grid, kThreads, 0, s>>>(a); return cudaGetLastError();
                case 3: sddmm_kernel<VEC, LPE, CPL, 1, 2, 4><<<grid, kThreads, 0, s>>>(a); return cudaGetLastError();
                default: break;
            }
        }
    }
    switch (cph) {
        case 1: sddmm_kernel<VEC, LPE, CPL, 1><<<grid, kThreads, 0, s>>>(a); break;
        case 2: sddmm_kernel<VEC, LPE, CPL, (LPE >= 2 ? 2 : 1)><<<grid, kThreads, 0, s>>>(a); break;
        case 4: sddmm_kernel<VEC, LPE, CPL, (LPE >= 4 ? 4 : 1)><<<grid, kThreads, 0, s>>>(a); break;
        case 8: sddmm_kernel<VEC, LPE, CPL, (LPE >= 8 ? 8 : 1)><<<grid, kThreads, 0, s>>>(a); break;
        case 16: sddmm_kernel<VEC, LPE, CPL, (LPE >= 16 ? 16 : 1)><<<grid, kThreads, 0, s>>>(a); break;
        default: sddmm_kernel<VEC, LPE, CPL, 32><<<grid, kThreads, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

template <int VEC>
cudaError_t sddmm_dispatch(const SddmmArgs &a, int cph, cudaStream_t s) {
    const int64_t nch = ceil_div(a.H * a.Fh, VEC);
    if (nch <= 16) {
        // the lanes of one edge must cover a whole head: lpe >= cph
        int lpe = pow2ceil(nch < 2 ? 2 : nch);
        if (lpe < cph) lpe = cph;
        if (lpe == 2) return sddmm_go_cph<VEC, 2, 1>(a, cph, 1, s);
        if (lpe == 4) return sddmm_go_cph<VEC, 4, 1>(a, cph, 1, s);
        if (lpe == 8) return sddmm_go_cph<VEC, 8, 1>(a, cph, 1, s);
        if (lpe == 16) return sddmm_go_cph<VEC, 16, 1>(a, cph, 1, s);
    }
    constexpr int MAXCPL = VEC >= 8 ? 2 : 4;
    const int64_t slabs = ceil_div(nch, 32 * MAXCPL);
    const int64_t cpl = ceil_div(nch, 32 * slabs);
    switch (cpl) {
        case 1: return sddmm_go_cph<VEC, 32, 1>(a, cph, slabs, s);
        case 2: return sddmm_go_cph<VEC, 32, 2>(a, cph, slabs, s);
        default: return sddmm_go_cph<VEC, 32, MAXCPL>(a, cph, slabs, s);
    }
}

}  // namespace

cudaError_t launch_spmm(const SpmmArgs &a, int mode, cudaStream_t s) {
    if (a.nrows == 0 || a.F == 0) return cudaSuccess;
    const bool wmode = mode == kSpmmWeightedFwd || mode == kSpmmWeightedRev;
    if (wmode && a.H > kHMax) return cudaErrorNotSupported;   // api.cu rejects H > 16 first
    auto ok_vec = [&](int v) {
        return a.F >= v && a.ldx % v == 0 && a.ldo % 4 == 0 && aligned(a.X, 4 * v) && aligned(a.out, 16) &&
               (!wmode || a.Fh % v == 0);
    };
    if (ok_vec(8)) return spmm_dispatch<8, 2>(a, mode, s);
    if (ok_vec(4)) return spmm_dispatch<4, 4>(a, mode, s);
    return spmm_dispatch<1, 4>(a, mode, s);
}

cudaError_t launch_sddmm(const SddmmArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    auto is_pow2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
    auto ok_vec = [&](int v) {
        return a.Fh % v == 0 && is_pow2(a.Fh / v) && a.Fh / v <= 32 && a.ldx % v == 0 && a.ldy % v == 0 &&
               aligned(a.X, 4 * v) && aligned(a.Y, 4 * v);
    };
    if (ok_vec(8)) return sddmm_dispatch<8>(a, (int)(a.Fh / 8), s);
    if (ok_vec(4)) return sddmm_dispatch<4>(a, (int)(a.Fh / 4), s);
    if (ok_vec(1)) return sddmm_dispatch<1>(a, (int)a.Fh, s);
    SddmmArgs g = a;
    g.n_heavy = 0;
    sddmm_generic_kernel<<<row_grid(a.nrows, 0, 1), kThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_softmax(const SoftmaxArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool contiguous = a.lde == a.H && a.ldo == a.H && a.H <= 32 && (32 % a.H) == 0;
    if (contiguous) {
        const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
        if (a.H % 4 == 0 && aligned(a.e, 16) && aligned(a.out, 16)) softmax_kernel<4><<<grid, kThreads, 0, s>>>(a);
        else softmax_kernel<1><<<grid, kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    SoftmaxArgs g = a;
    g.n_heavy = 0;
    softmax_generic_kernel<<<row_grid(a.nrows, 0, 1), kThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_softmax_bwd(const SoftmaxBwdArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool fast = a.lda == a.H && a.ldd == a.H && a.ldo == a.H && a.H % 4 == 0 && a.H <= 32 && (32 % a.H) == 0 &&
                      aligned(a.alpha, 16) && aligned(a.dalpha, 16) && aligned(a.out, 16);
    if (fast) {
        softmax_bwd_kernel<<<row_grid(a.nrows, a.n_heavy, 1), kThreads, 0, s>>>(a);
    } else {
        SoftmaxBwdArgs g = a;
        g.n_heavy = 0;
        softmax_bwd_generic_kernel<<<row_grid(a.nrows, 0, 1), kThreads, 0, s>>>(g);
    }
    return cudaGetLastError();
}

bool gat_fused_supported(const GatArgs &a) {
    const int64_t H = a.H;
    const bool h_ok = H == 2 || H == 4 || H == 8 || H == 16 || H == 32;
    return h_ok && a.ldx % 8 == 0 && a.ldy % 8 == 0 && a.ldv % 8 == 0 && a.ldo % 4 == 0 && aligned(a.X, 32) &&
           aligned(a.Y, 32) && aligned(a.Vt, 32) && aligned(a.out, 16) && aligned(a.alpha, 16);
}

cudaError_t launch_gat_fused(const GatArgs &a, cudaStream_t s) {
    if (a.nrows == 0) return cudaSuccess;
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    const bool same = a.Vt == a.Y && a.ldv == a.ldy;
#define GSP_GAT_CASE(HH)                                                         \
    case HH:                                                                     \
        if (same) gat_fused_kernel<HH, true><<<grid, kThreads, 0, s>>>(a);       \
        else gat_fused_kernel<HH, false><<<grid, kThreads, 0, s>>>(a);           \
        break;
    switch (a.H) {
        GSP_GAT_CASE(2)
        GSP_GAT_CASE(4)
        GSP_GAT_CASE(8)
        GSP_GAT_CASE(16)
        default:
            if (same) gat_fused_kernel<32, true><<<grid, kThreads, 0, s>>>(a);
            else gat_fused_kernel<32, false><<<grid, kThreads, 0, s>>>(a);
    }
#undef GSP_GAT_CASE
    return cudaGetLastError();
}

cudaError_t launch_spmm_e(const SpmmEArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    spmm_e_kernel<<<(unsigned)ceil_div(a.nrows, kWarps), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sddmm_ve(const SddmmVeArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    sddmm_ve_kernel<<<(unsigned)ceil_div(a.nrows, kWarps), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gather_scale(const int32_t *col, int64_t nnz, const float *scale, float *out, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    const int64_t blocks = ceil_div(nnz, 256) < 8192 ? ceil_div(nnz, 256) : 8192;
    gather_scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(col, nnz, scale, out);
    return cudaGetLastError();
}

cudaError_t launch_degree_scales(const int64_t *deg, int64_t n, float *inv, float *rsq, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int64_t blocks = ceil_div(n, 256) < 4096 ? ceil_div(n, 256) : 4096;
    degree_scales_kernel<<<(unsigned)blocks, 256, 0, s>>>(deg, n, inv, rsq);
    return cudaGetLastError();
}

}  // namespace gsp
