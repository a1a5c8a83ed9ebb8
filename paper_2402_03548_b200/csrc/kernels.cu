// sm_100a kernels of the GraphPy sparse hot path (arxiv 2402.03548).
//
// All three families are sparse gather-reduces (no dense contraction), so they
// run on the LSU/L2 path, not on tensor cores.  Common
// structure:
//   * rows come from a degree-ordered schedule built at graph create (rows by
//     descending degree; LPT order): the first n_heavy rows (degree > 1024)
//     get a whole CTA (8 warps split the row's edge list, deterministic smem
//     combine), the rest one warp each (8 rows per CTA);
//   * a warp reads 32 column ids (and edge ids / scales) with one coalesced
//     load and broadcasts them with __shfl_sync;
//   * feature rows are gathered with 128-bit __ldg (read-only path) by groups
//     of LPE lanes, G = 32/LPE edges at a time, U edges unrolled per lane for
//     memory-level parallelism; partial sums are combined by xor-shuffles.
// No atomics; every output element is written exactly once per call.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "kernels.h"

namespace gsp {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr unsigned kFull = 0xffffffffu;

template <int VEC>
struct Vec {
    float v[VEC];
};

template <int VEC>
__device__ __forceinline__ void vload(Vec<VEC> &r, const float *p) {
    if constexpr (VEC == 4) {
        float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
    } else {
#pragma unroll
        for (int k = 0; k < VEC; k++) r.v[k] = __ldg(p + k);
    }
}
template <int VEC>
__device__ __forceinline__ void vzero(Vec<VEC> &r) {
#pragma unroll
    for (int k = 0; k < VEC; k++) r.v[k] = 0.f;
}
// store the first `lim` (<= VEC) elements; full vector store when lim == VEC
template <int VEC>
__device__ __forceinline__ void vstore(float *p, const Vec<VEC> &r, int64_t lim) {
    if constexpr (VEC == 4) {
        if (lim >= 4) {
            *reinterpret_cast<float4 *>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
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
template <int VEC, int LPE, int CPL, int MODE>
__global__ void __launch_bounds__(kThreads, (CPL <= 2 ? 4 : 2)) spmm_kernel(const SpmmArgs a) {
    constexpr int G = 32 / LPE;
    constexpr int U = CPL >= 3 ? 1 : (CPL == 2 ? 2 : 4);
    constexpr int NACC = U >= 2 ? 2 : 1;
    constexpr int SW = VEC * LPE * CPL;  // feature slab handled by this CTA
    __shared__ float red[kWarps][SW];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, sub = lane % LPE;
    const int64_t f0 = (int64_t)blockIdx.y * SW;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;

    // Summation: each 32-edge tile is summed
    // plainly into `tile` (<= 32/G terms per lane), and tile sums are folded
    // into a Kahan-compensated running sum (acc, cmp).  The error is then
    // O(32/G * u) relative to sum|terms|, independent of the row length, so
    // hub rows of any degree stay far inside 1e-5 * (sum|terms| + 1).
    Vec<VEC> acc[CPL], cmp[CPL];
#pragma unroll
    for (int q = 0; q < CPL; q++) { vzero(acc[q]); vzero(cmp[q]); }

    for (int64_t base = b; base < e; base += 32) {
        const int n = (int)(e - base < 32 ? e - base : 32);
        int c = 0, ev = 0;
        float sc = 1.f;
        if (lane < n) {
            c = __ldg(a.col + base + lane);
            if constexpr (MODE == kSpmmScaled) {
                if (a.col_scale) sc = __ldg(a.col_scale + c);
            } else if constexpr (MODE == kSpmmWeightedFwd) {
                ev = (int)(base + lane);
            } else {
                ev = __ldg(a.eid + base + lane);
            }
        }
        Vec<VEC> tile[NACC][CPL];
#pragma unroll
        for (int s2 = 0; s2 < NACC; s2++)
#pragma unroll
            for (int q = 0; q < CPL; q++) vzero(tile[s2][q]);
        for (int k = 0; k < n; k += G * U) {
            Vec<VEC> x[U][CPL];
            float wt[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int ei = k + u * G + g;
                const bool ok = ei < n;
                const int cu = __shfl_sync(kFull, c, ei & 31);
                float su = 1.f;
                int eu = 0;
                if constexpr (MODE == kSpmmScaled) su = __shfl_sync(kFull, sc, ei & 31);
                else eu = __shfl_sync(kFull, ev, ei & 31);
#pragma unroll
                for (int q = 0; q < CPL; q++) {
                    const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
                    if (ok && f < a.F) {
                        vload(x[u][q], a.X + (int64_t)cu * a.ldx + f);
                        if constexpr (MODE == kSpmmScaled) wt[u][q] = su;
                        else wt[u][q] = __ldg(a.w + (int64_t)eu * a.ldw + f / a.Fh);
                    } else {
                        vzero(x[u][q]);
                        wt[u][q] = 0.f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < CPL; q++)
#pragma unroll
                    for (int t = 0; t < VEC; t++)
                        tile[u % NACC][q].v[t] = fmaf(wt[u][q], x[u][q].v[t], tile[u % NACC][q].v[t]);
        }
#pragma unroll
        for (int q = 0; q < CPL; q++)
#pragma unroll
            for (int t = 0; t < VEC; t++) {
                float y = tile[0][q].v[t];
                if constexpr (NACC == 2) y += tile[1][q].v[t];
                y -= cmp[q].v[t];
                const float sum = acc[q].v[t] + y;
                cmp[q].v[t] = (sum - acc[q].v[t]) - y;
                acc[q].v[t] = sum;
            }
    }
    // compensated totals, then the G edge groups of the warp (xor tree)
#pragma unroll
    for (int q = 0; q < CPL; q++)
#pragma unroll
        for (int t = 0; t < VEC; t++) {
            float v = acc[q].v[t] - cmp[q].v[t];
#pragma unroll
            for (int o = LPE; o < 32; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
            acc[q].v[t] = v;
        }

    float rs = 1.f;
    if constexpr (MODE == kSpmmScaled)
        if (a.row_scale) rs = __ldg(a.row_scale + row);

    if (!heavy) {
        if (g == 0) {
#pragma unroll
            for (int q = 0; q < CPL; q++) {
                const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
                if (f < a.F) {
                    Vec<VEC> r;
#pragma unroll
                    for (int t = 0; t < VEC; t++) r.v[t] = rs * acc[q].v[t];
                    vstore(a.out + row * a.ldo + f, r, a.F - f);
                }
            }
        }
        return;
    }
    // heavy row: deterministic cross-warp combine in warp order
    if (g == 0) {
#pragma unroll
        for (int q = 0; q < CPL; q++)
#pragma unroll
            for (int t = 0; t < VEC; t++) red[warp][(sub + q * LPE) * VEC + t] = acc[q].v[t];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < SW; t += kThreads) {
        const int64_t f = f0 + t;
        if (f < a.F) {
            float v = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; w++) v += red[w][t];
            a.out[row * a.ldo + f] = rs * v;
        }
    }
}

// ================================================================ gSDDMMvv
// out[j, h] = <X[row_base + v, head h], Y[col_j, head h]>, CPH = Fh / VEC lanes per head.
template <int VEC, int LPE, int CPL, int CPH>
__global__ void __launch_bounds__(kThreads) sddmm_kernel(const SddmmArgs a) {
    constexpr int G = 32 / LPE;
    constexpr int U = CPL >= 3 ? 1 : (CPL == 2 ? 2 : 4);
    constexpr int SW = VEC * LPE * CPL;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, sub = lane % LPE;
    const int64_t F = a.H * a.Fh;
    const int64_t f0 = (int64_t)blockIdx.y * SW;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    if (b >= e) return;

    // the row's features are fetched once and reused for every edge
    Vec<VEC> xv[CPL];
    const float *xr = a.X + (a.row_base + row) * a.ldx;
#pragma unroll
    for (int q = 0; q < CPL; q++) {
        const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
        if (f < F) vload(xv[q], xr + f);
        else vzero(xv[q]);
    }
    for (int64_t base = b; base < e; base += 32) {
        const int n = (int)(e - base < 32 ? e - base : 32);
        int c = 0;
        if (lane < n) c = __ldg(a.col + base + lane);
        for (int k = 0; k < n; k += G * U) {
            Vec<VEC> y[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int ei = k + u * G + g;
                const int cu = __shfl_sync(kFull, c, ei & 31);
#pragma unroll
                for (int q = 0; q < CPL; q++) {
                    const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
                    if (ei < n && f < F) vload(y[u][q], a.Y + (int64_t)cu * a.ldy + f);
                    else vzero(y[u][q]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int ei = k + u * G + g;
#pragma unroll
                for (int q = 0; q < CPL; q++) {
                    float p = 0.f;
#pragma unroll
                    for (int t = 0; t < VEC; t++) p = fmaf(xv[q].v[t], y[u][q].v[t], p);
#pragma unroll
                    for (int o = 1; o < CPH; o <<= 1) p += __shfl_xor_sync(kFull, p, o);
                    const int64_t f = f0 + (int64_t)(sub + q * LPE) * VEC;
                    if (ei < n && (sub % CPH) == 0 && f < F)
                        a.out[(base + ei) * a.ldo + f / a.Fh] = p;
                }
            }
        }
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
__device__ __forceinline__ void online_merge(float &m, float &s, float mo, float so) {
    const float mn = fmaxf(m, mo);
    if (mn == -INFINITY) return;  // both empty
    const float a = (m == -INFINITY) ? 0.f : s * expf(m - mn);
    const float b = (mo == -INFINITY) ? 0.f : so * expf(mo - mn);
    m = mn;
    s = a + b;
}

// Fast path: e, out contiguous [E, H] (ld == H), H divides 32*VEC/ (so every
// lane always sees the same VEC heads).  HPL = H / VEC lanes per head period.
template <int VEC>
__global__ void __launch_bounds__(kThreads) softmax_kernel(const SoftmaxArgs a) {
    __shared__ float sm_m[kWarps][32];
    __shared__ float sm_s[kWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = (int)a.H;
    const int HPL = H / VEC > 0 ? H / VEC : 1;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.off, a.order, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;

    float m[VEC], s[VEC];
#pragma unroll
    for (int t = 0; t < VEC; t++) { m[t] = -INFINITY; s[t] = 0.f; }
    const int64_t lo = b * H, hi = e * H;
    for (int64_t i = lo + (int64_t)lane * VEC; i < hi; i += 32 * VEC) {
        Vec<VEC> x;
        vload(x, a.e + i);
#pragma unroll
        for (int t = 0; t < VEC; t++) online_push(m[t], s[t], x.v[t]);
    }
#pragma unroll
    for (int t = 0; t < VEC; t++)
        for (int o = HPL; o < 32; o <<= 1) {
            const float mo = __shfl_xor_sync(kFull, m[t], o);
            const float so = __shfl_xor_sync(kFull, s[t], o);
            online_merge(m[t], s[t], mo, so);
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
            for (int w = 0; w < kWarps; w++) online_merge(mm, ss, sm_m[w][hl * VEC + t], sm_s[w][hl * VEC + t]);
            m[t] = mm;
            s[t] = ss;
        }
    }
    for (int64_t i = lo + (int64_t)lane * VEC; i < hi; i += 32 * VEC) {
        Vec<VEC> x, r;
        vload(x, a.e + i);
#pragma unroll
        for (int t = 0; t < VEC; t++) r.v[t] = expf(x.v[t] - m[t]) / s[t];
        vstore(a.out + i, r, VEC);
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

__global__ void degree_scales_kernel(const int64_t *deg, int64_t n, float *inv, float *rsq) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = deg[i] < 1 ? 1.0 : (double)deg[i];   // clamp d^ = max(d, 1)
        inv[i] = (float)(1.0 / d);
        rsq[i] = (float)(1.0 / sqrt(d));
    }
}

// ---------------------------------------------------------------- dispatch
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int pow2ceil(int64_t x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline dim3 row_grid(int64_t nrows, int64_t n_heavy, int64_t slabs) {
    return dim3((unsigned)(n_heavy + ceil_div(nrows - n_heavy, kWarps)), (unsigned)slabs, 1);
}

template <int VEC, int LPE, int CPL>
cudaError_t spmm_go(const SpmmArgs &a, int mode, int64_t slabs, cudaStream_t s) {
    dim3 grid = row_grid(a.nrows, a.n_heavy, slabs);
    if (mode == kSpmmScaled) spmm_kernel<VEC, LPE, CPL, kSpmmScaled><<<grid, kThreads, 0, s>>>(a);
    else if (mode == kSpmmWeightedFwd) spmm_kernel<VEC, LPE, CPL, kSpmmWeightedFwd><<<grid, kThreads, 0, s>>>(a);
    else spmm_kernel<VEC, LPE, CPL, kSpmmWeightedRev><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int VEC>
cudaError_t spmm_dispatch(const SpmmArgs &a, int mode, cudaStream_t s) {
    const int64_t nch = ceil_div(a.F, VEC);
    if (nch <= 16) {
        const int lpe = pow2ceil(nch < 4 ? 4 : nch);
        if (lpe == 4) return spmm_go<VEC, 4, 1>(a, mode, 1, s);
        if (lpe == 8) return spmm_go<VEC, 8, 1>(a, mode, 1, s);
        return spmm_go<VEC, 16, 1>(a, mode, 1, s);
    }
    const int64_t cpl_need = ceil_div(nch, 32);
    if (cpl_need <= 8) {
        switch (cpl_need) {
            case 1: return spmm_go<VEC, 32, 1>(a, mode, 1, s);
            case 2: return spmm_go<VEC, 32, 2>(a, mode, 1, s);
            case 3: return spmm_go<VEC, 32, 3>(a, mode, 1, s);
            case 4: return spmm_go<VEC, 32, 4>(a, mode, 1, s);
            case 5: return spmm_go<VEC, 32, 5>(a, mode, 1, s);
            case 6: return spmm_go<VEC, 32, 6>(a, mode, 1, s);
            case 7: return spmm_go<VEC, 32, 7>(a, mode, 1, s);
            default: return spmm_go<VEC, 32, 8>(a, mode, 1, s);
        }
    }
    return spmm_go<VEC, 32, 8>(a, mode, ceil_div(nch, 32 * 8), s);
}

template <int VEC, int LPE, int CPL>
cudaError_t sddmm_go_cph(const SddmmArgs &a, int cph, int64_t slabs, cudaStream_t s) {
    dim3 grid = row_grid(a.nrows, a.n_heavy, slabs);
    switch (cph) {
        case 1: sddmm_kernel<VEC, LPE, CPL, 1><<<grid, kThreads, 0, s>>>(a); break;
        case 2: if (LPE >= 2) sddmm_kernel<VEC, LPE, CPL, 2><<<grid, kThreads, 0, s>>>(a); break;
        case 4: if (LPE >= 4) sddmm_kernel<VEC, LPE, CPL, 4><<<grid, kThreads, 0, s>>>(a); break;
        case 8: if (LPE >= 8) sddmm_kernel<VEC, LPE, CPL, 8><<<grid, kThreads, 0, s>>>(a); break;
        case 16: if (LPE >= 16) sddmm_kernel<VEC, LPE, CPL, 16><<<grid, kThreads, 0, s>>>(a); break;
        default: sddmm_kernel<VEC, LPE, CPL, 32><<<grid, kThreads, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

template <int VEC>
cudaError_t sddmm_dispatch(const SddmmArgs &a, int cph, cudaStream_t s) {
    const int64_t nch = ceil_div(a.H * a.Fh, VEC);
    if (nch <= 16) {
        const int lpe = pow2ceil(nch < 4 ? 4 : nch);
        if (lpe == 4) return sddmm_go_cph<VEC, 4, 1>(a, cph, 1, s);
        if (lpe == 8) return sddmm_go_cph<VEC, 8, 1>(a, cph, 1, s);
        return sddmm_go_cph<VEC, 16, 1>(a, cph, 1, s);
    }
    const int64_t cpl_need = ceil_div(nch, 32);
    switch (cpl_need) {
        case 1: return sddmm_go_cph<VEC, 32, 1>(a, cph, 1, s);
        case 2: return sddmm_go_cph<VEC, 32, 2>(a, cph, 1, s);
        case 3: case 4: return sddmm_go_cph<VEC, 32, 4>(a, cph, 1, s);
        default: return sddmm_go_cph<VEC, 32, 8>(a, cph, ceil_div(nch, 32 * 8), s);
    }
}

}  // namespace

cudaError_t launch_spmm(const SpmmArgs &a, int mode, cudaStream_t s) {
    if (a.nrows == 0 || a.F == 0) return cudaSuccess;
    bool v4 = (a.ldx % 4 == 0) && (a.ldo % 4 == 0) && aligned16(a.X) && aligned16(a.out) && a.F >= 4;
    if (mode != kSpmmScaled) v4 = v4 && (a.Fh % 4 == 0);
    return v4 ? spmm_dispatch<4>(a, mode, s) : spmm_dispatch<1>(a, mode, s);
}

cudaError_t launch_sddmm(const SddmmArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    auto is_pow2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
    const bool v4 = (a.Fh % 4 == 0) && is_pow2(a.Fh / 4) && a.Fh / 4 <= 32 && (a.ldx % 4 == 0) &&
                    (a.ldy % 4 == 0) && aligned16(a.X) && aligned16(a.Y);
    if (v4) return sddmm_dispatch<4>(a, (int)(a.Fh / 4), s);
    if (is_pow2(a.Fh) && a.Fh <= 32) return sddmm_dispatch<1>(a, (int)a.Fh, s);
    dim3 grid = row_grid(a.nrows, 0, 1);
    SddmmArgs g = a;
    g.n_heavy = 0;
    sddmm_generic_kernel<<<grid, kThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_softmax(const SoftmaxArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool contiguous = a.lde == a.H && a.ldo == a.H && a.H <= 32 && (32 % a.H) == 0;
    if (contiguous) {
        dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
        if (a.H % 4 == 0 && aligned16(a.e) && aligned16(a.out)) softmax_kernel<4><<<grid, kThreads, 0, s>>>(a);
        else softmax_kernel<1><<<grid, kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    SoftmaxArgs g = a;
    g.n_heavy = 0;
    softmax_generic_kernel<<<row_grid(a.nrows, 0, 1), kThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_degree_scales(const int64_t *deg, int64_t n, float *inv, float *rsq, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int64_t blocks = ceil_div(n, 256) < 4096 ? ceil_div(n, 256) : 4096;
    degree_scales_kernel<<<(unsigned)blocks, 256, 0, s>>>(deg, n, inv, rsq);
    return cudaGetLastError();
}

}  // namespace gsp
