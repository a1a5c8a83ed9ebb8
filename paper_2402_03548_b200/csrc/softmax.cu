// Edge softmax and its backward.
#include "common.cuh"

namespace gsp {
namespace {

// ============================================================ edge softmax
__device__ __forceinline__ void online_push(float &m, float &s, float x) {
    if (x > m) {
        s = s * expf(m - x) + 1.f;
        m = x;
    } else {
        s += expf(x - m);
    }
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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    for (int64_t h = lane; h < a.H; h += 32) {
        float m = -INFINITY, s = 0.f;
        for (int64_t j = b; j < e; j++) online_push(m, s, a.e[j * a.lde + h]);
        for (int64_t j = b; j < e; j++) {
            const float x = a.e[j * a.lde + h];
            a.out[j * a.ldo + h] = expf(x - m) / s;
        }
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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    for (int64_t h = lane; h < a.H; h += 32) {
        float d = 0.f;
        for (int64_t j = b; j < e; j++) d = fmaf(a.alpha[j * a.lda + h], a.dalpha[j * a.ldd + h], d);
        for (int64_t j = b; j < e; j++) {
            const float x = a.alpha[j * a.lda + h], y = a.dalpha[j * a.ldd + h];
            a.out[j * a.ldo + h] = x * (y - d);
        }
    }
}

}  // namespace

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

}  // namespace gsp
