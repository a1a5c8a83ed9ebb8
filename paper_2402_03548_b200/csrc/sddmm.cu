// gSDDMMvv (u.v scores) and gSDDMMve.
#include "common.cuh"

namespace gsp {
namespace {

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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
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
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
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

// ========================================================= gSDDMMve (NEXT-3)
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

// Vector path (H in {4, 8, 16, 32}, 16-B aligned rows): QH = H/4 lanes per edge,
// one float4 of heads each; destination-side X row loaded once per warp.
// In place (out == w) is safe: each element is read, then written, by the
// same thread, through coherent loads.
template <int QH, int OP, bool SRC>
__global__ void __launch_bounds__(kThreads) sddmm_ve_vec_kernel(const SddmmVeArgs a) {
    constexpr int EPW = 32 / QH, U = 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int eo = lane / QH, q = lane % QH;
    float4 xd = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!SRC && b < e) xd = __ldg(reinterpret_cast<const float4 *>(a.X + (a.row_base + row) * a.ldx + 4 * q));
    auto apply = [](float w, float x) {
        if constexpr (OP == 0) return w + x;
        else if constexpr (OP == 1) return w - x;
        else if constexpr (OP == 2) return w * x;
        else return w / x;
    };
    auto one = [&](int64_t jj, const float4 wv, const float4 x) {
        st_stream_f4(a.out + jj * a.ldo + 4 * q,
                     make_float4(apply(wv.x, x.x), apply(wv.y, x.y), apply(wv.z, x.z), apply(wv.w, x.w)), pol.stream);
    };
    int64_t j = b + eo;
    for (; j + (U - 1) * EPW < e; j += U * EPW) {
        float4 wv[U], x[U];
        if constexpr (SRC) {
            int c[U];
#pragma unroll
            for (int u = 0; u < U; u++) c[u] = __ldg(a.col + j + u * EPW);
#pragma unroll
            for (int u = 0; u < U; u++) x[u] = __ldg(reinterpret_cast<const float4 *>(a.X + (int64_t)c[u] * a.ldx + 4 * q));
        }
#pragma unroll
        for (int u = 0; u < U; u++) wv[u] = ld_f4(a.w + (j + u * EPW) * a.ldw + 4 * q, pol.stream);
#pragma unroll
        for (int u = 0; u < U; u++) one(j + u * EPW, wv[u], SRC ? x[u] : xd);
    }
    for (; j < e; j += EPW) {
        const float4 x = SRC ? __ldg(reinterpret_cast<const float4 *>(a.X + (int64_t)__ldg(a.col + j) * a.ldx + 4 * q)) : xd;
        one(j, ld_f4(a.w + j * a.ldw + 4 * q, pol.stream), x);
    }
}

template <int QH, int OP>
cudaError_t sddmm_ve_side(const SddmmVeArgs &a, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    if (a.side_src) sddmm_ve_vec_kernel<QH, OP, true><<<grid, kThreads, 0, s>>>(a);
    else sddmm_ve_vec_kernel<QH, OP, false><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int QH>
cudaError_t sddmm_ve_op(const SddmmVeArgs &a, cudaStream_t s) {
    switch (a.op) {
        case 0: return sddmm_ve_side<QH, 0>(a, s);
        case 1: return sddmm_ve_side<QH, 1>(a, s);
        case 2: return sddmm_ve_side<QH, 2>(a, s);
        default: return sddmm_ve_side<QH, 3>(a, s);
    }
}

// ============================================ NEXT-3: additive GAT scores
// out[j, h] = lrelu(el[u_j, h] + er[v, h]) (oracle C14; P:1329-1331 gSDDMM
// family, SPEC S:380 / S:411 additive attention with leaky ReLU): el is the
// source-side table, er the destination side (padded tables on partitions:
// er row row_base + r).  Scalar path: lanes stride over the row's (edge, head)
// pairs; vector path (H in {4, 8, 16, 32}, 16-B rows): QH = H/4 lanes per
// edge, one float4 of heads each, 4 edges in flight per lane, er[v] loaded
// once per lane; the score stream is written evict_first.
__device__ __forceinline__ float lrelu(float x, float slope) { return x > 0.f ? x : slope * x; }

__global__ void __launch_bounds__(kThreads) sddmm_add_kernel(const SddmmAddArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t idx = (int64_t)blockIdx.x * kWarps + warp;
    if (idx >= a.nrows) return;
    const int64_t row = a.order[idx], b = a.off[row], e = a.off[row + 1];
    const int64_t H = a.H;
    for (int64_t t = lane; t < (e - b) * H; t += 32) {
        const int64_t j = b + t / H, h = t % H;
        const float x = __ldg(a.el + (int64_t)__ldg(a.col + j) * a.lde + h) + __ldg(a.er + (a.row_base + row) * a.ldr + h);
        a.out[j * a.ldo + h] = lrelu(x, a.slope);
    }
}

template <int QH>
__global__ void __launch_bounds__(kThreads) sddmm_add_vec_kernel(const SddmmAddArgs a) {
    constexpr int EPW = 32 / QH, U = 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int eo = lane / QH, q = lane % QH;
    const float sl = a.slope;
    const float4 r = b < e ? __ldg(reinterpret_cast<const float4 *>(a.er + (a.row_base + row) * a.ldr + 4 * q))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    auto one = [&](int64_t jj, const float4 x) {
        st_stream_f4(a.out + jj * a.ldo + 4 * q,
                     make_float4(lrelu(x.x + r.x, sl), lrelu(x.y + r.y, sl), lrelu(x.z + r.z, sl), lrelu(x.w + r.w, sl)),
                     pol.stream);
    };
    int64_t j = b + eo;
    for (; j + (U - 1) * EPW < e; j += U * EPW) {
        int c[U];
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; u++) c[u] = ld_stream_i32(a.col + j + u * EPW, pol.stream);
#pragma unroll
        for (int u = 0; u < U; u++) x[u] = __ldg(reinterpret_cast<const float4 *>(a.el + (int64_t)c[u] * a.lde + 4 * q));
#pragma unroll
        for (int u = 0; u < U; u++) one(j + u * EPW, x[u]);
    }
    for (; j < e; j += EPW)
        one(j, __ldg(reinterpret_cast<const float4 *>(a.el + (int64_t)ld_stream_i32(a.col + j, pol.stream) * a.lde + 4 * q)));
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

cudaError_t launch_sddmm_ve(const SddmmVeArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool vec = (a.H == 4 || a.H == 8 || a.H == 16 || a.H == 32) && a.ldw % 4 == 0 && a.ldo % 4 == 0 &&
                     a.ldx % 4 == 0 && aligned(a.w, 16) && aligned(a.out, 16) && aligned(a.X, 16);
    if (!vec) {
        sddmm_ve_kernel<<<(unsigned)ceil_div(a.nrows, kWarps), kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    switch (a.H) {
        case 4: return sddmm_ve_op<1>(a, s);
        case 8: return sddmm_ve_op<2>(a, s);
        case 16: return sddmm_ve_op<4>(a, s);
        default: return sddmm_ve_op<8>(a, s);
    }
}

cudaError_t launch_sddmm_add(const SddmmAddArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool vec = (a.H == 4 || a.H == 8 || a.H == 16 || a.H == 32) && a.lde % 4 == 0 && a.ldr % 4 == 0 &&
                     a.ldo % 4 == 0 && aligned(a.el, 16) && aligned(a.er, 16) && aligned(a.out, 16);
    if (!vec) {
        sddmm_add_kernel<<<(unsigned)ceil_div(a.nrows, kWarps), kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    switch (a.H) {
        case 4: sddmm_add_vec_kernel<1><<<grid, kThreads, 0, s>>>(a); break;
        case 8: sddmm_add_vec_kernel<2><<<grid, kThreads, 0, s>>>(a); break;
        case 16: sddmm_add_vec_kernel<4><<<grid, kThreads, 0, s>>>(a); break;
        default: sddmm_add_vec_kernel<8><<<grid, kThreads, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

}  // namespace gsp
