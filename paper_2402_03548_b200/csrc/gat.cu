// Fused GAT forward (NEXT-2).
#include <atomic>

#include "common.cuh"

namespace gsp {
namespace {

// ===================================================== fused GAT forward
// NEXT-2 ("18 kernels in each layer"; a fused forward is
// legal only if it still materialises the state tensor alpha).  One pass per
// destination row v: for each in-edge j = (u -> v) and head h (one lane per
// head, Fh = 8 features per lane):
//   s = <X[v,h], Y[u,h]>          -> written to alpha (raw) ;
//   online softmax (m, S) and acc = sum exp(s - m) Vt[u,h]   (flash-style);
// then out[v,h] = acc / S and the row's raw scores are re-read and
// overwritten with alpha = exp(s - m) / S.  The first `cap` edges of each
// warp's slice keep their raw scores in shared memory (dynamic, cap * H floats
// per warp): only the excess of long rows makes the global round trip, so the
// in-flight score blocks no longer crowd the gathered table out of L2.  Y and
// Vt may be the same table (one gather serves both).  Heavy rows: CTA split +
// deterministic merge.
// MODE 0: s = <X[v,h], Y[u,h]>, Vt == Y (one gather); MODE 1: the same with a
// separate Vt; MODE 2 (NEXT-3, oracle C15): additive attention
// s = lrelu(Y[u,h] + X[v,h], slope) with Y = el, X = er one float per head
// ([ncols, H] tables) -- the standard GAT logit.
template <int LPE, int MODE, int UOVR = 0, int MINB = 2>
__global__ void __launch_bounds__(kThreads, MINB) gat_fused_kernel(const GatArgs a) {
    constexpr int VEC = 8;
    constexpr int G = 32 / LPE;
    constexpr int PER = LPE;
    constexpr bool SAME = MODE == 0, ADD = MODE == 2;
    constexpr int XV = ADD ? 1 : VEC;    // floats of the score operands per lane
    constexpr int U0 = UOVR ? UOVR : ((SAME || ADD) ? 8 : 4);
    constexpr int U = U0 > PER ? PER : U0;   // edges in flight per lane
    __shared__ __align__(16) int s_col[kWarps][32];
    // running Kahan state (acc, accc) per lane lives in smem: touched once per
    // tile (fold) and on the rare max increase (rescale), keeping registers for
    // the gathers in flight.  Reused for the heavy-row cross-warp merge.
    // [t][lane]: lane-minor, so the per-lane accesses are bank-conflict free
    __shared__ __align__(16) float s_run[kWarps][2 * VEC][32];
    __shared__ float sm_ms[kWarps][LPE][2];
    extern __shared__ __align__(16) float s_sc[];   // [kWarps][cap][H] raw scores
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, h = lane % LPE;   // head of this lane
    const int H = LPE;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int64_t cap = a.sc_cap;
    float *wsc = s_sc + (int64_t)warp * cap * LPE;

    Vec<XV> xv;
    ld_keep(xv, a.X + (a.row_base + row) * a.ldx + h * XV, pol.stream);
    const char *yl = reinterpret_cast<const char *>(a.Y + h * XV);
    const char *vl = reinterpret_cast<const char *>(a.Vt + h * VEC);
    const uint32_t ldyb = (uint32_t)(a.ldy * 4), ldvb = (uint32_t)(a.ldv * 4);

    // (m, S + Sc compensation) in registers; acc / accc in smem; tile sums in registers
    float m = -INFINITY, S = 0.f, Sc = 0.f, St = 0.f;
    auto run = [&](int t) -> float & { return s_run[warp][t][lane]; };
#pragma unroll
    for (int t = 0; t < 2 * VEC; t++) run(t) = 0.f;
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
        // raw scores of this tile: shared memory while the slice is within cap (whole
        // tiles: cap is a multiple of 32), else the alpha buffer itself
        const bool in_smem = base - b < cap;
        float *ab = in_smem ? wsc + (base - b + g) * H + h
                            : a.alpha + (base + g) * H + h;   // group g's i-th edge is tile edge g + G*i
        const int mcount = n == 32 ? PER : (n > g ? (n - g + G - 1) / G : 0);
        auto body = [&](int i, auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            Vec<XV> y[U];
            Vec<VEC> vv[SAME ? 1 : U];
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
                if constexpr (ADD) {
                    const float x = y[u].v[0] + xv.v[0];
                    sc[u] = x > 0.f ? x : a.slope * x;
                } else {
                    float s0 = 0.f, s1 = 0.f;   // even / odd features: one FFMA2 per pair
#pragma unroll
                    for (int t = 0; t < VEC; t += 2) fma2(s0, s1, xv.v[t], xv.v[t + 1], y[u].v[t], y[u].v[t + 1]);
                    sc[u] = s0 + s1;
                }
                if (FULL || i + u < mcount) {
                    ab[(int64_t)(G * (i + u)) * H] = sc[u];   // raw score (smem, or global with the default L2 policy)
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
                    run(t) *= r;
                    run(VEC + t) *= r;
                    acct.v[t] *= r;
                }
                m = mb;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const float pu = fast_exp(sc[u] - m);   // 0 for padding (-inf)
                St += pu;
                if constexpr (SAME) {
#pragma unroll
                    for (int t = 0; t < VEC; t += 2) fma2(acct.v[t], acct.v[t + 1], pu, pu, y[u].v[t], y[u].v[t + 1]);
                } else {
#pragma unroll
                    for (int t = 0; t < VEC; t += 2) fma2(acct.v[t], acct.v[t + 1], pu, pu, vv[u].v[t], vv[u].v[t + 1]);
                }
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
                const float ac = run(t), cc = run(VEC + t);
                y2 = acct.v[t] - cc;
                t2 = ac + y2;
                run(VEC + t) = (t2 - ac) - y2;
                run(t) = t2;
                acct.v[t] = 0.f;
            }
        }
    }
    S -= Sc;
    Vec<VEC> acc;
#pragma unroll
    for (int t = 0; t < VEC; t++) acc.v[t] = run(t) - run(VEC + t);
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
        float *xs = &s_run[0][0][0];   // [warp][head][t] scratch
        if (g == 0) {
            sm_ms[warp][h][0] = m;
            sm_ms[warp][h][1] = S;
#pragma unroll
            for (int t = 0; t < VEC; t++) xs[(warp * 32 + h) * VEC + t] = acc.v[t];
        }
        __syncthreads();
        m = -INFINITY;
        S = 0.f;
        vzero(acc);
        for (int w = 0; w < kWarps; w++) {
            Vec<VEC> ao;
#pragma unroll
            for (int t = 0; t < VEC; t++) ao.v[t] = xs[(w * 32 + h) * VEC + t];
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
    // normalise this warp's slice of raw scores into alpha: element i has head i % H;
    // [lo, mid) from shared memory, [mid, hi) in place in global memory
    __syncwarp();
    const int64_t lo = b * H, hi = e * H, mid = min(hi, lo + cap * H);
    if (H % 4 == 0) {
        float mh[4], rh[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int hh = (lane * 4 + t) % H;
            mh[t] = __shfl_sync(kFull, m, hh);
            rh[t] = __shfl_sync(kFull, rS, hh);
        }
        for (int64_t i0 = lo + (int64_t)lane * 4; i0 < mid; i0 += 128) {
            const float4 v = *reinterpret_cast<const float4 *>(wsc + (i0 - lo));
            st_stream_f4(a.alpha + i0,
                         make_float4(fast_exp(v.x - mh[0]) * rh[0], fast_exp(v.y - mh[1]) * rh[1],
                                     fast_exp(v.z - mh[2]) * rh[2], fast_exp(v.w - mh[3]) * rh[3]),
                         pol.stream);
        }
        constexpr int NU = 8;   // loads in flight per lane (the row block is L2-hot)
        for (int64_t i0 = mid + (int64_t)lane * 4; i0 < hi; i0 += 128 * NU) {
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
            const float v = i < mid ? wsc[i - lo] : ld_f32(a.alpha + i, pol.stream);
            st_stream_f32(a.alpha + i, fast_exp(v - mh) * rh, pol.stream);
        }
    }
}


// ================================================ fused GAT backward scores
// NEXT-1 ("Backward Computation"): the score
// gradient of one GAT layer in one pass per destination row v, one lane per
// head (Fh = 8 features per lane), a = GatArgs with X = dOut (destination
// side), Vt = the aggregated table, alpha = the forward state, out = ds:
//   dalpha[j,h] = <dOut[v,h], Vt[u_j,h]>                  (gSDDMM, C6)
//   ds[j,h]     = alpha[j,h] (dalpha[j,h] - c_h),  c_h = sum_j alpha[j,h] dalpha[j,h]   (C9)
// Phase 1 gathers Vt rows, computes dalpha and the per-head row sum c (tile
// sums folded with Kahan compensation); dalpha of the first `cap` edges of the
// warp slice stays in shared memory, the rest is parked in ds itself.  Phase 2
// (after c is complete, across warps for CTA-split rows) streams
// ds = alpha (dalpha - c).
template <int LPE>
__global__ void __launch_bounds__(kThreads, 2) gat_bwd_kernel(const GatArgs a) {
    constexpr int VEC = 8;
    constexpr int G = 32 / LPE;
    constexpr int PER = LPE;
    constexpr int U = PER >= 8 ? 8 : PER;
    __shared__ __align__(16) int s_col[kWarps][32];
    __shared__ float s_c[kWarps][32];
    extern __shared__ __align__(16) float s_sc[];   // [kWarps][cap][H] dalpha
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, h = lane % LPE;
    const int H = LPE;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int64_t cap = a.sc_cap;
    float *wsc = s_sc + (int64_t)warp * cap * LPE;
    const float *al = a.alpha;

    Vec<VEC> xv;
    ld_keep(xv, a.X + (a.row_base + row) * a.ldx + h * VEC, pol.stream);
    const char *vl = reinterpret_cast<const char *>(a.Vt + h * VEC);
    const uint32_t ldvb = (uint32_t)(a.ldv * 4);

    float c = 0.f, cc = 0.f, ct = 0.f;   // Kahan running sum of alpha * dalpha, tile sum
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
        const bool in_smem = base - b < cap;
        float *db = in_smem ? wsc + (base - b + g) * H + h : a.out + (base + g) * H + h;
        const float *ab = al + (base + g) * H + h;
        const int mcount = n == 32 ? PER : (n > g ? (n - g + G - 1) / G : 0);
#pragma unroll 1
        for (int i = 0; i < mcount; i += U) {
            Vec<VEC> y[U];
            float av[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (i + u < mcount) {
                    ld_keep(y[u], reinterpret_cast<const float *>(vl + (uint64_t)(uint32_t)gp[i + u] * ldvb), pol.keep);
                    av[u] = ld_f32(ab + (int64_t)(G * (i + u)) * H, pol.keep);   // re-read in phase 2
                } else {
                    vzero(y[u]);
                    av[u] = 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                float s0 = 0.f, s1 = 0.f;
#pragma unroll
                for (int t = 0; t < VEC; t += 2) {   // (FFMA2 here measured 3 % slower: 4.19 vs 4.05 ms)
                    s0 = fmaf(xv.v[t], y[u].v[t], s0);
                    s1 = fmaf(xv.v[t + 1], y[u].v[t + 1], s1);
                }
                const float d = s0 + s1;
                if (i + u < mcount) db[(int64_t)(G * (i + u)) * H] = d;
                ct = fmaf(av[u], d, ct);
            }
        }
        __syncwarp();
        if (++ntile == kFoldTiles || base + 32 >= e) {   // Kahan fold of the tile sum
            ntile = 0;
            const float y2 = ct - cc, t2 = c + y2;
            cc = (t2 - c) - y2;
            c = t2;
            ct = 0.f;
        }
    }
    c -= cc;
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1) c += __shfl_xor_sync(kFull, c, o);   // the G groups of head h
    if (heavy) {   // the CTA's warps hold slices of one row: sum in warp order
        if (g == 0) s_c[warp][h] = c;
        __syncthreads();
        c = 0.f;
        for (int w = 0; w < kWarps; w++) c += s_c[w][h];
    }
    // phase 2: ds = alpha (dalpha - c) over the warp's slice; element i has head i % H
    __syncwarp();
    const int64_t lo = b * H, hi = e * H, mid = min(hi, lo + cap * H);
    if (H % 4 == 0) {
        float ch[4];
#pragma unroll
        for (int t = 0; t < 4; t++) ch[t] = __shfl_sync(kFull, c, (lane * 4 + t) % H);
        constexpr int NU = 4;   // loads in flight per lane
        for (int64_t i0 = lo + (int64_t)lane * 4; i0 < hi; i0 += 128 * NU) {
            float4 d[NU], av[NU];
#pragma unroll
            for (int k = 0; k < NU; k++) {
                const int64_t i = i0 + 128 * k;
                if (i < hi) {
                    av[k] = ld_f4(al + i, pol.stream);
                    d[k] = i < mid ? *reinterpret_cast<const float4 *>(wsc + (i - lo)) : ld_f4(a.out + i, pol.stream);
                }
            }
#pragma unroll
            for (int k = 0; k < NU; k++) {
                const int64_t i = i0 + 128 * k;
                if (i < hi)
                    st_stream_f4(a.out + i, make_float4(av[k].x * (d[k].x - ch[0]), av[k].y * (d[k].y - ch[1]),
                                                        av[k].z * (d[k].z - ch[2]), av[k].w * (d[k].w - ch[3])),
                                 pol.stream);
            }
        }
    } else {
        const float chh = __shfl_sync(kFull, c, lane % H);
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const float d = i < mid ? wsc[i - lo] : ld_f32(a.out + i, pol.stream);
            st_stream_f32(a.out + i, ld_f32(al + i, pol.stream) * (d - chh), pol.stream);
        }
    }
}
}  // namespace

bool gat_fused_supported(const GatArgs &a) {
    const int64_t H = a.H;
    const bool h_ok = H == 2 || H == 4 || H == 8 || H == 16 || H == 32;
    const bool xy_ok = a.additive ? (aligned(a.X, 4) && aligned(a.Y, 4))
                                  : (a.ldx % 8 == 0 && a.ldy % 8 == 0 && aligned(a.X, 32) && aligned(a.Y, 32));
    return h_ok && xy_ok && a.ldv % 8 == 0 && a.ldo % 4 == 0 && aligned(a.Vt, 32) && aligned(a.out, 16) &&
           aligned(a.alpha, 16);
}

// shared-memory score block per warp (bytes); GSP_GAT_SMEM_KB overrides (0: off, A/B)
static int64_t gat_score_bytes() {
    static const int64_t v = [] {
        const char *e = getenv("GSP_GAT_SMEM_KB");
        return (e ? atoll(e) : int64_t(7)) << 10;   // 7 KB (224 edges at H = 8): 3.26 -> 2.93 ms on Reddit 8x8; 11 KB: 4.2 ms (L1 squeezed)
    }();
    return v;
}

// Opt a kernel in to > 48 KB of dynamic shared memory once per device.  The
// per-(kernel, device) flags are atomics: concurrent first calls on different
// threads / streams (gsp.h: compute calls are thread-safe) at worst both set the
// (idempotent) attribute; no data race.
using AttrFlags = std::atomic<int>[64];
template <class K>
cudaError_t opt_in_smem(K kernel, size_t dyn, AttrFlags &flags) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && flags[dev].load(std::memory_order_acquire) >= (int)dyn) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    if (dev < 64) {
        int cur = flags[dev].load(std::memory_order_relaxed);
        while (cur < (int)dyn && !flags[dev].compare_exchange_weak(cur, (int)dyn, std::memory_order_release)) {
        }
    }
    return cudaSuccess;
}
template <int HH, int MODE, int UO, int MB>
AttrFlags &gat_fused_attr() {
    static AttrFlags f{};
    return f;
}
template <int HH>
AttrFlags &gat_bwd_attr() {
    static AttrFlags f{};
    return f;
}

template <int HH, int MODE, int UO = 0, int MB = 2>
cudaError_t launch_gat_v(GatArgs a, dim3 grid, cudaStream_t s, int64_t score_bytes = -1) {
    a.sc_cap = ((score_bytes >= 0 ? score_bytes : gat_score_bytes()) / (4 * HH)) & ~int64_t(31);   // whole 32-edge tiles
    const size_t dyn = (size_t)(kWarps * a.sc_cap * HH * 4);
    cudaError_t e = opt_in_smem(gat_fused_kernel<HH, MODE, UO, MB>, dyn, gat_fused_attr<HH, MODE, UO, MB>());
    if (e != cudaSuccess) return e;
    gat_fused_kernel<HH, MODE, UO, MB><<<grid, kThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

// tuning knob for H = 8 (GSP_TUNE_GAT: (edges in flight per lane, CTAs per SM)); read once
static int tune_gat() {
    static int v = [] {
        const char *e = getenv("GSP_TUNE_GAT");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <int HH, int MODE>
cudaError_t launch_gat_h(GatArgs a, dim3 grid, cudaStream_t s) {
    if constexpr (HH == 8) {
        // light graphs (mean degree < 32, e.g. Pubmed): rows are one or two tiles, so rows in
        // flight decide -- 2 edges in flight per lane at 4 CTAs/SM with a 2 KB score block
        // (64 edges per warp): Pubmed 8 x 8 34.8 -> 26.6 us (same-box A/B; 4 at 3 CTAs/SM with
        // 3 KB 28.7 us)
        if (a.light && tune_gat() == 0) return launch_gat_v<HH, MODE, 2, 4>(a, grid, s, 2048);
        switch (tune_gat()) {
            case 1: return launch_gat_v<HH, MODE, 4, 3>(a, grid, s);
            case 2: return launch_gat_v<HH, MODE, 4, 2>(a, grid, s);
            case 3: return launch_gat_v<HH, MODE, 2, 4>(a, grid, s);
            case 4: return launch_gat_v<HH, MODE, 8, 3>(a, grid, s);
            default: break;
        }
    }
    return launch_gat_v<HH, MODE>(a, grid, s);
}

cudaError_t launch_gat_fused(const GatArgs &a, cudaStream_t s) {
    if (a.nrows == 0) return cudaSuccess;
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    const int mode = a.additive ? 2 : ((a.Vt == a.Y && a.ldv == a.ldy) ? 0 : 1);
#define GSP_GAT_CASE(HH)                                                      \
    case HH:                                                                  \
        return mode == 0 ? launch_gat_h<HH, 0>(a, grid, s)                    \
                         : (mode == 1 ? launch_gat_h<HH, 1>(a, grid, s) : launch_gat_h<HH, 2>(a, grid, s));
    switch (a.H) {
        GSP_GAT_CASE(2)
        GSP_GAT_CASE(4)
        GSP_GAT_CASE(8)
        GSP_GAT_CASE(16)
        GSP_GAT_CASE(32)
        default: return cudaErrorNotSupported;
    }
#undef GSP_GAT_CASE
}

template <int HH>
cudaError_t launch_gat_bwd_h(GatArgs a, dim3 grid, cudaStream_t s) {
    a.sc_cap = (gat_score_bytes() / (4 * HH)) & ~int64_t(31);
    const size_t dyn = (size_t)(kWarps * a.sc_cap * HH * 4);
    cudaError_t e = opt_in_smem(gat_bwd_kernel<HH>, dyn, gat_bwd_attr<HH>());
    if (e != cudaSuccess) return e;
    gat_bwd_kernel<HH><<<grid, kThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gat_bwd(const GatArgs &a, cudaStream_t s) {
    if (a.nrows == 0) return cudaSuccess;
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    switch (a.H) {
        case 2: return launch_gat_bwd_h<2>(a, grid, s);
        case 4: return launch_gat_bwd_h<4>(a, grid, s);
        case 8: return launch_gat_bwd_h<8>(a, grid, s);
        case 16: return launch_gat_bwd_h<16>(a, grid, s);
        default: return launch_gat_bwd_h<32>(a, grid, s);
    }
}

}  // namespace gsp
