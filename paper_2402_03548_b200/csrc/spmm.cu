// gSpMM family: gSpMMv + norm, gSpMMve / gSpMMve^T, min / max, gSpMMe (+ degree / edge scales).
#include "common.cuh"

#ifndef GSP_MAXCPL4
#define GSP_MAXCPL4 5   // 128-bit path: max 16-B chunks per lane before the row splits into feature slabs (F = 602: 5 -> one slab, 19.9 ms; 4 -> two slabs, 23.6 ms)
#endif
#ifndef GSP_TUNE_V4
#define GSP_TUNE_V4 0   // 1: formula default for the F = 65-128 float4 path (A/B)
#endif
#ifndef GSP_PAIR_LAYOUT
#define GSP_PAIR_LAYOUT 1
#endif

namespace gsp {
namespace {

// ============================================================ gSpMM family
// MODE kSpmmScaled      : out[r] = rs(r) * sum_j cs(col_j) * X[col_j]          (gSpMMv + norm)
// MODE kSpmmWeightedFwd : out[r, h-block] = sum_j w[j, h] * X[col_j, h-block]   (gSpMMve)
// MODE kSpmmWeightedRev : out[r, h-block] = sum_k w[eid_k, h] * X[col_k, ...]   (gSpMMve^T via eid)
template <int VEC, int LPE, int CPL, int MODE, bool HAS_CS, int UOVR = 0, int MINB = 0, bool HOT = false>
__global__ void __launch_bounds__(kThreads, (MINB ? MINB : (VEC * CPL <= 8 ? 3 : 2))) spmm_kernel(const SpmmArgs a) {
    constexpr int G = 32 / LPE;           // edge groups per warp
    constexpr int PER = LPE;              // edges per group per 32-edge tile
    constexpr int UB = 32 / (VEC * CPL);  // loads in flight per lane: ~32 floats
    constexpr int U0 = UOVR ? UOVR : (UB < 2 ? 2 : (UB > 4 ? 4 : UB));
    constexpr int U = U0 > PER ? PER : U0;
    constexpr int SW = VEC * LPE * CPL;   // feature slab handled by this CTA
    constexpr bool W = MODE == kSpmmWeightedFwd || MODE == kSpmmWeightedRev;
    constexpr bool MM = MODE == kSpmmMin || MODE == kSpmmMax;   // min / max reductions (NEXT-3)
#ifndef GSP_FF2_WIDE
#define GSP_FF2_WIDE 1   // FFMA2 on the multi-chunk 128-bit path (Reddit F = 602: 20.0 -> 19.8 ms same box)
#endif
    constexpr bool FF2 = VEC >= 8 || (GSP_FF2_WIDE && VEC == 4 && CPL >= 2);
    constexpr float ID = MODE == kSpmmMin ? INFINITY : (MODE == kSpmmMax ? -INFINITY : 0.f);
    auto comb = [](float x, float y) {
        if constexpr (MODE == kSpmmMin) return fminf(x, y);
        else if constexpr (MODE == kSpmmMax) return fmaxf(x, y);
        else return x + y;
    };
    constexpr int RED = kWarps * SW;
    // double-buffered weight rows; each edge group's rows start 8 words (one
    // bank octet) after the previous group's, so the 32/LPE groups of a warp
    // read their per-edge weights from distinct banks (no 4-way conflicts)
    constexpr int WP = G <= 4 ? 8 : 4;   // group padding (words, keeps 16-B rows); narrower for many groups (48 KB static smem)
    constexpr int WSW = 32 * kHMax + WP * G;
    constexpr int WS = W ? 2 * kWarps * WSW : 0;
    __shared__ __align__(16) int2 s_pair[kWarps][32];
    __shared__ __align__(16) float s_raw[RED > WS ? RED : WS];   // weights during the walk, then heavy combine
    // Kahan compensation of narrow lanes lives in smem (touched once per fold):
    // the registers go to gathers in flight
    constexpr bool CMP_SMEM = VEC * CPL <= 8 && !MM;
    __shared__ __align__(16) float s_cmp[CMP_SMEM ? kWarps : 1][CMP_SMEM ? VEC * CPL : 1][CMP_SMEM ? 32 : 1];   // lane-minor: conflict-free

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPE, sub = lane % LPE;
    const int64_t f0 = (int64_t)blockIdx.y * SW;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
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
        if constexpr (CMP_SMEM) return s_cmp[warp][q * VEC + t][lane];
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
    const int wpos = (lane % G) * (PER * H + WP) + (lane / G) * H;   // this lane's weight row in s_w
    // (col, scale) pairs of group g's edges i, i+1 (i even) sit in one 16-B
    // chunk, the G groups' chunks side by side: one LDS.128 per two edges reads
    // 16*G contiguous bytes, conflict-free
#if GSP_PAIR_LAYOUT == 0
    const int ppos = (lane % G) * PER + lane / G;
#else
    const int ppos = ((lane / G) >> 1) * 2 * G + 2 * (lane % G) + ((lane / G) & 1);
#endif
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
    uint64_t wp = pol.stream;
    if constexpr (W) {
        if (a.wpol == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(wp));
        else if (a.wpol == 2) wp = pol.keep;
    }
    auto load_w8 = [&](int64_t tb, int ev, float *d) {
        if constexpr (W) {
            if (tb + lane < e) ld_stream_v8(d, a.w + (int64_t)ev * 8, wp);
            else {
#pragma unroll
                for (int t = 0; t < 8; t++) d[t] = 0.f;
            }
        }
    };
    auto issue_w = [&](int64_t tb, int ev, int buf) {
        if constexpr (W) {
            if (w8) return;
            float *dst = s_raw + (buf * kWarps + warp) * WSW + wpos;
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
    // L2 prefetch of the streamed edge arrays a.pf tiles ahead (lane 0, one
    // bulk request per stream and tile)
    const bool pfw = MODE == kSpmmWeightedFwd && (a.ldw % 4 == 0);
    auto prefetch = [&](int64_t tb, int64_t n) {
        if (lane != 0 || tb >= e) return;
        n = n < e - tb ? n : e - tb;
        prefetch_l2(a.col + tb, (uint32_t)(n * 4));
        if constexpr (MODE == kSpmmScaled)
            if (a.edge_scale) prefetch_l2(a.edge_scale + tb, (uint32_t)(n * 4));
        if constexpr (MODE == kSpmmWeightedRev) prefetch_l2(a.eid + tb, (uint32_t)(n * 4));
        if (pfw) prefetch_l2(a.w + tb * a.ldw, (uint32_t)(n * a.ldw * 4));
    };
    if (a.pf) prefetch(b, (int64_t)a.pf * 32);
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
        if (a.pf) prefetch(base + (int64_t)a.pf * 32, 32);
        s_pair[warp][ppos] = make_int2(c1, __float_as_int(wv1));
        // ---- advance the pipeline before this tile's gathers
        int c3, e3;
        load_idx(base + 64, c3, e3);
        const float wv2 = load_scale(base + 32, c2);
        float w8b[W ? 8 : 1];
        if constexpr (W) {
            if (w8) {
                float *dst = s_raw + (buf * kWarps + warp) * WSW + wpos;
                reinterpret_cast<float4 *>(dst)[0] = make_float4(w8a[0], w8a[1], w8a[2], w8a[3]);
                reinterpret_cast<float4 *>(dst)[1] = make_float4(w8a[4], w8a[5], w8a[6], w8a[7]);
                load_w8(base + 32, e2, w8b);
            } else {
                issue_w(base + 32, e2, buf ^ 1);
                cp_async_wait<1>();   // this tile's weight rows have landed
            }
        }
        const float *s_w = s_raw + (buf * kWarps + warp) * WSW;
        __syncwarp();
#if GSP_PAIR_LAYOUT == 0
        const int2 *gp = &s_pair[warp][g * PER];
#else
        const int2 *gp = &s_pair[warp][2 * g];
#endif
        const float *gw = s_w + g * (PER * H + WP);

        auto body = [&](int i, bool full, int m) {
            Vec<VEC> x[U][CPL];
            float wt[U][CPL];
#pragma unroll
            for (int u = 0; u < U; u += 2) {
#if GSP_PAIR_LAYOUT == 0
                const int4 pp = *reinterpret_cast<const int4 *>(gp + i + u);
#else
                const int4 pp = *reinterpret_cast<const int4 *>(gp + (i + u) * G);
#endif
                const int cc[2] = {pp.x, pp.z};
                const float ww[2] = {__int_as_float(pp.y), __int_as_float(pp.w)};
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const bool ok = full || (i + u + k < m);
#pragma unroll
                    for (int q = 0; q < CPL; q++) {
                        if (ok && fv[q]) {
                            // hot-row policy (scaled mode, BOTH norm; api.cu hot_scale_for): a source
                            // whose column scale d^-1/2 is below a.hot_scale (degree above the hot
                            // threshold) keeps its row in L2 (evict_last), cold rows stream (evict_first)
                            // (a separate instantiation: the all-evict_last kernels stay as they were)
                            uint64_t gp_pol = pol.keep;
                            if constexpr (HOT && MODE == kSpmmScaled && HAS_CS)
                                if (ww[k] >= a.hot_scale) gp_pol = pol.stream;
                            ld_keep(x[u + k][q],
                                    reinterpret_cast<const float *>(xl[q] + (uint64_t)(uint32_t)cc[k] * ldxb),
                                    gp_pol);
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
                    for (int t = 0; t < VEC; t += (FF2 && !MM ? 2 : 1))
                        if constexpr (MM) tile[u % NT][q].v[t] = comb(tile[u % NT][q].v[t], x[u][q].v[t]);
                        else if constexpr (FF2)   // FFMA2: two features per instruction (the 256-bit
                            // path; on the 128-bit DRAM-bound path, e.g. products F = 100, it measured
                            // 8 % slower: 9.97 vs 9.18 ms same box)
                            fma2(tile[u % NT][q].v[t], tile[u % NT][q].v[t + 1], wt[u][q], wt[u][q], x[u][q].v[t],
                                 x[u][q].v[t + 1]);
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
                    float *o = a.out + row * a.ldo + f;
                    if (a.out_vec) {
                        vstore(o, r, a.F - f);
                    } else {   // odd output stride: the gathers stay vectorised, the row store is scalar
#pragma unroll
                        for (int t = 0; t < VEC; t++)
                            if (f + t < a.F) o[t] = r.v[t];
                    }
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

// Vector path (H in {4, 8, 16, 32}, 16-B aligned rows): QH = H/4 lanes per edge,
// one float4 of heads each, EPW = 32/QH edges per warp step, 4 steps in
// flight; the LPT schedule of the other kernels (heavy rows: one CTA, warps
// combined in a fixed order through shared memory -> deterministic).
template <int QH, int RED, bool EID>
__global__ void __launch_bounds__(kThreads) spmm_e_vec_kernel(const SpmmEArgs a) {
    constexpr int EPW = 32 / QH, U = 4;
    __shared__ double part[kWarps][4 * QH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const int eo = lane / QH, q = lane % QH;
    auto comb = [](double x, double y) {
        if constexpr (RED == 1) return y < x ? y : x;
        else if constexpr (RED == 2) return y > x ? y : x;
        else return x + y;
    };
    constexpr double ID = RED == 1 ? INFINITY : (RED == 2 ? -INFINITY : 0.0);
    double acc[4] = {ID, ID, ID, ID};
    const float *wq = a.w + 4 * q;
    auto addv = [&](const float4 v) {
        acc[0] = comb(acc[0], (double)v.x); acc[1] = comb(acc[1], (double)v.y);
        acc[2] = comb(acc[2], (double)v.z); acc[3] = comb(acc[3], (double)v.w);
    };
    int64_t j = b + eo;
    for (; j + (U - 1) * EPW < e; j += U * EPW) {
        int64_t ei[U];
#pragma unroll
        for (int u = 0; u < U; u++) ei[u] = EID ? (int64_t)ld_stream_i32(a.eid + j + u * EPW, pol.stream) : j + u * EPW;
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = ld_stream_f4(wq + ei[u] * a.ldw, pol.stream);
#pragma unroll
        for (int u = 0; u < U; u++) addv(v[u]);
    }
    for (; j < e; j += EPW) {
        const int64_t ei = EID ? (int64_t)ld_stream_i32(a.eid + j, pol.stream) : j;
        addv(ld_stream_f4(wq + ei * a.ldw, pol.stream));
    }
#pragma unroll
    for (int o = QH; o < 32; o <<= 1) {
#pragma unroll
        for (int k = 0; k < 4; k++) acc[k] = comb(acc[k], __shfl_xor_sync(kFull, acc[k], o));
    }
    if (!heavy) {
        if (eo == 0) {
            float *o = a.out + row * a.ldo + 4 * q;
#pragma unroll
            for (int k = 0; k < 4; k++) o[k] = b == e ? 0.f : (float)acc[k];
        }
        return;
    }
    if (eo == 0) {
#pragma unroll
        for (int k = 0; k < 4; k++) part[warp][4 * q + k] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < 4 * QH) {
        double v = ID;
#pragma unroll
        for (int w = 0; w < kWarps; w++) v = comb(v, part[w][threadIdx.x]);
        a.out[row * a.ldo + threadIdx.x] = (float)v;
    }
}

template <int QH>
cudaError_t spmm_e_red(const SpmmEArgs &a, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    const bool eid = a.eid != nullptr;
    switch (a.red) {
        case 1:
            if (eid) spmm_e_vec_kernel<QH, 1, true><<<grid, kThreads, 0, s>>>(a);
            else spmm_e_vec_kernel<QH, 1, false><<<grid, kThreads, 0, s>>>(a);
            break;
        case 2:
            if (eid) spmm_e_vec_kernel<QH, 2, true><<<grid, kThreads, 0, s>>>(a);
            else spmm_e_vec_kernel<QH, 2, false><<<grid, kThreads, 0, s>>>(a);
            break;
        default:
            if (eid) spmm_e_vec_kernel<QH, 0, true><<<grid, kThreads, 0, s>>>(a);
            else spmm_e_vec_kernel<QH, 0, false><<<grid, kThreads, 0, s>>>(a);
            break;
    }
    return cudaGetLastError();
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

template <int VEC, int LPE, int CPL, int UOVR = 0, int MINB = 0>
cudaError_t spmm_go_v(const SpmmArgs &a, int mode, int64_t slabs, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, slabs);
    if (mode == kSpmmScaled) {
        if ((a.col_scale || a.edge_scale) && a.hot_scale > 0.f)
            spmm_kernel<VEC, LPE, CPL, kSpmmScaled, true, UOVR, MINB, true><<<grid, kThreads, 0, s>>>(a);
        else if (a.col_scale || a.edge_scale) spmm_kernel<VEC, LPE, CPL, kSpmmScaled, true, UOVR, MINB><<<grid, kThreads, 0, s>>>(a);
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
            case 0:   // measured best on B200 (Reddit-shaped F = 64, tools/opbench.py): the scaled
                      // gSpMM 4 gathers in flight per lane at 3 CTAs/SM (1.63 ms; 4 CTAs/SM 1.63-1.66,
                      // 8 at 2 CTAs/SM 1.69); the weighted modes 8 at 2 CTAs/SM (wfwd 2.01 vs 2.39,
                      // wrev 2.84 vs 3.72 ms at 4 / 4)
                if (mode == kSpmmScaled) return spmm_go_v<VEC, LPE, CPL, 4, 3>(a, mode, slabs, s);
                return spmm_go_v<VEC, LPE, CPL, 8, 2>(a, mode, slabs, s);
            case 7: return spmm_go_v<VEC, LPE, CPL, 4, 3>(a, mode, slabs, s);
            case 5: return spmm_go_v<VEC, LPE, CPL>(a, mode, slabs, s);
            case 6: return spmm_go_v<VEC, LPE, CPL, 4, 2>(a, mode, slabs, s);
            case 1: return spmm_go_v<VEC, LPE, CPL, 8, 2>(a, mode, slabs, s);
            case 2: return spmm_go_v<VEC, LPE, CPL, 4, 4>(a, mode, slabs, s);
            case 3: return spmm_go_v<VEC, LPE, CPL, 2, 4>(a, mode, slabs, s);
            case 4: return spmm_go_v<VEC, LPE, CPL, 8, 3>(a, mode, slabs, s);
            default: break;
        }
    }
    if constexpr (VEC == 8 && LPE == 16 && CPL == 1) {   // F = 65-128 with 32-B rows (ogbn-arxiv F = 128)
        // light graphs (mean degree < 32): a row is a few 2-edge gather instructions, so the
        // launch is bound by rows in flight x per-row latency -- 2 gathers in flight per lane
        // at 4 CTAs/SM (more warps) beat 4 at 3: arxiv 127 -> 103 us (same-box A/B; 2 at 6
        // CTAs/SM 205, 4 at 4 137, 8 at 2 164 us)
        if (mode == kSpmmScaled && a.light) return spmm_go_v<VEC, LPE, CPL, 2, 4>(a, mode, slabs, s);
    }
    if constexpr (VEC == 4 && LPE == 32 && CPL == 1) {   // rows of 17-32 float4 chunks (e.g. F = 100)
        // scaled gSpMM on a DRAM-resident table (ogbn-products F = 100): 8 gathers in flight
        // per lane at 3 CTAs/SM, 9.92 -> 9.18 ms (2 CTAs/SM: 10.6; U = 16: 10.3)
        if (mode == kSpmmScaled && GSP_TUNE_V4 == 0) return spmm_go_v<VEC, LPE, CPL, 8, 3>(a, mode, slabs, s);
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

}  // namespace

static int prefetch_tiles() {
    static int v = [] {
        const char *e = getenv("GSP_PF");
        return e ? atoi(e) : 0;
    }();
    return v;
}

// L2 policy of the edge-ID indirected weight rows of the weighted reverse (GSP_WREV_POL for A/B):
// rev rows of one id window read runs of adjacent alpha rows in each destination's block,
// so the rows are reused by the window's other sources
static int wrev_policy() {
    static int v = [] {
        const char *e = getenv("GSP_WREV_POL");
        return e ? atoi(e) : 0;
    }();
    return v;
}

cudaError_t launch_spmm(const SpmmArgs &a_in, int mode, cudaStream_t s) {
    if (a_in.nrows == 0 || a_in.F == 0) return cudaSuccess;
    SpmmArgs a = a_in;
    a.pf = prefetch_tiles();
    a.wpol = mode == kSpmmWeightedRev ? wrev_policy() : 0;

    const bool wmode = mode == kSpmmWeightedFwd || mode == kSpmmWeightedRev;
    if (wmode && a.H > kHMax) return cudaErrorNotSupported;   // api.cu rejects H > 16 first
    // the gather width depends on X only; an output stride that is not a multiple of 4
    // (e.g. F = 602 written densely) just makes the row stores scalar
    a.out_vec = a.ldo % 4 == 0 && aligned(a.out, 16);
    auto ok_vec = [&](int v) {
        return a.F >= v && a.ldx % v == 0 && aligned(a.X, 4 * v) && (!wmode || a.Fh % v == 0);
    };
    if (ok_vec(8)) return spmm_dispatch<8, 2>(a, mode, s);
    if (ok_vec(4)) return spmm_dispatch<4, GSP_MAXCPL4>(a, mode, s);
    return spmm_dispatch<1, 4>(a, mode, s);
}

cudaError_t launch_spmm_e(const SpmmEArgs &a, cudaStream_t s) {
    if (a.nrows == 0 || a.H == 0) return cudaSuccess;
    const bool vec = (a.H == 4 || a.H == 8 || a.H == 16 || a.H == 32) && a.ldw % 4 == 0 && aligned(a.w, 16);
    if (!vec) {
        spmm_e_kernel<<<(unsigned)ceil_div(a.nrows, kWarps), kThreads, 0, s>>>(a);
        return cudaGetLastError();
    }
    switch (a.H) {
        case 4: return spmm_e_red<1>(a, s);
        case 8: return spmm_e_red<2>(a, s);
        case 16: return spmm_e_red<4>(a, s);
        default: return spmm_e_red<8>(a, s);
    }
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
