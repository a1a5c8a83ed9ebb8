// Weighted gSpMM (gSpMMve / gSpMMve^T via eid) for the GAT head shape H = 8
// heads x Fh = 8 features (F = 64): the A7 / A8 rows of SURVEY §8(a).
//
// Same schedule, lane mapping and summation as spmm_kernel's weighted modes
// (common.cuh: degree-ordered rows, CTA-split heavy rows, 32-edge tiles, 8
// lanes per edge = one head each, LDG.256 feature slices, Kahan-folded tile
// sums), but with TWO tiles of feature gathers in flight per warp instead of
// one: even tiles land in registers (ld.global.nc.v8), odd tiles in a per-warp
// shared-memory buffer (cp.async, LDGSTS), and the gathers of tile t+2 are
// issued as soon as tile t has been consumed.  The register file alone holds
// one 8 KB tile per warp (128 registers, 2 CTAs/SM) and the kernel was bound
// by bytes in flight x latency (ncu: ~45 % of warp samples waiting on the
// gathers); the shared-memory buffer doubles the bytes in flight per SM
// without registers (DESIGN.md §6 "Two tiles in flight").
#include <atomic>

#include "common.cuh"

namespace gsp {
namespace {

constexpr int kWG = 4;        // edge groups per warp (8 lanes per edge)
constexpr int kWPer = 8;      // edges per group per 32-edge tile
constexpr int kWRow = kWPer * 8 + 8;   // one group's weight block (floats): 8 edges x 8 heads + 8 pad

struct W8Smem {
    // odd tiles' feature rows: [warp][edge i][group g][16 chunks of 16 B], chunk c of the
    // 256-B row stored at c ^ (c >> 3 & 1) -- each cp.async instruction copies 128 contiguous
    // bytes of a row per group (whole L2 sectors), each 16-B read of the consume hits every
    // bank quad exactly four times (no conflicts)
    float4 x[kWarps][kWPer][kWG][16];
    // weight rows of tiles t .. t+3 (ring, filled by cp.async three tiles ahead): edge L of a
    // tile at group L % 4, slot L / 4 (group blocks padded by 8 floats)
    float w[4][kWarps][kWG * kWRow];
    int col[2][kWarps][32];            // column ids of the tile whose gathers are being issued
    float cmp[kWarps][8][32];          // Kahan compensation, lane-minor
};

__device__ __forceinline__ void cp_async16_hint(void *sdst, const void *gsrc, int src_size, uint64_t pol) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(sa), "l"(gsrc),
                 "r"(src_size), "l"(pol)
                 : "memory");
}

template <bool REV>
__global__ void __launch_bounds__(kThreads, 2) wspmm8_kernel(const SpmmArgs a) {
    extern __shared__ __align__(16) unsigned char w8_smem_raw[];
    W8Smem &S = *reinterpret_cast<W8Smem *>(w8_smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 3, h = lane & 7;

    int64_t row, b, e;
    bool heavy;
    if (!warp_task(a.task, a.nrows, a.n_heavy, warp, row, b, e, heavy)) return;
    const Pol pol = make_pol();
    const char *xl = reinterpret_cast<const char *>(a.X + h * 8);   // this lane's head slice
    const char *xc = reinterpret_cast<const char *>(a.X) + h * 16;  // this lane's copy chunks
    const uint32_t ldxb = (uint32_t)(a.ldx * 4);
    const int ntiles = (int)((e - b + 31) >> 5);
    const int nfull = (int)((e - b) >> 5);   // tiles [0, nfull) hold 32 edges

    // (column id, edge id) of this lane's edge (tile edge `lane`) of tile t
    auto load_idx = [&](int t, int &c, int &ev) {
        c = 0;
        ev = 0;
        const int64_t j = b + (int64_t)t * 32 + lane;
        if (j < e) {
            c = ld_stream_i32(a.col + j, pol.stream);
            ev = REV ? ld_stream_i32(a.eid + j, pol.stream) : (int)j;
        }
    };
    // weight rows of tile t into ring slot t & 3: two lanes per 32-B row (halves), rows
    // 16 k + (lane >> 1); `ev` = the edge id register of tile t (lane r holds edge r's)
    auto issue_w = [&](int t, int ev) {
        const int p = lane & 1;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int r = 16 * k + (lane >> 1);
            const int er = __shfl_sync(kFull, ev, r);
            const bool ok = b + (int64_t)t * 32 + r < e;
            float *dst = &S.w[t & 3][warp][(r & 3) * kWRow + (r >> 2) * 8 + p * 4];
            cp_async16_hint(dst, a.w + (int64_t)(ok ? er : 0) * 8 + p * 4, ok ? 16 : 0, pol.stream);
        }
    };
    // stage the column ids of tile t (this lane holds edge `lane`, i.e. group lane % 4, slot lane / 4)
    auto stage_col = [&](int t, int c) { S.col[t & 1][warp][(lane & 3) * kWPer + (lane >> 2)] = c; };
    // number of valid edges of this lane's group in tile t (edge g + 4 i)
    auto group_count = [&](int t) {
        const int64_t n = e - (b + (int64_t)t * 32);
        return n >= 32 ? kWPer : (n > g ? (int)((n - g + kWG - 1) / kWG) : 0);
    };
    auto tile_cols = [&](int t, int *cc) {
        const int4 c0 = *reinterpret_cast<const int4 *>(&S.col[t & 1][warp][g * kWPer]);
        const int4 c1 = *reinterpret_cast<const int4 *>(&S.col[t & 1][warp][g * kWPer + 4]);
        cc[0] = c0.x; cc[1] = c0.y; cc[2] = c0.z; cc[3] = c0.w;
        cc[4] = c1.x; cc[5] = c1.y; cc[6] = c1.z; cc[7] = c1.w;
    };

    Vec<8> xr[kWPer];   // even tiles' gathers
    auto issue_reg = [&](int t) {
        int cc[8];
        tile_cols(t, cc);
        if (t < nfull) {
#pragma unroll
            for (int i = 0; i < kWPer; i++)
                ld_keep(xr[i], reinterpret_cast<const float *>(xl + (uint64_t)(uint32_t)cc[i] * ldxb), pol.keep);
        } else {
            const int m = group_count(t);
#pragma unroll
            for (int i = 0; i < kWPer; i++) {
                if (i < m) ld_keep(xr[i], reinterpret_cast<const float *>(xl + (uint64_t)(uint32_t)cc[i] * ldxb), pol.keep);
                else vzero(xr[i]);
            }
        }
    };
    auto issue_smem = [&](int t) {
        int cc[8];
        tile_cols(t, cc);
        const int m = group_count(t);
#pragma unroll
        for (int i = 0; i < kWPer; i++) {
            // this lane copies chunks h and 8 + h of the row (whole-sector requests per group)
            const char *src = xc + (uint64_t)(uint32_t)(i < m ? cc[i] : 0) * ldxb;
            float4 *dst = &S.x[warp][i][g][0];
            cp_async16_hint(dst + h, src, i < m ? 16 : 0, pol.keep);
            cp_async16_hint(dst + ((8 + h) ^ 1), src + 128, i < m ? 16 : 0, pol.keep);
        }
    };

    Vec<8> acc, tile;
    vzero(acc);
    vzero(tile);
#pragma unroll
    for (int k = 0; k < 8; k++) S.cmp[warp][k][lane] = 0.f;
    int nfold = 0;
    auto fold = [&]() {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const float y = tile.v[k] - S.cmp[warp][k][lane];
            const float sum = acc.v[k] + y;
            S.cmp[warp][k][lane] = (sum - acc.v[k]) - y;
            acc.v[k] = sum;
            tile.v[k] = 0.f;
        }
    };
    auto edge = [&](int t, int i, auto from_smem) {
        constexpr bool SM = decltype(from_smem)::value;
        const float wt = S.w[t & 3][warp][g * kWRow + i * 8 + h];
        Vec<8> x;
        if constexpr (SM) {
            const float4 *rw = &S.x[warp][i][g][0];
            const int c = 2 * h, sw = (c >> 3) & 1;   // the lane's chunks 2h, 2h + 1 at c ^ (c >> 3 & 1)
            const float4 lo = rw[c ^ sw], hi = rw[(c + 1) ^ sw];
            x.v[0] = lo.x; x.v[1] = lo.y; x.v[2] = lo.z; x.v[3] = lo.w;
            x.v[4] = hi.x; x.v[5] = hi.y; x.v[6] = hi.z; x.v[7] = hi.w;
        } else {
            x = xr[i];
        }
#pragma unroll
        for (int k = 0; k < 8; k += 2) fma2(tile.v[k], tile.v[k + 1], wt, wt, x.v[k], x.v[k + 1]);
    };
    auto consume = [&](int t, auto from_smem) {
        if (t < nfull) {
#pragma unroll
            for (int i = 0; i < kWPer; i++) edge(t, i, from_smem);
        } else {
            const int m = group_count(t);
#pragma unroll
            for (int i = 0; i < kWPer; i++)
                if (i < m) edge(t, i, from_smem);
        }
        if (++nfold == kFoldTiles || t + 1 == ntiles) {
            nfold = 0;
            fold();
        }
    };

    // ---- prologue.  cp.async groups: P0 = {w(0)}, P1 = {w(1), w(2), x(1)}, then one group per
    // iteration t = {w(t+3), x(t+2) if t+2 is odd}; at iteration t everything but the newest
    // group is complete after wait_group 1 -- which covers w(t) and (odd t) x(t).
    // Index queue: (column id, edge id) of tile u in slot u % 4, loaded 4 tiles ahead; the loop
    // is unrolled by 4 so every slot is a fixed register (a rotating queue would MOV registers
    // whose loads are still in flight and stall on them every tile).
    int qc[4], qe[4];
#pragma unroll
    for (int k = 0; k < 4; k++) load_idx(k, qc[k], qe[k]);
    stage_col(0, qc[0]);
    stage_col(1, qc[1]);
    __syncwarp();
    if (ntiles > 0) issue_w(0, qe[0]);
    cp_async_commit();
    if (ntiles > 1) issue_w(1, qe[1]);
    if (ntiles > 2) issue_w(2, qe[2]);
    if (ntiles > 1) issue_smem(1);
    cp_async_commit();
    if (ntiles > 0) issue_reg(0);

    auto step = [&](int t, auto kk) {
        constexpr int K = decltype(kk)::value;   // t % 4
        cp_async_wait<1>();
        __syncwarp();
        consume(t, std::integral_constant<bool, (K & 1) == 1>{});
        __syncwarp();   // done with S.x, S.col[t & 1] and ring slot t & 3 of tile t
        if (t + 3 < ntiles) issue_w(t + 3, qe[(K + 3) & 3]);
        if (t + 2 < ntiles) {
            stage_col(t + 2, qc[(K + 2) & 3]);
            __syncwarp();
            if constexpr ((K & 1) == 0) issue_reg(t + 2);
            else issue_smem(t + 2);
        }
        cp_async_commit();
        load_idx(t + 4, qc[K], qe[K]);   // slot K held tile t: no longer needed
    };
#pragma unroll 1
    for (int t = 0; t < ntiles; t += 4) {
        step(t, std::integral_constant<int, 0>{});
        if (t + 1 >= ntiles) break;
        step(t + 1, std::integral_constant<int, 1>{});
        if (t + 2 >= ntiles) break;
        step(t + 2, std::integral_constant<int, 2>{});
        if (t + 3 >= ntiles) break;
        step(t + 3, std::integral_constant<int, 3>{});
    }
    cp_async_wait<0>();

    // compensated totals, then the 4 edge groups (xor over lanes 8, 16)
#pragma unroll
    for (int k = 0; k < 8; k++) {
        float v = acc.v[k] - S.cmp[warp][k][lane];
        v += __shfl_xor_sync(kFull, v, 8);
        v += __shfl_xor_sync(kFull, v, 16);
        acc.v[k] = v;
    }
    if (!heavy) {
        if (g == 0) vstore(a.out + row * a.ldo + h * 8, acc, 8);
        return;
    }
    // heavy row: deterministic cross-warp combine in warp order (reuses the weight ring)
    __syncthreads();
    float *red = &S.w[0][0][0];
    if (g == 0) {
#pragma unroll
        for (int k = 0; k < 8; k++) red[warp * 64 + h * 8 + k] = acc.v[k];
    }
    __syncthreads();
    if (threadIdx.x < 64) {
        float v = 0.f;
        for (int w = 0; w < kWarps; w++) v += red[w * 64 + threadIdx.x];
        a.out[row * a.ldo + threadIdx.x] = v;
    }
}

}  // namespace

static int wspmm8_mode() {   // GSP_WSPMM8=0 disables the two-tile kernel (A/B against spmm_kernel)
    static const int v = [] {
        const char *e = getenv("GSP_WSPMM8");
        return e ? atoi(e) : 1;
    }();
    return v;
}

bool wspmm8_supported(const SpmmArgs &a, int mode) {
    return wspmm8_mode() != 0 && (mode == kSpmmWeightedFwd || mode == kSpmmWeightedRev) && a.H == 8 &&
           a.Fh == 8 && a.F == 64 && a.ldx % 8 == 0 && aligned(a.X, 32) && a.ldw == 8 && aligned(a.w, 32) &&
           a.ldo % 4 == 0 && aligned(a.out, 16);
}

cudaError_t launch_wspmm8(const SpmmArgs &a, int mode, cudaStream_t s) {
    const dim3 grid = row_grid(a.nrows, a.n_heavy, 1);
    static const size_t pad = [] {   // GSP_W8_SMEM_KB: request this much (forces lower occupancy; A/B)
        const char *e = getenv("GSP_W8_SMEM_KB");
        return e ? (size_t)atoi(e) << 10 : (size_t)0;
    }();
    const size_t dyn = pad > sizeof(W8Smem) ? pad : sizeof(W8Smem);
    static std::atomic<int> attr_done[2][64];   // per (kernel, device): idempotent opt-in
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int k = mode == kSpmmWeightedRev ? 1 : 0;
    if (dev >= 64 || !attr_done[k][dev].load(std::memory_order_acquire)) {
        e = k ? cudaFuncSetAttribute(wspmm8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn)
              : cudaFuncSetAttribute(wspmm8_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
        if (dev < 64) attr_done[k][dev].store(1, std::memory_order_release);
    }
    if (k) wspmm8_kernel<true><<<grid, kThreads, dyn, s>>>(a);
    else wspmm8_kernel<false><<<grid, kThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

}  // namespace gsp
