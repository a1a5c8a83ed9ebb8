// Host-side launchers of the sm_100a kernels (spmm.cu, sddmm.cu, softmax.cu, gat.cu).  Internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace gsp {

// One pass of a gather-reduce over a structure (gSpMMv / gSpMMve / gSpMMve^T).
struct SpmmArgs {
    const int64_t *off;
    const int32_t *col;
    const int32_t *eid;      // MODE weighted-rev: explicit edge IDs; else unused
    const int32_t *order;    // degree-ordered rows
    const int32_t *task;     // per schedule slot {row, degree, first slot lo, hi} (16 B; DevStructure::task)
    int64_t nrows, n_heavy;
    const float *X;
    int64_t ldx;
    float *out;
    int64_t ldo;
    int64_t F;
    const float *row_scale;  // may be null (1.0)
    const float *col_scale;  // may be null (1.0)
    const float *edge_scale; // per-slot column scale (precomputed, streamed); overrides col_scale
    const float *w;          // weighted modes
    int64_t ldw;
    int64_t H, Fh;
    int pf;                  // L2 prefetch distance of the edge streams, in 32-edge tiles (0 = off)
    int wpol;                // L2 policy of the weight rows: 0 evict_first (streamed once), 1 evict_normal, 2 evict_last
    int light;               // mean degree < 32 (set by the caller): launch shapes that favour rows in flight
    int out_vec;             // out rows 16-B aligned (ldo % 4 == 0): vector stores, else scalar (set by launch_spmm)
    float hot_scale;         // scaled mode: column scale below which a source row is "hot" (L2 evict_last; 0 = all)
};

enum SpmmMode { kSpmmScaled = 0, kSpmmWeightedFwd = 1, kSpmmWeightedRev = 2, kSpmmMin = 3, kSpmmMax = 4 };

cudaError_t launch_spmm(const SpmmArgs &a, int mode, cudaStream_t s);

struct SddmmArgs {
    const int64_t *off;
    const int32_t *col;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy;
    int64_t row_base;        // X row of local row r is row_base + r
    const float *X;
    int64_t ldx;
    const float *Y;
    int64_t ldy;
    float *out;
    int64_t ldo;
    int64_t H, Fh;
};
cudaError_t launch_sddmm(const SddmmArgs &a, cudaStream_t s);

struct SoftmaxArgs {
    const int64_t *off;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy;
    const float *e;
    int64_t lde;
    float *out;
    int64_t ldo;
    int64_t H;
};
cudaError_t launch_softmax(const SoftmaxArgs &a, cudaStream_t s);

// Edge-softmax backward: ds = alpha * (dalpha - sum_row alpha*dalpha).
struct SoftmaxBwdArgs {
    const int64_t *off;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy;
    const float *alpha;
    int64_t lda;
    const float *dalpha;
    int64_t ldd;
    float *out;
    int64_t ldo;
    int64_t H;
};
cudaError_t launch_softmax_bwd(const SoftmaxBwdArgs &a, cudaStream_t s);

// Fused GAT forward: alpha = edge_softmax(gsddmm(X, Y)),
// out = gspmm_weighted(Vt, alpha), one pass per destination row, alpha still
// written (state tensor).  Fast path: Fh == 8, H in {2,..,32} power of two.
struct GatArgs {
    const int64_t *off;
    const int32_t *col;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy, row_base;
    const float *X;
    int64_t ldx;
    const float *Y;
    int64_t ldy;
    const float *Vt;
    int64_t ldv;
    float *alpha;      // [E, H], ld == H
    float *out;
    int64_t ldo;
    int64_t H;
    int64_t sc_cap;    // edges per warp slice whose raw scores stay in shared memory (set by the launcher)
    int light;         // mean degree < 32 (set by the caller): launch shape favouring rows in flight
    int additive;      // 0: scores <X[v], Y[u]> (Fh = 8); 1: lrelu(Y[u,h] + X[v,h], slope) (X = er, Y = el: [ncols, H])
    float slope;
};
bool gat_fused_supported(const GatArgs &a);
cudaError_t launch_gat_fused(const GatArgs &a, cudaStream_t s);
// fused GAT backward scores (NEXT-1): X = dOut (destination side), Vt, alpha (read), out = ds [E, H]
cudaError_t launch_gat_bwd(const GatArgs &a, cudaStream_t s);

// NEXT-3 (Table 1 surface): gSpMMe / gSpMMeid and gSDDMMve.
struct SpmmEArgs {
    const int64_t *off;
    const int32_t *eid;      // null: implicit (slot = edge id)
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy;  // rows in LPT order; the first n_heavy get a CTA each
    const float *w;
    int64_t ldw;
    float *out;
    int64_t ldo;
    int64_t H;
    int red;                 // 0 sum, 1 min, 2 max
};
cudaError_t launch_spmm_e(const SpmmEArgs &a, cudaStream_t s);

struct SddmmVeArgs {
    const int64_t *off;
    const int32_t *col;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy, row_base;
    const float *X;
    int64_t ldx;
    const float *w;
    int64_t ldw;
    float *out;
    int64_t ldo;
    int64_t H;
    int op;                  // 0 add, 1 sub, 2 mul, 3 div
    int side_src;            // 1: X indexed by the column (source), 0: by the row (destination)
};
cudaError_t launch_sddmm_ve(const SddmmVeArgs &a, cudaStream_t s);

// NEXT-3 additive GAT scores (oracle C14): out[j,h] = lrelu(el[col_j,h] + er[row_base+row,h], slope)
struct SddmmAddArgs {
    const int64_t *off;
    const int32_t *col;
    const int32_t *order;
    const int32_t *task;
    int64_t nrows, n_heavy, row_base;
    const float *el;         // source side [ncols, H]
    int64_t lde;
    const float *er;         // destination side [ncols, H]
    int64_t ldr;
    float *out;              // [E, H]
    int64_t ldo;
    int64_t H;
    float slope;
};
cudaError_t launch_sddmm_add(const SddmmAddArgs &a, cudaStream_t s);

// out[j] = scale[col[j]] for j < nnz (per-edge column scales, built once at create)
cudaError_t launch_gather_scale(const int32_t *col, int64_t nnz, const float *scale, float *out, cudaStream_t s);

// fp32 degree scales from (clamped) integer degrees: inv = 1/d^, rsq = d^^-1/2
// computed in fp64 then rounded once.
cudaError_t launch_degree_scales(const int64_t *deg, int64_t n, float *inv, float *rsq, cudaStream_t s);

}  // namespace gsp
