/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU reference for the GraphPy sparse hot path
 * (arxiv 2402.03548).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code with the CUDA path (paper_2402_03548_b200/) and never reads anything the
 * CUDA path produced.
 *
 * Every float result is accumulated in fp64 from the fp32 inputs (exact in
 * fp64); alongside each value the oracle returns T = sum of |terms| so the
 * tests can apply the acceptance bound |gpu - oracle| <= 1e-5 (T + 1)
 * (BASELINE.json north_star).  The method is exact (it reaches the plain
 * definitions), so each function is the definition written out; there is no
 * blocking, fusion or reordering.
 *
 * Notation (SURVEY.md §8 / DESIGN.md): an input edge i is (src[i] -> dst[i]),
 * i.e. A[dst][src] = 1.  The "fwd" structure groups edges by destination
 * (CSR rows, §Background), the "rev" structure groups them by
 * source (CSC / transpose, P:1318, P:1497-1498 SYS-P2).
 *
 * Pins: tests/test_oracle.py (hand examples SPEC S:80-82, S:152-155, S:196-198;
 * closed form D^-1/2 A D^-1/2 X on dense adjacency; brute-force dense
 * products on <=64 vertices; adjoint / bilinear identities; softmax
 * characterisation).  Parity pinned for every function below.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { OR_NORM_NONE = 0, OR_NORM_RIGHT = 1, OR_NORM_BOTH = 2 };

/* ------------------------------------------------------------------ C1 --- */
/* Graph build, §Storage Format ("COO ... arranged in CSR-style",
 * "CSR and COO ... allocated consecutive edge IDs", "CSC requires an explicit
 * edge ID array") and DESIGN.md readings L5/L6/L7:
 *   order  = positions i sorted by (dst[i], src[i], i)       (ties: input order)
 *   fwd_off[v] = #{i : dst[i] < v};  fwd_col[j] = src[order[j]];
 *   coo_to_eid[order[j]] = j          (the edge ID of fwd slot j is j)
 *   rorder = slots j sorted by (src_j, dst_j, j)
 *   rev_off[u] = #{j : src_j < u};  rev_col[k] = dst_{rorder[k]};  rev_eid[k] = rorder[k]
 */
typedef struct { int64_t k1, k2, idx; } key3;

static int cmp_key3(const void *a, const void *b) {
    const key3 *x = (const key3 *)a, *y = (const key3 *)b;
    if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
    if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
    if (x->idx != y->idx) return x->idx < y->idx ? -1 : 1;
    return 0;
}

/* returns 0 ok, -1 bad vertex id, -2 out of memory */
int oracle_build(int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                 int64_t *fwd_off, int32_t *fwd_col, int64_t *rev_off, int32_t *rev_col,
                 int32_t *rev_eid, int32_t *coo_to_eid) {
    for (int64_t i = 0; i < E; i++)
        if (src[i] < 0 || src[i] >= V || dst[i] < 0 || dst[i] >= V) return -1;
    key3 *a = (key3 *)malloc(sizeof(key3) * (size_t)(E > 0 ? E : 1));
    int64_t *cnt = (int64_t *)calloc((size_t)V + 1, sizeof(int64_t));
    if (!a || !cnt) { free(a); free(cnt); return -2; }

    /* fwd: sort positions by (dst, src, position) */
    for (int64_t i = 0; i < E; i++) { a[i].k1 = dst[i]; a[i].k2 = src[i]; a[i].idx = i; }
    qsort(a, (size_t)E, sizeof(key3), cmp_key3);
    for (int64_t i = 0; i < E; i++) cnt[dst[i] + 1]++;         /* fwd_off[v] = #{i: dst[i] < v} */
    fwd_off[0] = 0;
    for (int64_t v = 0; v < V; v++) fwd_off[v + 1] = fwd_off[v] + cnt[v + 1];
    for (int64_t j = 0; j < E; j++) {
        fwd_col[j] = (int32_t)src[a[j].idx];
        coo_to_eid[a[j].idx] = (int32_t)j;
    }
    /* rev: sort fwd slots j by (src_j, dst_j, j); dst_j = dst[order[j]] */
    for (int64_t j = 0; j < E; j++) { a[j].k1 = src[a[j].idx]; a[j].k2 = dst[a[j].idx]; a[j].idx = j; }
    qsort(a, (size_t)E, sizeof(key3), cmp_key3);
    memset(cnt, 0, sizeof(int64_t) * ((size_t)V + 1));
    for (int64_t i = 0; i < E; i++) cnt[src[i] + 1]++;         /* rev_off[u] = #{j: src_j < u} */
    rev_off[0] = 0;
    for (int64_t u = 0; u < V; u++) rev_off[u + 1] = rev_off[u] + cnt[u + 1];
    for (int64_t k = 0; k < E; k++) {
        rev_col[k] = (int32_t)a[k].k2;
        rev_eid[k] = (int32_t)a[k].idx;
    }
    free(a); free(cnt);
    return 0;
}

/* ---------------------------------------------------------------- C2/C3 --- */
/* Degrees with the clamp d^ = max(d,1) (§Requirement Mismatch, "sets
 * the degree to 1.0").  d_in(v) = fwd row length, d_out(u) = rev
 * row length (L2).  Scales per DESIGN.md L1 / SURVEY §8(c) C3:
 *   NONE : s_dst = 1,              s_src = 1
 *   RIGHT: s_dst = 1/d^_in(v),     s_src = 1          (D_in^-1 A)
 *   BOTH : s_dst = d^_in(v)^-1/2,  s_src = d^_out(u)^-1/2   (D^-1/2 A D^-1/2, BJ) */
static double clamp_deg(int64_t d) { return d < 1 ? 1.0 : (double)d; }
static double s_dst(int norm, const int64_t *fwd_off, int64_t v) {
    double d = clamp_deg(fwd_off[v + 1] - fwd_off[v]);
    if (norm == OR_NORM_RIGHT) return 1.0 / d;
    if (norm == OR_NORM_BOTH) return 1.0 / sqrt(d);
    return 1.0;
}
static double s_src(int norm, const int64_t *rev_off, int64_t u) {
    double d = clamp_deg(rev_off[u + 1] - rev_off[u]);
    if (norm == OR_NORM_BOTH) return 1.0 / sqrt(d);
    return 1.0;
}

/* Degree scales as arrays (tests check C2/C3 against the SPEC degrees). */
void oracle_scales(int64_t V, const int64_t *fwd_off, const int64_t *rev_off, int norm,
                   double *sdst, double *ssrc) {
    for (int64_t v = 0; v < V; v++) {
        sdst[v] = s_dst(norm, fwd_off, v);
        ssrc[v] = s_src(norm, rev_off, v);
    }
}

/* ------------------------------------------------------------------ C4 --- */
/* gSpMMv with fused degree normalisation (Table 1; P:607-612;
 * P:2024-2027 §Kernel Design "gSpMMv^T"; P:1333-1335 Class B):
 *   fwd: out[v,f] = s_dst(v) * sum_{j in fwd row v} s_src(fwd_col[j]) * X[fwd_col[j], f]
 *   rev: out[u,f] = s_src(u) * sum_{k in rev row u} s_dst(rev_col[k]) * X[rev_col[k], f]
 * (rev is the exact adjoint of fwd; "Backward Computation",
 *  P:1536-1540 SYS-P3: the column-side scale is applied per non-zero).
 * T[v,f] = row scale * sum |col scale * X|.
 * sel: NULL -> all V rows (out has V rows); else the nsel listed rows in order. */
int oracle_gspmm(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col,
                 const int64_t *rev_off, const int32_t *rev_col,
                 const float *X, int64_t F, int64_t ldx, int norm, int reverse,
                 int64_t nsel, const int64_t *sel, double *out, double *T) {
    int64_t n = sel ? nsel : V;
    for (int64_t r = 0; r < n; r++) {
        int64_t v = sel ? sel[r] : r;
        if (v < 0 || v >= V) return -1;
        const int64_t *off = reverse ? rev_off : fwd_off;
        const int32_t *col = reverse ? rev_col : fwd_col;
        double rs = reverse ? s_src(norm, rev_off, v) : s_dst(norm, fwd_off, v);
        for (int64_t f = 0; f < F; f++) {
            double acc = 0.0, tacc = 0.0;
            for (int64_t j = off[v]; j < off[v + 1]; j++) {
                int64_t u = col[j];
                double cs = reverse ? s_dst(norm, fwd_off, u) : s_src(norm, rev_off, u);
                double term = cs * (double)X[u * ldx + f];
                acc += term;
                tacc += fabs(term);
            }
            out[r * F + f] = rs * acc;
            if (T) T[r * F + f] = rs * tacc;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ C5 --- */
/* Weighted gSpMM, multi-head (gSpMMve P:1329, "vector feature for
 * each edge"; its transpose gSpMMve^T fetches the edge value through the edge
 * ID, §Kernel Design, P:564 gSpMMveid).  Head layout (DESIGN.md
 * L10): vertex tensors [V, H*Fh], head h = columns [h*Fh, (h+1)*Fh); edge
 * tensor w [E, H] indexed by edge ID.
 *   fwd: out[v, h*Fh+f] = sum_{j in fwd row v} w[j, h] * X[fwd_col[j], h*Fh+f]
 *   rev: out[u, h*Fh+f] = sum_{k in rev row u} w[rev_eid[k], h] * X[rev_col[k], h*Fh+f]
 * T = sum |w * X|. */
int oracle_gspmm_weighted(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col,
                          const int64_t *rev_off, const int32_t *rev_col, const int32_t *rev_eid,
                          const float *X, int64_t F, int64_t ldx, const float *w, int64_t H,
                          int reverse, int64_t nsel, const int64_t *sel, double *out, double *T) {
    if (H <= 0 || F % H != 0) return -2;
    int64_t Fh = F / H, n = sel ? nsel : V;
    for (int64_t r = 0; r < n; r++) {
        int64_t v = sel ? sel[r] : r;
        if (v < 0 || v >= V) return -1;
        for (int64_t c = 0; c < F; c++) {
            int64_t h = c / Fh;
            double acc = 0.0, tacc = 0.0;
            if (!reverse) {
                for (int64_t j = fwd_off[v]; j < fwd_off[v + 1]; j++) {
                    double term = (double)w[j * H + h] * (double)X[(int64_t)fwd_col[j] * ldx + c];
                    acc += term; tacc += fabs(term);
                }
            } else {
                for (int64_t k = rev_off[v]; k < rev_off[v + 1]; k++) {
                    double term = (double)w[(int64_t)rev_eid[k] * H + h] * (double)X[(int64_t)rev_col[k] * ldx + c];
                    acc += term; tacc += fabs(term);
                }
            }
            out[r * F + c] = acc;
            if (T) T[r * F + c] = tacc;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ C6 --- */
/* gSDDMMvv (Table 1; "the vertex-level features of row ID and
 * column ID of each non-zero element ... perform dot product"):
 * X is indexed by the row (destination), Y by the column (source) (L8):
 *   out[j, h] = sum_{f < Fh} X[v, h*Fh+f] * Y[fwd_col[j], h*Fh+f]   for slot j of row v.
 * Output is indexed by edge ID (= fwd slot).  With sel, the edges of the
 * selected rows are packed row after row (each row's slots in order). */
int oracle_gsddmm(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col,
                  const float *X, int64_t ldx, const float *Y, int64_t ldy, int64_t F, int64_t H,
                  int64_t nsel, const int64_t *sel, double *out, double *T) {
    if (H <= 0 || F % H != 0) return -2;
    int64_t Fh = F / H, n = sel ? nsel : V, o = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t v = sel ? sel[r] : r;
        if (v < 0 || v >= V) return -1;
        for (int64_t j = fwd_off[v]; j < fwd_off[v + 1]; j++, o++) {
            int64_t u = fwd_col[j];
            for (int64_t h = 0; h < H; h++) {
                double acc = 0.0, tacc = 0.0;
                for (int64_t f = 0; f < Fh; f++) {
                    double term = (double)X[v * ldx + h * Fh + f] * (double)Y[u * ldy + h * Fh + f];
                    acc += term; tacc += fabs(term);
                }
                out[o * H + h] = acc;
                if (T) T[o * H + h] = tacc;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ C7 --- */
/* Edge softmax grouped by destination (fwd row) -- part of GAT's layer
 * (P:197), composite defined in SPEC S:217-225 and DESIGN.md L9:
 *   m = max_j e[j,h];  S = sum_j exp(e[j,h] - m);  out[j,h] = exp(e[j,h] - m) / S
 * over the slots j of row v.  Empty rows produce nothing. */
int oracle_edge_softmax(int64_t V, const int64_t *fwd_off, const float *e, int64_t H,
                        int64_t nsel, const int64_t *sel, double *out) {
    int64_t n = sel ? nsel : V, o = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t v = sel ? sel[r] : r;
        if (v < 0 || v >= V) return -1;
        int64_t b = fwd_off[v], en = fwd_off[v + 1];
        for (int64_t h = 0; h < H; h++) {
            double m = -INFINITY;
            for (int64_t j = b; j < en; j++) if ((double)e[j * H + h] > m) m = (double)e[j * H + h];
            double S = 0.0;
            for (int64_t j = b; j < en; j++) S += exp((double)e[j * H + h] - m);
            for (int64_t j = b; j < en; j++) out[(o + (j - b)) * H + h] = exp((double)e[j * H + h] - m) / S;
        }
        o += en - b;
    }
    return 0;
}

/* ------------------------------------------------------------------ C9 --- */
/* Edge-softmax backward (GAT backward chain; the chain
 * rule through C7 -- P:1340-1341 "Backward Computation"):
 *   ds[j,h] = alpha[j,h] * (dalpha[j,h] - sum_{j' in row v} alpha[j',h] * dalpha[j',h])
 * T[j,h] = |alpha dalpha| + alpha * sum |alpha dalpha|.  Packed like C6/C7 with sel. */
int oracle_edge_softmax_backward(int64_t V, const int64_t *fwd_off, const float *alpha, const float *dalpha,
                                 int64_t H, int64_t nsel, const int64_t *sel, double *out, double *T) {
    int64_t n = sel ? nsel : V, o = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t v = sel ? sel[r] : r;
        if (v < 0 || v >= V) return -1;
        int64_t b = fwd_off[v], en = fwd_off[v + 1];
        for (int64_t h = 0; h < H; h++) {
            double d = 0.0, dabs = 0.0;
            for (int64_t j = b; j < en; j++) {
                double t = (double)alpha[j * H + h] * (double)dalpha[j * H + h];
                d += t;
                dabs += fabs(t);
            }
            for (int64_t j = b; j < en; j++) {
                double a = (double)alpha[j * H + h], g = (double)dalpha[j * H + h];
                out[(o + (j - b)) * H + h] = a * (g - d);
                if (T) T[(o + (j - b)) * H + h] = fabs(a * g) + fabs(a) * dabs;
            }
        }
        o += en - b;
    }
    return 0;
}

/* ----------------------------------------------------------------- C10 --- */
/* GAT forward as one definition (P:1329 Class A):
 * for each destination row v and head h, over the slots j of row v (u = col_j):
 *   s_j   = sum_{f < Fh} X[v, h*Fh+f] * Y[u, h*Fh+f]                      (C6)
 *   a_j   = exp(s_j - max s) / sum exp(s - max s)                          (C7)
 *   out[v, h*Fv+f] = sum_j a_j * Vt[u, h*Fv+f]                             (C5)
 * all in fp64 (no fp32 hand-off between the steps).  alpha is written by
 * edge ID; T_out = sum_j a_j |Vt|.  The scratch s (size = max degree) is the
 * caller's. */
int oracle_gat_forward(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col, const float *X, int64_t ldx,
                       const float *Y, int64_t ldy, int64_t F, const float *Vt, int64_t ldv, int64_t Fv, int64_t H,
                       double *alpha, double *out, double *Tout, double *scratch) {
    if (H <= 0 || F % H != 0 || Fv % H != 0) return -2;
    int64_t Fh = F / H, Fvh = Fv / H;
    for (int64_t v = 0; v < V; v++) {
        int64_t b = fwd_off[v], e = fwd_off[v + 1];
        for (int64_t h = 0; h < H; h++) {
            double m = -INFINITY;
            for (int64_t j = b; j < e; j++) {
                int64_t u = fwd_col[j];
                double sc = 0.0;
                for (int64_t f = 0; f < Fh; f++) sc += (double)X[v * ldx + h * Fh + f] * (double)Y[u * ldy + h * Fh + f];
                scratch[j - b] = sc;
                if (sc > m) m = sc;
            }
            double S = 0.0;
            for (int64_t j = b; j < e; j++) S += exp(scratch[j - b] - m);
            for (int64_t j = b; j < e; j++) alpha[j * H + h] = exp(scratch[j - b] - m) / S;
            for (int64_t f = 0; f < Fvh; f++) {
                double acc = 0.0, tacc = 0.0;
                for (int64_t j = b; j < e; j++) {
                    double t = alpha[j * H + h] * (double)Vt[(int64_t)fwd_col[j] * ldv + h * Fvh + f];
                    acc += t;
                    tacc += fabs(t);
                }
                out[v * Fv + h * Fvh + f] = acc;
                if (Tout) Tout[v * Fv + h * Fvh + f] = tacc;
            }
        }
    }
    return 0;
}

/* ----------------------------------------------------------- C11-C13 --- */
/* Table 1's remaining API surface:
 * reductions sum / min / max ("various reduction operations (e.g. sum,
 * min, max"), empty rows -> 0 (SPEC S:237 design decision). */
enum { OR_RED_SUM = 0, OR_RED_MIN = 1, OR_RED_MAX = 2 };
static double red_init(int r) { return r == OR_RED_MIN ? INFINITY : (r == OR_RED_MAX ? -INFINITY : 0.0); }
static double red_apply(int r, double acc, double x) {
    if (r == OR_RED_MIN) return x < acc ? x : acc;
    if (r == OR_RED_MAX) return x > acc ? x : acc;
    return acc + x;
}

/* C11 gSpMMv with a reduction ("gSpMMv(g, in, out, eFn, Flag)"
 * "reduction operation type, such as sum, min, max"), no normalisation:
 *   fwd: out[v,f] = RED_{j in fwd row v} X[fwd_col[j], f];  rev: over rev row u of X[rev_col[k], f]. */
int oracle_gspmm_reduce(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col, const int64_t *rev_off,
                        const int32_t *rev_col, const float *X, int64_t F, int64_t ldx, int red, int reverse,
                        double *out, double *T) {
    const int64_t *off = reverse ? rev_off : fwd_off;
    const int32_t *col = reverse ? rev_col : fwd_col;
    for (int64_t v = 0; v < V; v++)
        for (int64_t f = 0; f < F; f++) {
            double acc = red_init(red), tacc = 0.0;
            for (int64_t j = off[v]; j < off[v + 1]; j++) {
                double x = (double)X[(int64_t)col[j] * ldx + f];
                acc = red_apply(red, acc, x);
                tacc += fabs(x);
            }
            out[v * F + f] = off[v] == off[v + 1] ? 0.0 : acc;
            if (T) T[v * F + f] = red == OR_RED_SUM ? tacc : 0.0;   /* min / max are exact */
        }
    return 0;
}

/* C12 gSpMMe / gSpMMeid ("gSpMMeid(g, in, out, eFn, Flag)"): an
 * edge-level tensor reduced per row, fetched through the edge ID:
 *   fwd: out[v,h] = RED_{j in fwd row v} w[j, h];  rev: out[u,h] = RED_{k in rev row u} w[rev_eid[k], h]. */
int oracle_gspmm_e(int64_t V, const int64_t *fwd_off, const int64_t *rev_off, const int32_t *rev_eid,
                   const float *w, int64_t H, int red, int reverse, double *out, double *T) {
    for (int64_t v = 0; v < V; v++)
        for (int64_t h = 0; h < H; h++) {
            double acc = red_init(red), tacc = 0.0;
            int64_t b = reverse ? rev_off[v] : fwd_off[v], e = reverse ? rev_off[v + 1] : fwd_off[v + 1];
            for (int64_t k = b; k < e; k++) {
                int64_t eid = reverse ? rev_eid[k] : k;
                double x = (double)w[eid * H + h];
                acc = red_apply(red, acc, x);
                tacc += fabs(x);
            }
            out[v * H + h] = b == e ? 0.0 : acc;
            if (T) T[v * H + h] = red == OR_RED_SUM ? tacc : 0.0;
        }
    return 0;
}

/* C13 gSDDMMve ("gSDDMMve(g, in, in, out, eFn, Flag)"
 * "vertex-level and edge-level tensors are accessed using the graph"; SPEC
 * S:199-207): for slot j of fwd row v with column u,
 *   out[j,h] = w[j,h] OP X[side ? u : v, h],  OP in {add, sub, mul, div}. */
enum { OR_OP_ADD = 0, OR_OP_SUB = 1, OR_OP_MUL = 2, OR_OP_DIV = 3 };
int oracle_gsddmm_ve(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col, const float *X, const float *w,
                     int64_t H, int op, int side_src, double *out) {
    for (int64_t v = 0; v < V; v++)
        for (int64_t j = fwd_off[v]; j < fwd_off[v + 1]; j++) {
            int64_t vx = side_src ? fwd_col[j] : v;
            for (int64_t h = 0; h < H; h++) {
                double a = (double)w[j * H + h], x = (double)X[vx * H + h], r;
                if (op == OR_OP_ADD) r = a + x;
                else if (op == OR_OP_SUB) r = a - x;
                else if (op == OR_OP_MUL) r = a * x;
                else r = a / x;
                out[j * H + h] = r;
            }
        }
    return 0;
}

/* ----------------------------------------------------- C4/C1 from COO --- */
/* The same definitions evaluated straight from the COO list for a few
 * selected rows (billion-edge graphs, where sorting the whole edge list in the
 * oracle is impractical).  Degrees by counting; every COO edge whose
 * destination (reverse: source) is a selected row contributes once:
 *   fwd: out[r,f] = s_dst(v) * sum_{i: dst[i]=v} s_src(src[i]) X[src[i], f]   (C4)
 * and the row's fwd slots are its COO edges sorted by (src, position) (C1). */
int oracle_gspmm_rows_coo(int64_t V, int64_t E, const int64_t *src, const int64_t *dst, const float *X, int64_t F,
                          int64_t ldx, int norm, int reverse, int64_t nsel, const int64_t *sel, double *out,
                          double *T) {
    int64_t *din = (int64_t *)calloc((size_t)V, sizeof(int64_t)), *dout = (int64_t *)calloc((size_t)V, sizeof(int64_t));
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    if (!din || !dout || !slot) { free(din); free(dout); free(slot); return -2; }
    for (int64_t i = 0; i < E; i++) { din[dst[i]]++; dout[src[i]]++; }
    for (int64_t v = 0; v < V; v++) slot[v] = -1;
    for (int64_t r = 0; r < nsel; r++) slot[sel[r]] = (int32_t)r;
    for (int64_t r = 0; r < nsel * F; r++) { out[r] = 0.0; if (T) T[r] = 0.0; }
    for (int64_t i = 0; i < E; i++) {
        int64_t row = reverse ? src[i] : dst[i], c = reverse ? dst[i] : src[i];
        int32_t r = slot[row];
        if (r < 0) continue;
        /* column-side scale: fwd -> s_src(c) from d_out; rev -> s_dst(c) from d_in */
        double dc = (double)(reverse ? din[c] : dout[c]);
        if (dc < 1.0) dc = 1.0;
        double cs = 1.0;
        if (norm == OR_NORM_BOTH) cs = 1.0 / sqrt(dc);
        else if (norm == OR_NORM_RIGHT && reverse) cs = 1.0 / dc;
        for (int64_t f = 0; f < F; f++) {
            double t = cs * (double)X[c * ldx + f];
            out[r * F + f] += t;
            if (T) T[r * F + f] += fabs(t);
        }
    }
    for (int64_t r = 0; r < nsel; r++) {
        int64_t v = sel[r];
        double dr = (double)(reverse ? dout[v] : din[v]);
        if (dr < 1.0) dr = 1.0;
        double rs = 1.0;
        if (norm == OR_NORM_BOTH) rs = 1.0 / sqrt(dr);
        else if (norm == OR_NORM_RIGHT && !reverse) rs = 1.0 / dr;
        for (int64_t f = 0; f < F; f++) { out[r * F + f] *= rs; if (T) T[r * F + f] *= rs; }
    }
    free(din); free(dout); free(slot);
    return 0;
}

/* For each selected destination row, its in-edges from the COO list as
 * (src, position) pairs sorted by (src, position) = the row's fwd slots (C1),
 * plus fwd_off[v] = #{i : dst[i] < v}.  pairs has room for the rows' degrees. */
static int cmp_pair(const void *a, const void *b) {
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}
int oracle_rows_coo(int64_t V, int64_t E, const int64_t *dst_, const int64_t *src_, int64_t nsel, const int64_t *sel,
                    int64_t *row_off /* nsel+1, prefix of degrees */, int64_t *first_slot /* nsel */,
                    int64_t *pairs /* 2 * sum deg */) {
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * (size_t)V);
    int64_t *cnt = (int64_t *)calloc((size_t)nsel, sizeof(int64_t));
    int64_t *hist = (int64_t *)calloc((size_t)V + 1, sizeof(int64_t));
    if (!slot || !cnt || !hist) { free(slot); free(cnt); free(hist); return -2; }
    for (int64_t v = 0; v < V; v++) slot[v] = -1;
    for (int64_t r = 0; r < nsel; r++) slot[sel[r]] = (int32_t)r;
    for (int64_t i = 0; i < E; i++) {
        hist[dst_[i] + 1]++;                      /* fwd_off[v] = #{i : dst[i] < v} */
        int32_t r = slot[dst_[i]];
        if (r >= 0) cnt[r]++;
    }
    for (int64_t v = 0; v < V; v++) hist[v + 1] += hist[v];
    for (int64_t r = 0; r < nsel; r++) first_slot[r] = hist[sel[r]];
    free(hist);
    row_off[0] = 0;
    for (int64_t r = 0; r < nsel; r++) row_off[r + 1] = row_off[r] + cnt[r];
    for (int64_t r = 0; r < nsel; r++) cnt[r] = 0;
    for (int64_t i = 0; i < E; i++) {
        int32_t r = slot[dst_[i]];
        if (r < 0) continue;
        int64_t k = row_off[r] + cnt[r]++;
        pairs[2 * k] = src_[i];
        pairs[2 * k + 1] = i;
    }
    for (int64_t r = 0; r < nsel; r++)
        qsort(pairs + 2 * row_off[r], (size_t)(row_off[r + 1] - row_off[r]), 2 * sizeof(int64_t), cmp_pair);
    free(slot); free(cnt);
    return 0;
}

/* ------------------------------------------------------------------ C8 --- */
/* Edge-balanced contiguous row partition (BJ north_star
 * "destination-row partitioner"):  b_0 = 0, b_P = V,
 *   b_p = min { v : off[v] >= ceil(p * E / P) }   for 0 < p < P. */
int oracle_partition_bounds(int64_t V, const int64_t *off, int64_t nparts, int64_t *bounds) {
    if (nparts < 1) return -2;
    int64_t E = off[V];
    bounds[0] = 0;
    for (int64_t p = 1; p < nparts; p++) {
        /* ceil(p*E/P) in exact integer arithmetic */
        __int128 num = (__int128)p * E;
        int64_t target = (int64_t)((num + nparts - 1) / nparts);
        int64_t v = 0;
        while (v < V && off[v] < target) v++;
        bounds[p] = v;
    }
    bounds[nparts] = V;
    return 0;
}

/* The partition's structure in the padded rank-major layout (DESIGN.md
 * "Multi-GPU"): R = max_p (b_{p+1} - b_p); partition `part` owns rows
 * [b_part, b_part+1); local row r has the edges of global row b_part + r, in
 * the same order; every column id v is remapped to p(v)*R + (v - b_{p(v)}),
 * where p(v) is the part holding v.  Rows [nrows_local, R) are empty.
 * loc_off has R+1 entries, loc_col has off[b_{part+1}] - off[b_part]. */
int oracle_partition_structure(int64_t V, const int64_t *off, const int32_t *col,
                               int64_t nparts, const int64_t *bounds, int64_t part,
                               int64_t *loc_off, int32_t *loc_col) {
    int64_t R = 0;
    for (int64_t p = 0; p < nparts; p++)
        if (bounds[p + 1] - bounds[p] > R) R = bounds[p + 1] - bounds[p];
    int64_t b = bounds[part], e = bounds[part + 1], base = off[b];
    for (int64_t r = 0; r <= R; r++) {
        int64_t g = b + r < e ? b + r : e;
        loc_off[r] = off[g] - base;
    }
    for (int64_t j = off[b]; j < off[e]; j++) {
        int64_t v = col[j], p = 0;
        while (!(bounds[p] <= v && v < bounds[p + 1])) p++;
        loc_col[j - base] = (int32_t)(p * R + (v - bounds[p]));
    }
    return 0;
}

/* ---------------------------------------------------------- C14, C15 --- */
/* Additive (GAT) attention scores: Table 1's gSDDMM family with an add instead
 * of a dot product ("gSDDMMve ... vertex-level and
 * edge-level tensors ... to arrive at the resultant edge-level tensor", here
 * the u_add_v form of both endpoints' per-head vertex scalars), followed by the
 * leaky ReLU of the standard GAT attention ("edge logit[j,h] =
 * leaky_relu(<a_src, z[.]> + <a_dst, z[.]>, slope)", slope 0.2 at S:411):
 *   C14: out[j,h] = lrelu(el[u_j, h] + er[v, h]),  lrelu(x) = x if x > 0 else slope * x
 * for slot j of fwd row v with column (source) u_j.  el [V, lde] is the source
 * side, er [V, lde] the destination side (H columns used), both fp32; the sum
 * and the product are taken in fp64. */
int oracle_gsddmm_add_leaky(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col, const float *el,
                            const float *er, int64_t lde, int64_t H, double slope, double *out) {
    for (int64_t v = 0; v < V; v++)
        for (int64_t j = fwd_off[v]; j < fwd_off[v + 1]; j++) {
            int64_t u = fwd_col[j];
            for (int64_t h = 0; h < H; h++) {
                double x = (double)el[u * lde + h] + (double)er[v * lde + h];
                out[j * H + h] = x > 0.0 ? x : slope * x;
            }
        }
    return 0;
}

/* C15: the fused additive GAT forward (NEXT-3 + NEXT-2): alpha = C7(C14(el,
 * er)) and out[v, h*Fvh+f] = sum_j alpha[j,h] Vt[u_j, h*Fvh+f] (C5), all in
 * fp64 with no fp32 hand-off between the steps; T_out = sum_j alpha |Vt|. */
int oracle_gat_forward_additive(int64_t V, const int64_t *fwd_off, const int32_t *fwd_col, const float *el,
                                const float *er, int64_t lde, const float *Vt, int64_t ldv, int64_t Fv, int64_t H,
                                double slope, double *alpha, double *out, double *Tout, double *scratch) {
    if (H <= 0 || Fv % H != 0) return -2;
    int64_t Fvh = Fv / H;
    for (int64_t v = 0; v < V; v++) {
        int64_t b = fwd_off[v], e = fwd_off[v + 1];
        for (int64_t h = 0; h < H; h++) {
            double m = -INFINITY;
            for (int64_t j = b; j < e; j++) {
                double x = (double)el[(int64_t)fwd_col[j] * lde + h] + (double)er[v * lde + h];
                double sc = x > 0.0 ? x : slope * x;
                scratch[j - b] = sc;
                if (sc > m) m = sc;
            }
            double S = 0.0;
            for (int64_t j = b; j < e; j++) S += exp(scratch[j - b] - m);
            for (int64_t j = b; j < e; j++) alpha[j * H + h] = exp(scratch[j - b] - m) / S;
            for (int64_t f = 0; f < Fvh; f++) {
                double acc = 0.0, tacc = 0.0;
                for (int64_t j = b; j < e; j++) {
                    double t = alpha[j * H + h] * (double)Vt[(int64_t)fwd_col[j] * ldv + h * Fvh + f];
                    acc += t;
                    tacc += fabs(t);
                }
                out[v * Fv + h * Fvh + f] = acc;
                if (Tout) Tout[v * Fv + h * Fvh + f] = tacc;
            }
        }
    }
    return 0;
}
