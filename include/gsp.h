/*
 * gsp.h -- C ABI of the B200-native GraphPy sparse hot path (arxiv 2402.03548).
 *
 * The calls follow the paper's system-API table (Table 1:
 * "status gSpMMv(g, in, out, eFn, Flag)", "gSpMMveid", "gSDDMMvv"; listings
 * P:733) and its graph APIs (wrap_graph, get_vcount,
 * get_ecount).  Mapping: gsp_gspmm = gSpMMv with the normalisation flag
 * generalised to `norm`, reverse = !Forward; gsp_gspmm_weighted
 * = gSpMMve (reverse=0) / gSpMMveid = gSpMMve^T through the edge ID
 * (reverse=1); gsp_gsddmm = gSDDMMvv;
 * gsp_edge_softmax = the per-destination softmax of GAT.
 *
 * Conventions (every call):
 *  - Every call returns gsp_status; nothing aborts or throws across the ABI.
 *    On error nothing is written and nothing is launched; a detail string is
 *    available from gsp_last_error_detail() (thread-local).
 *  - Ownership follows the paper's "Half DLPack" borrowing (P:697-704,
 *    P:1014-1017): the CALLER allocates every tensor, including outputs, and
 *    the library never retains a tensor pointer after the call returns.  The
 *    graph object is library-owned until gsp_graph_destroy.
 *  - Compute calls allocate nothing and are asynchronous on `stream`
 *    (GSP_OK means "enqueued"); kernel faults surface as sticky CUDA errors at
 *    the caller's next synchronisation.  The graph is immutable after create,
 *    so concurrent compute calls on different streams are safe.
 *  - Outputs are fully overwritten (rows with no edges become 0), so callers
 *    need not zero them (the paper's th.zeros, is unnecessary).
 *  - Edge (u -> v) means A[v][u] = 1; v = destination = "fwd" row, u = source
 *    = "fwd" column.  The fwd structure groups edges by
 *    destination (CSR, implicit consecutive edge IDs), the rev structure groups
 *    them by source (CSC, explicit edge-ID array) -- P:2001-2005 §Storage
 *    Format "novel edge ID reordering".  Edge tensors are indexed by edge ID.
 */
#ifndef GSP_H
#define GSP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gsp_graph gsp_graph;          /* opaque; owned by the library */
typedef struct CUstream_st *gsp_stream;      /* == cudaStream_t; NULL = legacy default stream */

/* Borrowed dense fp32 matrix, row-major: element (r, c) is data[r*ld + c].
 * ld >= cols (elements).  The buffer spans rows*ld floats (padding columns
 * [cols, ld) may be read but are never written).  The paper's array_t. */
typedef struct {
    void *data;
    int64_t rows, cols, ld;
} gsp_tensor;

typedef enum {
    GSP_OK = 0,
    GSP_ERR_NULL = 1,          /* a required pointer is NULL */
    GSP_ERR_ARG = 2,           /* bad enum / flag / count, no device, stream on another device */
    GSP_ERR_VERTEX_RANGE = 3,  /* a COO id is outside [0, V) */
    GSP_ERR_SHAPE = 4,         /* rows/cols/ld inconsistent with the graph or each other */
    GSP_ERR_ALIAS = 5,         /* output overlaps an input (edge_softmax allows out == e exactly) */
    GSP_ERR_NO_REVERSE = 6,    /* reverse op on a graph built without the rev structure */
    GSP_ERR_OVERFLOW = 7,      /* V or E >= 2^31 (int32 column ids / edge ids) */
    GSP_ERR_OOM = 8,           /* host or device allocation failed */
    GSP_ERR_CUDA = 9           /* a CUDA runtime call failed (detail has the CUDA error) */
} gsp_status;

/* norm ("normalization by degree", reading L1; d^ = max(d,1)):
 *   NONE : out[v] = sum_u X[u]
 *   RIGHT: out[v] = 1/d^_in(v) * sum_u X[u]                      (D_in^-1 A, the paper/SPEC form)
 *   BOTH : out[v] = d^_in(v)^-1/2 * sum_u d^_out(u)^-1/2 X[u]     (D_in^-1/2 A D_out^-1/2, GCN) */
enum { GSP_NORM_NONE = 0, GSP_NORM_RIGHT = 1, GSP_NORM_BOTH = 2 };

/* gsp_graph_create flags */
enum {
    GSP_BUILD_REVERSE = 1u << 0,          /* build the rev (CSC) structure + rev_eid (needed for reverse=1) */
    GSP_BUILD_SHARE_SYMMETRIC = 1u << 1,  /* if the edge multiset is symmetric, keep ONE topology for
                                             fwd and rev ("one copy of the topology"); rev_eid
                                             is still stored */
    GSP_BUILD_EDGE_SCALES = 1u << 2,      /* precompute the per-edge column-side degree scale of the BOTH
                                             norm (4 B per edge per structure; one array when symmetric)
                                             so gsp_gspmm streams it instead of gathering d^-1/2 per edge */
    GSP_BUILD_L2_PERSIST = 1u << 3,       /* opt-in: raise the device's persisting-L2 set-aside
                                             (cudaLimitPersistingL2CacheSize, device-wide, never lowered)
                                             to min(device maximum, 48 MiB; env GSP_L2_SETASIDE_MB
                                             overrides).  The gathered feature tables are loaded with an
                                             L2 evict_last policy, which only protects lines inside the
                                             set-aside from the edge-tensor streams: gSDDMM and the fused
                                             GAT forward gain ~5 %, but edge softmax (+10-15 %), its
                                             backward and gSDDMMve lose the L2 capacity they reuse
                                             (DESIGN.md §6).  A failure to set it is ignored (cache hint) */
    GSP_BUILD_NO_EDGE_IDS = 1u << 4       /* GCN-lean device format ("For GCN, GraphPy need only
                                             (|V|+|E|)"): no explicit edge-ID array on the device.  With
                                             GSP_BUILD_SHARE_SYMMETRIC a symmetric graph then stores ONE
                                             topology (fwd_off + fwd_col) that serves gsp_gspmm in both
                                             directions; a directed graph stores fwd + rev topology.  The
                                             edge-ID indirected reverse ops (gsp_gspmm_weighted /
                                             gsp_gspmm_e with reverse = 1) return GSP_ERR_NO_REVERSE.
                                             The host structure (gsp_graph_export) is unchanged */
};

/* gsp_graph_partition flags */
enum { GSP_PART_REVERSE = 1u << 0 };     /* partition the rev structure (rows = sources) */

/* ------------------------------------------------------------------ graph */

/* Build the kernel-graph from a host COO list (src[i] -> dst[i], i < E) --
 * GraphPy-SM's get_csr + GraphPy-GNN's wrap_graph in one call.
 *  fwd: rows = destinations, slots ordered by (dst, src, input position);
 *       edge ID of slot j is j (implicit).
 *  rev: rows = sources, slots ordered by (src, dst, edge ID); rev_eid[k] is
 *       the edge ID of rev slot k.
 * Duplicates and self-loops are kept as distinct edges (L7).
 * device >= 0: upload to that CUDA device and precompute the degree scales
 *   and degree-binned row schedules (synchronous: returns after the upload).
 * device == -1: host-only graph (structure + export + partitioning; compute
 *   calls return GSP_ERR_ARG).  src/dst are only read during the call.
 * Errors: NULL (g_out, or src/dst with E > 0), ARG (V < 0, E < 0, unknown
 * flags, device out of range), VERTEX_RANGE, OVERFLOW, OOM, CUDA. */
gsp_status gsp_graph_create(int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                            uint32_t flags, int device, gsp_graph **g_out);

/* NULL is a no-op.  Not thread-safe against in-flight compute calls on g:
 * synchronise the streams that use g first. */
gsp_status gsp_graph_destroy(gsp_graph *g);

/* get_vcount / get_ecount.  For a partition graph V is the local
 * row count R (padded) and E the local edge count.  Any output may be NULL.
 * device_bytes = bytes this graph holds on the device (topology, edge IDs,
 * scales, schedules); symmetric = 1 if the topology is shared fwd/rev. */
gsp_status gsp_graph_info(const gsp_graph *g, int64_t *V, int64_t *E, int64_t *device_bytes,
                          int *symmetric);

/* Device bytes of g by kind (any output may be NULL): topology = offsets + column
 * ids of every stored structure (the paper's |V|+|E| words per structure, P:2012;
 * a symmetric shared graph stores one), edge_ids = explicit edge-ID arrays
 * (rev_eid; partitions: the local-rev edge ids), edge_scales = GSP_BUILD_EDGE_SCALES
 * arrays, vertex_arrays = O(V) degree scales and row schedules.  The four sum to
 * gsp_graph_info's device_bytes.  Host-only graphs report zeros. */
gsp_status gsp_graph_memory(const gsp_graph *g, int64_t *topology, int64_t *edge_ids, int64_t *edge_scales,
                            int64_t *vertex_arrays);

/* Copy the canonical structure into caller-allocated HOST arrays (bit-exact
 * checks).  fwd_off[V+1], fwd_col[E], rev_off[V+1], rev_col[E], rev_eid[E],
 * coo_to_eid[E] (coo_to_eid[i] = edge ID of input COO edge i).  Any NULL is
 * skipped.  rev_* on a graph without rev -> GSP_ERR_NO_REVERSE.  Partition
 * graphs: fwd_* is the partition's own structure (R+1 offsets, padded column
 * ids); for a fwd partition rev_* is its local-rev structure (ncols+1 offsets:
 * its own edges grouped by padded source; rev_col = padded destination,
 * rev_eid = local edge id); coo_to_eid -> GSP_ERR_ARG. */
gsp_status gsp_graph_export(const gsp_graph *g, int64_t *fwd_off, int32_t *fwd_col, int64_t *rev_off,
                            int32_t *rev_col, int32_t *rev_eid, int32_t *coo_to_eid);

/* ---------------------------------------------------------------- compute */

/* gSpMMv with fused degree normalisation.
 *  reverse = 0: out[v,f] = s_dst(v) * sum_{slots j of fwd row v} s_src(col_j) * X[col_j, f]
 *  reverse = 1: out[u,f] = s_src(u) * sum_{slots k of rev row u} s_dst(rcol_k) * X[rcol_k, f]
 *  (reverse=1 is the exact adjoint of reverse=0 under the same norm: GCN
 *  backward, with the column-side degree applied per non-zero -- P:1536-1540.)
 * Shapes: X [ncols, F], out [nrows, F] with F = X->cols = out->cols >= 0;
 * ncols = nrows = V for a full graph (partition graphs: see gsp_graph_partition).
 * Cache hint: with norm = BOTH and an X table larger than 6x the device's L2,
 * rows of the highest-degree sources are gathered L2 evict_last and the rest
 * evict_first (DESIGN.md §6 "Hot rows"; env GSP_HOT=0 disables).  Results are
 * unaffected.
 * Errors: NULL, ARG (bad norm/reverse, host-only graph), SHAPE, ALIAS (out
 * overlaps X), NO_REVERSE, CUDA (launch failure). */
gsp_status gsp_gspmm(const gsp_graph *g, const gsp_tensor *X, int norm, gsp_tensor *out,
                     int reverse, gsp_stream stream);

/* Weighted multi-head gSpMM (gSpMMve P:598-601; gSpMMve^T via the
 * edge ID P:2017-2021).  H = w->cols, Fh = X->cols / H (X->cols % H == 0);
 * head h of a vertex row is columns [h*Fh, (h+1)*Fh) (L10).
 *  reverse = 0: out[v, h*Fh+f] = sum_{j in fwd row v} w[j, h] * X[col_j, h*Fh+f]
 *  reverse = 1: out[u, h*Fh+f] = sum_{k in rev row u} w[rev_eid_k, h] * X[rcol_k, h*Fh+f]
 * w is [E, H] indexed by edge ID (no eShuffle, no O(E) temporary).
 * Errors as gsp_gspmm; SHAPE also when w->rows != E, H > 16 or X->cols % H != 0.
 * Partition graphs: see gsp_graph_partition (reverse = 1 gives per-source partials). */
gsp_status gsp_gspmm_weighted(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *w,
                              gsp_tensor *out, int reverse, gsp_stream stream);

/* gSDDMMvv: for every slot j of fwd row v,
 *   out[j, h] = sum_{f < Fh} X[v, h*Fh+f] * Y[col_j, h*Fh+f],   H = out->cols, Fh = X->cols / H.
 * X is the destination (row) side, Y the source (column) side; X == Y allowed
 * (L8).  X and Y are [ncols, H*Fh] (for a partition graph, local row
 * r reads X row row_base + r of the padded table); out is [E, H] by edge ID.
 * Errors: NULL, ARG, SHAPE, ALIAS (out overlaps X or Y), CUDA. */
gsp_status gsp_gsddmm(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *Y, gsp_tensor *out,
                      gsp_stream stream);

/* Edge softmax over each destination's incoming edges (fwd row), per head
 * (L9):
 *   out[j,h] = exp(e[j,h] - m_v,h) / sum_{j' in row v} exp(e[j',h] - m_v,h),  m = row max.
 * e, out are [E, H]; out == e exactly (same data and ld) is allowed (in place),
 * any other overlap is GSP_ERR_ALIAS.  Non-finite inputs propagate (IEEE). */
gsp_status gsp_edge_softmax(const gsp_graph *g, const gsp_tensor *e, gsp_tensor *out, gsp_stream stream);

/* Edge-softmax backward (GAT backward chain; the
 * softmax Jacobian-vector product, "Backward Computation"):
 *   dscore[j,h] = alpha[j,h] * (dalpha[j,h] - sum_{j' in fwd row of j} alpha[j',h] * dalpha[j',h])
 * alpha = the forward edge_softmax output (state tensor), dalpha
 * its gradient; all [E, H] by edge ID.  dscore == dalpha exactly is allowed
 * (in place); any other overlap with dalpha, or any overlap with alpha, is
 * GSP_ERR_ALIAS.  The rest of the GAT backward uses existing calls:
 * dalpha = gsp_gsddmm(g, dOut, Z) and dZ = gsp_gspmm_weighted(reverse = 1). */
gsp_status gsp_edge_softmax_backward(const gsp_graph *g, const gsp_tensor *alpha, const gsp_tensor *dalpha,
                                     gsp_tensor *dscore, gsp_stream stream);

/* Fused GAT forward (the fusion P:197 / P:1472-1484 asks
 * for, that still materialises the state tensor alpha):
 *   alpha = edge_softmax(gsddmm(X, Y))   [E, H] by edge ID   (as gsp_gsddmm + gsp_edge_softmax)
 *   out   = gspmm_weighted(Vt, alpha)    [nrows, Vt->cols]   (as gsp_gspmm_weighted, reverse = 0)
 * computed in one pass per destination row (online softmax) when the head
 * width is 8 (X->cols = Vt->cols = 8 H, H in {2,4,8,16}, alpha->ld == H,
 * 32-byte aligned tables), else by the three kernels in sequence.  Vt == Y
 * (AGNN-style) is allowed and gathered once.  1 <= H <= 16.  Errors: NULL,
 * ARG, SHAPE, ALIAS (out or alpha overlapping an input, out overlapping
 * alpha), CUDA. */
gsp_status gsp_gat_forward(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *Y, const gsp_tensor *Vt,
                           gsp_tensor *alpha, gsp_tensor *out, gsp_stream stream);

/* Fused GAT backward scores ("Backward
 * Computation"; P:1458-1518 the state tensor alpha): the gradient of the
 * attention scores of one GAT layer out = gspmm_weighted(Vt, alpha), in one
 * pass per destination row:
 *   dalpha[j,h] = <dOut[v, head h], Vt[u_j, head h]>          (as gsp_gsddmm(dOut, Vt))
 *   ds[j,h]     = alpha[j,h] (dalpha[j,h] - sum_{j' in row v} alpha[j',h] dalpha[j',h])
 *                                                              (as gsp_edge_softmax_backward)
 * dOut, Vt [ncols, F] (dOut by destination, like gsddmm's X; partitions: the
 * padded tables), alpha, ds [E, H] by edge ID.  Fused when F = 8 H, H in
 * {2, 4, 8, 16}, alpha->ld = ds->ld = H and 32-byte aligned tables; else the
 * two kernels in sequence.  The rest of the layer's backward: dZ through the
 * aggregation = gsp_gspmm_weighted(dOut, alpha, reverse = 1); the score
 * inputs' gradients = gsp_gspmm_weighted(Y, ds) and (X, ds, reverse = 1).
 * Errors: NULL, ARG, SHAPE (1 <= H <= 16, F % H == 0), ALIAS (ds overlapping
 * any input), CUDA. */
gsp_status gsp_gat_backward_scores(const gsp_graph *g, const gsp_tensor *dOut, const gsp_tensor *Vt,
                                   const gsp_tensor *alpha, gsp_tensor *ds, gsp_stream stream);

/* ---------------------------------------- Table 1 surface (NEXT-3, §8(f)) */
enum { GSP_REDUCE_SUM = 0, GSP_REDUCE_MIN = 1, GSP_REDUCE_MAX = 2 };
enum { GSP_OP_ADD = 0, GSP_OP_SUB = 1, GSP_OP_MUL = 2, GSP_OP_DIV = 3 };
enum { GSP_SIDE_DST = 0, GSP_SIDE_SRC = 1 };

/* gSpMMv with a reduction ("reduction operation type, such as
 * sum, min, max"), no normalisation (norm only with sum):
 *   reverse = 0: out[v,f] = RED_{j in fwd row v} X[col_j, f]   (rev: over rev row u)
 * Empty rows -> 0.  reduce = SUM is gsp_gspmm(norm = NONE).
 * Shapes / errors as gsp_gspmm; ARG for an unknown reduce. */
gsp_status gsp_gspmm_reduce(const gsp_graph *g, const gsp_tensor *X, int reduce, gsp_tensor *out, int reverse,
                            gsp_stream stream);

/* gSpMMe / gSpMMeid: an edge tensor reduced per row, fetched
 * through the edge ID:  reverse = 0: out[v,h] = RED_{j in fwd row v} w[j,h];
 * reverse = 1: out[u,h] = RED_{k in rev row u} w[rev_eid_k, h].  w [E,H] by
 * edge ID, out [nrows, H] (fwd partitions, reverse = 1: [ncols, H] partials
 * over the partition's own edges, as gsp_gspmm_weighted).  Empty rows -> 0;
 * sums accumulate in fp64.  Errors as gsp_gspmm_weighted. */
gsp_status gsp_gspmm_e(const gsp_graph *g, const gsp_tensor *w, int reduce, gsp_tensor *out, int reverse,
                       gsp_stream stream);

/* gSDDMMve: for slot j of fwd row v with
 * column u,  out[j,h] = w[j,h] OP X[side == GSP_SIDE_SRC ? u : v, h].
 * X [ncols, H] (partitions: the padded table), w/out [E, H]; out == w exactly
 * is allowed (in place).  Additive GAT scores e = a_dst[v] + a_src[u] are two
 * calls: (w = 0) ADD DST, then in place ADD SRC.  IEEE semantics for DIV. */
gsp_status gsp_gsddmm_ve(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *w, int op, int side,
                         gsp_tensor *out, gsp_stream stream);

/* Additive GAT attention scores (NEXT-3; the u_add_v form of Table 1's gSDDMM
 * family, P:562-568 / P:1329-1331, followed by the standard GAT leaky ReLU,
 * SPEC S:380 "edge logit = leaky_relu(<a_src, z[.]> + <a_dst, z[.]>, slope)",
 * slope 0.2 at S:411).  For slot j of fwd row v with column (source) u_j:
 *   out[j, h] = lrelu(el[u_j, h] + er[v, h]),  lrelu(x) = x > 0 ? x : slope * x
 * el = source-side, er = destination-side per-head vertex scalars, both
 * [ncols, H] (partitions: the padded tables, er read at row row_base + r);
 * out [E, H] by edge ID.  fp32 add and multiply (oracle C14 in fp64).
 * Errors: NULL, ARG (non-finite slope, host-only graph), SHAPE, ALIAS (out
 * overlapping el or er), CUDA. */
gsp_status gsp_gsddmm_add_leaky(const gsp_graph *g, const gsp_tensor *el, const gsp_tensor *er, float slope,
                                gsp_tensor *out, gsp_stream stream);

/* Fused additive GAT forward (NEXT-3 + NEXT-2; oracle C15): the standard GAT
 * layer's attention and aggregation in one pass per destination row, alpha
 * still materialised:
 *   alpha = edge_softmax(gsddmm_add_leaky(el, er, slope))   [E, H] by edge ID
 *   out   = gspmm_weighted(Vt, alpha)                         [nrows, Vt->cols]
 * One pass (online softmax) when Vt->cols = 8 H, H in {2, 4, 8, 16},
 * alpha->ld == H and a 32-byte aligned Vt; else the three kernels in sequence.
 * 1 <= H <= 16.  Errors: NULL, ARG, SHAPE, ALIAS (out or alpha overlapping an
 * input, out overlapping alpha), CUDA. */
gsp_status gsp_gat_forward_additive(const gsp_graph *g, const gsp_tensor *el, const gsp_tensor *er,
                                    const gsp_tensor *Vt, float slope, gsp_tensor *alpha, gsp_tensor *out,
                                    gsp_stream stream);

/* -------------------------------------------------------------- multi-GPU */

/* Edge-balanced contiguous row bounds:
 * bounds[0] = 0, bounds[nparts] = V, bounds[p] = min{ v : off[v] >= ceil(p*E/nparts) },
 * off = fwd_off (reverse = 0) or rev_off (reverse = 1).  bounds has nparts+1
 * entries (caller-allocated, host).  Empty parts are allowed. */
gsp_status gsp_partition_bounds(const gsp_graph *g, int nparts, int reverse, int64_t *bounds);

/* Partition `part` of `nparts` of a full graph g (rows [b_part, b_part+1) of
 * the fwd structure, or of the rev structure with GSP_PART_REVERSE), in the
 * padded rank-major layout: R = max_p (b_{p+1} - b_p); the partition has R
 * rows (rows past the local count are empty) and every column id v is
 * remapped to p(v)*R + (v - b_p(v)), so X tables are [nparts*R, F] and one
 * all-gather of the [R, F] outputs forms the next layer's input.  Local edge
 * IDs are global edge IDs minus fwd_off[b_part] (fwd partitions).
 * Compute on a partition graph:
 *  gsp_gspmm(reverse = 0) on a fwd partition / reverse = 1 on a
 *  GSP_PART_REVERSE partition gives rows [b_p, b_p+1) of the full op; on a
 *  symmetric shared graph a fwd partition also serves reverse = 1 (its own
 *  rows).  reverse = 1 on a fwd partition of a DIRECTED graph gives, like the
 *  weighted reverse below, out [ncols, F]: the contribution of this
 *  partition's edges to every padded source row, the source-side scale s_src
 *  already applied; the sum over partitions (one reduce-scatter) is the full
 *  reverse (adjoint) gSpMMv in the same padded layout.
 *  gsp_gsddmm / gsp_edge_softmax / gsp_gspmm_weighted(reverse=0): fwd
 *  partitions only; the destination-side table of gsddmm is the padded table.
 *  gsp_gspmm_weighted(reverse=1) on a fwd partition: out is [ncols, F], the
 *  contribution of this partition's edges to every (padded) source row; the
 *  sum over partitions (one reduce-scatter) equals the full gSpMMve^T rows.
 * device as in gsp_graph_create (-1 = host-only).  flags: GSP_PART_REVERSE.
 * Errors: NULL, ARG (nparts < 1, part out of range, g is itself a partition),
 * NO_REVERSE, OOM, CUDA. */
gsp_status gsp_graph_partition(const gsp_graph *g, int nparts, int part, int device, uint32_t flags,
                               gsp_graph **out);

/* Chunked partition for communication / computation overlap:
 * the rows are cut into Q = nparts * nchunks edge-balanced C8 blocks
 * (gsp_partition_bounds with Q parts); block q = part * nchunks + chunk is
 * partition (part, chunk), so rank `part` owns the same rows as with
 * gsp_graph_partition, split into nchunks consecutive sub-blocks.  The padded
 * layout is CHUNK-MAJOR: block q sits at slot s(q) = chunk * nparts + part,
 * R = max_q rows, column v -> s(q(v)) * R + (v - b_q(v)), ncols = Q * R.  For
 * each chunk c the nparts ranks' [R, F] outputs are therefore the contiguous
 * rows [c*nparts*R, (c+1)*nparts*R) of the next layer's input: one all-gather
 * per chunk, issued as soon as that chunk's kernel is done while the next
 * chunk computes.  Destination-side tables of gsddmm / gat calls are read at
 * row row_base + r, row_base = s(q) * R (gsp_partition_chunk_info).
 * nchunks = 1 is exactly gsp_graph_partition.  Compute semantics as above.
 * Errors as gsp_graph_partition; ARG also for chunk outside [0, nchunks). */
gsp_status gsp_graph_partition_chunked(const gsp_graph *g, int nparts, int nchunks, int part, int chunk,
                                       int device, uint32_t flags, gsp_graph **out);

/* Chunk geometry of a partition (any output may be NULL): nchunks, chunk, and
 * row_base = the padded row of local row 0.  Full graph: 1, 0, 0. */
gsp_status gsp_partition_chunk_info(const gsp_graph *g, int *nchunks, int *chunk, int64_t *row_base);

/* Partition geometry (any output may be NULL): nparts, part, global row range
 * [row_begin, row_end), padded rows R, ncols = nparts*R, reverse = 1 for a
 * GSP_PART_REVERSE partition.  For a full graph: nparts = 1, part = 0,
 * [0, V), R = V, ncols = V, reverse = 0. */
gsp_status gsp_partition_info(const gsp_graph *g, int *nparts, int *part, int64_t *row_begin,
                              int64_t *row_end, int64_t *R, int64_t *ncols, int *reverse);

/* ------------------------------------------------------------------ misc */
const char *gsp_status_string(gsp_status st);
const char *gsp_last_error_detail(void);      /* thread-local; "" if none */
int gsp_version(void);                          /* (major << 16) | minor */

#ifdef __cplusplus
}
#endif
#endif /* GSP_H */
