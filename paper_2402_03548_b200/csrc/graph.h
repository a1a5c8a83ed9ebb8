// Internal types of libgsp (not part of the ABI; see include/gsp.h).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "gsp.h"

namespace gsp {

// ---------------------------------------------------------------- host side
// Canonical host structure produced by the builder.
struct HostGraph {
    int64_t V = 0, E = 0;
    std::vector<int64_t> fwd_off;      // [V+1]
    std::vector<int32_t> fwd_col;      // [E]   source id of fwd slot j (edge ID j)
    std::vector<int64_t> rev_off;      // [V+1] (empty when no rev)
    std::vector<int32_t> rev_col;      // [E]   destination id of rev slot k
    std::vector<int32_t> rev_eid;      // [E]   edge ID of rev slot k
    std::vector<int32_t> coo_to_eid;   // [E]
    bool has_rev = false;
    bool symmetric = false;            // rev topology == fwd topology
};

// Builds the structure of gsp_graph_create (threads: deterministic result for
// any thread count).  Returns GSP_OK / GSP_ERR_VERTEX_RANGE / GSP_ERR_OOM.
gsp_status build_host_graph(int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                            bool want_rev, HostGraph &hg, std::string &detail);

// Rows ordered by descending degree (ties: ascending row id); heavy rows
// (degree > heavy_threshold) come first.  Returned counts: n_heavy.
void degree_order(const int64_t *off, int64_t nrows, int64_t heavy_threshold,
                  std::vector<int32_t> &order, int64_t &n_heavy);

// --------------------------------------------------------------- device side
// One CSR-like structure on the device: `nrows` rows over a column space of
// `ncols` vertices.  eid == nullptr means implicit edge IDs (slot + eid_base).
struct DevStructure {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    const int64_t *off = nullptr;
    const int32_t *col = nullptr;
    const int32_t *eid = nullptr;
    // degree scales per norm: index 0 NONE (null), 1 RIGHT, 2 BOTH; null => 1.0
    const float *row_scale[3] = {nullptr, nullptr, nullptr};
    const float *col_scale[3] = {nullptr, nullptr, nullptr};
    // optional per-slot column scales (GSP_BUILD_EDGE_SCALES): edge_scale[n][j] = col_scale[n][col[j]]
    const float *edge_scale[3] = {nullptr, nullptr, nullptr};
    // degree-binned schedule: rows by descending degree; the first n_heavy
    // rows get a whole CTA each, the rest one warp each.
    const int32_t *order = nullptr;
    // the same schedule as 16-B records {row, degree, off[row] lo, hi}: one
    // vector load gives a warp its whole task (no order -> off round trip)
    const int32_t *task = nullptr;
    // structures with explicit edge ids (rev, lrev): the same heavy rows first,
    // then the light rows in windows of consecutive row ids (by descending degree
    // inside a window, so a CTA's 8 warps get rows of similar length).  Rows in
    // flight together then cover a narrow range of ids, so the edge-ID indirected
    // reads of a destination's edge block (w[eid]: contiguous per destination,
    // ordered by source id) hit the same lines close in time.
    const int32_t *task_id = nullptr;
    int64_t n_heavy = 0;
    int64_t max_deg = 0;
    bool present = false;
};

constexpr int64_t kHeavyThreshold = 2048;   // edges; DESIGN.md §6 "Work decomposition" (1024 -> 2048: gSpMM -2 %, GAT -2 %)

}  // namespace gsp

struct gsp_graph {
    int device = -1;
    int64_t nrows = 0, ncols = 0, E = 0;       // nrows = V (full) or R (partition)
    int64_t V_global = 0;
    bool symmetric = false;
    // partition geometry (chunked: sub-block q = part*nchunks + chunk of nparts*nchunks
    // C8 blocks sits at padded slot chunk*nparts + part; row_base = slot*R)
    bool is_partition = false;
    int nparts = 1, part = 0, part_reverse = 0, nchunks = 1, chunk = 0;
    int64_t row_begin = 0, row_end = 0, R = 0, row_base = 0;
    // host mirror (full graphs: HostGraph; fwd partitions: local fwd + local rev (lrev))
    gsp::HostGraph host;
    // device.  lrev (fwd partitions only): the partition's OWN edges grouped by
    // padded source row (rows = ncols), explicit local edge ids -- the weighted
    // reverse on a partition yields per-source partial sums to reduce-scatter.
    gsp::DevStructure fwd, rev, lrev;
    std::vector<void *> dev_allocs;
    int64_t device_bytes = 0;
    // device bytes by kind (gsp_graph_memory): topology (offsets + column ids, the
    // paper's |V|+|E| words per stored structure), explicit edge ids,
    // per-edge scales, vertex arrays (degree scales, row schedules)
    int64_t bytes_by[4] = {0, 0, 0, 0};
    bool edge_scales = false;
    bool edge_ids = true;      // false: GSP_BUILD_NO_EDGE_IDS (no rev_eid / lrev on the device)
    // column degrees of the fwd / rev structure sorted descending (host): the hot-row L2
    // policy of the scaled gSpMM on tables larger than L2 (api.cu hot_scale_for)
    // (shared, immutable: partitions point at their parent's)
    std::shared_ptr<const std::vector<int32_t>> col_deg_fwd, col_deg_rev;
};
