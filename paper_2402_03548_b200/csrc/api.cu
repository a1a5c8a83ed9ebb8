// C ABI of libgsp (include/gsp.h): host-side validation, the device graph
// object (upload, degree scales, degree-binned schedules, partitions) and the
// dispatch of the sm_100a kernels.  No exception or abort crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <string>
#include <vector>

#include "graph.h"
#include "gsp.h"
#include "kernels.h"

namespace {

thread_local std::string g_detail;

gsp_status fail(gsp_status st, const std::string &msg) {
    g_detail = msg;
    return st;
}
gsp_status cuda_fail(cudaError_t e, const char *what) {
    return fail(GSP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// kinds of device bytes (gsp_graph::bytes_by, gsp_graph_memory)
enum { kTopo = 0, kEid = 1, kEscale = 2, kVertex = 3 };

template <class T>
gsp_status dev_upload(gsp_graph *g, const T *h, size_t n, const T **out, int kind) {
    *out = nullptr;
    if (n == 0) return GSP_OK;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GSP_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    g->dev_allocs.push_back(p);
    g->device_bytes += (int64_t)(n * sizeof(T));
    g->bytes_by[kind] += (int64_t)(n * sizeof(T));
    e = cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
    *out = static_cast<const T *>(p);
    return GSP_OK;
}

gsp_status dev_alloc_f32(gsp_graph *g, size_t n, float **out, int kind) {
    *out = nullptr;
    if (n == 0) return GSP_OK;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, n * sizeof(float));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GSP_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    g->dev_allocs.push_back(p);
    g->device_bytes += (int64_t)(n * sizeof(float));
    g->bytes_by[kind] += (int64_t)(n * sizeof(float));
    *out = static_cast<float *>(p);
    return GSP_OK;
}

void free_device(gsp_graph *g) {
    if (g->device >= 0) {
        DeviceGuard dg(g->device);
        for (void *p : g->dev_allocs) cudaFree(p);
    }
    g->dev_allocs.clear();
}

// fp32 degree scales (1/d^, d^^-1/2) of an integer degree vector, on the device.
gsp_status make_scales(gsp_graph *g, const std::vector<int64_t> &deg, const float **inv, const float **rsq) {
    *inv = *rsq = nullptr;
    if (deg.empty()) return GSP_OK;
    const int64_t *d_deg = nullptr;
    gsp_status st = dev_upload(g, deg.data(), deg.size(), &d_deg, kVertex);
    if (st != GSP_OK) return st;
    float *pi = nullptr, *pr = nullptr;
    if ((st = dev_alloc_f32(g, deg.size(), &pi, kVertex)) != GSP_OK) return st;
    if ((st = dev_alloc_f32(g, deg.size(), &pr, kVertex)) != GSP_OK) return st;
    cudaError_t e = gsp::launch_degree_scales(d_deg, (int64_t)deg.size(), pi, pr, 0);
    if (e != cudaSuccess) return cuda_fail(e, "degree_scales launch");
    // the integer degrees are only an input of the scale kernel: release them
    // (cudaFree waits for the kernel) so the graph keeps O(V) fp32 scales only
    e = cudaFree(const_cast<int64_t *>(d_deg));
    if (e != cudaSuccess) return cuda_fail(e, "cudaFree");
    g->dev_allocs.erase(std::find(g->dev_allocs.begin(), g->dev_allocs.end(), (void *)d_deg));
    g->device_bytes -= (int64_t)(deg.size() * sizeof(int64_t));
    g->bytes_by[kVertex] -= (int64_t)(deg.size() * sizeof(int64_t));
    *inv = pi;
    *rsq = pr;
    return GSP_OK;
}

// rows above this degree get a whole CTA (graph.h kHeavyThreshold; env GSP_HEAVY for A/B)
int64_t heavy_threshold() {
    static const int64_t v = [] {
        const char *e = getenv("GSP_HEAVY");
        return e ? atoll(e) : gsp::kHeavyThreshold;
    }();
    return v;
}

gsp_status upload_structure(gsp_graph *g, gsp::DevStructure &S, int64_t nrows, int64_t ncols,
                            const std::vector<int64_t> &off, const std::vector<int32_t> &col,
                            const std::vector<int32_t> *eid, const int32_t *shared_order,
                            int64_t shared_n_heavy, const gsp::DevStructure *share_topology) {
    S.nrows = nrows;
    S.ncols = ncols;
    S.nnz = off.empty() ? 0 : off.back();
    S.present = true;
    gsp_status st;
    S.max_deg = 0;
    for (int64_t r = 0; r < nrows; r++) S.max_deg = std::max<int64_t>(S.max_deg, off[r + 1] - off[r]);
    if (share_topology) {
        S.off = share_topology->off;
        S.col = share_topology->col;
    } else {
        if ((st = dev_upload(g, off.data(), off.size(), &S.off, kTopo)) != GSP_OK) return st;
        if ((st = dev_upload(g, col.data(), col.size(), &S.col, kTopo)) != GSP_OK) return st;
    }
    if (eid && (st = dev_upload(g, eid->data(), eid->size(), &S.eid, kEid)) != GSP_OK) return st;
    auto make_task = [&](const std::vector<int32_t> &order, const int32_t **dst) {
        std::vector<int32_t> task((size_t)nrows * 4);
        for (int64_t i = 0; i < nrows; i++) {
            const int64_t r = order[i], b = off[r];
            task[4 * i] = (int32_t)r;
            task[4 * i + 1] = (int32_t)(off[r + 1] - b);   // degree < 2^31 (E < 2^31)
            task[4 * i + 2] = (int32_t)(uint32_t)((uint64_t)b & 0xffffffffu);
            task[4 * i + 3] = (int32_t)(uint32_t)((uint64_t)b >> 32);
        }
        return dev_upload(g, task.data(), task.size(), dst, kVertex);
    };
    std::vector<int32_t> order;
    if (shared_order) {   // same offsets (symmetric topology): same schedule
        S.order = shared_order;
        S.task = share_topology->task;
        S.n_heavy = shared_n_heavy;
        if (eid) gsp::degree_order(off.data(), nrows, heavy_threshold(), order, S.n_heavy);
    } else {
        gsp::degree_order(off.data(), nrows, heavy_threshold(), order, S.n_heavy);
        if ((st = dev_upload(g, order.data(), order.size(), &S.order, kVertex)) != GSP_OK) return st;
        if ((st = make_task(order, &S.task)) != GSP_OK) return st;
    }
    static const int64_t win = [] {   // GSP_EID_WIN: id window of the locality schedule (0: off)
        const char *e = getenv("GSP_EID_WIN");
        return e ? atoll(e) : int64_t(2048);
    }();
    if (eid && win > 0) {   // locality schedule for the edge-ID indirected reverse (graph.h)
        std::sort(order.begin() + S.n_heavy, order.end(), [&](int32_t a, int32_t b) {
            const int64_t wa = a / win, wb = b / win;
            if (wa != wb) return wa < wb;
            const int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
            return da != db ? da > db : a < b;
        });
        if ((st = make_task(order, &S.task_id)) != GSP_OK) return st;
    }
    return GSP_OK;
}

// Hot-row L2 policy of the scaled gSpMM (DESIGN.md §6 "Hot rows"): when the gathered
// table is many times larger than L2, the rows of the highest-degree sources -- the ones gathered
// most often -- are loaded evict_last and all others evict_first, so the streaming
// cold rows stop pushing the reused rows out.  The BOTH norm's column scale d^-1/2 is
// already in the kernel's registers per edge, so "degree above T" is the test
// scale < T^-1/2: T is the degree of the k-th hottest column, k = the rows that fit in
// ~1.3x L2 (GSP_HOT_MB overrides the budget; GSP_HOT=0 turns the policy off).  Returns
// 0 (everything evict_last, as for L2-resident tables) when it does not apply.
float hot_scale_for(const gsp_graph *g, int norm, int reverse, const gsp_tensor *X) {
    static const int on = [] {
        const char *e = getenv("GSP_HOT");
        return e ? atoi(e) : 1;
    }();
    if (!on || norm != GSP_NORM_BOTH) return 0.f;
    const auto &dp = reverse ? g->col_deg_rev : g->col_deg_fwd;
    if (!dp || dp->empty()) return 0.f;
    const std::vector<int32_t> &deg = *dp;
    static const int64_t l2 = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
            cudaGetLastError();
            return int64_t(0);
        }
        return (int64_t)v;
    }();
    static const int64_t budget = [] {
        const char *e = getenv("GSP_HOT_MB");
        return e ? (int64_t)atoll(e) << 20 : int64_t(0);
    }();
    // only tables several times the L2: at 4.5x (Reddit F = 602, 561 MB) plain LRU already
    // serves 63 % of the gathers and the hint costs 19.4 -> 29.0 ms; at 7.8x (ogbn-products,
    // 980 MB, 9 % hits) it saves 4 %, at 160x (Kron-25) 5 %
    const int64_t row_bytes = X->ld * 4, table = X->rows * row_bytes;
    if (l2 <= 0 || row_bytes <= 0 || table <= 6 * l2) return 0.f;
    const int64_t k = std::min<int64_t>((int64_t)deg.size() - 1, (budget ? budget : l2 * 13 / 10) / row_bytes);
    const int32_t T = std::max<int32_t>(deg[(size_t)k], 1);
    return (float)(1.0 / std::sqrt((double)T));
}

// schedule of the edge-ID indirected reverse ops (graph.h task_id)
const int32_t *eid_task(const gsp::DevStructure &S) { return S.task_id ? S.task_id : S.task; }

std::vector<int64_t> degrees_of(const std::vector<int64_t> &off) {
    std::vector<int64_t> d(off.empty() ? 0 : off.size() - 1);
    for (size_t i = 0; i + 1 < off.size(); i++) d[i] = off[i + 1] - off[i];
    return d;
}

// ---------------------------------------------------------------- checks
// Exact overlap test of two strided fp32 regions {data + 4*(i*ld + c) : i < rows, c < cols}.
// Regions with the same row stride (e.g. disjoint column slices X = B[:, :F], out = B[:, F:]
// of one buffer) are resolved exactly; otherwise the exact byte extents are compared.
bool overlaps(const gsp_tensor *a, const gsp_tensor *b) {
    if (!a || !b || !a->data || !b->data) return false;
    if (a->rows == 0 || b->rows == 0 || a->cols == 0 || b->cols == 0) return false;
    const int64_t A0 = (int64_t)reinterpret_cast<uintptr_t>(a->data), B0 = (int64_t)reinterpret_cast<uintptr_t>(b->data);
    const int64_t hi_a = A0 + ((a->rows - 1) * a->ld + a->cols) * 4, hi_b = B0 + ((b->rows - 1) * b->ld + b->cols) * 4;
    if (!(A0 < hi_b && B0 < hi_a)) return false;               // disjoint extents
    if (a->ld != b->ld || (B0 - A0) % 4 != 0) return true;      // conservative beyond this point
    const int64_t L = a->ld, d = (B0 - A0) / 4;
    // B row j starts at element d + j*L of A's frame: row q + j, column r (floor division)
    int64_t q = d / L, r = d % L;
    if (r < 0) { r += L; q -= 1; }
    auto rows_meet = [&](int64_t shift) {   // some j in [0, b.rows) with A row q + j + shift in [0, a.rows)
        const int64_t lo = std::max<int64_t>(0, -(q + shift)), hi = std::min<int64_t>(b->rows, a->rows - (q + shift));
        return lo < hi;
    };
    if (r < a->cols && rows_meet(0)) return true;               // B's row segment [r, r+cb) meets A's [0, ca)
    if (r + b->cols > L && rows_meet(1)) return true;           // ... or spills into A's next row
    return false;
}

gsp_status check_tensor(const gsp_graph *g, const gsp_tensor *t, const char *name, int64_t rows, int64_t cols) {
    if (!t) return fail(GSP_ERR_NULL, std::string(name) + " is NULL");
    if (t->rows < 0 || t->cols < 0 || t->ld < t->cols)
        return fail(GSP_ERR_SHAPE, std::string(name) + ": need rows >= 0, cols >= 0, ld >= cols");
    if (rows >= 0 && t->rows != rows)
        return fail(GSP_ERR_SHAPE, std::string(name) + ".rows = " + std::to_string(t->rows) + ", expected " +
                                       std::to_string(rows));
    if (cols >= 0 && t->cols != cols)
        return fail(GSP_ERR_SHAPE, std::string(name) + ".cols = " + std::to_string(t->cols) + ", expected " +
                                       std::to_string(cols));
    if (t->rows > 0 && t->cols > 0) {
        if (!t->data) return fail(GSP_ERR_NULL, std::string(name) + ".data is NULL");
        cudaPointerAttributes at;
        cudaError_t e = cudaPointerGetAttributes(&at, t->data);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(GSP_ERR_ARG, std::string(name) + ": not a CUDA pointer");
        }
        if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
            return fail(GSP_ERR_ARG, std::string(name) + ": not device memory");
        if (at.type == cudaMemoryTypeDevice && at.device != g->device)
            return fail(GSP_ERR_ARG, std::string(name) + ": on device " + std::to_string(at.device) +
                                         ", graph on device " + std::to_string(g->device));
    }
    return GSP_OK;
}

gsp_status check_compute_graph(const gsp_graph *g) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    if (g->device < 0) return fail(GSP_ERR_ARG, "host-only graph (device = -1) cannot run compute calls");
    return GSP_OK;
}

gsp_status check_stream(const gsp_graph *g, gsp_stream s) {
    if (!s) return GSP_OK;
    // during CUDA-graph capture the stream cannot be queried (and the capture
    // would be invalidated): skip the device check, everything else is capturable
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)s, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
        return GSP_OK;
    cudaGetLastError();
    int dev = -1;
    cudaError_t e = cudaStreamGetDevice((cudaStream_t)s, &dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GSP_ERR_ARG, std::string("invalid stream: ") + cudaGetErrorString(e));
    }
    if (dev != g->device)
        return fail(GSP_ERR_ARG, "stream on device " + std::to_string(dev) + ", graph on device " +
                                     std::to_string(g->device));
    return GSP_OK;
}

}  // namespace

extern "C" {

const char *gsp_status_string(gsp_status st) {
    switch (st) {
        case GSP_OK: return "GSP_OK";
        case GSP_ERR_NULL: return "GSP_ERR_NULL";
        case GSP_ERR_ARG: return "GSP_ERR_ARG";
        case GSP_ERR_VERTEX_RANGE: return "GSP_ERR_VERTEX_RANGE";
        case GSP_ERR_SHAPE: return "GSP_ERR_SHAPE";
        case GSP_ERR_ALIAS: return "GSP_ERR_ALIAS";
        case GSP_ERR_NO_REVERSE: return "GSP_ERR_NO_REVERSE";
        case GSP_ERR_OVERFLOW: return "GSP_ERR_OVERFLOW";
        case GSP_ERR_OOM: return "GSP_ERR_OOM";
        case GSP_ERR_CUDA: return "GSP_ERR_CUDA";
    }
    return "GSP_ERR_UNKNOWN";
}

const char *gsp_last_error_detail(void) { return g_detail.c_str(); }

int gsp_version(void) { return (1 << 16) | 0; }

static gsp_status upload_full(gsp_graph *g) {
    const gsp::HostGraph &h = g->host;
    DeviceGuard dg(g->device);
    if (!dg.ok) return fail(GSP_ERR_ARG, "cannot select device " + std::to_string(g->device));
    gsp_status st;
    std::vector<int64_t> din = degrees_of(h.fwd_off), dout;
    if (h.has_rev) dout = degrees_of(h.rev_off);
    else {
        dout.assign((size_t)h.V, 0);
        for (int32_t u : h.fwd_col) dout[u]++;
    }
    auto sorted_desc = [](const std::vector<int64_t> &d) {
        auto s = std::make_shared<std::vector<int32_t>>(d.begin(), d.end());
        std::sort(s->begin(), s->end(), std::greater<int32_t>());
        return std::shared_ptr<const std::vector<int32_t>>(std::move(s));
    };
    g->col_deg_fwd = sorted_desc(dout);   // fwd columns are sources
    g->col_deg_rev = sorted_desc(din);    // rev columns are destinations
    const float *inv_in, *rsq_in, *inv_out, *rsq_out;
    if ((st = make_scales(g, din, &inv_in, &rsq_in)) != GSP_OK) return st;
    if ((st = make_scales(g, dout, &inv_out, &rsq_out)) != GSP_OK) return st;
    (void)inv_out;
    if ((st = upload_structure(g, g->fwd, h.V, h.V, h.fwd_off, h.fwd_col, nullptr, nullptr, 0, nullptr)) != GSP_OK)
        return st;
    g->fwd.row_scale[GSP_NORM_RIGHT] = inv_in;
    g->fwd.row_scale[GSP_NORM_BOTH] = rsq_in;
    g->fwd.col_scale[GSP_NORM_BOTH] = rsq_out;
    if (h.has_rev) {
        // GSP_BUILD_NO_EDGE_IDS: the GCN-lean format keeps no explicit edge ids on
        // the device; a symmetric graph then holds ONE topology (|V|+|E| words) for both directions
        const std::vector<int32_t> *rev_eid = g->edge_ids ? &h.rev_eid : nullptr;
        if (h.symmetric)
            st = upload_structure(g, g->rev, h.V, h.V, h.rev_off, h.rev_col, rev_eid, g->fwd.order,
                                  g->fwd.n_heavy, &g->fwd);
        else
            st = upload_structure(g, g->rev, h.V, h.V, h.rev_off, h.rev_col, rev_eid, nullptr, 0, nullptr);
        if (st != GSP_OK) return st;
        g->rev.row_scale[GSP_NORM_BOTH] = rsq_out;
        g->rev.col_scale[GSP_NORM_RIGHT] = inv_in;
        g->rev.col_scale[GSP_NORM_BOTH] = rsq_in;
    }
    if (g->edge_scales) {
        float *es = nullptr;
        if ((st = dev_alloc_f32(g, (size_t)h.E, &es, kEscale)) != GSP_OK) return st;
        cudaError_t e0 = gsp::launch_gather_scale(g->fwd.col, h.E, rsq_out, es, 0);
        if (e0 != cudaSuccess) return cuda_fail(e0, "edge scales");
        g->fwd.edge_scale[GSP_NORM_BOTH] = es;
        if (h.has_rev) {
            if (h.symmetric) {
                g->rev.edge_scale[GSP_NORM_BOTH] = es;   // d_in == d_out: the same values
            } else {
                float *er = nullptr;
                if ((st = dev_alloc_f32(g, (size_t)h.E, &er, kEscale)) != GSP_OK) return st;
                e0 = gsp::launch_gather_scale(g->rev.col, h.E, rsq_in, er, 0);
                if (e0 != cudaSuccess) return cuda_fail(e0, "edge scales");
                g->rev.edge_scale[GSP_NORM_BOTH] = er;
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "graph upload");
    return GSP_OK;
}

// GSP_BUILD_L2_PERSIST (include/gsp.h): a cache hint, so failures are ignored
void raise_l2_setaside(int device) {
    DeviceGuard dg(device);
    int maxp = 0;
    if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device) != cudaSuccess || maxp <= 0) {
        cudaGetLastError();
        return;
    }
    const char *env = getenv("GSP_L2_SETASIDE_MB");
    size_t want = (size_t)(env ? atoll(env) : 48) << 20;
    if (want > (size_t)maxp) want = (size_t)maxp;
    size_t cur = 0;
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess && cur < want)
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    cudaGetLastError();
}

gsp_status gsp_graph_create(int64_t V, int64_t E, const int64_t *src, const int64_t *dst, uint32_t flags,
                            int device, gsp_graph **g_out) {
    if (!g_out) return fail(GSP_ERR_NULL, "g_out is NULL");
    *g_out = nullptr;
    if (E > 0 && (!src || !dst)) return fail(GSP_ERR_NULL, "src/dst is NULL");
    if (V < 0 || E < 0) return fail(GSP_ERR_ARG, "V and E must be >= 0");
    if (flags & ~(uint32_t)(GSP_BUILD_REVERSE | GSP_BUILD_SHARE_SYMMETRIC | GSP_BUILD_EDGE_SCALES |
                            GSP_BUILD_L2_PERSIST | GSP_BUILD_NO_EDGE_IDS))
        return fail(GSP_ERR_ARG, "unknown flags");
    if (V >= (int64_t(1) << 31) || E >= (int64_t(1) << 31))
        return fail(GSP_ERR_OVERFLOW, "V and E must be < 2^31 (int32 column and edge ids)");
    if (device < -1) return fail(GSP_ERR_ARG, "device must be >= -1");
    if (device >= 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || device >= n) {
            cudaGetLastError();
            return fail(GSP_ERR_ARG, "device " + std::to_string(device) + " not available");
        }
    }
    gsp_graph *g = new (std::nothrow) gsp_graph();
    if (!g) return fail(GSP_ERR_OOM, "host allocation failed");
    std::string detail;
    gsp_status st = gsp::build_host_graph(V, E, src, dst, (flags & GSP_BUILD_REVERSE) != 0, g->host, detail);
    if (st != GSP_OK) {
        delete g;
        return fail(st, detail);
    }
    if (!(flags & GSP_BUILD_SHARE_SYMMETRIC)) g->host.symmetric = false;
    g->nrows = g->ncols = g->V_global = V;
    g->E = E;
    g->row_begin = 0;
    g->row_end = V;
    g->R = V;
    g->symmetric = g->host.symmetric;
    g->device = device;
    g->edge_scales = (flags & GSP_BUILD_EDGE_SCALES) != 0;
    g->edge_ids = (flags & GSP_BUILD_NO_EDGE_IDS) == 0;
    if (device >= 0 && (flags & GSP_BUILD_L2_PERSIST)) raise_l2_setaside(device);
    if (device >= 0) {
        st = upload_full(g);
        if (st != GSP_OK) {
            std::string keep = g_detail;
            free_device(g);
            delete g;
            return fail(st, keep);
        }
    }
    *g_out = g;
    return GSP_OK;
}

gsp_status gsp_graph_destroy(gsp_graph *g) {
    if (!g) return GSP_OK;
    free_device(g);
    delete g;
    return GSP_OK;
}

gsp_status gsp_graph_info(const gsp_graph *g, int64_t *V, int64_t *E, int64_t *device_bytes, int *symmetric) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    if (V) *V = g->nrows;
    if (E) *E = g->E;
    if (device_bytes) *device_bytes = g->device_bytes;
    if (symmetric) *symmetric = g->symmetric ? 1 : 0;
    return GSP_OK;
}

gsp_status gsp_graph_export(const gsp_graph *g, int64_t *fwd_off, int32_t *fwd_col, int64_t *rev_off,
                            int32_t *rev_col, int32_t *rev_eid, int32_t *coo_to_eid) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    const gsp::HostGraph &h = g->host;
    if (g->is_partition && coo_to_eid) return fail(GSP_ERR_ARG, "partition graphs have no coo_to_eid");
    if ((rev_off || rev_col || rev_eid) && !h.has_rev) return fail(GSP_ERR_NO_REVERSE, "graph has no rev structure");
    if (fwd_off) std::memcpy(fwd_off, h.fwd_off.data(), sizeof(int64_t) * h.fwd_off.size());
    if (fwd_col && !h.fwd_col.empty()) std::memcpy(fwd_col, h.fwd_col.data(), sizeof(int32_t) * h.fwd_col.size());
    if (rev_off) std::memcpy(rev_off, h.rev_off.data(), sizeof(int64_t) * h.rev_off.size());
    if (rev_col && !h.rev_col.empty()) std::memcpy(rev_col, h.rev_col.data(), sizeof(int32_t) * h.rev_col.size());
    if (rev_eid && !h.rev_eid.empty()) std::memcpy(rev_eid, h.rev_eid.data(), sizeof(int32_t) * h.rev_eid.size());
    if (coo_to_eid && !h.coo_to_eid.empty())
        std::memcpy(coo_to_eid, h.coo_to_eid.data(), sizeof(int32_t) * h.coo_to_eid.size());
    return GSP_OK;
}

// ---------------------------------------------------------------- compute
gsp_status gsp_gspmm(const gsp_graph *g, const gsp_tensor *X, int norm, gsp_tensor *out, int reverse,
                     gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    if (norm < GSP_NORM_NONE || norm > GSP_NORM_BOTH) return fail(GSP_ERR_ARG, "norm must be 0, 1 or 2");
    if (reverse != 0 && reverse != 1) return fail(GSP_ERR_ARG, "reverse must be 0 or 1");
    // reverse = 1 on a fwd partition of a directed graph: per-source partials over the
    // partition's own edges (lrev, [ncols, F]); one reduce-scatter completes them (gsp.h)
    const bool partials = reverse && !g->rev.present && g->is_partition && g->lrev.present;
    const gsp::DevStructure &S = reverse ? (partials ? g->lrev : g->rev) : g->fwd;
    if (!S.present)
        return reverse ? fail(GSP_ERR_NO_REVERSE, "graph has no rev structure (GSP_BUILD_REVERSE)")
                       : fail(GSP_ERR_ARG, "this partition only serves reverse = 1");
    if (!X || !out) return fail(GSP_ERR_NULL, "X/out is NULL");
    if ((st = check_tensor(g, X, "X", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", S.nrows, X->cols)) != GSP_OK) return st;
    if (overlaps(X, out)) return fail(GSP_ERR_ALIAS, "out overlaps X");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SpmmArgs a{};
    a.off = S.off; a.col = S.col; a.eid = nullptr; a.order = S.order; a.task = S.task;
    a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.X = static_cast<const float *>(X->data); a.ldx = X->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.F = X->cols;
    a.row_scale = S.row_scale[norm]; a.col_scale = S.col_scale[norm]; a.edge_scale = S.edge_scale[norm];
    a.H = 1; a.Fh = X->cols > 0 ? X->cols : 1;
    a.light = S.nnz < 32 * S.nrows;
    a.hot_scale = hot_scale_for(g, norm, reverse, X);
    cudaError_t e = gsp::launch_spmm(a, gsp::kSpmmScaled, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gspmm launch");
    return GSP_OK;
}

gsp_status gsp_gspmm_weighted(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *w, gsp_tensor *out,
                              int reverse, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    if (reverse != 0 && reverse != 1) return fail(GSP_ERR_ARG, "reverse must be 0 or 1");
    // fwd partitions: reverse = 1 runs over the partition's own edges grouped by
    // source (lrev) and yields partial sums for every padded source row
    const gsp::DevStructure &S = reverse ? (g->is_partition ? g->lrev : g->rev) : g->fwd;
    if (!S.present || (reverse && !S.eid))
        return reverse ? fail(GSP_ERR_NO_REVERSE, "no rev structure with edge ids on this graph")
                       : fail(GSP_ERR_ARG, "this partition only serves reverse = 1");
    if (!X || !w || !out) return fail(GSP_ERR_NULL, "X/w/out is NULL");
    if ((st = check_tensor(g, w, "w", g->E, -1)) != GSP_OK) return st;
    const int64_t H = w->cols;
    if (H < 1 || H > 16) return fail(GSP_ERR_SHAPE, "w must have 1 <= H <= 16 columns (heads)");
    if ((st = check_tensor(g, X, "X", S.ncols, -1)) != GSP_OK) return st;
    if (X->cols % H != 0) return fail(GSP_ERR_SHAPE, "X.cols must be a multiple of H = w.cols");
    if ((st = check_tensor(g, out, "out", S.nrows, X->cols)) != GSP_OK) return st;
    if (overlaps(X, out) || overlaps(w, out)) return fail(GSP_ERR_ALIAS, "out overlaps X or w");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SpmmArgs a{};
    a.off = S.off; a.col = S.col; a.eid = S.eid; a.order = S.order; a.task = reverse ? eid_task(S) : S.task;
    a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.X = static_cast<const float *>(X->data); a.ldx = X->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.F = X->cols;
    a.w = static_cast<const float *>(w->data); a.ldw = w->ld;
    a.H = H; a.Fh = X->cols / H > 0 ? X->cols / H : 1;
    cudaError_t e = gsp::launch_spmm(a, reverse ? gsp::kSpmmWeightedRev : gsp::kSpmmWeightedFwd, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gspmm_weighted launch");
    return GSP_OK;
}

gsp_status gsp_gsddmm(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *Y, gsp_tensor *out,
                      gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "gsddmm needs the fwd structure (not a reverse partition)");
    if (!X || !Y || !out) return fail(GSP_ERR_NULL, "X/Y/out is NULL");
    if ((st = check_tensor(g, out, "out", g->E, -1)) != GSP_OK) return st;
    const int64_t H = out->cols;
    if (H < 1) return fail(GSP_ERR_SHAPE, "out must have H >= 1 columns");
    if ((st = check_tensor(g, X, "X", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, Y, "Y", S.ncols, X->cols)) != GSP_OK) return st;
    if (X->cols % H != 0) return fail(GSP_ERR_SHAPE, "X.cols must be a multiple of H = out.cols");
    if (overlaps(X, out) || overlaps(Y, out)) return fail(GSP_ERR_ALIAS, "out overlaps X or Y");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SddmmArgs a{};
    a.off = S.off; a.col = S.col; a.order = S.order; a.task = S.task;
    a.nrows = S.nrows; a.n_heavy = S.n_heavy; a.row_base = g->row_base;
    a.X = static_cast<const float *>(X->data); a.ldx = X->ld;
    a.Y = static_cast<const float *>(Y->data); a.ldy = Y->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.H = H; a.Fh = X->cols / H;
    if (a.Fh == 0) {
        // F = 0: every dot product is empty -> write zeros
        cudaError_t e = cudaMemset2DAsync(out->data, (size_t)out->ld * 4, 0, (size_t)H * 4, (size_t)g->E,
                                          (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "gsddmm memset");
        return GSP_OK;
    }
    cudaError_t e = gsp::launch_sddmm(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gsddmm launch");
    return GSP_OK;
}

gsp_status gsp_edge_softmax(const gsp_graph *g, const gsp_tensor *e_in, gsp_tensor *out, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "edge_softmax needs the fwd structure (not a reverse partition)");
    if (!e_in || !out) return fail(GSP_ERR_NULL, "e/out is NULL");
    if ((st = check_tensor(g, e_in, "e", g->E, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", g->E, e_in->cols)) != GSP_OK) return st;
    const bool same = e_in->data == out->data && e_in->ld == out->ld;
    if (!same && overlaps(e_in, out)) return fail(GSP_ERR_ALIAS, "out partially overlaps e");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SoftmaxArgs a{};
    a.off = S.off; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.e = static_cast<const float *>(e_in->data); a.lde = e_in->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.H = e_in->cols;
    cudaError_t err = gsp::launch_softmax(a, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "edge_softmax launch");
    return GSP_OK;
}

gsp_status gsp_edge_softmax_backward(const gsp_graph *g, const gsp_tensor *alpha, const gsp_tensor *dalpha,
                                     gsp_tensor *dscore, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "edge_softmax_backward needs the fwd structure");
    if (!alpha || !dalpha || !dscore) return fail(GSP_ERR_NULL, "alpha/dalpha/dscore is NULL");
    if ((st = check_tensor(g, alpha, "alpha", g->E, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, dalpha, "dalpha", g->E, alpha->cols)) != GSP_OK) return st;
    if ((st = check_tensor(g, dscore, "dscore", g->E, alpha->cols)) != GSP_OK) return st;
    if (overlaps(alpha, dscore)) return fail(GSP_ERR_ALIAS, "dscore overlaps alpha");
    const bool same = dalpha->data == dscore->data && dalpha->ld == dscore->ld;
    if (!same && overlaps(dalpha, dscore)) return fail(GSP_ERR_ALIAS, "dscore partially overlaps dalpha");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SoftmaxBwdArgs a{};
    a.off = S.off; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.alpha = static_cast<const float *>(alpha->data); a.lda = alpha->ld;
    a.dalpha = static_cast<const float *>(dalpha->data); a.ldd = dalpha->ld;
    a.out = static_cast<float *>(dscore->data); a.ldo = dscore->ld;
    a.H = alpha->cols;
    cudaError_t e = gsp::launch_softmax_bwd(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "edge_softmax_backward launch");
    return GSP_OK;
}

gsp_status gsp_gat_forward(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *Y, const gsp_tensor *Vt,
                           gsp_tensor *alpha, gsp_tensor *out, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "gat_forward needs the fwd structure (not a reverse partition)");
    if (!X || !Y || !Vt || !alpha || !out) return fail(GSP_ERR_NULL, "X/Y/Vt/alpha/out is NULL");
    if ((st = check_tensor(g, alpha, "alpha", g->E, -1)) != GSP_OK) return st;
    const int64_t H = alpha->cols;
    if (H < 1 || H > 16) return fail(GSP_ERR_SHAPE, "alpha must have 1 <= H <= 16 columns (heads)");
    if ((st = check_tensor(g, X, "X", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, Y, "Y", S.ncols, X->cols)) != GSP_OK) return st;
    if ((st = check_tensor(g, Vt, "Vt", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", S.nrows, Vt->cols)) != GSP_OK) return st;
    if (X->cols % H != 0 || Vt->cols % H != 0) return fail(GSP_ERR_SHAPE, "X.cols and Vt.cols must be multiples of H");
    if (overlaps(out, X) || overlaps(out, Y) || overlaps(out, Vt) || overlaps(out, alpha))
        return fail(GSP_ERR_ALIAS, "out overlaps an input or alpha");
    if (overlaps(alpha, X) || overlaps(alpha, Y) || overlaps(alpha, Vt))
        return fail(GSP_ERR_ALIAS, "alpha overlaps X, Y or Vt");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    cudaStream_t cs = (cudaStream_t)stream;
    gsp::GatArgs ga{};
    ga.off = S.off; ga.col = S.col; ga.order = S.order; ga.task = S.task; ga.nrows = S.nrows; ga.n_heavy = S.n_heavy;
    ga.row_base = g->row_base;
    ga.light = S.nnz < 32 * S.nrows;
    ga.X = static_cast<const float *>(X->data); ga.ldx = X->ld;
    ga.Y = static_cast<const float *>(Y->data); ga.ldy = Y->ld;
    ga.Vt = static_cast<const float *>(Vt->data); ga.ldv = Vt->ld;
    ga.alpha = static_cast<float *>(alpha->data);
    ga.out = static_cast<float *>(out->data); ga.ldo = out->ld;
    ga.H = H;
    const bool fused = X->cols == 8 * H && Vt->cols == 8 * H && alpha->ld == H && gsp::gat_fused_supported(ga);
    cudaError_t e;
    if (fused) {
        e = gsp::launch_gat_fused(ga, cs);
    } else {
        // any other shape: the three kernels in sequence (same results within the bound)
        gsp::SddmmArgs sa{};
        sa.off = S.off; sa.col = S.col; sa.order = S.order; sa.task = S.task; sa.nrows = S.nrows; sa.n_heavy = S.n_heavy;
        sa.row_base = g->row_base;
        sa.X = ga.X; sa.ldx = X->ld; sa.Y = ga.Y; sa.ldy = Y->ld;
        sa.out = ga.alpha; sa.ldo = alpha->ld; sa.H = H; sa.Fh = X->cols / H;
        e = sa.Fh > 0 ? gsp::launch_sddmm(sa, cs)
                      : cudaMemset2DAsync(alpha->data, (size_t)alpha->ld * 4, 0, (size_t)H * 4, (size_t)g->E, cs);
        if (e == cudaSuccess) {
            gsp::SoftmaxArgs xa{};
            xa.off = S.off; xa.order = S.order; xa.task = S.task; xa.nrows = S.nrows; xa.n_heavy = S.n_heavy;
            xa.e = ga.alpha; xa.lde = alpha->ld; xa.out = ga.alpha; xa.ldo = alpha->ld; xa.H = H;
            e = gsp::launch_softmax(xa, cs);
        }
        if (e == cudaSuccess) {
            gsp::SpmmArgs wa{};
            wa.off = S.off; wa.col = S.col; wa.order = S.order; wa.task = S.task; wa.nrows = S.nrows; wa.n_heavy = S.n_heavy;
            wa.X = ga.Vt; wa.ldx = Vt->ld; wa.out = ga.out; wa.ldo = out->ld; wa.F = Vt->cols;
            wa.w = ga.alpha; wa.ldw = alpha->ld; wa.H = H; wa.Fh = Vt->cols / H > 0 ? Vt->cols / H : 1;
            e = gsp::launch_spmm(wa, gsp::kSpmmWeightedFwd, cs);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "gat_forward launch");
    return GSP_OK;
}

gsp_status gsp_gat_backward_scores(const gsp_graph *g, const gsp_tensor *dOut, const gsp_tensor *Vt,
                                   const gsp_tensor *alpha, gsp_tensor *ds, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "gat_backward_scores needs the fwd structure (not a reverse partition)");
    if (!dOut || !Vt || !alpha || !ds) return fail(GSP_ERR_NULL, "dOut/Vt/alpha/ds is NULL");
    if ((st = check_tensor(g, alpha, "alpha", g->E, -1)) != GSP_OK) return st;
    const int64_t H = alpha->cols;
    if (H < 1 || H > 16) return fail(GSP_ERR_SHAPE, "alpha must have 1 <= H <= 16 columns (heads)");
    if ((st = check_tensor(g, ds, "ds", g->E, H)) != GSP_OK) return st;
    if ((st = check_tensor(g, dOut, "dOut", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, Vt, "Vt", S.ncols, dOut->cols)) != GSP_OK) return st;
    if (dOut->cols % H != 0) return fail(GSP_ERR_SHAPE, "dOut.cols must be a multiple of H");
    if (overlaps(ds, alpha) || overlaps(ds, dOut) || overlaps(ds, Vt))
        return fail(GSP_ERR_ALIAS, "ds overlaps alpha, dOut or Vt");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    cudaStream_t cs = (cudaStream_t)stream;
    gsp::GatArgs ga{};
    ga.off = S.off; ga.col = S.col; ga.order = S.order; ga.task = S.task; ga.nrows = S.nrows; ga.n_heavy = S.n_heavy;
    ga.row_base = g->row_base;
    ga.light = S.nnz < 32 * S.nrows;
    ga.X = static_cast<const float *>(dOut->data); ga.ldx = dOut->ld;
    ga.Y = ga.X; ga.ldy = dOut->ld;
    ga.Vt = static_cast<const float *>(Vt->data); ga.ldv = Vt->ld;
    ga.alpha = static_cast<float *>(alpha->data);   // read only
    ga.out = static_cast<float *>(ds->data); ga.ldo = ds->ld;
    ga.H = H;
    const bool fused = dOut->cols == 8 * H && alpha->ld == H && ds->ld == H && H != 1 && gsp::gat_fused_supported(ga);
    cudaError_t e;
    if (fused) {
        e = gsp::launch_gat_bwd(ga, cs);
    } else {
        // any other shape: gSDDMM into ds (as dalpha), then the softmax backward in place
        gsp::SddmmArgs sa{};
        sa.off = S.off; sa.col = S.col; sa.order = S.order; sa.task = S.task; sa.nrows = S.nrows; sa.n_heavy = S.n_heavy;
        sa.row_base = g->row_base;
        sa.X = ga.X; sa.ldx = dOut->ld; sa.Y = ga.Vt; sa.ldy = Vt->ld;
        sa.out = ga.out; sa.ldo = ds->ld; sa.H = H; sa.Fh = dOut->cols / H;
        e = sa.Fh > 0 ? gsp::launch_sddmm(sa, cs)
                      : cudaMemset2DAsync(ds->data, (size_t)ds->ld * 4, 0, (size_t)H * 4, (size_t)g->E, cs);
        if (e == cudaSuccess) {
            gsp::SoftmaxBwdArgs a{};
            a.off = S.off; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
            a.alpha = ga.alpha; a.lda = alpha->ld;
            a.dalpha = ga.out; a.ldd = ds->ld;
            a.out = ga.out; a.ldo = ds->ld;
            a.H = H;
            e = gsp::launch_softmax_bwd(a, cs);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "gat_backward_scores launch");
    return GSP_OK;
}

// ------------------------------------- NEXT-3: additive GAT attention (C14, C15)
static gsp_status check_additive(const gsp_graph *g, const gsp_tensor *el, const gsp_tensor *er, float slope,
                                 int64_t *H) {
    gsp_status st;
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "needs the fwd structure (not a reverse partition)");
    if (!el || !er) return fail(GSP_ERR_NULL, "el/er is NULL");
    if (!std::isfinite(slope)) return fail(GSP_ERR_ARG, "slope must be finite");
    if ((st = check_tensor(g, el, "el", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, er, "er", S.ncols, el->cols)) != GSP_OK) return st;
    *H = el->cols;
    if (*H < 1) return fail(GSP_ERR_SHAPE, "el/er must have H >= 1 columns");
    return GSP_OK;
}

gsp_status gsp_gsddmm_add_leaky(const gsp_graph *g, const gsp_tensor *el, const gsp_tensor *er, float slope,
                                gsp_tensor *out, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    int64_t H = 0;
    if ((st = check_additive(g, el, er, slope, &H)) != GSP_OK) return st;
    if (!out) return fail(GSP_ERR_NULL, "out is NULL");
    if ((st = check_tensor(g, out, "out", g->E, H)) != GSP_OK) return st;
    if (overlaps(out, el) || overlaps(out, er)) return fail(GSP_ERR_ALIAS, "out overlaps el or er");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    const gsp::DevStructure &S = g->fwd;
    gsp::SddmmAddArgs a{};
    a.off = S.off; a.col = S.col; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.row_base = g->row_base;
    a.el = static_cast<const float *>(el->data); a.lde = el->ld;
    a.er = static_cast<const float *>(er->data); a.ldr = er->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.H = H; a.slope = slope;
    cudaError_t e = gsp::launch_sddmm_add(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gsddmm_add_leaky launch");
    return GSP_OK;
}

gsp_status gsp_gat_forward_additive(const gsp_graph *g, const gsp_tensor *el, const gsp_tensor *er,
                                    const gsp_tensor *Vt, float slope, gsp_tensor *alpha, gsp_tensor *out,
                                    gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    int64_t H = 0;
    if ((st = check_additive(g, el, er, slope, &H)) != GSP_OK) return st;
    if (!Vt || !alpha || !out) return fail(GSP_ERR_NULL, "Vt/alpha/out is NULL");
    const gsp::DevStructure &S = g->fwd;
    if (H > 16) return fail(GSP_ERR_SHAPE, "1 <= H <= 16 heads");
    if ((st = check_tensor(g, alpha, "alpha", g->E, H)) != GSP_OK) return st;
    if ((st = check_tensor(g, Vt, "Vt", S.ncols, -1)) != GSP_OK) return st;
    if (Vt->cols % H != 0) return fail(GSP_ERR_SHAPE, "Vt.cols must be a multiple of H");
    if ((st = check_tensor(g, out, "out", S.nrows, Vt->cols)) != GSP_OK) return st;
    if (overlaps(out, el) || overlaps(out, er) || overlaps(out, Vt) || overlaps(out, alpha))
        return fail(GSP_ERR_ALIAS, "out overlaps an input or alpha");
    if (overlaps(alpha, el) || overlaps(alpha, er) || overlaps(alpha, Vt))
        return fail(GSP_ERR_ALIAS, "alpha overlaps el, er or Vt");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    cudaStream_t cs = (cudaStream_t)stream;
    gsp::GatArgs ga{};
    ga.off = S.off; ga.col = S.col; ga.order = S.order; ga.task = S.task; ga.nrows = S.nrows; ga.n_heavy = S.n_heavy;
    ga.row_base = g->row_base;
    ga.light = S.nnz < 32 * S.nrows;
    ga.X = static_cast<const float *>(er->data); ga.ldx = er->ld;
    ga.Y = static_cast<const float *>(el->data); ga.ldy = el->ld;
    ga.Vt = static_cast<const float *>(Vt->data); ga.ldv = Vt->ld;
    ga.alpha = static_cast<float *>(alpha->data);
    ga.out = static_cast<float *>(out->data); ga.ldo = out->ld;
    ga.H = H; ga.additive = 1; ga.slope = slope;
    cudaError_t e;
    if (Vt->cols == 8 * H && alpha->ld == H && gsp::gat_fused_supported(ga)) {
        e = gsp::launch_gat_fused(ga, cs);
    } else {   // any other shape: scores, softmax in place, weighted aggregate (same results within the bound)
        gsp::SddmmAddArgs sa{};
        sa.off = S.off; sa.col = S.col; sa.order = S.order; sa.task = S.task; sa.nrows = S.nrows;
        sa.n_heavy = S.n_heavy; sa.row_base = g->row_base;
        sa.el = ga.Y; sa.lde = el->ld; sa.er = ga.X; sa.ldr = er->ld;
        sa.out = ga.alpha; sa.ldo = alpha->ld; sa.H = H; sa.slope = slope;
        e = gsp::launch_sddmm_add(sa, cs);
        if (e == cudaSuccess) {
            gsp::SoftmaxArgs xa{};
            xa.off = S.off; xa.order = S.order; xa.task = S.task; xa.nrows = S.nrows; xa.n_heavy = S.n_heavy;
            xa.e = ga.alpha; xa.lde = alpha->ld; xa.out = ga.alpha; xa.ldo = alpha->ld; xa.H = H;
            e = gsp::launch_softmax(xa, cs);
        }
        if (e == cudaSuccess) {
            gsp::SpmmArgs wa{};
            wa.off = S.off; wa.col = S.col; wa.order = S.order; wa.task = S.task; wa.nrows = S.nrows; wa.n_heavy = S.n_heavy;
            wa.X = ga.Vt; wa.ldx = Vt->ld; wa.out = ga.out; wa.ldo = out->ld; wa.F = Vt->cols;
            wa.w = ga.alpha; wa.ldw = alpha->ld; wa.H = H; wa.Fh = Vt->cols / H > 0 ? Vt->cols / H : 1;
            e = gsp::launch_spmm(wa, gsp::kSpmmWeightedFwd, cs);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "gat_forward_additive launch");
    return GSP_OK;
}

// ------------------------------------------------ NEXT-3: Table 1 surface
gsp_status gsp_gspmm_reduce(const gsp_graph *g, const gsp_tensor *X, int reduce, gsp_tensor *out, int reverse,
                            gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    if (reduce < GSP_REDUCE_SUM || reduce > GSP_REDUCE_MAX) return fail(GSP_ERR_ARG, "reduce must be 0, 1 or 2");
    if (reduce == GSP_REDUCE_SUM) return gsp_gspmm(g, X, GSP_NORM_NONE, out, reverse, stream);
    if (reverse != 0 && reverse != 1) return fail(GSP_ERR_ARG, "reverse must be 0 or 1");
    const gsp::DevStructure &S = reverse ? g->rev : g->fwd;
    if (!S.present)
        return reverse ? fail(GSP_ERR_NO_REVERSE, "graph has no rev structure (GSP_BUILD_REVERSE)")
                       : fail(GSP_ERR_ARG, "this partition only serves reverse = 1");
    if (!X || !out) return fail(GSP_ERR_NULL, "X/out is NULL");
    if ((st = check_tensor(g, X, "X", S.ncols, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", S.nrows, X->cols)) != GSP_OK) return st;
    if (overlaps(X, out)) return fail(GSP_ERR_ALIAS, "out overlaps X");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SpmmArgs a{};
    a.off = S.off; a.col = S.col; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.X = static_cast<const float *>(X->data); a.ldx = X->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.F = X->cols; a.H = 1; a.Fh = X->cols > 0 ? X->cols : 1;
    cudaError_t e = gsp::launch_spmm(a, reduce == GSP_REDUCE_MIN ? gsp::kSpmmMin : gsp::kSpmmMax, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gspmm_reduce launch");
    return GSP_OK;
}

gsp_status gsp_gspmm_e(const gsp_graph *g, const gsp_tensor *w, int reduce, gsp_tensor *out, int reverse,
                       gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    if (reduce < GSP_REDUCE_SUM || reduce > GSP_REDUCE_MAX) return fail(GSP_ERR_ARG, "reduce must be 0, 1 or 2");
    if (reverse != 0 && reverse != 1) return fail(GSP_ERR_ARG, "reverse must be 0 or 1");
    const gsp::DevStructure &S = reverse ? (g->is_partition ? g->lrev : g->rev) : g->fwd;
    if (!S.present || (reverse && !S.eid))
        return reverse ? fail(GSP_ERR_NO_REVERSE, "no rev structure with edge ids on this graph")
                       : fail(GSP_ERR_ARG, "this partition only serves reverse = 1");
    if (!w || !out) return fail(GSP_ERR_NULL, "w/out is NULL");
    if ((st = check_tensor(g, w, "w", g->E, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", S.nrows, w->cols)) != GSP_OK) return st;
    if (overlaps(w, out)) return fail(GSP_ERR_ALIAS, "out overlaps w");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SpmmEArgs a{};
    a.off = S.off; a.eid = reverse ? S.eid : nullptr; a.order = S.order; a.task = reverse ? eid_task(S) : S.task;
    a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.w = static_cast<const float *>(w->data); a.ldw = w->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.H = w->cols; a.red = reduce;
    cudaError_t e = gsp::launch_spmm_e(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gspmm_e launch");
    return GSP_OK;
}

gsp_status gsp_gsddmm_ve(const gsp_graph *g, const gsp_tensor *X, const gsp_tensor *w, int op, int side,
                         gsp_tensor *out, gsp_stream stream) {
    gsp_status st;
    if ((st = check_compute_graph(g)) != GSP_OK) return st;
    if (op < GSP_OP_ADD || op > GSP_OP_DIV) return fail(GSP_ERR_ARG, "op must be 0..3");
    if (side != GSP_SIDE_DST && side != GSP_SIDE_SRC) return fail(GSP_ERR_ARG, "side must be 0 or 1");
    const gsp::DevStructure &S = g->fwd;
    if (!S.present) return fail(GSP_ERR_ARG, "gsddmm_ve needs the fwd structure (not a reverse partition)");
    if (!X || !w || !out) return fail(GSP_ERR_NULL, "X/w/out is NULL");
    if ((st = check_tensor(g, w, "w", g->E, -1)) != GSP_OK) return st;
    if ((st = check_tensor(g, X, "X", S.ncols, w->cols)) != GSP_OK) return st;
    if ((st = check_tensor(g, out, "out", g->E, w->cols)) != GSP_OK) return st;
    if (overlaps(X, out)) return fail(GSP_ERR_ALIAS, "out overlaps X");
    const bool same = w->data == out->data && w->ld == out->ld;
    if (!same && overlaps(w, out)) return fail(GSP_ERR_ALIAS, "out partially overlaps w");
    if ((st = check_stream(g, stream)) != GSP_OK) return st;
    DeviceGuard dg(g->device);
    gsp::SddmmVeArgs a{};
    a.off = S.off; a.col = S.col; a.order = S.order; a.task = S.task; a.nrows = S.nrows; a.n_heavy = S.n_heavy;
    a.row_base = g->row_base;
    a.X = static_cast<const float *>(X->data); a.ldx = X->ld;
    a.w = static_cast<const float *>(w->data); a.ldw = w->ld;
    a.out = static_cast<float *>(out->data); a.ldo = out->ld;
    a.H = w->cols; a.op = op; a.side_src = side;
    cudaError_t e = gsp::launch_sddmm_ve(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gsddmm_ve launch");
    return GSP_OK;
}

// -------------------------------------------------------------- partition
static void bounds_of(const std::vector<int64_t> &off, int64_t V, int nparts, int64_t *bounds) {
    const int64_t E = off[V];
    bounds[0] = 0;
    for (int p = 1; p < nparts; p++) {
        const int64_t target = (int64_t)(((__int128)p * E + nparts - 1) / nparts);  // ceil(p*E/P)
        bounds[p] = std::lower_bound(off.begin(), off.begin() + V + 1, target) - off.begin();
    }
    bounds[nparts] = V;
}

gsp_status gsp_partition_bounds(const gsp_graph *g, int nparts, int reverse, int64_t *bounds) {
    if (!g || !bounds) return fail(GSP_ERR_NULL, "graph/bounds is NULL");
    if (g->is_partition) return fail(GSP_ERR_ARG, "graph is already a partition");
    if (nparts < 1) return fail(GSP_ERR_ARG, "nparts must be >= 1");
    if (reverse != 0 && reverse != 1) return fail(GSP_ERR_ARG, "reverse must be 0 or 1");
    if (reverse && !g->host.has_rev) return fail(GSP_ERR_NO_REVERSE, "graph has no rev structure");
    bounds_of(reverse ? g->host.rev_off : g->host.fwd_off, g->host.V, nparts, bounds);
    return GSP_OK;
}

// Partition (part, chunk) of a full graph: sub-block q = part*nchunks + chunk of the
// nparts*nchunks edge-balanced C8 blocks, placed at padded slot chunk*nparts + part
// (chunk-major), so that for every chunk the nparts ranks' [R, F] outputs are one
// contiguous [nparts*R, F] range of the padded table (one all-gather per chunk).
static gsp_status partition_impl(const gsp_graph *g, int nparts, int nchunks, int part, int chunk, int device,
                                 uint32_t flags, gsp_graph **out) {
    if (!g || !out) return fail(GSP_ERR_NULL, "graph/out is NULL");
    *out = nullptr;
    if (g->is_partition) return fail(GSP_ERR_ARG, "graph is already a partition");
    if (nparts < 1 || part < 0 || part >= nparts) return fail(GSP_ERR_ARG, "need 0 <= part < nparts");
    if (nchunks < 1 || chunk < 0 || chunk >= nchunks) return fail(GSP_ERR_ARG, "need 0 <= chunk < nchunks");
    if ((int64_t)nparts * nchunks >= (int64_t(1) << 31)) return fail(GSP_ERR_ARG, "nparts * nchunks too large");
    if (flags & ~(uint32_t)GSP_PART_REVERSE) return fail(GSP_ERR_ARG, "unknown flags");
    if (device < -1) return fail(GSP_ERR_ARG, "device must be >= -1");
    const bool prev = (flags & GSP_PART_REVERSE) != 0;
    const gsp::HostGraph &h = g->host;
    if (prev && !h.has_rev) return fail(GSP_ERR_NO_REVERSE, "graph has no rev structure");
    if (device >= 0) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
            cudaGetLastError();
            return fail(GSP_ERR_ARG, "device " + std::to_string(device) + " not available");
        }
    }
    const std::vector<int64_t> &off = prev ? h.rev_off : h.fwd_off;
    const std::vector<int32_t> &col = prev ? h.rev_col : h.fwd_col;
    const int64_t V = h.V;
    const int Q = nparts * nchunks;
    std::vector<int64_t> b((size_t)Q + 1);
    bounds_of(off, V, Q, b.data());
    int64_t R = 0;
    for (int q = 0; q < Q; q++) R = std::max<int64_t>(R, b[q + 1] - b[q]);
    if ((__int128)Q * R >= ((__int128)1 << 31)) return fail(GSP_ERR_OVERFLOW, "padded column space >= 2^31");
    gsp_graph *pg = new (std::nothrow) gsp_graph();
    if (!pg) return fail(GSP_ERR_OOM, "host allocation failed");
    try {
        const int q0 = part * nchunks + chunk;
        auto slot = [&](int q) { return (int64_t)(q % nchunks) * nparts + q / nchunks; };
        const int64_t rb = b[q0], re = b[q0 + 1], nloc = re - rb, base = off[rb], row_base = slot(q0) * R;
        std::vector<int32_t> pmap((size_t)V);
        for (int q = 0; q < Q; q++)
            for (int64_t v = b[q]; v < b[q + 1]; v++) pmap[v] = q;
        auto padded = [&](int64_t v) { return slot(pmap[v]) * R + (v - b[pmap[v]]); };
        const int64_t NC = (int64_t)Q * R;
        pg->col_deg_fwd = g->col_deg_fwd;   // global degrees: the scales are the full graph's
        pg->col_deg_rev = g->col_deg_rev;
        gsp::HostGraph &lh = pg->host;
        lh.V = R;
        lh.E = off[re] - base;
        lh.fwd_off.resize((size_t)R + 1);
        for (int64_t r = 0; r <= R; r++) lh.fwd_off[r] = off[rb + std::min(r, nloc)] - base;
        lh.fwd_col.resize((size_t)lh.E);
        for (int64_t j = 0; j < lh.E; j++) lh.fwd_col[j] = (int32_t)padded(col[base + j]);
        if (!prev) {
            // local rev: this partition's edges grouped by padded source, stable in local edge id
            lh.rev_off.assign((size_t)NC + 1, 0);
            lh.rev_col.resize((size_t)lh.E);
            lh.rev_eid.resize((size_t)lh.E);
            for (int64_t j = 0; j < lh.E; j++) lh.rev_off[(size_t)lh.fwd_col[j] + 1]++;
            for (int64_t u = 0; u < NC; u++) lh.rev_off[u + 1] += lh.rev_off[u];
            std::vector<int64_t> pos(lh.rev_off.begin(), lh.rev_off.end() - 1);
            for (int64_t r = 0; r < nloc; r++)
                for (int64_t j = lh.fwd_off[r]; j < lh.fwd_off[r + 1]; j++) {
                    const int64_t k = pos[lh.fwd_col[j]]++;
                    lh.rev_col[k] = (int32_t)(row_base + r);
                    lh.rev_eid[k] = (int32_t)j;
                }
            lh.has_rev = true;
        }
        pg->is_partition = true;
        pg->nparts = nparts;
        pg->part = part;
        pg->nchunks = nchunks;
        pg->chunk = chunk;
        pg->part_reverse = prev ? 1 : 0;
        pg->row_begin = rb;
        pg->row_end = re;
        pg->R = R;
        pg->row_base = row_base;
        pg->nrows = R;
        pg->ncols = NC;
        pg->V_global = V;
        pg->E = lh.E;
        pg->symmetric = h.symmetric;
        pg->device = device;
        pg->edge_ids = g->edge_ids;
        if (device >= 0) {
            DeviceGuard dg(device);
            gsp_status st;
            // global degrees; d_out from rev_off or by counting fwd columns
            std::vector<int64_t> din = degrees_of(h.fwd_off), dout;
            if (h.has_rev) dout = degrees_of(h.rev_off);
            else {
                dout.assign((size_t)V, 0);
                for (int32_t u : h.fwd_col) dout[u]++;
            }
            std::vector<int64_t> loc_in((size_t)R, 1), loc_out((size_t)R, 1);
            std::vector<int64_t> pad_in((size_t)NC, 1), pad_out((size_t)NC, 1);
            for (int64_t r = 0; r < nloc; r++) { loc_in[r] = din[rb + r]; loc_out[r] = dout[rb + r]; }
            for (int64_t v = 0; v < V; v++) { pad_in[padded(v)] = din[v]; pad_out[padded(v)] = dout[v]; }
            const float *li_inv, *li_rsq, *lo_inv, *lo_rsq, *pi_inv, *pi_rsq, *po_inv, *po_rsq;
            if ((st = make_scales(pg, loc_in, &li_inv, &li_rsq)) != GSP_OK ||
                (st = make_scales(pg, loc_out, &lo_inv, &lo_rsq)) != GSP_OK ||
                (st = make_scales(pg, pad_in, &pi_inv, &pi_rsq)) != GSP_OK ||
                (st = make_scales(pg, pad_out, &po_inv, &po_rsq)) != GSP_OK) {
                std::string keep = g_detail;
                free_device(pg);
                delete pg;
                return fail(st, keep);
            }
            (void)lo_inv; (void)po_inv;
            gsp::DevStructure *fw = prev ? nullptr : &pg->fwd;
            if (fw) {
                st = upload_structure(pg, *fw, R, NC, lh.fwd_off, lh.fwd_col, nullptr, nullptr, 0, nullptr);
                if (st == GSP_OK) {
                    fw->row_scale[GSP_NORM_RIGHT] = li_inv;
                    fw->row_scale[GSP_NORM_BOTH] = li_rsq;
                    fw->col_scale[GSP_NORM_BOTH] = po_rsq;
                }
            }
            // rev view: a GSP_PART_REVERSE partition, or the shared topology of a symmetric graph
            if (st == GSP_OK && (prev || h.symmetric)) {
                if (prev)
                    st = upload_structure(pg, pg->rev, R, NC, lh.fwd_off, lh.fwd_col, nullptr, nullptr, 0, nullptr);
                else
                    st = upload_structure(pg, pg->rev, R, NC, lh.fwd_off, lh.fwd_col, nullptr, pg->fwd.order,
                                          pg->fwd.n_heavy, &pg->fwd);
                if (st == GSP_OK) {
                    pg->rev.eid = nullptr;  // weighted reverse on partitions: the lrev partials (below)
                    pg->rev.row_scale[GSP_NORM_BOTH] = lo_rsq;
                    pg->rev.col_scale[GSP_NORM_RIGHT] = pi_inv;
                    pg->rev.col_scale[GSP_NORM_BOTH] = pi_rsq;
                }
            }
            // local rev (fwd partitions): per-source partials of the weighted reverse
            // (explicit local edge ids) and, on a directed graph, of the scaled reverse
            // gSpMMv (rows = padded sources: s_src = d_out^-1/2, columns = this part's
            // destinations: s_dst = 1/d_in or d_in^-1/2).  GSP_BUILD_NO_EDGE_IDS keeps
            // only what the scaled reverse needs: nothing on a symmetric graph (its
            // reverse is the shared topology above), the topology on a directed one.
            if (st == GSP_OK && !prev && (g->edge_ids || !h.symmetric)) {
                st = upload_structure(pg, pg->lrev, NC, NC, lh.rev_off, lh.rev_col, g->edge_ids ? &lh.rev_eid : nullptr,
                                      nullptr, 0, nullptr);
                if (st == GSP_OK) {
                    pg->lrev.row_scale[GSP_NORM_BOTH] = po_rsq;
                    pg->lrev.col_scale[GSP_NORM_RIGHT] = pi_inv;
                    pg->lrev.col_scale[GSP_NORM_BOTH] = pi_rsq;
                }
            }
            if (st == GSP_OK && g->edge_scales && lh.E > 0) {
                pg->edge_scales = true;
                float *es = nullptr;
                if ((st = dev_alloc_f32(pg, (size_t)lh.E, &es, kEscale)) == GSP_OK) {
                    // fwd partition: column side = sources (d_out); reverse partition: destinations (d_in)
                    const gsp::DevStructure &own = prev ? pg->rev : pg->fwd;
                    cudaError_t e0 = gsp::launch_gather_scale(own.col, lh.E, prev ? pi_rsq : po_rsq, es, 0);
                    if (e0 != cudaSuccess) st = cuda_fail(e0, "edge scales");
                    if (prev) pg->rev.edge_scale[GSP_NORM_BOTH] = es;
                    else {
                        pg->fwd.edge_scale[GSP_NORM_BOTH] = es;
                        if (h.symmetric) pg->rev.edge_scale[GSP_NORM_BOTH] = es;   // same values (d_in == d_out)
                    }
                }
            }
            if (st == GSP_OK) {
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) st = cuda_fail(e, "partition upload");
            }
            if (st != GSP_OK) {
                std::string keep = g_detail;
                free_device(pg);
                delete pg;
                return fail(st, keep);
            }
        }
    } catch (const std::bad_alloc &) {
        free_device(pg);
        delete pg;
        return fail(GSP_ERR_OOM, "host allocation failed in partition");
    }
    *out = pg;
    return GSP_OK;
}

gsp_status gsp_graph_partition(const gsp_graph *g, int nparts, int part, int device, uint32_t flags,
                               gsp_graph **out) {
    return partition_impl(g, nparts, 1, part, 0, device, flags, out);
}

gsp_status gsp_graph_partition_chunked(const gsp_graph *g, int nparts, int nchunks, int part, int chunk, int device,
                                       uint32_t flags, gsp_graph **out) {
    return partition_impl(g, nparts, nchunks, part, chunk, device, flags, out);
}

gsp_status gsp_partition_chunk_info(const gsp_graph *g, int *nchunks, int *chunk, int64_t *row_base) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    if (nchunks) *nchunks = g->nchunks;
    if (chunk) *chunk = g->chunk;
    if (row_base) *row_base = g->row_base;
    return GSP_OK;
}

gsp_status gsp_graph_memory(const gsp_graph *g, int64_t *topology, int64_t *edge_ids, int64_t *edge_scales,
                            int64_t *vertex_arrays) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    if (topology) *topology = g->bytes_by[kTopo];
    if (edge_ids) *edge_ids = g->bytes_by[kEid];
    if (edge_scales) *edge_scales = g->bytes_by[kEscale];
    if (vertex_arrays) *vertex_arrays = g->bytes_by[kVertex];
    return GSP_OK;
}

gsp_status gsp_partition_info(const gsp_graph *g, int *nparts, int *part, int64_t *row_begin, int64_t *row_end,
                              int64_t *R, int64_t *ncols, int *reverse) {
    if (!g) return fail(GSP_ERR_NULL, "graph is NULL");
    if (nparts) *nparts = g->nparts;
    if (part) *part = g->part;
    if (row_begin) *row_begin = g->row_begin;
    if (row_end) *row_end = g->row_end;
    if (R) *R = g->R;
    if (ncols) *ncols = g->ncols;
    if (reverse) *reverse = g->part_reverse;
    return GSP_OK;
}

}  // extern "C"
