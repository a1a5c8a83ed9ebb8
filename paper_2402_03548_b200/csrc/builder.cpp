// Host graph builder (GraphPy-SM's role): COO -> fwd
// (CSR, rows = destinations, implicit consecutive edge IDs) + rev (CSC, rows =
// sources, explicit edge-ID array) -- P:2001-2005 §Storage Format.
//
// Order (L6): fwd slots sorted by (dst, src, input position); rev
// slots sorted by (src, dst, edge ID).  Both are produced by LSD stable
// counting sorts, parallel over contiguous chunks with per-chunk histograms, so
// the result is identical for any thread count ("deterministic").
#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <thread>

#include "graph.h"

namespace gsp {
namespace {

int pick_threads(int64_t n, int64_t nkeys) {
    unsigned hc = std::thread::hardware_concurrency();
    int t = (int)std::min<unsigned>(hc ? hc : 1, 16);
    if (n < (1 << 16)) t = 1;
    // keep the per-thread histograms (t * nkeys * 4 B) under ~2 GB
    while (t > 1 && (double)t * (double)nkeys * 4.0 > 2e9) t--;
    return std::max(t, 1);
}

template <class F>
void parallel_for(int nthreads, int64_t n, F &&fn) {  // fn(tid, begin, end)
    if (nthreads <= 1) { fn(0, 0, n); return; }
    std::vector<std::thread> th;
    th.reserve(nthreads);
    for (int t = 0; t < nthreads; t++) {
        int64_t b = n * t / nthreads, e = n * (t + 1) / nthreads;
        th.emplace_back([&, t, b, e] { fn(t, b, e); });
    }
    for (auto &x : th) x.join();
}

// Stable counting sort of the sequence item(0..n-1) by key(t) in [0, nkeys):
// out[...] receives item(t) in key order, ties in sequence order.  Also
// returns the per-key totals in `count` (size nkeys) when non-null.
template <class KeyF, class ItemF>
bool stable_counting_sort(int64_t n, int64_t nkeys, KeyF key, ItemF item, int32_t *out,
                          std::vector<int64_t> *count) {
    int T = pick_threads(n, nkeys);
    std::vector<uint32_t> hist;
    try {
        hist.assign((size_t)T * (size_t)nkeys, 0u);
    } catch (...) {
        return false;
    }
    parallel_for(T, n, [&](int t, int64_t b, int64_t e) {
        uint32_t *h = hist.data() + (size_t)t * nkeys;
        for (int64_t i = b; i < e; i++) h[key(i)]++;
    });
    if (count) count->assign((size_t)nkeys, 0);
    // exclusive positions, key-major then chunk order (stability)
    uint32_t run = 0;
    for (int64_t k = 0; k < nkeys; k++) {
        uint32_t tot = 0;
        for (int t = 0; t < T; t++) {
            uint32_t c = hist[(size_t)t * nkeys + k];
            hist[(size_t)t * nkeys + k] = run;
            run += c;
            tot += c;
        }
        if (count) (*count)[k] = tot;
    }
    parallel_for(T, n, [&](int t, int64_t b, int64_t e) {
        uint32_t *pos = hist.data() + (size_t)t * nkeys;
        for (int64_t i = b; i < e; i++) out[pos[key(i)]++] = item(i);
    });
    return true;
}

}  // namespace

gsp_status build_host_graph(int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                            bool want_rev, HostGraph &hg, std::string &detail) {
    // validation (before any allocation of the structure)
    {
        int T = pick_threads(E, 1);
        std::atomic<int64_t> bad{-1};
        parallel_for(T, E, [&](int, int64_t b, int64_t e) {
            for (int64_t i = b; i < e; i++) {
                if (src[i] < 0 || src[i] >= V || dst[i] < 0 || dst[i] >= V) {
                    int64_t cur = bad.load();
                    while ((cur < 0 || i < cur) && !bad.compare_exchange_weak(cur, i)) {}
                    return;
                }
            }
        });
        if (bad.load() >= 0) {
            int64_t i = bad.load();
            detail = "edge " + std::to_string(i) + " (" + std::to_string(src[i]) + " -> " +
                     std::to_string(dst[i]) + ") outside [0, " + std::to_string(V) + ")";
            return GSP_ERR_VERTEX_RANGE;
        }
    }
    try {
        hg.V = V;
        hg.E = E;
        hg.fwd_off.assign((size_t)V + 1, 0);
        hg.fwd_col.resize((size_t)E);
        hg.coo_to_eid.resize((size_t)E);
        std::vector<int32_t> perm((size_t)E), order((size_t)E);
        std::vector<int64_t> cnt;
        // pass 1: positions stably by src; pass 2: that sequence stably by dst
        // => order = positions sorted by (dst, src, position)
        if (!stable_counting_sort(E, V, [&](int64_t i) { return src[i]; },
                                  [&](int64_t i) { return (int32_t)i; }, perm.data(), nullptr))
            return GSP_ERR_OOM;
        if (!stable_counting_sort(E, V, [&](int64_t t) { return dst[perm[t]]; },
                                  [&](int64_t t) { return perm[t]; }, order.data(), &cnt))
            return GSP_ERR_OOM;
        for (int64_t v = 0; v < V; v++) hg.fwd_off[v + 1] = hg.fwd_off[v] + cnt[v];
        {
            int T = pick_threads(E, 1);
            parallel_for(T, E, [&](int, int64_t b, int64_t e) {
                for (int64_t j = b; j < e; j++) {
                    int32_t i = order[j];
                    hg.fwd_col[j] = (int32_t)src[i];
                    hg.coo_to_eid[i] = (int32_t)j;
                }
            });
        }
        hg.has_rev = want_rev;
        hg.symmetric = false;
        if (want_rev) {
            // slot destinations (row of slot j), reuse `perm` storage
            std::vector<int32_t> &slot_dst = perm;
            {
                int T = pick_threads(E, 1);
                parallel_for(T, E, [&](int, int64_t b, int64_t e) {
                    for (int64_t j = b; j < e; j++) slot_dst[j] = (int32_t)dst[order[j]];
                });
            }
            hg.rev_eid.resize((size_t)E);
            hg.rev_col.resize((size_t)E);
            hg.rev_off.assign((size_t)V + 1, 0);
            // slots j (already in (dst, src, pos) order) stably by src => (src, dst, j)
            if (!stable_counting_sort(E, V, [&](int64_t j) { return (int64_t)hg.fwd_col[j]; },
                                      [&](int64_t j) { return (int32_t)j; }, hg.rev_eid.data(), &cnt))
                return GSP_ERR_OOM;
            for (int64_t u = 0; u < V; u++) hg.rev_off[u + 1] = hg.rev_off[u] + cnt[u];
            int T = pick_threads(E, 1);
            parallel_for(T, E, [&](int, int64_t b, int64_t e) {
                for (int64_t k = b; k < e; k++) hg.rev_col[k] = slot_dst[hg.rev_eid[k]];
            });
            bool sym = hg.rev_off == hg.fwd_off;
            if (sym) {
                std::atomic<bool> same{true};
                parallel_for(T, E, [&](int, int64_t b, int64_t e) {
                    if (std::memcmp(hg.rev_col.data() + b, hg.fwd_col.data() + b,
                                    sizeof(int32_t) * (size_t)(e - b)) != 0)
                        same = false;
                });
                sym = same.load();
            }
            hg.symmetric = sym;
        }
    } catch (const std::bad_alloc &) {
        detail = "host allocation failed in graph build";
        return GSP_ERR_OOM;
    }
    return GSP_OK;
}

void degree_order(const int64_t *off, int64_t nrows, int64_t heavy_threshold,
                  std::vector<int32_t> &order, int64_t &n_heavy) {
    order.resize((size_t)nrows);
    for (int64_t r = 0; r < nrows; r++) order[r] = (int32_t)r;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
        return da != db ? da > db : a < b;
    });
    n_heavy = 0;
    while (n_heavy < nrows && off[order[n_heavy] + 1] - off[order[n_heavy]] > heavy_threshold) n_heavy++;
}

}  // namespace gsp
