"""Thin ctypes binding of libgsp.so (include/gsp.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only turns torch tensors into ``gsp_tensor`` descriptors (the paper's
"Half DLPack" borrowing: pointer + shape, no ownership), allocates
outputs when the caller passes none (as GraphPy-Workflow does) and maps
status codes to exceptions.  There is no CPU fallback: if the shared library
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# GSP_LIB_OVERRIDE: another in-tree build of the same library (A/B timing tools only)
_SO = os.environ.get("GSP_LIB_OVERRIDE") or os.path.join(_PKG, "libgsp.so")

NORM_NONE, NORM_RIGHT, NORM_BOTH = 0, 1, 2
REDUCE_SUM, REDUCE_MIN, REDUCE_MAX = 0, 1, 2
OP_ADD, OP_SUB, OP_MUL, OP_DIV = 0, 1, 2, 3
SIDE_DST, SIDE_SRC = 0, 1
BUILD_REVERSE, BUILD_SHARE_SYMMETRIC, BUILD_EDGE_SCALES, BUILD_L2_PERSIST, BUILD_NO_EDGE_IDS = 1, 2, 4, 8, 16
PART_REVERSE = 1

STATUS = {0: "GSP_OK", 1: "GSP_ERR_NULL", 2: "GSP_ERR_ARG", 3: "GSP_ERR_VERTEX_RANGE", 4: "GSP_ERR_SHAPE",
          5: "GSP_ERR_ALIAS", 6: "GSP_ERR_NO_REVERSE", 7: "GSP_ERR_OVERFLOW", 8: "GSP_ERR_OOM", 9: "GSP_ERR_CUDA"}

# the exported C symbols (include/gsp.h), checked by tests/test_abi.py
SYMBOLS = ["gsp_graph_create", "gsp_graph_destroy", "gsp_graph_info", "gsp_graph_export", "gsp_gspmm",
           "gsp_gspmm_weighted", "gsp_gsddmm", "gsp_edge_softmax", "gsp_edge_softmax_backward",
           "gsp_gat_forward", "gsp_gat_backward_scores", "gsp_gspmm_reduce", "gsp_gspmm_e", "gsp_gsddmm_ve", "gsp_partition_bounds", "gsp_graph_partition",
           "gsp_graph_partition_chunked", "gsp_partition_chunk_info", "gsp_graph_memory",
           "gsp_gsddmm_add_leaky", "gsp_gat_forward_additive",
           "gsp_partition_info", "gsp_status_string", "gsp_last_error_detail", "gsp_version"]


class gsp_tensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("ld", ctypes.c_int64)]


class GspError(RuntimeError):
    def __init__(self, status, detail):
        self.status = status
        self.name = STATUS.get(status, f"GSP_ERR_{status}")
        super().__init__(f"{self.name}: {detail}")


def _load():
    if not os.path.exists(_SO):
        raise ImportError(f"libgsp.so not built ({_SO}); run __graft_entry__.build() "
                          f"or python paper_2402_03548_b200/_build.py")
    lib = ctypes.CDLL(_SO)
    p, i64, u32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int
    P = ctypes.POINTER
    T = P(gsp_tensor)
    sig = {
        "gsp_graph_create": ([i64, i64, p, p, u32, ci, P(p)], ci),
        "gsp_graph_destroy": ([p], ci),
        "gsp_graph_info": ([p, P(i64), P(i64), P(i64), P(ci)], ci),
        "gsp_graph_export": ([p, p, p, p, p, p, p], ci),
        "gsp_gspmm": ([p, T, ci, T, ci, p], ci),
        "gsp_gspmm_weighted": ([p, T, T, T, ci, p], ci),
        "gsp_gsddmm": ([p, T, T, T, p], ci),
        "gsp_edge_softmax": ([p, T, T, p], ci),
        "gsp_edge_softmax_backward": ([p, T, T, T, p], ci),
        "gsp_gat_forward": ([p, T, T, T, T, T, p], ci),
        "gsp_gat_backward_scores": ([p, T, T, T, T, p], ci),
        "gsp_gspmm_reduce": ([p, T, ci, T, ci, p], ci),
        "gsp_gspmm_e": ([p, T, ci, T, ci, p], ci),
        "gsp_gsddmm_ve": ([p, T, T, ci, ci, T, p], ci),
        "gsp_partition_bounds": ([p, ci, ci, p], ci),
        "gsp_graph_partition": ([p, ci, ci, ci, u32, P(p)], ci),
        "gsp_graph_partition_chunked": ([p, ci, ci, ci, ci, ci, u32, P(p)], ci),
        "gsp_partition_chunk_info": ([p, P(ci), P(ci), P(i64)], ci),
        "gsp_graph_memory": ([p, P(i64), P(i64), P(i64), P(i64)], ci),
        "gsp_gsddmm_add_leaky": ([p, T, T, ctypes.c_float, T, p], ci),
        "gsp_gat_forward_additive": ([p, T, T, T, ctypes.c_float, T, T, p], ci),
        "gsp_partition_info": ([p, P(ci), P(ci), P(i64), P(i64), P(i64), P(i64), P(ci)], ci),
        "gsp_status_string": ([ci], ctypes.c_char_p),
        "gsp_last_error_detail": ([], ctypes.c_char_p),
        "gsp_version": ([], ci),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def _check(st):
    if st != 0:
        raise GspError(st, lib.gsp_last_error_detail().decode())


def _desc(t):
    """gsp_tensor for a 2-D fp32 torch tensor with unit column stride."""
    import torch
    if t.dtype != torch.float32:
        raise TypeError("gsp tensors are fp32")
    if t.dim() != 2:
        raise ValueError("gsp tensors are 2-D [rows, cols]")
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise ValueError("gsp tensors need unit column stride")
    if t.shape[0] > 1:
        # the row stride goes through unchanged: a broadcast / overlapping-row view
        # (stride(0) < cols, e.g. expand()) is rejected here and by the library's SHAPE check
        if t.stride(0) < t.shape[1]:
            raise ValueError(f"gsp tensors need row stride >= cols (got stride {t.stride(0)} for "
                             f"{t.shape[1]} columns: broadcast or overlapping rows)")
        ld = t.stride(0)
    else:   # a single row: any stride is valid, report the tightest one
        ld = max(t.shape[1], t.stride(0))
    return gsp_tensor(t.data_ptr(), t.shape[0], t.shape[1], ld)


def _stream(stream, device):
    import torch
    if stream is None:
        # a host tensor is rejected by the library (GSP_ERR_ARG); pick any valid stream
        stream = torch.cuda.current_stream(device if device.type == "cuda" else None)
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class Graph:
    """Kernel-graph handle (GraphPy's `g`) owning a libgsp graph."""

    def __init__(self, V=None, src=None, dst=None, *, reverse=True, share_symmetric=True, edge_scales=True,
                 l2_persist=False, edge_ids=True, device=0, _handle=None):
        self._h = ctypes.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            src = np.ascontiguousarray(np.asarray(src), dtype=np.int64)
            dst = np.ascontiguousarray(np.asarray(dst), dtype=np.int64)
            if src.shape != dst.shape or src.ndim != 1:
                raise ValueError("src and dst must be 1-D arrays of equal length")
            flags = (BUILD_REVERSE if reverse else 0) | (BUILD_SHARE_SYMMETRIC if share_symmetric else 0) | \
                (BUILD_EDGE_SCALES if edge_scales else 0) | (BUILD_L2_PERSIST if l2_persist else 0) | \
                (0 if edge_ids else BUILD_NO_EDGE_IDS)
            _check(lib.gsp_graph_create(int(V), src.shape[0], src.ctypes.data, dst.ctypes.data, flags,
                                        int(device), ctypes.byref(self._h)))
        V_, E_, b_, s_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _check(lib.gsp_graph_info(self._h, ctypes.byref(V_), ctypes.byref(E_), ctypes.byref(b_), ctypes.byref(s_)))
        self.V, self.E, self.device_bytes, self.symmetric = V_.value, E_.value, b_.value, bool(s_.value)
        info = self.partition_info()
        self.nparts, self.part, self.row_begin, self.row_end, self.R, self.ncols, self.part_reverse = info
        nc, ch, rb = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(lib.gsp_partition_chunk_info(self._h, ctypes.byref(nc), ctypes.byref(ch), ctypes.byref(rb)))
        self.nchunks, self.chunk, self.row_base = nc.value, ch.value, rb.value
        self.is_partition = _handle is not None   # handles come from partition()
        self.device = device

    def close(self):
        if self._h:
            lib.gsp_graph_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------- structure
    def export(self, rev=True, coo=True):
        n = self.V
        nr = self.ncols   # full graph: V; fwd partition: local rev over the padded sources
        out = {"fwd_off": np.empty(n + 1, np.int64), "fwd_col": np.empty(self.E, np.int32)}
        if rev:
            out.update(rev_off=np.empty(nr + 1, np.int64), rev_col=np.empty(self.E, np.int32),
                       rev_eid=np.empty(self.E, np.int32))
        if coo:
            out["coo_to_eid"] = np.empty(self.E, np.int32)
        g = lambda k: out[k].ctypes.data if k in out else None
        _check(lib.gsp_graph_export(self._h, g("fwd_off"), g("fwd_col"), g("rev_off"), g("rev_col"), g("rev_eid"),
                                    g("coo_to_eid")))
        return out

    def partition_info(self):
        a = [ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(),
             ctypes.c_int()]
        _check(lib.gsp_partition_info(self._h, *[ctypes.byref(x) for x in a]))
        return tuple(x.value for x in a)

    def partition_bounds(self, nparts, reverse=False):
        b = np.empty(nparts + 1, np.int64)
        _check(lib.gsp_partition_bounds(self._h, int(nparts), int(bool(reverse)), b.ctypes.data))
        return b

    def partition(self, nparts, part, device=0, reverse=False, nchunks=1, chunk=0):
        """Partition `part` of `nparts` (gsp_graph_partition); with nchunks > 1 the
        chunk `chunk` of it in the chunk-major padded layout (gsp_graph_partition_chunked)."""
        h = ctypes.c_void_p()
        _check(lib.gsp_graph_partition_chunked(self._h, int(nparts), int(nchunks), int(part), int(chunk),
                                               int(device), PART_REVERSE if reverse else 0, ctypes.byref(h)))
        return Graph(_handle=h, device=device)

    def memory(self):
        """Device bytes by kind (gsp_graph_memory): topology, edge_ids, edge_scales, vertex_arrays."""
        a = [ctypes.c_int64() for _ in range(4)]
        _check(lib.gsp_graph_memory(self._h, *[ctypes.byref(x) for x in a]))
        return dict(zip(("topology", "edge_ids", "edge_scales", "vertex_arrays"), (x.value for x in a)))

    # ------------------------------------------------------------ compute
    def _alloc(self, rows, cols, like):
        import torch
        return torch.empty((rows, cols), dtype=torch.float32, device=like.device)

    def reverse_gives_partials(self):
        """reverse = 1 gSpMMv on this graph yields per-source partials [ncols, F]
        (a fwd partition of a directed graph; gsp.h gsp_graph_partition)."""
        return self.is_partition and not self.part_reverse and not self.symmetric

    def gspmm(self, X, norm=NORM_BOTH, out=None, reverse=False, stream=None):
        if out is None:
            rows = self.ncols if (reverse and self.reverse_gives_partials()) else self.V
            out = self._alloc(rows, X.shape[1], X)
        dx, do = _desc(X), _desc(out)
        _check(lib.gsp_gspmm(self._h, ctypes.byref(dx), int(norm), ctypes.byref(do), int(bool(reverse)),
                             _stream(stream, X.device)))
        return out

    def gspmm_weighted(self, X, w, out=None, reverse=False, stream=None):
        if out is None:
            rows = self.ncols if reverse else self.V   # fwd partition, reverse: per-source partials
            out = self._alloc(rows, X.shape[1], X)
        dx, dw, do = _desc(X), _desc(w), _desc(out)
        _check(lib.gsp_gspmm_weighted(self._h, ctypes.byref(dx), ctypes.byref(dw), ctypes.byref(do),
                                      int(bool(reverse)), _stream(stream, X.device)))
        return out

    def gsddmm(self, X, Y, H=None, out=None, stream=None):
        if out is None:
            out = self._alloc(self.E, 1 if H is None else H, X)
        dx, dy, do = _desc(X), _desc(Y), _desc(out)
        _check(lib.gsp_gsddmm(self._h, ctypes.byref(dx), ctypes.byref(dy), ctypes.byref(do),
                              _stream(stream, X.device)))
        return out

    def edge_softmax(self, e, out=None, stream=None):
        if out is None:
            out = self._alloc(self.E, e.shape[1], e)
        de, do = _desc(e), _desc(out)
        _check(lib.gsp_edge_softmax(self._h, ctypes.byref(de), ctypes.byref(do), _stream(stream, e.device)))
        return out


def _edge_softmax_backward(self, alpha, dalpha, out=None, stream=None):
    if out is None:
        out = self._alloc(self.E, alpha.shape[1], alpha)
    da, dd, do = _desc(alpha), _desc(dalpha), _desc(out)
    _check(lib.gsp_edge_softmax_backward(self._h, ctypes.byref(da), ctypes.byref(dd), ctypes.byref(do),
                                         _stream(stream, alpha.device)))
    return out


Graph.edge_softmax_backward = _edge_softmax_backward


def _gat_forward(self, X, Y, Vt, H, alpha=None, out=None, stream=None):
    """alpha = edge_softmax(gsddmm(X, Y)); out = gspmm_weighted(Vt, alpha) -- fused (NEXT-2)."""
    if alpha is None:
        alpha = self._alloc(self.E, H, X)
    if out is None:
        out = self._alloc(self.V, Vt.shape[1], X)
    dx, dy, dv, da, do = _desc(X), _desc(Y), _desc(Vt), _desc(alpha), _desc(out)
    _check(lib.gsp_gat_forward(self._h, ctypes.byref(dx), ctypes.byref(dy), ctypes.byref(dv), ctypes.byref(da),
                               ctypes.byref(do), _stream(stream, X.device)))
    return alpha, out


Graph.gat_forward = _gat_forward


def _gat_backward_scores(self, dOut, Vt, alpha, out=None, stream=None):
    """ds = edge_softmax_backward(alpha, gsddmm(dOut, Vt)) -- fused (NEXT-1)."""
    if out is None:
        out = self._alloc(self.E, alpha.shape[1], alpha)
    dd, dv, da, do = _desc(dOut), _desc(Vt), _desc(alpha), _desc(out)
    _check(lib.gsp_gat_backward_scores(self._h, ctypes.byref(dd), ctypes.byref(dv), ctypes.byref(da),
                                       ctypes.byref(do), _stream(stream, alpha.device)))
    return out


Graph.gat_backward_scores = _gat_backward_scores


def _gspmm_reduce(self, X, reduce, out=None, reverse=False, stream=None):
    if out is None:
        out = self._alloc(self.V, X.shape[1], X)
    dx, do = _desc(X), _desc(out)
    _check(lib.gsp_gspmm_reduce(self._h, ctypes.byref(dx), int(reduce), ctypes.byref(do), int(bool(reverse)),
                                _stream(stream, X.device)))
    return out


def _gspmm_e(self, w, reduce, out=None, reverse=False, stream=None):
    if out is None:
        out = self._alloc(self.ncols if reverse else self.V, w.shape[1], w)
    dw, do = _desc(w), _desc(out)
    _check(lib.gsp_gspmm_e(self._h, ctypes.byref(dw), int(reduce), ctypes.byref(do), int(bool(reverse)),
                           _stream(stream, w.device)))
    return out


def _gsddmm_ve(self, X, w, op, side, out=None, stream=None):
    if out is None:
        out = self._alloc(self.E, w.shape[1], w)
    dx, dw, do = _desc(X), _desc(w), _desc(out)
    _check(lib.gsp_gsddmm_ve(self._h, ctypes.byref(dx), ctypes.byref(dw), int(op), int(side), ctypes.byref(do),
                             _stream(stream, w.device)))
    return out


def _gsddmm_add_leaky(self, el, er, slope=0.2, out=None, stream=None):
    """out[j,h] = leaky_relu(el[u_j,h] + er[v,h], slope) -- additive GAT scores (NEXT-3)."""
    if out is None:
        out = self._alloc(self.E, el.shape[1], el)
    de, dr, do = _desc(el), _desc(er), _desc(out)
    _check(lib.gsp_gsddmm_add_leaky(self._h, ctypes.byref(de), ctypes.byref(dr), float(slope), ctypes.byref(do),
                                    _stream(stream, el.device)))
    return out


def _gat_forward_additive(self, el, er, Vt, slope=0.2, alpha=None, out=None, stream=None):
    """alpha = edge_softmax(gsddmm_add_leaky(el, er)); out = gspmm_weighted(Vt, alpha) -- fused."""
    if alpha is None:
        alpha = self._alloc(self.E, el.shape[1], el)
    if out is None:
        out = self._alloc(self.V, Vt.shape[1], el)
    de, dr, dv, da, do = _desc(el), _desc(er), _desc(Vt), _desc(alpha), _desc(out)
    _check(lib.gsp_gat_forward_additive(self._h, ctypes.byref(de), ctypes.byref(dr), ctypes.byref(dv), float(slope),
                                        ctypes.byref(da), ctypes.byref(do), _stream(stream, el.device)))
    return alpha, out


Graph.gsddmm_add_leaky = _gsddmm_add_leaky
Graph.gat_forward_additive = _gat_forward_additive
Graph.gspmm_reduce = _gspmm_reduce
Graph.gspmm_e = _gspmm_e
Graph.gsddmm_ve = _gsddmm_ve


def version():
    v = lib.gsp_version()
    return (v >> 16, v & 0xFFFF)
