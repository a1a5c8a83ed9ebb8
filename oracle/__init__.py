"""CPU oracle for the GraphPy sparse hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2402_03548_b200``) never imports it and shares no code with
it.  The arithmetic lives in ``oracle.c`` (plain single-threaded C, fp64
accumulation); this module only marshals numpy arrays through ctypes.

Parity is pinned for every function (tests/test_oracle.py); see the header of
oracle.c and DESIGN.md "Oracle".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

NORM_NONE, NORM_RIGHT, NORM_BOTH = 0, 1, 2
RED_SUM, RED_MIN, RED_MAX = 0, 1, 2
OP_ADD, OP_SUB, OP_MUL, OP_DIV = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, no fast-math: IEEE fp64 throughout)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        ci = ctypes.c_int
        lib.oracle_build.argtypes = [i64, i64, p, p, p, p, p, p, p, p]
        lib.oracle_build.restype = ci
        lib.oracle_scales.argtypes = [i64, p, p, ci, p, p]
        lib.oracle_scales.restype = None
        lib.oracle_gspmm.argtypes = [i64, p, p, p, p, p, i64, i64, ci, ci, i64, p, p, p]
        lib.oracle_gspmm.restype = ci
        lib.oracle_gspmm_weighted.argtypes = [i64, p, p, p, p, p, p, i64, i64, p, i64, ci, i64, p, p, p]
        lib.oracle_gspmm_weighted.restype = ci
        lib.oracle_gsddmm.argtypes = [i64, p, p, p, i64, p, i64, i64, i64, i64, p, p, p]
        lib.oracle_gsddmm.restype = ci
        lib.oracle_edge_softmax.argtypes = [i64, p, p, i64, i64, p, p]
        lib.oracle_edge_softmax.restype = ci
        lib.oracle_edge_softmax_backward.argtypes = [i64, p, p, p, i64, i64, p, p, p]
        lib.oracle_edge_softmax_backward.restype = ci
        lib.oracle_gat_forward.argtypes = [i64, p, p, p, i64, p, i64, i64, p, i64, i64, i64, p, p, p, p]
        lib.oracle_gat_forward.restype = ci
        lib.oracle_gspmm_reduce.argtypes = [i64, p, p, p, p, p, i64, i64, ci, ci, p, p]
        lib.oracle_gspmm_reduce.restype = ci
        lib.oracle_gspmm_e.argtypes = [i64, p, p, p, p, i64, ci, ci, p, p]
        lib.oracle_gspmm_e.restype = ci
        lib.oracle_gsddmm_ve.argtypes = [i64, p, p, p, p, i64, ci, ci, p]
        lib.oracle_gsddmm_ve.restype = ci
        lib.oracle_gspmm_rows_coo.argtypes = [i64, i64, p, p, p, i64, i64, ci, ci, i64, p, p, p]
        lib.oracle_gspmm_rows_coo.restype = ci
        lib.oracle_rows_coo.argtypes = [i64, i64, p, p, i64, p, p, p, p]
        lib.oracle_rows_coo.restype = ci
        lib.oracle_partition_bounds.argtypes = [i64, p, i64, p]
        lib.oracle_partition_bounds.restype = ci
        lib.oracle_partition_structure.argtypes = [i64, p, p, i64, p, i64, p, p]
        lib.oracle_partition_structure.restype = ci
        d = ctypes.c_double
        lib.oracle_gsddmm_add_leaky.argtypes = [i64, p, p, p, p, i64, i64, d, p]
        lib.oracle_gsddmm_add_leaky.restype = ci
        lib.oracle_gat_forward_additive.argtypes = [i64, p, p, p, p, i64, p, i64, i64, i64, d, p, p, p, p]
        lib.oracle_gat_forward_additive.restype = ci
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Graph:
    """The oracle's own build of a COO graph (C1).  Arrays are numpy."""

    def __init__(self, V, src, dst):
        src = _c(src, np.int64)
        dst = _c(dst, np.int64)
        E = int(src.shape[0])
        assert dst.shape[0] == E
        self.V, self.E = int(V), E
        self.fwd_off = np.empty(V + 1, np.int64)
        self.fwd_col = np.empty(E, np.int32)
        self.rev_off = np.empty(V + 1, np.int64)
        self.rev_col = np.empty(E, np.int32)
        self.rev_eid = np.empty(E, np.int32)
        self.coo_to_eid = np.empty(E, np.int32)
        rc = _L().oracle_build(V, E, _ptr(src), _ptr(dst), _ptr(self.fwd_off), _ptr(self.fwd_col),
                               _ptr(self.rev_off), _ptr(self.rev_col), _ptr(self.rev_eid),
                               _ptr(self.coo_to_eid))
        if rc == -1:
            raise ValueError("vertex id out of range")
        if rc != 0:
            raise MemoryError("oracle_build failed")

    # --- C2/C3
    def scales(self, norm):
        sd = np.empty(self.V, np.float64)
        ss = np.empty(self.V, np.float64)
        _L().oracle_scales(self.V, _ptr(self.fwd_off), _ptr(self.rev_off), norm, _ptr(sd), _ptr(ss))
        return sd, ss

    def _sel(self, rows):
        if rows is None:
            return 0, None, self.V
        rows = _c(rows, np.int64)
        return rows.shape[0], rows, rows.shape[0]

    # --- C4
    def gspmm(self, X, norm, reverse=False, rows=None, F=None):
        """Returns (out fp64 [n,F], T fp64 [n,F]); X is fp32 [V, ld] (first F columns used)."""
        X = _c(X, np.float32)
        F = X.shape[1] if F is None else F
        nsel, sel, n = self._sel(rows)
        out = np.empty((n, F), np.float64)
        T = np.empty((n, F), np.float64)
        rc = _L().oracle_gspmm(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(self.rev_off),
                               _ptr(self.rev_col), _ptr(X), F, X.shape[1], norm, int(bool(reverse)),
                               nsel, _ptr(sel), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    # --- C5
    def gspmm_weighted(self, X, w, reverse=False, rows=None, F=None):
        X = _c(X, np.float32)
        w = _c(w, np.float32)
        F = X.shape[1] if F is None else F
        H = w.shape[1]
        assert w.shape[0] == self.E
        nsel, sel, n = self._sel(rows)
        out = np.empty((n, F), np.float64)
        T = np.empty((n, F), np.float64)
        rc = _L().oracle_gspmm_weighted(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(self.rev_off),
                                        _ptr(self.rev_col), _ptr(self.rev_eid), _ptr(X), F, X.shape[1],
                                        _ptr(w), H, int(bool(reverse)), nsel, _ptr(sel), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    def _nedges(self, rows):
        if rows is None:
            return self.E
        rows = np.asarray(rows, np.int64)
        return int((self.fwd_off[rows + 1] - self.fwd_off[rows]).sum())

    # --- C6
    def gsddmm(self, X, Y, H, rows=None, F=None):
        """Returns (out [m,H], T [m,H]); m = E (rows None) or the selected rows' edges, packed."""
        X = _c(X, np.float32)
        Y = _c(Y, np.float32)
        F = X.shape[1] if F is None else F
        nsel, sel, _ = self._sel(rows)
        m = self._nedges(rows)
        out = np.empty((m, H), np.float64)
        T = np.empty((m, H), np.float64)
        rc = _L().oracle_gsddmm(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(X), X.shape[1],
                                _ptr(Y), Y.shape[1], F, H, nsel, _ptr(sel), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    # --- C7
    def edge_softmax(self, e, rows=None):
        e = _c(e, np.float32)
        H = e.shape[1]
        assert e.shape[0] == self.E
        nsel, sel, _ = self._sel(rows)
        m = self._nedges(rows)
        out = np.empty((m, H), np.float64)
        rc = _L().oracle_edge_softmax(self.V, _ptr(self.fwd_off), _ptr(e), H, nsel, _ptr(sel), _ptr(out))
        assert rc == 0, rc
        return out

    # --- C9 (NEXT-1)
    def edge_softmax_backward(self, alpha, dalpha, rows=None):
        alpha = _c(alpha, np.float32)
        dalpha = _c(dalpha, np.float32)
        H = alpha.shape[1]
        assert alpha.shape == dalpha.shape and alpha.shape[0] == self.E
        nsel, sel, _ = self._sel(rows)
        m = self._nedges(rows)
        out = np.empty((m, H), np.float64)
        T = np.empty((m, H), np.float64)
        rc = _L().oracle_edge_softmax_backward(self.V, _ptr(self.fwd_off), _ptr(alpha), _ptr(dalpha), H, nsel,
                                               _ptr(sel), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    # --- C10 (NEXT-2)
    def gat_forward(self, X, Y, Vt, H):
        """(alpha [E,H], out [V,Fv], T_out) in fp64: softmax(gsddmm(X,Y)) then weighted sum of Vt."""
        X = _c(X, np.float32)
        Y = _c(Y, np.float32)
        Vt = _c(Vt, np.float32)
        F, Fv = X.shape[1], Vt.shape[1]
        alpha = np.empty((self.E, H), np.float64)
        out = np.empty((self.V, Fv), np.float64)
        T = np.empty((self.V, Fv), np.float64)
        maxdeg = int(np.max(np.diff(self.fwd_off))) if self.V else 0
        scratch = np.empty(max(maxdeg, 1), np.float64)
        rc = _L().oracle_gat_forward(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(X), X.shape[1], _ptr(Y),
                                     Y.shape[1], F, _ptr(Vt), Vt.shape[1], Fv, H, _ptr(alpha), _ptr(out), _ptr(T),
                                     _ptr(scratch))
        assert rc == 0, rc
        return alpha, out, T

    # --- C14, C15 (NEXT-3: additive GAT attention)
    def gsddmm_add_leaky(self, el, er, slope=0.2):
        """C14: out[j,h] = leaky_relu(el[u_j,h] + er[v,h], slope) fp64 [E,H]; el/er fp32 [V,H]."""
        el = _c(el, np.float32)
        er = _c(er, np.float32)
        assert el.shape == er.shape
        H = el.shape[1]
        out = np.empty((self.E, H), np.float64)
        rc = _L().oracle_gsddmm_add_leaky(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(el), _ptr(er), H, H,
                                          float(slope), _ptr(out))
        assert rc == 0, rc
        return out

    def gat_forward_additive(self, el, er, Vt, slope=0.2):
        """C15: (alpha [E,H], out [V,Fv], T_out) in fp64: softmax(C14(el, er)) then weighted sum of Vt."""
        el = _c(el, np.float32)
        er = _c(er, np.float32)
        Vt = _c(Vt, np.float32)
        H, Fv = el.shape[1], Vt.shape[1]
        alpha = np.empty((self.E, H), np.float64)
        out = np.empty((self.V, Fv), np.float64)
        T = np.empty((self.V, Fv), np.float64)
        maxdeg = int(np.max(np.diff(self.fwd_off))) if self.V else 0
        scratch = np.empty(max(maxdeg, 1), np.float64)
        rc = _L().oracle_gat_forward_additive(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(el), _ptr(er), H,
                                              _ptr(Vt), Fv, Fv, H, float(slope), _ptr(alpha), _ptr(out), _ptr(T),
                                              _ptr(scratch))
        assert rc == 0, rc
        return alpha, out, T

    # --- C11-C13 (NEXT-3)
    def gspmm_reduce(self, X, red, reverse=False):
        X = _c(X, np.float32)
        F = X.shape[1]
        out = np.empty((self.V, F), np.float64)
        T = np.empty((self.V, F), np.float64)
        rc = _L().oracle_gspmm_reduce(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(self.rev_off),
                                      _ptr(self.rev_col), _ptr(X), F, F, red, int(bool(reverse)), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    def gspmm_e(self, w, red, reverse=False):
        w = _c(w, np.float32)
        H = w.shape[1]
        out = np.empty((self.V, H), np.float64)
        T = np.empty((self.V, H), np.float64)
        rc = _L().oracle_gspmm_e(self.V, _ptr(self.fwd_off), _ptr(self.rev_off), _ptr(self.rev_eid), _ptr(w), H,
                                 red, int(bool(reverse)), _ptr(out), _ptr(T))
        assert rc == 0, rc
        return out, T

    def gsddmm_ve(self, X, w, op, side_src):
        X = _c(X, np.float32)
        w = _c(w, np.float32)
        H = w.shape[1]
        assert X.shape[1] == H
        out = np.empty((self.E, H), np.float64)
        rc = _L().oracle_gsddmm_ve(self.V, _ptr(self.fwd_off), _ptr(self.fwd_col), _ptr(X), _ptr(w), H, op,
                                   int(bool(side_src)), _ptr(out))
        assert rc == 0, rc
        return out

    # --- C8
    def partition_bounds(self, nparts, reverse=False):
        b = np.empty(nparts + 1, np.int64)
        off = self.rev_off if reverse else self.fwd_off
        rc = _L().oracle_partition_bounds(self.V, _ptr(off), nparts, _ptr(b))
        assert rc == 0, rc
        return b

    def partition_structure(self, nparts, part, reverse=False):
        """(loc_off [R+1], loc_col, R, bounds) of partition `part` in the padded layout."""
        b = self.partition_bounds(nparts, reverse)
        R = int(np.max(b[1:] - b[:-1])) if nparts > 0 else 0
        off = self.rev_off if reverse else self.fwd_off
        col = self.rev_col if reverse else self.fwd_col
        ne = int(off[b[part + 1]] - off[b[part]])
        loc_off = np.empty(R + 1, np.int64)
        loc_col = np.empty(ne, np.int32)
        rc = _L().oracle_partition_structure(self.V, _ptr(off), _ptr(col), nparts, _ptr(b), part,
                                             _ptr(loc_off), _ptr(loc_col))
        assert rc == 0, rc
        return loc_off, loc_col, R, b

    def row_edges(self, rows):
        """Edge-ID slices of the given rows, concatenated (for packing GPU edge tensors)."""
        rows = np.asarray(rows, np.int64)
        return np.concatenate([np.arange(self.fwd_off[v], self.fwd_off[v + 1]) for v in rows]) \
            if len(rows) else np.zeros(0, np.int64)


def bound(T):
    """Acceptance bound of BASELINE.json: 1e-5 * (sum|terms| + 1) per element."""
    return 1e-5 * (np.asarray(T) + 1.0)


# ------------------------------------------------ row-sampled oracle from COO
def gspmm_rows_coo(V, src, dst, X, norm, rows, reverse=False, F=None):
    """C4 for the selected rows straight from the COO list (no build)."""
    src = _c(src, np.int64)
    dst = _c(dst, np.int64)
    X = _c(X, np.float32)
    F = X.shape[1] if F is None else F
    rows = _c(rows, np.int64)
    out = np.empty((len(rows), F), np.float64)
    T = np.empty((len(rows), F), np.float64)
    rc = _L().oracle_gspmm_rows_coo(V, len(src), _ptr(src), _ptr(dst), _ptr(X), F, X.shape[1], norm,
                                    int(bool(reverse)), len(rows), _ptr(rows), _ptr(out), _ptr(T))
    assert rc == 0, rc
    return out, T


def rows_coo(V, src, dst, rows):
    """C1 for the selected destination rows from the COO list: per row the
    sorted (src, position) pairs of its in-edges and its first fwd slot."""
    src = _c(src, np.int64)
    dst = _c(dst, np.int64)
    rows = _c(rows, np.int64)
    off = np.empty(len(rows) + 1, np.int64)
    first = np.empty(len(rows), np.int64)
    tot = int(sum(int(np.count_nonzero(dst == v)) for v in rows)) if len(src) < (1 << 24) else \
        int(np.bincount(dst, minlength=V)[rows].sum())
    pairs = np.empty(2 * max(tot, 1), np.int64)
    rc = _L().oracle_rows_coo(V, len(src), _ptr(dst), _ptr(src), len(rows), _ptr(rows), _ptr(off), _ptr(first),
                              _ptr(pairs))
    assert rc == 0, rc
    return [(int(first[r]), pairs[2 * off[r]:2 * off[r + 1]].reshape(-1, 2)) for r in range(len(rows))]
