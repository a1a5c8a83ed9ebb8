"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench).

Holds none of the method's arithmetic: it only draws COO edge lists and
feature matrices.  The five workload shapes are BASELINE.json's configs
(Cora-, Pubmed-, ogbn-arxiv-, Reddit-, ogbn-products-shaped; sizes as in
BASELINE.json, structure calibrated per SURVEY.md §8(d)); the recipe is stated
in DESIGN.md "Input recipe".  The C generator (gen.c) is compiled on first use
or by ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgspgen.so")
_SRC = os.path.join(_HERE, "gen.c")


def build(force: bool = False) -> str:
    """Compile gen.c into libgspgen.so (gcc, -O2)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, dbl, p64 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.gen_chung_lu.argtypes = [i64, i64, dbl, u64, p64, p64]
        lib.gen_chung_lu.restype = ctypes.c_int
        lib.gen_rmat.argtypes = [ctypes.c_int, i64, i64, dbl, dbl, dbl, u64, p64, p64]
        lib.gen_rmat.restype = ctypes.c_int
        lib.gen_kron.argtypes = [ctypes.c_int, i64, dbl, dbl, dbl, u64, p64, p64]
        lib.gen_kron.restype = ctypes.c_int
        lib.gen_uniform_f32.argtypes = [u64, i64, i64, i64, ctypes.c_float, ctypes.c_float, p64]
        lib.gen_uniform_f32.restype = None
        _lib = lib
    return _lib


def chung_lu(V: int, npairs: int, beta: float, seed: int):
    """Symmetric simple power-law graph: 2*npairs directed edges (int64 src, dst)."""
    src = np.empty(2 * npairs, dtype=np.int64)
    dst = np.empty(2 * npairs, dtype=np.int64)
    rc = _L().gen_chung_lu(V, npairs, beta, seed, src.ctypes.data, dst.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"gen_chung_lu failed rc={rc}")
    return src, dst


def rmat(scale: int, V: int, E: int, seed: int, a=0.57, b=0.19, c=0.19):
    """Directed simple R-MAT graph with exactly E edges, ids < V (int64 src, dst)."""
    src = np.empty(E, dtype=np.int64)
    dst = np.empty(E, dtype=np.int64)
    rc = _L().gen_rmat(scale, V, E, a, b, c, seed, src.ctypes.data, dst.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"gen_rmat failed rc={rc}")
    return src, dst


def kron(scale: int, npairs: int, seed: int, a=0.57, b=0.19, c=0.19):
    """Graph500-style Kronecker graph: 2*npairs directed edges (duplicates and
    self-loops kept), 2^scale vertices, seeded relabelling."""
    src = np.empty(2 * npairs, dtype=np.int64)
    dst = np.empty(2 * npairs, dtype=np.int64)
    rc = _L().gen_kron(scale, npairs, a, b, c, seed, src.ctypes.data, dst.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"gen_kron failed rc={rc}")
    return src, dst


def uniform(seed: int, rows: int, cols: int, ld: int | None = None, lo: float = -1.0, hi: float = 1.0,
            out: np.ndarray | None = None) -> np.ndarray:
    """Counter-based U[lo,hi) fp32 matrix [rows, ld] (padding columns are 0)."""
    ld = cols if ld is None else ld
    assert ld >= cols
    if out is None:
        out = np.empty((rows, ld), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (rows, ld)
    _L().gen_uniform_f32(seed, rows, cols, ld, lo, hi, out.ctypes.data)
    return out


def random_multigraph(V: int, E: int, seed: int, self_loops: bool = True):
    """Tiny random directed multigraph (duplicates and self-loops allowed) for brute-force tests."""
    rng = np.random.Generator(np.random.Philox(seed))
    src = rng.integers(0, V, size=E, dtype=np.int64) if V > 0 else np.zeros(0, np.int64)
    dst = rng.integers(0, V, size=E, dtype=np.int64) if V > 0 else np.zeros(0, np.int64)
    if not self_loops and V > 1:
        m = src == dst
        dst[m] = (dst[m] + 1) % V
    return src, dst


def skewed_multigraph(V: int, E: int, seed: int, alpha: float = 1.2):
    """Random directed multigraph with Zipf-skewed destinations (heavy rows) and sources."""
    rng = np.random.Generator(np.random.Philox(seed))
    w = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** alpha
    w /= w.sum()
    dst = rng.choice(V, size=E, p=w).astype(np.int64)
    src = rng.choice(V, size=E, p=w[::-1]).astype(np.int64)
    perm = rng.permutation(V).astype(np.int64)
    return perm[src], perm[dst]


# --------------------------------------------------------------- tiny graphs
def t4():
    """SPEC.md S:80-82 graph T4: undirected {(0,1),(0,2),(1,2),(2,3)}, |E|=8.
    COO order as SURVEY.md Appendix A: (0→1),(1→0),(0→2),(2→0),(1→2),(2→1),(2→3),(3→2)."""
    src = np.array([0, 1, 0, 2, 1, 2, 2, 3], dtype=np.int64)
    dst = np.array([1, 0, 2, 0, 2, 1, 3, 2], dtype=np.int64)
    return 4, src, dst


def d4():
    """SURVEY.md Appendix A graph D4: directed, a duplicate (e6 = e2), a self-loop (e5),
    vertex 3 has no in-edges."""
    src = np.array([0, 2, 0, 3, 1, 2, 0], dtype=np.int64)
    dst = np.array([1, 0, 2, 2, 2, 2, 2], dtype=np.int64)
    return 4, src, dst


# ---------------------------------------------------------- BASELINE configs
@dataclass(frozen=True)
class GraphConfig:
    name: str
    kind: str          # "chung_lu" | "rmat"
    V: int
    E: int             # directed edge count (BASELINE.json)
    beta: float = 0.0  # Chung-Lu exponent
    scale: int = 0     # R-MAT scale
    seed: int = 0
    F: int = 0         # feature width used by the config's ops
    ld: int = 0        # row stride of X (>= F)
    H: int = 0         # heads for the GAT chain (0 = no GAT ops)
    Fh: int = 0


CONFIGS = {
    # BASELINE.json configs[0..4]; seeds and Chung-Lu exponents per SURVEY.md §8(d)
    "cora": GraphConfig("cora", "chung_lu", 2708, 10556, beta=0.5832, seed=0xC04A, F=16, ld=16),
    "pubmed": GraphConfig("pubmed", "chung_lu", 19717, 88648, beta=0.4234, seed=0x9BED, F=64, ld=64, H=8, Fh=8),
    "arxiv": GraphConfig("arxiv", "rmat", 169343, 1166243, scale=18, seed=0xA5C1, F=128, ld=128),
    "reddit": GraphConfig("reddit", "chung_lu", 232965, 114615892, beta=0.3398, seed=0x2EDD, F=64, ld=64, H=8, Fh=8),
    "products": GraphConfig("products", "chung_lu", 2449029, 123718280, beta=0.4364, seed=0x960D, F=100, ld=100),
    # the paper's billion-edge Kron-25 (Table 2): Graph500 Kronecker,
    # 2^25 vertices, 2^29 draws emitted in both directions = 2^30 edges, F = 150 (ld 152)
    "kron25": GraphConfig("kron25", "kron", 1 << 25, 1 << 30, scale=25, seed=0xC125, F=150, ld=152),
}


def make_graph(cfg: GraphConfig | str):
    """(V, src, dst) for a BASELINE config (deterministic in cfg.seed)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.kind == "chung_lu":
        assert cfg.E % 2 == 0
        src, dst = chung_lu(cfg.V, cfg.E // 2, cfg.beta, cfg.seed)
    elif cfg.kind == "kron":
        src, dst = kron(cfg.scale, cfg.E // 2, cfg.seed)
    else:
        src, dst = rmat(cfg.scale, cfg.V, cfg.E, cfg.seed)
    return cfg.V, src, dst
