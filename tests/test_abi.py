"""C-ABI library checks that need no GPU: libgsp.so loads, exports every symbol
include/gsp.h declares, and its HOST logic (the graph builder, partition
bounds and padded partition structure of a device = -1 graph) is bit-exact
against the oracle.  No compute call runs here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import datagen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gsp():
    from conftest import build_lib
    build_lib()
    import paper_2402_03548_b200 as m
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gsp.h")).read()
    return sorted(set(re.findall(r"\b(gsp_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(gsp):
    declared = header_symbols()
    assert len(declared) >= 14
    nm = subprocess.run(["nm", "-D", "--defined-only", gsp.gsp._SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gsp_\w+)", nm))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(gsp.gsp.SYMBOLS) == declared
    for s in declared:
        getattr(gsp.lib, s)
    assert gsp.version() == (1, 0)


def test_status_strings(gsp):
    for code, name in gsp.gsp.STATUS.items():
        assert gsp.lib.gsp_status_string(code).decode() == name


def host_graph(gsp, V, src, dst, **kw):
    return gsp.Graph(V, src, dst, device=-1, **kw)


def assert_same_structure(G, og, rev=True):
    ex = G.export(rev=rev)
    assert np.array_equal(ex["fwd_off"], og.fwd_off)
    assert np.array_equal(ex["fwd_col"], og.fwd_col)
    assert np.array_equal(ex["coo_to_eid"], og.coo_to_eid)
    if rev:
        assert np.array_equal(ex["rev_off"], og.rev_off)
        assert np.array_equal(ex["rev_col"], og.rev_col)
        assert np.array_equal(ex["rev_eid"], og.rev_eid)


def test_build_golden(gsp, golden):
    for name in ("t4.json", "d4.json"):
        g = golden(name)
        G = host_graph(gsp, g["V"], g["src"], g["dst"])
        og = oracle.Graph(g["V"], g["src"], g["dst"])
        assert_same_structure(G, og)
        assert G.symmetric == (name == "t4.json")


@pytest.mark.parametrize("seed", range(40))
def test_build_random_bitexact(gsp, seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(1, 300))
    E = int(rng.integers(0, 3000))
    src, dst = datagen.random_multigraph(V, E, seed)
    G = host_graph(gsp, V, src, dst)
    assert_same_structure(G, oracle.Graph(V, src, dst))


@pytest.mark.parametrize("seed", range(4))
def test_build_skewed_multithreaded_bitexact(gsp, seed):
    # > 65536 edges: the builder's parallel counting sorts are used
    V, E = 5000, 200_000
    src, dst = datagen.skewed_multigraph(V, E, seed)
    G = host_graph(gsp, V, src, dst)
    assert_same_structure(G, oracle.Graph(V, src, dst))


@pytest.mark.parametrize("name", ["cora", "pubmed", "arxiv"])
def test_build_configs_bitexact(gsp, name):
    V, src, dst = datagen.make_graph(name)
    G = host_graph(gsp, V, src, dst)
    og = oracle.Graph(V, src, dst)
    assert_same_structure(G, og)
    assert G.symmetric == (name != "arxiv")


def test_build_without_reverse(gsp, golden):
    g = golden("d4.json")
    G = host_graph(gsp, g["V"], g["src"], g["dst"], reverse=False)
    ex = G.export(rev=False)
    assert ex["fwd_col"].tolist() == g["fwd_col"]
    with pytest.raises(gsp.GspError) as ei:
        G.export(rev=True)
    assert ei.value.name == "GSP_ERR_NO_REVERSE"


def test_share_symmetric_flag(gsp, golden):
    g = golden("t4.json")
    assert host_graph(gsp, g["V"], g["src"], g["dst"]).symmetric
    assert not host_graph(gsp, g["V"], g["src"], g["dst"], share_symmetric=False).symmetric


def test_build_errors(gsp):
    with pytest.raises(gsp.GspError) as ei:
        host_graph(gsp, 3, [0, 3], [1, 1])
    assert ei.value.name == "GSP_ERR_VERTEX_RANGE"
    with pytest.raises(gsp.GspError) as ei:
        host_graph(gsp, 3, [0, -1], [1, 1])
    assert ei.value.name == "GSP_ERR_VERTEX_RANGE"
    with pytest.raises(gsp.GspError) as ei:
        host_graph(gsp, 1 << 31, [0], [0])
    assert ei.value.name == "GSP_ERR_OVERFLOW"
    with pytest.raises(gsp.GspError) as ei:
        host_graph(gsp, -1, [], [])
    assert ei.value.name == "GSP_ERR_ARG"
    h = ctypes.c_void_p()
    assert gsp.lib.gsp_graph_create(3, 2, None, None, 0, -1, ctypes.byref(h)) == 1   # GSP_ERR_NULL
    assert gsp.lib.gsp_graph_create(3, 0, None, None, 1 << 7, -1, ctypes.byref(h)) == 2  # unknown flag
    assert gsp.lib.gsp_graph_destroy(None) == 0


def test_empty_graphs(gsp):
    G = host_graph(gsp, 5, np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert G.V == 5 and G.E == 0
    assert G.export()["fwd_off"].tolist() == [0] * 6
    G0 = host_graph(gsp, 0, np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert G0.export()["fwd_off"].tolist() == [0]


def test_compute_on_host_graph_is_rejected(gsp, golden):
    g = golden("t4.json")
    G = host_graph(gsp, g["V"], g["src"], g["dst"])
    t = gsp.gsp_tensor(None, 4, 1, 1)
    o = gsp.gsp_tensor(None, 4, 1, 1)
    st = gsp.lib.gsp_gspmm(G.handle, ctypes.byref(t), 2, ctypes.byref(o), 0, None)
    assert st == 2  # GSP_ERR_ARG: host-only graph
    assert "host-only" in gsp.lib.gsp_last_error_detail().decode()


# ---------------------------------------------------------------- partitions
def test_partition_bounds_golden(gsp, golden):
    for gf, cf in [("t4.json", "t4_chain.json"), ("d4.json", "d4.json")]:
        g, c = golden(gf), golden(cf)
        G = host_graph(gsp, g["V"], g["src"], g["dst"])
        for P, ref in c["partition_bounds"].items():
            assert G.partition_bounds(int(P)).tolist() == ref


@pytest.mark.parametrize("seed", range(15))
def test_partition_structure_bitexact(gsp, seed):
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(1, 200))
    E = int(rng.integers(0, 1500))
    src, dst = datagen.random_multigraph(V, E, seed)
    G = host_graph(gsp, V, src, dst)
    og = oracle.Graph(V, src, dst)
    for P in (1, 2, 3, 4, 8):
        for rev in (False, True):
            assert np.array_equal(G.partition_bounds(P, rev), og.partition_bounds(P, rev))
            for p in range(P):
                pg = G.partition(P, p, device=-1, reverse=rev)
                lo, lc, R, b = og.partition_structure(P, p, rev)
                ex = pg.export(rev=False, coo=False)
                assert np.array_equal(ex["fwd_off"], lo) and np.array_equal(ex["fwd_col"], lc)
                assert (pg.nparts, pg.part, pg.row_begin, pg.row_end, pg.R, pg.ncols, pg.part_reverse) == \
                    (P, p, b[p], b[p + 1], R, P * R, int(rev))


def test_partition_errors(gsp, golden):
    g = golden("d4.json")
    G = host_graph(gsp, g["V"], g["src"], g["dst"], reverse=False)
    with pytest.raises(gsp.GspError) as ei:
        G.partition(2, 0, device=-1, reverse=True)
    assert ei.value.name == "GSP_ERR_NO_REVERSE"
    with pytest.raises(gsp.GspError) as ei:
        G.partition(2, 2, device=-1)
    assert ei.value.name == "GSP_ERR_ARG"
    pg = G.partition(2, 0, device=-1)
    with pytest.raises(gsp.GspError):
        pg.partition(2, 0, device=-1)


@pytest.mark.parametrize("seed", range(8))
def test_partition_local_rev_bitexact(gsp, seed):
    """Local rev of a fwd partition: its own edges grouped by padded source,
    stable in local edge id (brute force with a stable numpy argsort)."""
    rng = np.random.default_rng(300 + seed)
    V = int(rng.integers(2, 150))
    E = int(rng.integers(0, 1200))
    src, dst = datagen.random_multigraph(V, E, seed)
    G = host_graph(gsp, V, src, dst)
    og = oracle.Graph(V, src, dst)
    for P in (1, 2, 3):
        for p in range(P):
            pg = G.partition(P, p, device=-1)
            lo, lc, R, b = og.partition_structure(P, p)
            ex = pg.export(rev=True, coo=False)
            rows = np.repeat(np.arange(R), np.diff(lo))
            order = np.argsort(lc, kind="stable")
            assert np.array_equal(ex["rev_eid"], order.astype(np.int32))
            assert np.array_equal(ex["rev_col"], (p * R + rows[order]).astype(np.int32))
            assert np.array_equal(ex["rev_off"], np.concatenate([[0], np.cumsum(np.bincount(lc, minlength=P * R))]))


# ------------------------------------------------------- chunked partitions
def chunked_expected(og, P, C, p, c, reverse=False):
    """Brute force of the chunk-major layout (include/gsp.h gsp_graph_partition_chunked):
    blocks = oracle C8 bounds with Q = P*C parts, block q = p*C + c at slot (q % C)*P + q // C."""
    Q = P * C
    b = og.partition_bounds(Q, reverse)
    R = int(np.max(np.diff(b)))
    off = og.rev_off if reverse else og.fwd_off
    col = og.rev_col if reverse else og.fwd_col
    qmap = np.searchsorted(b, np.arange(og.V), side="right") - 1      # block of every vertex
    slot = (qmap % C) * P + qmap // C
    padded = slot * R + (np.arange(og.V) - b[qmap])
    q = p * C + c
    lo, hi = b[q], b[q + 1]
    loc_off = off[np.minimum(lo + np.arange(R + 1), hi)] - off[lo]
    loc_col = padded[col[off[lo]:off[hi]]].astype(np.int32)
    return loc_off, loc_col, R, b, ((q % C) * P + q // C) * R


@pytest.mark.parametrize("seed", range(10))
def test_chunked_partition_structure_bitexact(gsp, seed):
    rng = np.random.default_rng(700 + seed)
    V = int(rng.integers(1, 300))
    E = int(rng.integers(0, 2500))
    src, dst = datagen.random_multigraph(V, E, seed)
    G = host_graph(gsp, V, src, dst)
    og = oracle.Graph(V, src, dst)
    for P, C in ((1, 3), (2, 2), (2, 3), (3, 4), (4, 1)):
        for rev in (False, True):
            # the rows a rank owns are those of the unchunked partition
            bP = og.partition_bounds(P, rev)
            assert np.array_equal(G.partition_bounds(P * C, rev)[::C], bP)
            seen = 0
            for p in range(P):
                for c in range(C):
                    pg = G.partition(P, p, device=-1, reverse=rev, nchunks=C, chunk=c)
                    lo, lc, R, b, rb = chunked_expected(og, P, C, p, c, rev)
                    ex = pg.export(rev=False, coo=False)
                    assert np.array_equal(ex["fwd_off"], lo) and np.array_equal(ex["fwd_col"], lc)
                    q = p * C + c
                    assert (pg.nparts, pg.part, pg.nchunks, pg.chunk, pg.row_begin, pg.row_end, pg.R, pg.ncols,
                            pg.row_base) == (P, p, C, c, b[q], b[q + 1], R, P * C * R, rb)
                    seen += pg.E
            assert seen == og.E
            if C == 1:   # nchunks = 1 is exactly gsp_graph_partition
                for p in range(P):
                    a = G.partition(P, p, device=-1, reverse=rev).export(rev=False, coo=False)
                    lo, lc, R, b = og.partition_structure(P, p, rev)
                    assert np.array_equal(a["fwd_off"], lo) and np.array_equal(a["fwd_col"], lc)


def test_chunked_partition_local_rev(gsp):
    """Local rev of a chunk: its own edges grouped by padded source, rev_col = row_base + local row."""
    src, dst = datagen.random_multigraph(120, 900, 3)
    G = host_graph(gsp, 120, src, dst)
    og = oracle.Graph(120, src, dst)
    P, C = 2, 3
    for p in range(P):
        for c in range(C):
            pg = G.partition(P, p, device=-1, nchunks=C, chunk=c)
            lo, lc, R, b, rb = chunked_expected(og, P, C, p, c)
            ex = pg.export(rev=True, coo=False)
            rows = np.repeat(np.arange(R), np.diff(lo))
            order = np.argsort(lc, kind="stable")
            assert np.array_equal(ex["rev_eid"], order.astype(np.int32))
            assert np.array_equal(ex["rev_col"], (rb + rows[order]).astype(np.int32))


def test_chunked_partition_errors(gsp, golden):
    g = golden("d4.json")
    G = host_graph(gsp, g["V"], g["src"], g["dst"])
    for P, C, p, c in ((2, 0, 0, 0), (2, 2, 0, 2), (2, 2, 0, -1), (2, 2, 2, 0)):
        with pytest.raises(gsp.GspError) as ei:
            G.partition(P, p, device=-1, nchunks=C, chunk=c)
        assert ei.value.name == "GSP_ERR_ARG"


def test_no_edge_ids_flag_host(gsp, golden):
    """GSP_BUILD_NO_EDGE_IDS changes only the device format: the host structure
    (export) is the canonical one, and a host-only graph holds no device bytes."""
    for gf in ("t4.json", "d4.json"):
        g = golden(gf)
        G = host_graph(gsp, g["V"], g["src"], g["dst"], edge_ids=False)
        ex = G.export()
        assert ex["fwd_col"].tolist() == g["fwd_col"] and ex["rev_eid"].tolist() == g["rev_eid"]
        assert G.memory() == {"topology": 0, "edge_ids": 0, "edge_scales": 0, "vertex_arrays": 0}
        assert G.device_bytes == 0
