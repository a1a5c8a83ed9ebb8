"""N > 1 host path on CPU (gloo, world size 2): every rank builds its destination-
row partition with libgsp (device = -1: builder + partitioner only), computes its
local rows of the GCN aggregation from the padded structure, and the ranks
all-gather the [R, F] blocks into the padded [P*R, F] table -- the exchange the
bench performs with NCCL.  The un-padded result must equal the single-process
oracle.  (The CUDA kernels themselves are covered by the GPU tests.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, norm, q):
    import sys
    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    import paper_2402_03548_b200 as gsp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, src, dst = datagen.make_graph(name)
        G = gsp.Graph(V, src, dst, device=-1)
        pg = G.partition(world, rank, device=-1)
        b = G.partition_bounds(world)
        R = pg.R
        ex = pg.export(rev=False, coo=False)
        F = 8
        X = datagen.uniform(3, V, F).astype(np.float64)
        # global degree scales (oracle C3) placed in the padded layout
        og = oracle.Graph(V, src, dst)
        sdst, ssrc = og.scales(norm)
        pad = np.zeros((world * R, F))
        spad = np.zeros(world * R)
        for p in range(world):
            pad[p * R:p * R + b[p + 1] - b[p]] = X[b[p]:b[p + 1]]
            spad[p * R:p * R + b[p + 1] - b[p]] = ssrc[b[p]:b[p + 1]]
        loc = np.zeros((R, F))
        for r in range(b[rank + 1] - b[rank]):
            cols = ex["fwd_col"][ex["fwd_off"][r]:ex["fwd_off"][r + 1]]
            loc[r] = sdst[b[rank] + r] * (spad[cols, None] * pad[cols]).sum(0)
        assert np.all(ex["fwd_off"][b[rank + 1] - b[rank]:] == ex["fwd_off"][-1])   # padding rows empty
        gathered = torch.zeros((world * R, F), dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, torch.from_numpy(loc))
        g = gathered.numpy()
        got = np.concatenate([g[p * R:p * R + b[p + 1] - b[p]] for p in range(world)])
        ref, T = og.gspmm(X.astype(np.float32), norm, False)
        err = float(np.max(np.abs(got - ref) / (1e-9 * (T + 1)))) if got.size else 0.0
        q.put((rank, err, int(R), [int(x) for x in b]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,norm", [("cora", 2), ("cora", 0), ("pubmed", 1)])
def test_gloo_two_rank_partition_allgather(name, norm):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, norm, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, err, R, b in res:
        assert err <= 1.0, (rank, err)
    assert res[0][3] == res[1][3]


def _worker_wrev(rank, world, port, q):
    """Weighted reverse across ranks: each rank sums its own edges per padded
    source row (from libgsp's local-rev structure) and the ranks reduce the
    partials (bench: reduce_scatter_tensor on NCCL; here all_reduce + own slice,
    gloo)."""
    import sys
    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    import paper_2402_03548_b200 as gsp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, src, dst = datagen.make_graph("pubmed")
        G = gsp.Graph(V, src, dst, device=-1)
        og = oracle.Graph(V, src, dst)
        pg = G.partition(world, rank, device=-1)
        b = G.partition_bounds(world)
        R = pg.R
        H, Fh = 4, 2
        X = datagen.uniform(7, V, H * Fh).astype(np.float64)
        w = datagen.uniform(8, og.E, H, lo=0, hi=1)
        e0 = og.fwd_off[b[rank]]
        wl = w[e0:og.fwd_off[b[rank + 1]]].astype(np.float64)
        pad = np.zeros((world * R, H * Fh))
        for p in range(world):
            pad[p * R:p * R + b[p + 1] - b[p]] = X[b[p]:b[p + 1]]
        ex = pg.export(rev=True, coo=False)
        partial = np.zeros((world * R, H * Fh))
        for u in range(world * R):
            for k in range(ex["rev_off"][u], ex["rev_off"][u + 1]):
                wrow = np.repeat(wl[ex["rev_eid"][k]], Fh)
                partial[u] += wrow * pad[ex["rev_col"][k]]
        t = torch.from_numpy(partial)
        dist.all_reduce(t)
        mine = t.numpy()[rank * R: rank * R + b[rank + 1] - b[rank]]
        ref, T = og.gspmm_weighted(X.astype(np.float32), w, True, rows=np.arange(b[rank], b[rank + 1]))
        err = float(np.max(np.abs(mine - ref) / (1e-9 * (T + 1)))) if mine.size else 0.0
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_weighted_reverse_reduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_wrev, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, err in res:
        assert err <= 1.0, (rank, err)


def _worker_chunked(rank, world, port, name, C, q):
    """Chunked layer exchange (bench.py GCN configs at N > 1): every rank computes
    its C chunks one after another and all-gathers chunk c into rows
    [c*P*R, (c+1)*P*R) of the chunk-major padded table as soon as it is done;
    un-padding the table must give the single-process oracle result (fwd and,
    on a symmetric graph, the reverse over the shared topology)."""
    import sys
    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    import paper_2402_03548_b200 as gsp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, src, dst = datagen.make_graph(name)
        G = gsp.Graph(V, src, dst, device=-1)
        og = oracle.Graph(V, src, dst)
        parts = [G.partition(world, rank, device=-1, nchunks=C, chunk=c) for c in range(C)]
        R, NC = parts[0].R, parts[0].ncols
        b = G.partition_bounds(world * C)
        slot_of = lambda qq: (qq % C) * world + qq // C
        F = 6
        X = datagen.uniform(5, V, F).astype(np.float64)
        pad = np.zeros((NC, F))
        sin, sout = np.zeros(NC), np.zeros(NC)
        din = np.diff(og.fwd_off).clip(min=1).astype(np.float64)
        dout = np.diff(og.rev_off).clip(min=1).astype(np.float64)
        for qq in range(world * C):
            s0 = slot_of(qq) * R
            n = b[qq + 1] - b[qq]
            pad[s0:s0 + n] = X[b[qq]:b[qq + 1]]
            sin[s0:s0 + n] = din[b[qq]:b[qq + 1]] ** -0.5
            sout[s0:s0 + n] = dout[b[qq]:b[qq + 1]] ** -0.5
        res = []
        for rev in (False, True):
            gathered = torch.zeros((NC, F), dtype=torch.float64)
            for c, pg in enumerate(parts):
                ex = pg.export(rev=False, coo=False)
                loc = np.zeros((R, F))
                for r in range(pg.row_end - pg.row_begin):
                    cols = ex["fwd_col"][ex["fwd_off"][r]:ex["fwd_off"][r + 1]]
                    # symmetric graph: reverse = the same rows with the scale roles swapped (BOTH)
                    s_row = (sout if rev else sin)[pg.row_base + r]
                    s_col = (sin if rev else sout)[cols]
                    loc[r] = s_row * (s_col[:, None] * pad[cols]).sum(0)
                chunk_rows = gathered[c * world * R:(c + 1) * world * R]
                dist.all_gather_into_tensor(chunk_rows, torch.from_numpy(loc))
            g = gathered.numpy()
            got = np.concatenate([g[slot_of(qq) * R:slot_of(qq) * R + b[qq + 1] - b[qq]] for qq in range(world * C)])
            ref, T = og.gspmm(X.astype(np.float32), 2, rev)
            res.append(float(np.max(np.abs(got - ref) / (1e-9 * (T + 1)))) if got.size else 0.0)
        q.put((rank, max(res)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,C", [("cora", 3), ("pubmed", 2)])
def test_gloo_two_rank_chunked_allgather(name, C):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_chunked, args=(r, world, port, name, C, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, err in res:
        assert err <= 1.0, (rank, err)


def _worker_directed_reverse(rank, world, port, q):
    """Directed graph at N > 1 (bench.py arxiv): the reverse gSpMMv of a fwd
    partition is the per-source partial over its own edges (local rev, s_src
    applied); one reduce-scatter gives every rank its rows of the full reverse."""
    import sys
    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    import paper_2402_03548_b200 as gsp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V = 3000
        src, dst = datagen.rmat(12, V, 20000, 0xA5)
        G = gsp.Graph(V, src, dst, device=-1)
        og = oracle.Graph(V, src, dst)
        assert not G.symmetric
        pg = G.partition(world, rank, device=-1)
        R, NC = pg.R, pg.ncols
        b = G.partition_bounds(world)
        F = 5
        Y = datagen.uniform(9, V, F).astype(np.float64)
        din = np.diff(og.fwd_off).clip(min=1).astype(np.float64)
        dout = np.diff(og.rev_off).clip(min=1).astype(np.float64)
        pad, sin, sout = np.zeros((NC, F)), np.ones(NC), np.ones(NC)
        for p in range(world):
            n = b[p + 1] - b[p]
            pad[p * R:p * R + n] = Y[b[p]:b[p + 1]]
            sin[p * R:p * R + n] = din[b[p]:b[p + 1]] ** -0.5
            sout[p * R:p * R + n] = dout[b[p]:b[p + 1]] ** -0.5
        ex = pg.export(rev=True, coo=False)
        partial = np.zeros((NC, F))
        for u in range(NC):
            cols = ex["rev_col"][ex["rev_off"][u]:ex["rev_off"][u + 1]]
            partial[u] = sout[u] * (sin[cols][:, None] * pad[cols]).sum(0)
        t = torch.from_numpy(partial)
        dist.all_reduce(t)           # NCCL: reduce_scatter_tensor (each rank keeps its slot)
        mine = t.numpy()[rank * R:rank * R + b[rank + 1] - b[rank]]
        ref, T = og.gspmm(Y.astype(np.float32), 2, True, rows=np.arange(b[rank], b[rank + 1]))
        err = float(np.max(np.abs(mine - ref) / (1e-9 * (T + 1)))) if mine.size else 0.0
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_directed_reverse_partials():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_directed_reverse, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    for rank, err in res:
        assert err <= 1.0, (rank, err)
