"""Parity at BASELINE.json's full sizes (Reddit- and ogbn-products-shaped), in the
launch configuration bench.py times: the whole structure bit-exact against the
oracle's own build, float outputs on sampled rows the oracle computes one by
one (the heaviest rows -- CTA-split path --, random rows, the lightest rows),
plus properties that hold at any size (softmax rows sum to 1)."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def sample_rows(off, seed, n_heavy=16, n_rand=48, n_light=16):
    deg = np.diff(off)
    order = np.argsort(-deg, kind="stable")
    rng = np.random.default_rng(seed)
    rows = np.concatenate([order[:n_heavy], rng.choice(len(deg), n_rand, replace=False), order[-n_light:]])
    return np.unique(rows).astype(np.int64)


def within(gpu, ref, T, scale=1e-5):
    err = np.abs(np.asarray(gpu, np.float64) - ref)
    r = float(np.max(err / (scale * (np.asarray(T) + 1.0)))) if err.size else 0.0
    assert r <= 1.0, f"max err/bound {r:.3g}"
    return r


@pytest.fixture(scope="module")
def reddit():
    import paper_2402_03548_b200 as gsp
    cfg = datagen.CONFIGS["reddit"]
    V, src, dst = datagen.make_graph(cfg)
    G = gsp.Graph(V, src, dst, device=0)
    og = oracle.Graph(V, src, dst)
    return cfg, G, og


def test_reddit_structure_bitexact(reddit):
    cfg, G, og = reddit
    assert G.symmetric and G.E == cfg.E
    ex = G.export()
    for k in ("fwd_off", "fwd_col", "rev_off", "rev_col", "rev_eid", "coo_to_eid"):
        assert np.array_equal(ex[k], getattr(og, k)), k


@pytest.mark.parametrize("F,ld", [(64, 64), (602, 604)])
def test_reddit_gspmm_sampled(reddit, F, ld):
    cfg, G, og = reddit
    rows = sample_rows(og.fwd_off, F)
    buf = np.zeros((og.V, ld), np.float32)
    Xh = datagen.uniform(0x2EDD + F, og.V, F, ld=ld)
    buf[:] = Xh
    X = dev(buf)[:, :F]
    for rev in (0, 1):
        out = G.gspmm(X, 2, reverse=rev).cpu().numpy()
        ref, T = og.gspmm(Xh, 2, bool(rev), rows=rows, F=F)
        within(out[rows], ref, T)
    # non-negative inputs: the fp32 error-growth case
    Xp = datagen.uniform(5, og.V, F, ld=ld, lo=0.0, hi=1.0)
    out = G.gspmm(dev(Xp)[:, :F], 2).cpu().numpy()
    ref, T = og.gspmm(Xp, 2, False, rows=rows, F=F)
    within(out[rows], ref, T)


def test_reddit_gat_chain_sampled(reddit):
    cfg, G, og = reddit
    H, F = cfg.H, cfg.H * cfg.Fh
    rows = sample_rows(og.fwd_off, 77)
    eids = og.row_edges(rows)
    Zh = datagen.uniform(11, og.V, F)
    Z = dev(Zh)
    s = G.gsddmm(Z, Z, H=H)
    ref, T = og.gsddmm(Zh, Zh, H, rows=rows)
    within(s[torch.from_numpy(eids).cuda()].cpu().numpy(), ref, T)
    del s
    lh = datagen.uniform(12, og.E, H, lo=-8, hi=8)
    a = G.edge_softmax(dev(lh))
    within(a[torch.from_numpy(eids).cuda()].cpu().numpy(), og.edge_softmax(lh, rows=rows), 1.0)
    # every non-empty row sums to 1 (any size)
    rowsum = torch.zeros((og.V, H), dtype=torch.float64, device="cuda")
    rid = torch.repeat_interleave(torch.arange(og.V, device="cuda"), dev(np.diff(og.fwd_off)))
    rowsum.index_add_(0, rid, a.double())
    assert torch.allclose(rowsum, torch.ones_like(rowsum), atol=1e-4)
    del a, rowsum, rid
    wh = datagen.uniform(13, og.E, H, lo=0, hi=1)
    w = dev(wh)
    for rev in (0, 1):
        out = G.gspmm_weighted(Z, w, reverse=rev).cpu().numpy()
        ref, T = og.gspmm_weighted(Zh, wh, bool(rev), rows=rows)
        within(out[rows], ref, T)


def test_reddit_gat_forward_fused_sampled(reddit):
    """The fused GAT forward in bench.py's step configuration (gat_forward(Z, Z, Z),
    H = 8 x 8, alpha into a preallocated [E, H] buffer): alpha and the aggregate of
    sampled rows against oracle C10.  A row's results depend only on its own
    in-edges, so the oracle runs on the sub-graph of the sampled rows' in-edges
    (same vertex ids; its fwd slots are the rows' slots in order)."""
    cfg, G, og = reddit
    H, F = cfg.H, cfg.H * cfg.Fh
    rows = sample_rows(og.fwd_off, 91)
    eids = og.row_edges(rows)
    sub_dst = np.repeat(rows, og.fwd_off[rows + 1] - og.fwd_off[rows])
    sub = oracle.Graph(og.V, og.fwd_col[eids].astype(np.int64), sub_dst)
    assert np.array_equal(sub.fwd_col, og.fwd_col[eids])
    Zh = datagen.uniform(17, og.V, F)
    Z = dev(Zh)
    alpha = torch.empty((og.E, H), device="cuda")
    out = torch.empty((og.V, F), device="cuda")
    G.gat_forward(Z, Z, Z, H, alpha=alpha, out=out)
    a_ref, o_ref, T = sub.gat_forward(Zh, Zh, Zh, H)
    # tolerances as the small-size fused tests
    within(alpha[torch.from_numpy(eids).cuda()].cpu().numpy(), a_ref, 1.0)   # 2e-5 absolute
    within(out[torch.from_numpy(rows).cuda()].cpu().numpy(), o_ref[rows], T[rows])


def test_reddit_gat_forward_additive_sampled(reddit):
    """NEXT-3 at full size: the fused additive GAT forward (alpha = softmax(lrelu(el[u]
    + er[v])), aggregate of Z, H = 8 x 8) on sampled rows against oracle C15 on the
    sub-graph of those rows' in-edges."""
    cfg, G, og = reddit
    H, F = cfg.H, cfg.H * cfg.Fh
    rows = sample_rows(og.fwd_off, 95)
    eids = og.row_edges(rows)
    sub = oracle.Graph(og.V, og.fwd_col[eids].astype(np.int64),
                       np.repeat(rows, og.fwd_off[rows + 1] - og.fwd_off[rows]))
    elh = datagen.uniform(31, og.V, H, lo=-4, hi=4)
    erh = datagen.uniform(32, og.V, H, lo=-4, hi=4)
    Zh = datagen.uniform(33, og.V, F)
    alpha, out = G.gat_forward_additive(dev(elh), dev(erh), dev(Zh), 0.2)
    a_ref, o_ref, T = sub.gat_forward_additive(elh, erh, Zh, 0.2)
    within(alpha[torch.from_numpy(eids).cuda()].cpu().numpy(), a_ref, 1.0)
    within(out[torch.from_numpy(rows).cuda()].cpu().numpy(), o_ref[rows], T[rows])


def test_products_chunked_partitions_bench_layout():
    """ogbn-products in bench.py's N = 8 launch configuration: 8 ranks x 4 chunks of
    chunk-major partitions, run one after another on this GPU, each writing its
    [R, F] block into its chunk's all-gather range of the padded table (the NCCL
    all-gather replaced by the placement).  Un-padded rows, sampled (heaviest,
    random, lightest), against oracle C4 from the COO list; forward and the
    symmetric reverse."""
    import paper_2402_03548_b200 as gsp
    cfg = datagen.CONFIGS["products"]
    V, src, dst = datagen.make_graph(cfg)
    G = gsp.Graph(V, src, dst, device=0)
    P, C = 8, 4
    b = G.partition_bounds(P * C)
    slot = lambda q: (q % C) * P + q // C
    Xh = datagen.uniform(0x960D + 1, V, cfg.F)
    R = None
    tables = {}
    for p in range(P):
        for c in range(C):
            pg = G.partition(P, p, device=0, nchunks=C, chunk=c)
            if R is None:
                R = pg.R
                Xp = torch.zeros((pg.ncols, cfg.F), device="cuda")
                for q in range(P * C):
                    Xp[slot(q) * R:slot(q) * R + b[q + 1] - b[q]] = dev(Xh[b[q]:b[q + 1]])
                for r in (False, True):
                    tables[r] = torch.full((pg.ncols, cfg.F), float("nan"), device="cuda")
            for rev in (False, True):
                pg.gspmm(Xp, gsp.NORM_BOTH, out=tables[rev][(c * P + p) * R:(c * P + p + 1) * R], reverse=rev)
            torch.cuda.synchronize()
            del pg
    off = G.export(rev=False, coo=False)["fwd_off"]
    rows = sample_rows(off, 5)
    q_of = np.searchsorted(b, rows, side="right") - 1
    pos = torch.from_numpy(np.array([slot(q) * R + r - b[q] for q, r in zip(q_of, rows)])).cuda()
    for rev in (False, True):
        got = tables[rev][pos].cpu().numpy()
        ref, T = oracle.gspmm_rows_coo(V, src, dst, Xh, 2, rows, reverse=rev, F=cfg.F)
        within(got, ref, T)


def test_reddit_gat_backward_scores_sampled(reddit):
    """The fused GAT backward scores (NEXT-1) at full size, as bench.py's next_rows
    calls it (dOut, Z, alpha of the forward, H = 8 x 8): ds of sampled rows against
    the oracle composition C9 o C6 on the sub-graph of those rows' in-edges (a
    row's ds depends only on its own edges).  Bound as the small-size test."""
    cfg, G, og = reddit
    H, F = cfg.H, cfg.H * cfg.Fh
    rows = sample_rows(og.fwd_off, 93)
    eids = og.row_edges(rows)
    sub = oracle.Graph(og.V, og.fwd_col[eids].astype(np.int64),
                       np.repeat(rows, og.fwd_off[rows + 1] - og.fwd_off[rows]))
    Zh = datagen.uniform(21, og.V, F)
    dOh = datagen.uniform(22, og.V, F)
    Z, dO = dev(Zh), dev(dOh)
    alpha, _ = G.gat_forward(Z, Z, Z, H)
    ds = G.gat_backward_scores(dO, Z, alpha)
    e = torch.from_numpy(eids).cuda()
    ah = alpha[e].cpu().numpy()
    got = ds[e].cpu().numpy()
    del alpha, ds
    d64, T6 = sub.gsddmm(dOh, Zh, H)
    ref, T9 = sub.edge_softmax_backward(ah, d64.astype(np.float32))
    rid = np.repeat(np.arange(len(rows)), og.fwd_off[rows + 1] - og.fwd_off[rows])
    S = np.zeros((len(rows), H))
    np.add.at(S, rid, ah * T6)
    within(got, ref, T9 + ah * T6 + ah * S[rid])


def test_products_gspmm_sampled():
    import paper_2402_03548_b200 as gsp
    cfg = datagen.CONFIGS["products"]
    V, src, dst = datagen.make_graph(cfg)
    G = gsp.Graph(V, src, dst, device=0)
    og = oracle.Graph(V, src, dst)
    ex = G.export(rev=False, coo=False)
    assert np.array_equal(ex["fwd_off"], og.fwd_off) and np.array_equal(ex["fwd_col"], og.fwd_col)
    rows = sample_rows(og.fwd_off, 3)
    Xh = datagen.uniform(0x960D, V, cfg.F, ld=cfg.ld)
    out = G.gspmm(dev(Xh), 2).cpu().numpy()
    ref, T = og.gspmm(Xh, 2, False, rows=rows)
    within(out[rows], ref, T)


def test_kron25_billion_edges():
    """NEXT-4: the paper's billion-edge Kron-25 (2^25 vertices, 2^30 edges,
    F = 150) built and aggregated on ONE B200.  Structure of
    sampled rows bit-exact and GCN gSpMM (BOTH) on sampled rows within the
    bound, both against the oracle evaluated straight from the COO list."""
    import paper_2402_03548_b200 as gsp
    cfg = datagen.CONFIGS["kron25"]
    V, src, dst = datagen.make_graph(cfg)
    G = gsp.Graph(V, src, dst, device=0)
    assert G.E == 1 << 30 and G.symmetric
    ex = G.export(rev=False, coo=False)
    deg = np.diff(ex["fwd_off"])
    order = np.argsort(-deg, kind="stable")
    rng = np.random.default_rng(25)
    rows = np.unique(np.concatenate([order[:6], rng.choice(V, 20, replace=False), order[-4:]])).astype(np.int64)
    for (first, pairs), v in zip(oracle.rows_coo(V, src, dst, rows), rows):
        assert first == ex["fwd_off"][v]
        assert np.array_equal(pairs[:, 0], ex["fwd_col"][ex["fwd_off"][v]:ex["fwd_off"][v + 1]])
    del ex
    Xh = datagen.uniform(0xC125, V, cfg.F, ld=cfg.ld)
    X = torch.from_numpy(Xh).cuda()[:, :cfg.F]
    out = G.gspmm(X, gsp.NORM_BOTH)
    torch.cuda.synchronize()
    got = out[torch.from_numpy(rows).cuda()].cpu().numpy()
    del out, X
    ref, T = oracle.gspmm_rows_coo(V, src, dst, Xh, 2, rows, F=cfg.F)
    within(got, ref, T)


def test_bench_multi_rank_path_matches_single_gpu(tmp_path):
    """bench.py's N > 1 path (destination-row partitions, all-gathers of the GCN /
    GAT forward outputs, reduce-scatter of the GAT backward partials) run as 3
    ranks sharing this GPU (gloo, host-staged exchange) must reproduce the
    single-GPU results (--check)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GSP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "3",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"), "--gpus", "3",
           "--config", "pubmed", "--steps", "3", "--warmup", "3", "--check", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 3 and line["multi_gpu_check"]["ok"], line["multi_gpu_check"]


@pytest.mark.parametrize("config,ranks,chunks", [("cora", 2, 3), ("arxiv", 2, 0)])
def test_bench_gcn_multi_rank_paths(config, ranks, chunks):
    """bench.py's GCN-only step at N > 1 (gloo ranks sharing this GPU): the chunked
    chunk-major all-gather (Cora, 3 chunks per rank) and the directed graph's
    reverse as per-source partials + reduce-scatter (ogbn-arxiv-shaped); --check
    compares every exchanged output per element with the oracle on sampled rows."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GSP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(29540 + ranks + chunks), os.path.join(root, "bench.py"),
           "--gpus", str(ranks), "--config", config, "--steps", "3", "--warmup", "3", "--check", "--no-e2e",
           "--chunks", str(chunks)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == ranks and line["multi_gpu_check"]["ok"], line["multi_gpu_check"]
    if chunks > 1:
        assert f"{chunks} chunks per rank" in line["config"]["parallelism"]


@pytest.mark.parametrize("config,ranks,rank", [("products", 4, 2), ("reddit", 2, 1), ("arxiv", 2, 0)])
def test_bench_nccl_path_control_flow(config, ranks, rank):
    """The NCCL branch of bench.py's N > 1 step on this single GPU: one process plays
    rank `rank` of `ranks` with torch's fake process group, so the async all-gathers
    (chunked, chunk-major for products), reduce-scatters, the observer-stream layer
    timing and the pipelined e2e with collectives all run on CUDA tensors with the
    NCCL code path's shapes (the fake collectives move no data; parity of the
    exchanged outputs is the gloo --check tests' job)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GSP_BENCH_BACKEND="fake", WORLD_SIZE=str(ranks), RANK=str(rank), LOCAL_RANK="0")
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", str(ranks), "--config", config,
           "--steps", "3", "--warmup", "3", "--no-configs"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    if rank == 0:
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert line["n_gpus"] == ranks and line["e2e"]["value"] > 0 and line["value"] > 0
        assert "fake" in line["per_op"]["exchange"]["what"]


_HOT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import datagen, paper_2402_03548_b200 as gsp
V, E, F = 1_500_000, 15_000_000, 128             # table 768 MB > 6 x the B200's 126 MB L2
src, dst = datagen.skewed_multigraph(V, E, 17, alpha=0.8)
G = gsp.Graph(V, src, dst, device=0)
X = torch.from_numpy(datagen.uniform(5, V, F)).cuda()
outs = [G.gspmm(X, gsp.NORM_BOTH, reverse=r).cpu().numpy() for r in (0, 1)]
np.save(sys.argv[1], np.stack(outs))
"""


def test_hot_row_policy_is_bitwise_neutral(tmp_path):
    """The hot-row L2 policy (api.cu hot_scale_for: tables > 6x L2, BOTH norm) only
    changes cache hints: gSpMM fwd / rev with it and with GSP_HOT=0 agree bit for bit.
    (Accuracy of the hot path against the oracle: test_products_gspmm_sampled.)"""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for hot in ("1", "0"):
        out = tmp_path / f"hot{hot}.npy"
        env = dict(os.environ, GSP_HOT=hot)
        subprocess.run([sys.executable, "-c", _HOT_SCRIPT, str(out), root], env=env, check=True, timeout=600)
        res.append(np.load(out))
    assert np.array_equal(res[0], res[1])
