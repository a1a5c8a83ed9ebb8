"""GPU parity: the sm_100a kernels behind the C ABI vs the CPU oracle, element by
element, on the same seeded inputs.  Acceptance (BASELINE.json north_star):
structure bit-exact; |gpu - oracle| <= 1e-5 * (sum|terms| + 1) per fp32 element
(edge softmax: T := 1, i.e. 2e-5 absolute -- DESIGN.md "Tolerances")."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

NORMS = (0, 1, 2)


@pytest.fixture(scope="module")
def gsp():
    import paper_2402_03548_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def padded(a, ld):
    """fp32 [rows, ld] device tensor holding `a` in its first cols (padding = NaN:
    the kernels may read padding but must never use it)."""
    rows, cols = a.shape
    buf = np.full((rows, ld), np.nan, np.float32)
    buf[:, :cols] = a
    t = dev(buf)
    return t[:, :cols]


def assert_within(gpu, ref, T, what="", scale=1e-5):
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - ref)
    bound = scale * (np.asarray(T) + 1.0)
    ratio = float(np.max(err / bound)) if err.size else 0.0
    assert np.all(np.isfinite(gpu)), what
    assert ratio <= 1.0, f"{what}: max err/bound = {ratio:.3g}"
    return ratio


def graph_pair(gsp, V, src, dst, **kw):
    return gsp.Graph(V, src, dst, device=0, **kw), oracle.Graph(V, src, dst)


# ------------------------------------------------------------------ golden
def test_golden_t4_d4(gsp, golden):
    for gf, cf in [("t4.json", "t4_chain.json"), ("d4.json", "d4.json")]:
        g, c = golden(gf), golden(cf)
        G, og = graph_pair(gsp, g["V"], g["src"], g["dst"])
        X = dev(np.array(c["X"], np.float32)[:, None])
        Y = dev(np.array(c["Y"], np.float32)[:, None])
        for norm in NORMS:
            for rev in (0, 1):
                ref, T = og.gspmm(X.cpu().numpy(), norm, rev)
                assert_within(G.gspmm(X, norm, reverse=rev).cpu().numpy(), ref, T, f"{gf} n{norm} r{rev}")
        s = G.gsddmm(X, Y, H=1)
        assert np.array_equal(s.cpu().numpy()[:, 0], np.array(c["gsddmm_XY"], np.float32))
        a = G.edge_softmax(s / 100.0)
        assert np.allclose(a.cpu().numpy()[:, 0], c["edge_softmax_gsddmm_over_100"], atol=2e-5)
        f = G.gspmm_weighted(X, a).cpu().numpy()[:, 0]
        r = G.gspmm_weighted(X, a, reverse=True).cpu().numpy()[:, 0]
        assert np.allclose(f, c["weighted_fwd_alpha_X"], atol=1e-4)
        assert np.allclose(r, c["weighted_rev_alpha_X"], atol=1e-4)


def test_export_matches_oracle_on_device_graph(gsp):
    V, src, dst = datagen.make_graph("arxiv")
    G, og = graph_pair(gsp, V, src, dst)
    ex = G.export()
    for k in ("fwd_off", "fwd_col", "rev_off", "rev_col", "rev_eid", "coo_to_eid"):
        assert np.array_equal(ex[k], getattr(og, k)), k
    assert G.device_bytes > 0


# ------------------------------------------------------------- gspmm family
GSPMM_SHAPES = [(1, 1), (3, 3), (4, 4), (5, 8), (16, 16), (64, 64), (100, 100), (128, 132), (602, 604)]


@pytest.mark.parametrize("F,ld", GSPMM_SHAPES)
def test_gspmm_random_graphs(gsp, F, ld):
    for seed in range(3):
        rng = np.random.default_rng(seed * 7 + F)
        V = int(rng.integers(1, 3000))
        E = int(rng.integers(0, 40000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed != 1
                    else datagen.skewed_multigraph(V, E, seed))
        # seed 2: without precomputed per-edge scales (the per-edge gather path)
        G, og = graph_pair(gsp, V, src, dst, edge_scales=(seed != 2))
        Xh = datagen.uniform(seed + 11, V, F)
        X = padded(Xh, ld)
        for norm in NORMS:
            for rev in (0, 1):
                ref, T = og.gspmm(Xh, norm, rev)
                out = padded(np.zeros((V, F), np.float32), ld)
                G.gspmm(X, norm, out=out, reverse=rev)
                assert_within(out.cpu().numpy(), ref, T, f"V{V} E{E} F{F} n{norm} r{rev}")
                if ld > F:   # padding columns of out are never written
                    full = out.as_strided((V, ld), (ld, 1)).cpu().numpy()
                    assert np.all(np.isnan(full[:, F:]))


def test_gspmm_heavy_and_mega_rows(gsp):
    """Rows far above the 2048-edge CTA threshold (CTA-split path), rows in every
    degree bin, isolated vertices; non-negative inputs (the error-growth case of
    SURVEY Appendix B)."""
    V, E = 4000, 600_000
    src, dst = datagen.skewed_multigraph(V, E, 3, alpha=1.6)
    G, og = graph_pair(gsp, V, src, dst)
    deg = np.diff(og.fwd_off)
    assert deg.max() > 50_000
    # hub rows (degree > max(8192, E / 4096)) run as thread-block clusters of 8 CTAs
    assert (deg > max(8192, E // 4096)).sum() >= 3
    for F, ld in ((16, 16), (64, 64), (128, 128), (602, 604)):
        Xh = datagen.uniform(5, V, F, lo=0.0, hi=1.0)
        X = padded(Xh, ld)
        for norm in NORMS:
            for rev in (0, 1):
                ref, T = og.gspmm(Xh, norm, rev)
                assert_within(G.gspmm(X, norm, reverse=rev).cpu().numpy(), ref, T, f"F{F} n{norm} r{rev}")
        if F == 64:
            for red in (gsp.REDUCE_MIN, gsp.REDUCE_MAX):
                ref, _ = og.gspmm_reduce(Xh, red)
                assert np.array_equal(G.gspmm_reduce(X, red).cpu().numpy().astype(np.float64), ref)


@pytest.mark.parametrize("H,Fh,ld", [(1, 1, 1), (1, 3, 3), (2, 3, 6), (2, 4, 8), (8, 8, 64), (8, 8, 68),
                                     (4, 16, 64), (3, 5, 15), (1, 64, 64), (2, 64, 128)])
def test_weighted_random(gsp, H, Fh, ld):
    for seed in range(2):
        rng = np.random.default_rng(seed + 31 * H + Fh)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.4))
        G, og = graph_pair(gsp, V, src, dst)
        F = H * Fh
        Xh = datagen.uniform(seed + 3, V, F)
        wh = datagen.uniform(seed + 4, E, H, lo=0.0, hi=1.0) if E else np.zeros((0, H), np.float32)
        X, w = padded(Xh, ld), dev(wh)
        for rev in (0, 1):
            ref, T = og.gspmm_weighted(Xh, wh, rev)
            assert_within(G.gspmm_weighted(X, w, reverse=rev).cpu().numpy(), ref, T, f"H{H} Fh{Fh} r{rev}")


def test_weighted_heavy_rows(gsp):
    V, E = 3000, 400_000
    src, dst = datagen.skewed_multigraph(V, E, 9, alpha=1.6)
    G, og = graph_pair(gsp, V, src, dst)
    Xh = datagen.uniform(1, V, 64)
    wh = datagen.uniform(2, E, 8, lo=0.0, hi=1.0)
    for rev in (0, 1):
        ref, T = og.gspmm_weighted(Xh, wh, rev)
        assert_within(G.gspmm_weighted(dev(Xh), dev(wh), reverse=rev).cpu().numpy(), ref, T, f"r{rev}")


def test_weighted_8x8_every_tile_count(gsp):
    """The H = 8 x Fh = 8 weighted kernel (wspmm8.cu) alternates register and
    shared-memory tiles: rows of every degree 0..300 (tile counts 0..10, odd and
    even, every ragged tail), a CTA-split hub row, and an ld = 72 table, both
    directions (reverse through the edge ids), against oracle C5."""
    degs = list(range(0, 301)) + [5000]
    V = len(degs)
    rng = np.random.default_rng(5)
    dst = np.repeat(np.arange(V, dtype=np.int64), degs)
    src = rng.integers(0, V, size=dst.size).astype(np.int64)
    perm = rng.permutation(dst.size)
    src, dst = src[perm], dst[perm]
    G, og = graph_pair(gsp, V, src, dst)
    Xh = datagen.uniform(11, V, 64)
    wh = datagen.uniform(12, dst.size, 8, lo=0.0, hi=1.0)
    for ld in (64, 72):
        for rev in (0, 1):
            ref, T = og.gspmm_weighted(Xh, wh, rev)
            got = G.gspmm_weighted(padded(Xh, ld), dev(wh), reverse=rev).cpu().numpy()
            assert_within(got, ref, T, f"ld{ld} r{rev}")


# ------------------------------------------------------------------ gsddmm
@pytest.mark.parametrize("H,Fh,ld", [(1, 1, 1), (1, 3, 3), (2, 3, 6), (2, 4, 8), (8, 8, 64), (8, 8, 72),
                                     (1, 32, 32), (4, 16, 64), (1, 128, 128), (2, 256, 512), (3, 5, 16)])
def test_gsddmm_random(gsp, H, Fh, ld):
    for seed in range(2):
        rng = np.random.default_rng(seed + 7 * H + Fh)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.5))
        G, og = graph_pair(gsp, V, src, dst)
        F = H * Fh
        Xh = datagen.uniform(seed + 1, V, F)
        Yh = datagen.uniform(seed + 2, V, F)
        ref, T = og.gsddmm(Xh, Yh, H)
        out = G.gsddmm(padded(Xh, ld), padded(Yh, ld), H=H)
        assert_within(out.cpu().numpy(), ref, T, f"H{H} Fh{Fh}")


# ------------------------------------------------------------ edge softmax
@pytest.mark.parametrize("H,ld", [(1, 1), (2, 2), (3, 3), (4, 4), (8, 8), (8, 12), (16, 16), (32, 32), (5, 7)])
def test_softmax_random(gsp, H, ld):
    for seed in range(2):
        rng = np.random.default_rng(seed + H)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 40000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.7))
        G, og = graph_pair(gsp, V, src, dst)
        eh = datagen.uniform(seed, E, H, lo=-10.0, hi=10.0) if E else np.zeros((0, H), np.float32)
        ref = og.edge_softmax(eh)
        out = G.edge_softmax(padded(eh, ld))
        assert_within(out.cpu().numpy(), ref, 1.0, f"H{H} ld{ld}")


def test_softmax_in_place_and_rows_sum_to_one(gsp):
    V, E = 3000, 500_000
    src, dst = datagen.skewed_multigraph(V, E, 4, alpha=1.6)
    G, og = graph_pair(gsp, V, src, dst)
    eh = datagen.uniform(3, E, 8, lo=-10.0, hi=10.0)
    ref = og.edge_softmax(eh)
    e = dev(eh)
    G.edge_softmax(e, out=e)                                  # in place (out == e allowed)
    a = e.cpu().numpy()
    assert_within(a, ref, 1.0, "in-place")
    rows = np.repeat(np.arange(V), np.diff(og.fwd_off))
    sums = np.zeros((V, 8))
    np.add.at(sums, rows, a.astype(np.float64))
    nonempty = np.diff(og.fwd_off) > 0
    assert np.allclose(sums[nonempty], 1.0, atol=1e-4)


# ---------------------------------------------------------------- configs
def test_cora_gcn_fwd_bwd(gsp):
    cfg = datagen.CONFIGS["cora"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    Xh = datagen.uniform(1, V, cfg.F)
    dYh = datagen.uniform(2, V, cfg.F)
    ref, T = og.gspmm(Xh, 2, False)
    assert_within(G.gspmm(dev(Xh), 2).cpu().numpy(), ref, T, "cora fwd")
    ref, T = og.gspmm(dYh, 2, True)
    assert_within(G.gspmm(dev(dYh), 2, reverse=True).cpu().numpy(), ref, T, "cora bwd")


def test_pubmed_gat_chain(gsp):
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    H, F = cfg.H, cfg.H * cfg.Fh
    Zh = datagen.uniform(1, V, F)
    s_ref, sT = og.gsddmm(Zh, Zh, H)
    Z = dev(Zh)
    s = G.gsddmm(Z, Z, H=H)
    assert_within(s.cpu().numpy(), s_ref, sT, "pubmed gsddmm")
    lh = datagen.uniform(2, og.E, H, lo=-8, hi=8)
    assert_within(G.edge_softmax(dev(lh)).cpu().numpy(), og.edge_softmax(lh), 1.0, "pubmed softmax")
    wh = datagen.uniform(3, og.E, H, lo=0, hi=1)
    for rev in (0, 1):
        ref, T = og.gspmm_weighted(Zh, wh, rev)
        assert_within(G.gspmm_weighted(Z, dev(wh), reverse=rev).cpu().numpy(), ref, T, f"pubmed w r{rev}")
    # the chain itself (scores -> softmax -> aggregate) vs the oracle's chain, fp32 hand-off;
    # tolerance derived in DESIGN.md "Tolerances" (score error x softmax sensitivity)
    a = G.edge_softmax(s)
    out = G.gspmm_weighted(Z, a).cpu().numpy()
    a_ref = og.edge_softmax(s_ref.astype(np.float32))
    o_ref, oT = og.gspmm_weighted(Zh, a_ref.astype(np.float32))
    assert_within(out, o_ref, oT, "pubmed chain", scale=1e-3)


def test_arxiv_directed_fwd_bwd(gsp):
    cfg = datagen.CONFIGS["arxiv"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    assert not G.symmetric
    Xh = datagen.uniform(1, V, cfg.F)
    for norm in NORMS:
        for rev in (0, 1):
            ref, T = og.gspmm(Xh, norm, rev)
            assert_within(G.gspmm(dev(Xh), norm, reverse=rev).cpu().numpy(), ref, T, f"arxiv n{norm} r{rev}")


# ------------------------------------------------------------- partitions
@pytest.mark.parametrize("name", ["cora", "arxiv"])
def test_partitions_simulated_on_one_gpu(gsp, name):
    """P partitions run one after another on one GPU; the 'all-gather' is a copy
    into the padded [P*R, F] table.  Concatenated outputs == full oracle."""
    cfg = datagen.CONFIGS[name]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    F = 16
    Xh = datagen.uniform(7, V, F)
    for P in (2, 3, 4):
        for rev in ((0, 1) if not G.symmetric else (0,)):
            parts = [G.partition(P, p, device=0, reverse=bool(rev)) for p in range(P)]
            assert all(pg.device_bytes > 0 for pg in parts)
            R = parts[0].R
            b = G.partition_bounds(P, bool(rev))
            Xpad = torch.zeros((P * R, F), device="cuda")
            for p in range(P):
                Xpad[p * R:p * R + b[p + 1] - b[p]] = dev(Xh[b[p]:b[p + 1]])
            for norm in NORMS:
                full, T = og.gspmm(Xh, norm, bool(rev))
                gathered = torch.zeros((P * R, F), device="cuda")
                for p, pg in enumerate(parts):
                    pg.gspmm(Xpad, norm, out=gathered[p * R:(p + 1) * R], reverse=rev)
                    if G.symmetric:   # shared topology also serves the reverse op
                        ref_r, Tr = og.gspmm(Xh, norm, True)
                        o = pg.gspmm(Xpad, norm, reverse=1).cpu().numpy()
                        n = b[p + 1] - b[p]
                        assert_within(o[:n], ref_r[b[p]:b[p + 1]], Tr[b[p]:b[p + 1]], "sym rev part")
                        assert np.all(o[n:] == 0)
                g = gathered.cpu().numpy()
                got = np.concatenate([g[p * R:p * R + b[p + 1] - b[p]] for p in range(P)])
                assert_within(got, full, T, f"{name} P{P} n{norm} r{rev}")


def test_partition_gat_chain_blocks(gsp):
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    H, F, P = 8, 64, 3
    Zh = datagen.uniform(1, V, F)
    wh = datagen.uniform(2, og.E, H, lo=0, hi=1)
    lh = datagen.uniform(3, og.E, H, lo=-6, hi=6)
    s_ref, sT = og.gsddmm(Zh, Zh, H)
    a_ref = og.edge_softmax(lh)
    w_ref, wT = og.gspmm_weighted(Zh, wh, False)
    b = G.partition_bounds(P)
    parts = [G.partition(P, p, device=0) for p in range(P)]
    R = parts[0].R
    Zpad = torch.zeros((P * R, F), device="cuda")
    for p in range(P):
        Zpad[p * R:p * R + b[p + 1] - b[p]] = dev(Zh[b[p]:b[p + 1]])
    for p, pg in enumerate(parts):
        e0, e1 = og.fwd_off[b[p]], og.fwd_off[b[p + 1]]
        n = b[p + 1] - b[p]
        assert pg.E == e1 - e0
        assert_within(pg.gsddmm(Zpad, Zpad, H=H).cpu().numpy(), s_ref[e0:e1], sT[e0:e1], "part gsddmm")
        assert_within(pg.edge_softmax(dev(lh[e0:e1])).cpu().numpy(), a_ref[e0:e1], 1.0, "part softmax")
        o = pg.gspmm_weighted(Zpad, dev(wh[e0:e1])).cpu().numpy()
        assert_within(o[:n], w_ref[b[p]:b[p + 1]], wT[b[p]:b[p + 1]], "part weighted")


# ------------------------------------------------------------------ errors
def test_error_codes(gsp, golden):
    g = golden("d4.json")
    G = gsp.Graph(g["V"], g["src"], g["dst"], device=0)
    X = torch.ones((4, 8), device="cuda")
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm(X, 2, out=X)
    assert ei.value.name == "GSP_ERR_ALIAS"
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm(torch.ones((5, 8), device="cuda"), 2)
    assert ei.value.name == "GSP_ERR_SHAPE"
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm(X, 3)
    assert ei.value.name == "GSP_ERR_ARG"
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm(torch.ones((4, 8)), 2, out=torch.empty((4, 8), device="cuda"))   # host tensor
    assert ei.value.name == "GSP_ERR_ARG"
    Gnr = gsp.Graph(g["V"], g["src"], g["dst"], device=0, reverse=False)
    with pytest.raises(gsp.GspError) as ei:
        Gnr.gspmm(X, 2, reverse=True)
    assert ei.value.name == "GSP_ERR_NO_REVERSE"
    e = torch.ones((7, 2), device="cuda")
    with pytest.raises(gsp.GspError) as ei:
        G.edge_softmax(e, out=e[1:])
    assert ei.value.name in ("GSP_ERR_ALIAS", "GSP_ERR_SHAPE")
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm_weighted(X, torch.ones((7, 3), device="cuda"))
    assert ei.value.name == "GSP_ERR_SHAPE"
    torch.cuda.synchronize()


def test_empty_and_degenerate(gsp):
    G = gsp.Graph(6, np.zeros(0, np.int64), np.zeros(0, np.int64), device=0)
    X = torch.randn((6, 5), device="cuda")
    out = torch.full((6, 5), float("nan"), device="cuda")
    G.gspmm(X, 2, out=out)
    assert torch.all(out == 0)
    out.fill_(float("nan"))
    G.gspmm(X, 2, out=out, reverse=True)
    assert torch.all(out == 0)
    # zero-width features, zero heads
    G.gspmm(torch.empty((6, 0), device="cuda"), 2)
    torch.cuda.synchronize()


def test_partition_weighted_reverse_partials_sum_to_full(gsp):
    """Weighted reverse on fwd partitions: per-source partials over each
    partition's own edges; their sum (the reduce-scatter) == full gSpMMve^T."""
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    H, F = 8, 64
    Zh = datagen.uniform(5, V, F)
    wh = datagen.uniform(6, og.E, H, lo=0, hi=1)
    ref, T = og.gspmm_weighted(Zh, wh, True)
    for P in (2, 3):
        b = G.partition_bounds(P)
        parts = [G.partition(P, p, device=0) for p in range(P)]
        R = parts[0].R
        Zpad = torch.zeros((P * R, F), device="cuda")
        for p in range(P):
            Zpad[p * R:p * R + b[p + 1] - b[p]] = dev(Zh[b[p]:b[p + 1]])
        total = torch.zeros((P * R, F), device="cuda")
        for p, pg in enumerate(parts):
            e0, e1 = og.fwd_off[b[p]], og.fwd_off[b[p + 1]]
            total += pg.gspmm_weighted(Zpad, dev(wh[e0:e1]), reverse=True)
        t = total.cpu().numpy()
        got = np.concatenate([t[p * R:p * R + b[p + 1] - b[p]] for p in range(P)])
        assert_within(got, ref, T, f"P{P} weighted rev partials")


# ---------------------------------------------------- NEXT-1: softmax backward
@pytest.mark.parametrize("H,ld", [(1, 1), (4, 4), (8, 8), (8, 12), (32, 32), (3, 3)])
def test_softmax_backward_random(gsp, H, ld):
    for seed in range(2):
        rng = np.random.default_rng(seed + 11 * H)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 40000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.7))
        G, og = graph_pair(gsp, V, src, dst)
        if E == 0:
            continue
        ah = og.edge_softmax(datagen.uniform(seed, E, H, lo=-6, hi=6)).astype(np.float32)
        gh = datagen.uniform(seed + 1, E, H)
        ref, T = og.edge_softmax_backward(ah, gh)
        out = G.edge_softmax_backward(padded(ah, ld), padded(gh, ld))
        assert_within(out.cpu().numpy(), ref, T, f"H{H} ld{ld}")
        g = dev(gh)
        G.edge_softmax_backward(dev(ah), g, out=g)                 # in place on dalpha
        assert_within(g.cpu().numpy(), ref, T, f"H{H} in place")


# ---------------------------------------------------- NEXT-2: fused GAT forward
def _gat_check(gsp, V, src, dst, H, Fh, Fv, same, ld=None, seed=0):
    G, og = graph_pair(gsp, V, src, dst)
    Xh = datagen.uniform(seed + 1, V, H * Fh)
    Yh = datagen.uniform(seed + 2, V, H * Fh)
    Vh = Yh if same else datagen.uniform(seed + 3, V, H * Fv)
    a_ref, o_ref, T = og.gat_forward(Xh, Yh, Vh, H)
    X = padded(Xh, ld or H * Fh)
    Y = dev(Yh)
    Vt = Y if same else dev(Vh)
    alpha, out = G.gat_forward(X, Y, Vt, H)
    # north_star bound: alpha 1e-5 (1 + 1) absolute, out 1e-5 (T + 1)
    assert_within(alpha.cpu().numpy(), a_ref, 1.0, f"alpha H{H} Fh{Fh}")
    assert_within(out.cpu().numpy(), o_ref, T, f"out H{H} Fh{Fh}")


@pytest.mark.parametrize("H,Fh,Fv,same", [(8, 8, 8, True), (8, 8, 8, False), (2, 8, 8, True), (4, 8, 8, False),
                                          (16, 8, 8, True), (1, 8, 8, True), (3, 5, 4, False), (8, 4, 8, False)])
def test_gat_forward_random(gsp, H, Fh, Fv, same):
    if same and Fv != Fh:
        return
    for seed in range(2):
        rng = np.random.default_rng(seed + 13 * H + Fh)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.6))
        _gat_check(gsp, V, src, dst, H, Fh, Fv, same, seed=seed)


def test_gat_forward_heavy_rows_and_pubmed(gsp):
    V, E = 3000, 400_000
    src, dst = datagen.skewed_multigraph(V, E, 21, alpha=1.6)
    _gat_check(gsp, V, src, dst, 8, 8, 8, True, seed=3)
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    _gat_check(gsp, V, src, dst, 8, 8, 8, True, seed=4)


# ------------------------------------------- NEXT-3: Table 1 surface (min/max, gSpMMe, gSDDMMve)
@pytest.mark.parametrize("F,ld", [(1, 1), (5, 8), (16, 16), (64, 64), (100, 100), (602, 604)])
def test_gspmm_reduce_minmax(gsp, F, ld):
    for seed in range(2):
        rng = np.random.default_rng(seed + F)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.6))
        G, og = graph_pair(gsp, V, src, dst)
        Xh = datagen.uniform(seed + 3, V, F)
        X = padded(Xh, ld)
        for red in (gsp.REDUCE_MIN, gsp.REDUCE_MAX, gsp.REDUCE_SUM):
            for rev in (0, 1):
                ref, T = og.gspmm_reduce(Xh, red, bool(rev))
                out = G.gspmm_reduce(X, red, reverse=rev).cpu().numpy()
                if red == gsp.REDUCE_SUM:
                    assert_within(out, ref, T, f"sum r{rev}")
                else:   # min / max pick an input exactly
                    assert np.array_equal(out.astype(np.float64), ref), (red, rev)


@pytest.mark.parametrize("H", [1, 2, 4, 8, 16, 32, 5, 40])
def test_gspmm_e(gsp, H):
    for seed in range(2):
        rng = np.random.default_rng(seed + 3 * H)
        V = int(rng.integers(1, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.6))
        G, og = graph_pair(gsp, V, src, dst)
        wh = datagen.uniform(seed + 5, E, H) if E else np.zeros((0, H), np.float32)
        for red in (gsp.REDUCE_SUM, gsp.REDUCE_MIN, gsp.REDUCE_MAX):
            for rev in (0, 1):
                ref, T = og.gspmm_e(wh, red, bool(rev))
                out = G.gspmm_e(dev(wh), red, reverse=rev).cpu().numpy()
                if red == gsp.REDUCE_SUM:
                    assert_within(out, ref, T, f"gspmm_e sum r{rev}")
                else:
                    assert np.array_equal(out.astype(np.float64), ref), (red, rev)


@pytest.mark.parametrize("H", [1, 3, 4, 8, 16, 32])
def test_gsddmm_ve(gsp, H):
    rng = np.random.default_rng(H)
    V = int(rng.integers(1, 2500))
    E = int(rng.integers(1, 30000))
    src, dst = datagen.skewed_multigraph(V, E, H, alpha=1.5)
    G, og = graph_pair(gsp, V, src, dst)
    Xh = datagen.uniform(1, V, H, lo=0.5, hi=2.0)
    wh = datagen.uniform(2, E, H)
    for op in (gsp.OP_ADD, gsp.OP_SUB, gsp.OP_MUL, gsp.OP_DIV):
        for side in (gsp.SIDE_DST, gsp.SIDE_SRC):
            ref = og.gsddmm_ve(Xh, wh, op, side)
            out = G.gsddmm_ve(dev(Xh), dev(wh), op, side).cpu().numpy()
            # one IEEE fp32 operation on exact fp32 inputs: correctly rounded
            assert np.array_equal(out, ref.astype(np.float32)), (op, side)
    # additive GAT scores: e = a_dst[v] + a_src[u] as two calls, the second in place
    a_dst, a_src = datagen.uniform(3, V, H), datagen.uniform(4, V, H)
    e = G.gsddmm_ve(dev(a_dst), torch.zeros((E, H), device="cuda"), gsp.OP_ADD, gsp.SIDE_DST)
    G.gsddmm_ve(dev(a_src), e, gsp.OP_ADD, gsp.SIDE_SRC, out=e)
    row_of = np.repeat(np.arange(V), np.diff(og.fwd_off))
    ref = (a_dst[row_of].astype(np.float32) + a_src[og.fwd_col].astype(np.float32))
    assert np.array_equal(e.cpu().numpy(), ref)


@pytest.mark.parametrize("H,ld", [(8, 8), (8, 12), (8, 10), (16, 20), (4, 4)])
def test_next3_heavy_rows_and_strides(gsp, H, ld):
    """gSpMMe / gSDDMMve on a graph with CTA-split hub rows (degree 3000 and
    2049, just past the 2048-edge heavy threshold; 1025, a long warp row),
    empty rows and ragged light rows; edge-value rows padded to ld (NaN
    padding: never read)."""
    rng = np.random.default_rng(H * 100 + ld)
    V = 3100
    hub_src = rng.integers(0, V, 3000 + 1025 + 2049)
    hub_dst = np.concatenate([np.zeros(3000, np.int64), np.full(1025, 7, np.int64), np.full(2049, 11, np.int64)])
    m = 6000
    s2, d2 = rng.integers(0, V, m), rng.integers(20, V - 20, m)
    src = np.concatenate([hub_src, s2]).astype(np.int64)
    dst = np.concatenate([hub_dst, d2]).astype(np.int64)
    E = len(src)
    G, og = graph_pair(gsp, V, src, dst)
    wh = datagen.uniform(H + ld, E, H)
    w = padded(wh, ld)
    for red in (gsp.REDUCE_SUM, gsp.REDUCE_MIN, gsp.REDUCE_MAX):
        for rev in (0, 1):
            ref, T = og.gspmm_e(wh, red, bool(rev))
            out = G.gspmm_e(w, red, reverse=rev).cpu().numpy()
            if red == gsp.REDUCE_SUM:
                assert_within(out, ref, T, f"gspmm_e sum r{rev}")
            else:
                assert np.array_equal(out.astype(np.float64), ref), (red, rev)
    Xh = datagen.uniform(9, V, H, lo=0.5, hi=2.0)
    X = padded(Xh, ld)
    for op in (gsp.OP_ADD, gsp.OP_SUB, gsp.OP_MUL, gsp.OP_DIV):
        for side in (gsp.SIDE_DST, gsp.SIDE_SRC):
            ref = og.gsddmm_ve(Xh, wh, op, side).astype(np.float32)
            out = padded(np.zeros((E, H), np.float32), ld)
            G.gsddmm_ve(X, w, op, side, out=out)
            assert np.array_equal(out.cpu().numpy(), ref), (op, side)
            # in place: out aliases w
            w2 = padded(wh, ld)
            G.gsddmm_ve(X, w2, op, side, out=w2)
            assert np.array_equal(w2.cpu().numpy(), ref), (op, side, "in place")


# ------------------------------------------------ tile / bin boundary degrees
def _boundary_graph():
    """Destination rows with degrees exactly at the kernels' tile (32), fold
    (4 x 32) and heavy-bin (2048; formerly 1024) boundaries, plus empty rows; sources random."""
    degs = [0, 1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 1023, 1024, 1025, 2047, 2048, 2049, 4097, 0, 7]
    V = 300
    rng = np.random.default_rng(5)
    dst = np.concatenate([np.full(d, v, np.int64) for v, d in enumerate(degs)])
    src = rng.integers(0, V, size=len(dst)).astype(np.int64)
    perm = rng.permutation(len(dst))
    return V, src[perm], dst[perm]


def test_boundary_degrees_all_ops(gsp):
    V, src, dst = _boundary_graph()
    G, og = graph_pair(gsp, V, src, dst)
    E = og.E
    for F in (16, 64, 100):
        Xh = datagen.uniform(F, V, F, lo=0.0, hi=1.0)
        for norm in NORMS:
            for rev in (0, 1):
                ref, T = og.gspmm(Xh, norm, bool(rev))
                assert_within(G.gspmm(dev(Xh), norm, reverse=rev).cpu().numpy(), ref, T, f"F{F} n{norm} r{rev}")
        for red in (gsp.REDUCE_MIN, gsp.REDUCE_MAX):
            ref, _ = og.gspmm_reduce(Xh, red)
            assert np.array_equal(G.gspmm_reduce(dev(Xh), red).cpu().numpy().astype(np.float64), ref)
    H, Fh = 8, 8
    Zh = datagen.uniform(1, V, H * Fh)
    wh = datagen.uniform(2, E, H, lo=0, hi=1)
    for rev in (0, 1):
        ref, T = og.gspmm_weighted(Zh, wh, bool(rev))
        assert_within(G.gspmm_weighted(dev(Zh), dev(wh), reverse=rev).cpu().numpy(), ref, T, f"w r{rev}")
    ref, T = og.gsddmm(Zh, Zh, H)
    assert_within(G.gsddmm(dev(Zh), dev(Zh), H=H).cpu().numpy(), ref, T, "gsddmm")
    lh = datagen.uniform(3, E, H, lo=-9, hi=9)
    ah = og.edge_softmax(lh)
    assert_within(G.edge_softmax(dev(lh)).cpu().numpy(), ah, 1.0, "softmax")
    gh = datagen.uniform(4, E, H)
    ref, T = og.edge_softmax_backward(ah.astype(np.float32), gh)
    assert_within(G.edge_softmax_backward(dev(ah.astype(np.float32)), dev(gh)).cpu().numpy(), ref, T, "sbwd")
    a_ref, o_ref, T = og.gat_forward(Zh, Zh, Zh, H)
    alpha, out = G.gat_forward(dev(Zh), dev(Zh), dev(Zh), H)
    assert_within(alpha.cpu().numpy(), a_ref, 1.0, "gat alpha")
    assert_within(out.cpu().numpy(), o_ref, T, "gat out")


def test_cuda_graph_capture_replay(gsp):
    """Compute calls allocate nothing and never synchronise, so a whole GCN +
    GAT step can be captured into a CUDA graph (the launch-bound Cora / Pubmed
    regime, SURVEY §7 hard part 6) and replayed with identical results."""
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    G = gsp.Graph(V, src, dst, device=0)
    X = dev(datagen.uniform(1, V, 64))
    o1 = torch.empty((V, 64), device="cuda")
    o2 = torch.empty((V, 64), device="cuda")
    o3 = torch.empty((V, 64), device="cuda")
    s = torch.empty((G.E, 8), device="cuda")
    st = torch.cuda.Stream()

    def step():
        G.gspmm(X, gsp.NORM_BOTH, out=o1, stream=st)
        G.gspmm(o1, gsp.NORM_BOTH, out=o2, reverse=True, stream=st)
        G.gsddmm(X, X, out=s, stream=st)
        G.edge_softmax(s, out=s, stream=st)
        G.gspmm_weighted(X, s, out=o3, stream=st)

    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    ref = [t.clone() for t in (o1, o2, o3, s)]
    for t in (o1, o2, o3, s):
        t.zero_()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        step()
    gr.replay()
    torch.cuda.synchronize()
    for a, b in zip((o1, o2, o3, s), ref):
        assert torch.equal(a, b)


# ------------------------------------------- NEXT-1: fused GAT backward scores
def _gat_bwd_check(gsp, V, src, dst, H, Fh, seed=0):
    """ds = C9(alpha, C6(dOut, Vt)) composed from the oracle.  Bound 1e-5 (T + 1),
    T = C9's sum|terms| plus the propagation of dalpha's own fp32 dot error:
    alpha_j T6_j + alpha_j sum_j' alpha_j' T6_j' (T6 = C6's sum|terms|)."""
    G, og = graph_pair(gsp, V, src, dst)
    F = H * Fh
    dOh = datagen.uniform(seed + 1, V, F)
    Vh = datagen.uniform(seed + 2, V, F)
    ah = og.edge_softmax(datagen.uniform(seed + 3, og.E, H, lo=-4, hi=4)).astype(np.float32)
    d64, T6 = og.gsddmm(dOh, Vh, H)
    ref, T9 = og.edge_softmax_backward(ah, d64.astype(np.float32))
    rid = np.repeat(np.arange(V), np.diff(og.fwd_off))
    S = np.zeros((V, H))
    np.add.at(S, rid, ah * T6)
    T = T9 + ah * T6 + ah * S[rid]
    ds = G.gat_backward_scores(dev(dOh), dev(Vh), dev(ah))
    assert_within(ds.cpu().numpy(), ref, T, f"gat bwd H{H} Fh{Fh}")
    return G, og


@pytest.mark.parametrize("H,Fh", [(8, 8), (4, 8), (2, 8), (16, 8), (1, 8), (3, 5), (8, 4)])
def test_gat_backward_scores_random(gsp, H, Fh):
    for seed in range(2):
        rng = np.random.default_rng(seed + 10 * H + Fh)
        V = int(rng.integers(50, 2500))
        E = int(rng.integers(0, 30000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0 else datagen.skewed_multigraph(V, E, seed))
        _gat_bwd_check(gsp, V, src, dst, H, Fh, seed)


def test_gat_backward_scores_heavy_rows_pubmed_and_errors(gsp):
    V, E = 3000, 120_000   # CTA-split hub rows (> 2048 edges) and rows past the 224-edge score block
    src, dst = datagen.skewed_multigraph(V, E, 4, alpha=1.6)
    G, og = _gat_bwd_check(gsp, V, src, dst, 8, 8, seed=4)
    assert np.diff(og.fwd_off).max() > 2048
    cfg = datagen.CONFIGS["pubmed"]
    Vp, sp, dp = datagen.make_graph(cfg)
    _gat_bwd_check(gsp, Vp, sp, dp, cfg.H, cfg.Fh, seed=5)
    a = torch.rand((og.E, 8), device="cuda")
    X = torch.rand((V, 64), device="cuda")
    with pytest.raises(gsp.GspError) as ei:
        G.gat_backward_scores(X, X, a, out=a)
    assert ei.value.name == "GSP_ERR_ALIAS"
    with pytest.raises(gsp.GspError) as ei:
        G.gat_backward_scores(X[:, :60], X[:, :60], torch.rand((og.E, 8), device="cuda"))
    assert ei.value.name == "GSP_ERR_SHAPE"


def test_odd_output_stride_keeps_vector_gathers(gsp):
    """X rows 16-B aligned (vector gathers) but out rows not (ld % 4 != 0: F = 602
    written densely, odd padding): the row stores fall back to scalar, results
    unchanged -- gSpMM all norms / directions and weighted fwd / rev."""
    V, E = 2000, 60_000
    src, dst = datagen.skewed_multigraph(V, E, 8)
    G, og = graph_pair(gsp, V, src, dst)
    for F, ldx, ldo in [(602, 604, 602), (6, 8, 6), (64, 64, 65), (8, 8, 9)]:
        Xh = datagen.uniform(F + ldo, V, F)
        X = padded(Xh, ldx)
        for norm in NORMS:
            for rev in (0, 1):
                ref, T = og.gspmm(Xh, norm, rev)
                out = padded(np.full((V, F), np.nan, np.float32), ldo)
                G.gspmm(X, norm, out=out, reverse=rev)
                assert_within(out.cpu().numpy(), ref, T, f"F{F} ldx{ldx} ldo{ldo} n{norm} r{rev}")
    H, Fh, ldo = 2, 4, 9
    Xh = datagen.uniform(3, V, H * Fh)
    wh = datagen.uniform(4, og.E, H, lo=0.0, hi=1.0)
    for rev in (0, 1):
        ref, T = og.gspmm_weighted(Xh, wh, bool(rev))
        out = padded(np.full((V, H * Fh), np.nan, np.float32), ldo)
        G.gspmm_weighted(dev(Xh), dev(wh), out=out, reverse=rev)
        assert_within(out.cpu().numpy(), ref, T, f"weighted ldo{ldo} r{rev}")


# ------------------------------------------------- chunked partitions (A9)
def chunk_layout(G, P, C):
    """(bounds of the P*C blocks, slot of block q, R) of the chunk-major layout."""
    b = G.partition_bounds(P * C)
    R = int(np.max(np.diff(b)))
    return b, (lambda q: (q % C) * P + q // C), R


@pytest.mark.parametrize("name,P,C", [("pubmed", 2, 3), ("arxiv", 2, 2), ("cora", 3, 4)])
def test_chunked_partitions_simulated_on_one_gpu(gsp, name, P, C):
    """Every (rank, chunk) partition runs on one GPU, each writing its [R, F] block
    straight into its chunk's all-gather range [c*P*R, (c+1)*P*R) of the padded
    table (the NCCL all-gather replaced by the output placement).  Un-padded:
    == the oracle, element by element, for the three norms.  Reverse: symmetric
    graphs over the shared topology (own rows), directed graphs as per-source
    partials summed over all partitions (the reduce-scatter)."""
    V, src, dst = datagen.make_graph(name)
    G, og = graph_pair(gsp, V, src, dst)
    F = 16
    Xh = datagen.uniform(11, V, F)
    b, slot, R = chunk_layout(G, P, C)
    Q = P * C
    parts = {(p, c): G.partition(P, p, device=0, nchunks=C, chunk=c) for p in range(P) for c in range(C)}
    Xpad = torch.zeros((Q * R, F), device="cuda")
    for q in range(Q):
        Xpad[slot(q) * R:slot(q) * R + b[q + 1] - b[q]] = dev(Xh[b[q]:b[q + 1]])

    def unpad(t):
        g = t.cpu().numpy()
        return np.concatenate([g[slot(q) * R:slot(q) * R + b[q + 1] - b[q]] for q in range(Q)])

    for norm in NORMS:
        full, T = og.gspmm(Xh, norm, False)
        table = torch.full((Q * R, F), float("nan"), device="cuda")
        for (p, c), pg in parts.items():
            assert pg.row_base == slot(p * C + c) * R
            pg.gspmm(Xpad, norm, out=table[(c * P + p) * R:(c * P + p + 1) * R])
        assert_within(unpad(table), full, T, f"{name} chunked fwd n{norm}")
        ref_r, Tr = og.gspmm(Xh, norm, True)
        if G.symmetric:
            table.fill_(float("nan"))
            for (p, c), pg in parts.items():
                pg.gspmm(Xpad, norm, out=table[(c * P + p) * R:(c * P + p + 1) * R], reverse=True)
            assert_within(unpad(table), ref_r, Tr, f"{name} chunked sym rev n{norm}")
        else:
            acc = torch.zeros((Q * R, F), dtype=torch.float64, device="cuda")
            for pg in parts.values():
                assert pg.reverse_gives_partials()
                acc += pg.gspmm(Xpad, norm, reverse=True).double()
            assert_within(unpad(acc), ref_r, Tr, f"{name} chunked partial rev n{norm}")


def test_chunked_partition_gat_forward(gsp):
    """The fused GAT forward on chunked partitions reads its destination rows at
    row_base + r of the padded table; local edge ids are the block's global range."""
    cfg = datagen.CONFIGS["pubmed"]
    V, src, dst = datagen.make_graph(cfg)
    G, og = graph_pair(gsp, V, src, dst)
    H, F, P, C = 8, 64, 2, 2
    Zh = datagen.uniform(21, V, F)
    b, slot, R = chunk_layout(G, P, C)
    Zpad = torch.zeros((P * C * R, F), device="cuda")
    for q in range(P * C):
        Zpad[slot(q) * R:slot(q) * R + b[q + 1] - b[q]] = dev(Zh[b[q]:b[q + 1]])
    a_ref, o_ref, T = og.gat_forward(Zh, Zh, Zh, H)
    for p in range(P):
        for c in range(C):
            q = p * C + c
            pg = G.partition(P, p, device=0, nchunks=C, chunk=c)
            e0, e1 = og.fwd_off[b[q]], og.fwd_off[b[q + 1]]
            alpha, out = pg.gat_forward(Zpad, Zpad, Zpad, H)
            n = b[q + 1] - b[q]
            assert_within(alpha.cpu().numpy(), a_ref[e0:e1], 1.0, "chunk alpha")
            assert_within(out.cpu().numpy()[:n], o_ref[b[q]:b[q + 1]], T[b[q]:b[q + 1]], "chunk gat out")


# ---------------------------------------------------- GCN-lean device format
@pytest.mark.parametrize("name", ["pubmed", "arxiv"])
def test_no_edge_ids_graph(gsp, name):
    """GSP_BUILD_NO_EDGE_IDS ("For GCN, GraphPy need only (|V|+|E|)"): a
    symmetric graph holds one topology (8(V+1) + 4E bytes), a directed one two;
    no edge-id bytes; gSpMMv in both directions still matches the oracle; the
    edge-ID indirected reverse reports GSP_ERR_NO_REVERSE."""
    V, src, dst = datagen.make_graph(name)
    G = gsp.Graph(V, src, dst, device=0, edge_ids=False, edge_scales=False)
    og = oracle.Graph(V, src, dst)
    m = G.memory()
    per = 8 * (V + 1) + 4 * og.E
    assert m["topology"] == (per if G.symmetric else 2 * per)
    assert m["edge_ids"] == 0 and m["edge_scales"] == 0
    assert sum(m.values()) == G.device_bytes
    assert m["vertex_arrays"] < 64 * V          # O(V): scales + schedules
    Xh = datagen.uniform(4, V, 32)
    for norm in NORMS:
        for rev in (0, 1):
            ref, T = og.gspmm(Xh, norm, bool(rev))
            assert_within(G.gspmm(dev(Xh), norm, reverse=rev).cpu().numpy(), ref, T, f"lean n{norm} r{rev}")
    w = torch.rand((og.E, 1), device="cuda")
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm_weighted(dev(Xh), w, reverse=True)
    assert ei.value.name == "GSP_ERR_NO_REVERSE"
    # the default graph: edge ids and (on request) per-edge scales are accounted separately
    Gd = gsp.Graph(V, src, dst, device=0, edge_scales=True)
    md = Gd.memory()
    assert md["edge_ids"] == 4 * og.E and md["edge_scales"] == 4 * og.E * (1 if Gd.symmetric else 2)
    assert sum(md.values()) == Gd.device_bytes


# ------------------------------------------------ aliasing of strided views
def test_alias_exact_for_column_slices(gsp):
    """Disjoint column slices of one buffer are not aliases (exact strided test);
    interleaving or overlapping ones are; broadcast rows are rejected."""
    V, src, dst = datagen.make_graph("cora")
    G, og = graph_pair(gsp, V, src, dst)
    F = 8
    Xh = datagen.uniform(5, V, F)
    B = torch.zeros((V, 2 * F), device="cuda")
    B[:, :F] = dev(Xh)
    G.gspmm(B[:, :F], gsp.NORM_BOTH, out=B[:, F:])
    ref, T = og.gspmm(Xh, gsp.NORM_BOTH, False)
    assert_within(B[:, F:].cpu().numpy(), ref, T, "column-slice out")
    with pytest.raises(gsp.GspError) as ei:
        G.gspmm(B[:, :F], gsp.NORM_BOTH, out=B[:, F // 2:F // 2 + F])
    assert ei.value.name == "GSP_ERR_ALIAS"
    C = torch.zeros((V + 1, F), device="cuda")
    with pytest.raises(gsp.GspError) as ei:      # rows shifted by one: overlapping
        G.gspmm(C[:V], gsp.NORM_BOTH, out=C[1:])
    assert ei.value.name == "GSP_ERR_ALIAS"
    with pytest.raises(ValueError):
        G.gspmm(torch.zeros(F, device="cuda").expand(V, F), gsp.NORM_BOTH)


# ------------------------------------- margin of approximate exp
def test_approx_exp_paths_keep_10x_margin(gsp, golden):
    """the kernels' exp is ex2.approx (edge softmax, fused GAT
    forward); allowed only if parity holds with >= 10x margin, i.e. max
    err/bound <= 0.1 on T4 / D4 / random graphs (brute-force sizes) and Pubmed."""
    graphs = []
    for gf in ("t4.json", "d4.json"):
        g = golden(gf)
        graphs.append((gf, g["V"], np.array(g["src"], np.int64), np.array(g["dst"], np.int64)))
    for seed in range(6):
        rng = np.random.default_rng(900 + seed)
        V = int(rng.integers(2, 64)) if seed < 3 else int(rng.integers(200, 3000))
        E = int(rng.integers(1, 40 * V))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed % 2 == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.5))
        graphs.append((f"random{seed}", V, src, dst))
    graphs.append(("pubmed",) + datagen.make_graph("pubmed"))
    worst = {"edge_softmax": 0.0, "gat_fused_alpha": 0.0, "gat_fused_out": 0.0}
    for name, V, src, dst in graphs:
        G, og = graph_pair(gsp, V, src, dst)
        for H in (1, 4, 8):
            lh = datagen.uniform(V + H, og.E, H, lo=-8, hi=8)
            r = assert_within(G.edge_softmax(dev(lh)).cpu().numpy(), og.edge_softmax(lh), 1.0, f"{name} sm H{H}")
            worst["edge_softmax"] = max(worst["edge_softmax"], r)
        for H in (2, 8):     # the fused (one pass) kernel: Fh = 8
            Zh = datagen.uniform(V + 7 * H, V, 8 * H)
            Vh = datagen.uniform(V + 9 * H, V, 8 * H)
            a_ref, o_ref, T = og.gat_forward(Zh, Zh, Vh, H)
            alpha, out = G.gat_forward(dev(Zh), dev(Zh), dev(Vh), H)
            worst["gat_fused_alpha"] = max(worst["gat_fused_alpha"],
                                           assert_within(alpha.cpu().numpy(), a_ref, 1.0, f"{name} a H{H}"))
            worst["gat_fused_out"] = max(worst["gat_fused_out"],
                                         assert_within(out.cpu().numpy(), o_ref, T, f"{name} out H{H}"))
    print("approx-exp margins (max err/bound):", worst)
    for k, v in worst.items():
        assert v <= 0.1, f"{k}: max err/bound {v:.3g} > 0.1 (SURVEY L18 10x margin)"


# ----------------------------------------- NEXT-3: additive GAT attention
def _additive_inputs(V, H, Fvh, seed):
    el = datagen.uniform(seed, V, H, lo=-4, hi=4)
    er = datagen.uniform(seed + 1, V, H, lo=-4, hi=4)
    Vh = datagen.uniform(seed + 2, V, H * Fvh)
    return el, er, Vh


@pytest.mark.parametrize("H", [1, 2, 3, 4, 8, 16])
def test_gsddmm_add_leaky_random(gsp, H):
    """C14 element by element; T = |el[u]| + |er[v]| (the sum's terms)."""
    for seed in range(3):
        rng = np.random.default_rng(40 + seed + H)
        V = int(rng.integers(1, 3000))
        E = int(rng.integers(0, 50000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed != 1
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.6))
        G, og = graph_pair(gsp, V, src, dst)
        el, er, _ = _additive_inputs(V, H, 1, seed)
        for slope in (0.2, 0.01):
            ref = og.gsddmm_add_leaky(el, er, slope)
            rid = np.repeat(np.arange(V), np.diff(og.fwd_off))
            T = np.abs(el[og.fwd_col]).astype(np.float64) + np.abs(er[rid])
            out = G.gsddmm_add_leaky(padded(el, H + 3), dev(er), slope)
            assert_within(out.cpu().numpy(), ref, T, f"add_leaky H{H} s{slope}")


def test_gsddmm_add_leaky_t4_golden_and_errors(gsp, golden):
    g, c = golden("t4.json"), golden("t4_additive.json")
    G = gsp.Graph(g["V"], g["src"], g["dst"], device=0)
    el = dev(np.array(c["el"], np.float32)[:, None])
    er = dev(np.array(c["er"], np.float32)[:, None])
    out = G.gsddmm_add_leaky(el, er, c["slope"]).cpu().numpy()[:, 0]
    assert np.allclose(out, c["scores"], rtol=1e-6, atol=1e-7)
    assert G.gsddmm_add_leaky(el, er, 1.0).cpu().numpy()[:, 0].tolist() == c["scores_slope1"]
    with pytest.raises(gsp.GspError) as ei:
        G.gsddmm_add_leaky(el, torch.zeros((4, 2), device="cuda"))
    assert ei.value.name == "GSP_ERR_SHAPE"
    with pytest.raises(gsp.GspError) as ei:
        G.gsddmm_add_leaky(el, er, float("nan"))
    assert ei.value.name == "GSP_ERR_ARG"


def _gat_add_check(gsp, V, src, dst, H, Fvh, seed=0, slope=0.2):
    G, og = graph_pair(gsp, V, src, dst)
    el, er, Vh = _additive_inputs(V, H, Fvh, seed)
    a_ref, o_ref, T = og.gat_forward_additive(el, er, Vh, slope)
    alpha, out = G.gat_forward_additive(dev(el), dev(er), dev(Vh), slope)
    ra = assert_within(alpha.cpu().numpy(), a_ref, 1.0, f"add alpha H{H} Fvh{Fvh}")
    ro = assert_within(out.cpu().numpy(), o_ref, T, f"add out H{H} Fvh{Fvh}")
    return ra, ro


@pytest.mark.parametrize("H,Fvh", [(8, 8), (2, 8), (4, 8), (16, 8), (1, 8), (3, 4), (8, 4)])
def test_gat_forward_additive_random(gsp, H, Fvh):
    """C15 (fused one-pass kernel for Fvh = 8, H in {2,4,8,16}; three kernels otherwise)."""
    for seed in range(2):
        rng = np.random.default_rng(60 + seed + 7 * H)
        V = int(rng.integers(2, 2500))
        E = int(rng.integers(0, 40000))
        src, dst = (datagen.random_multigraph(V, E, seed) if seed == 0
                    else datagen.skewed_multigraph(V, E, seed, alpha=1.7))
        _gat_add_check(gsp, V, src, dst, H, Fvh, seed)


def test_gat_forward_additive_heavy_and_boundary_rows(gsp):
    V, src, dst = _boundary_graph()
    _gat_add_check(gsp, V, src, dst, 8, 8, seed=3)
    V, E = 3000, 120_000      # CTA-split hub rows (> 2048 edges), rows past the smem score block
    src, dst = datagen.skewed_multigraph(V, E, 4, alpha=1.6)
    _gat_add_check(gsp, V, src, dst, 8, 8, seed=4, slope=0.01)
    cfg = datagen.CONFIGS["pubmed"]
    _gat_add_check(gsp, *datagen.make_graph(cfg), cfg.H, cfg.Fh, seed=5)


def test_gat_forward_additive_margin(gsp, golden):
    """SURVEY L18 margin (ex2.approx in the one-pass kernel): <= 0.1 of the bound."""
    worst = [0.0, 0.0]
    graphs = [datagen.make_graph("pubmed")]
    for gf in ("t4.json", "d4.json"):
        g = golden(gf)
        graphs.append((g["V"], np.array(g["src"], np.int64), np.array(g["dst"], np.int64)))
    for seed in range(4):
        rng = np.random.default_rng(990 + seed)
        V = int(rng.integers(2, 64)) if seed < 2 else int(rng.integers(200, 3000))
        graphs.append((V,) + datagen.random_multigraph(V, int(rng.integers(1, 40 * V)), seed))
    for i, (V, src, dst) in enumerate(graphs):
        for H in (2, 8):
            ra, ro = _gat_add_check(gsp, V, src, dst, H, 8, seed=i)
            worst = [max(worst[0], ra), max(worst[1], ro)]
    print("additive GAT margins (alpha, out):", worst)
    assert max(worst) <= 0.1, worst
