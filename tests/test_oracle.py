"""Pins for the CPU oracle (no GPU).  Each test ties an oracle function to
something other than itself: the worked examples SPEC.md / SURVEY.md print
(tests/golden/), the closed form D^-1/2 A D^-1/2 X on dense adjacency
(BASELINE.json north_star), brute-force dense products built straight from the
COO list with numpy (never from the oracle's CSR), the adjoint / bilinear
identities of P:1340-1341 "Backward Computation", and the softmax
characterisation (positive, sums to 1, ratios exp(e_j - e_k)) plus
scipy.special.softmax per row.
"""
import numpy as np
import pytest
import scipy.special

import datagen
import oracle
from oracle import NORM_BOTH, NORM_NONE, NORM_RIGHT


# ----------------------------------------------------------------- helpers
def dense_adj(V, src, dst, wts=None):
    """A[v, u] = sum over COO edges u->v of weight (multiplicity when wts is None)."""
    A = np.zeros((V, V), np.float64)
    np.add.at(A, (dst, src), 1.0 if wts is None else wts)
    return A


def dense_operator(V, src, dst, norm):
    """Matrix M of the forward op (fwd(X) = M X), from the COO list only."""
    A = dense_adj(V, src, dst)
    din = np.maximum(np.bincount(dst, minlength=V), 1).astype(np.float64)
    dout = np.maximum(np.bincount(src, minlength=V), 1).astype(np.float64)
    if norm == NORM_NONE:
        return A
    if norm == NORM_RIGHT:
        return A / din[:, None]
    return (din ** -0.5)[:, None] * A * (dout ** -0.5)[None, :]


def rand_graph(seed, Vmax=64, Emax=300):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(1, Vmax + 1))
    E = int(rng.integers(0, Emax + 1))
    src, dst = datagen.random_multigraph(V, E, seed)
    return V, src, dst


def check(out, T, ref):
    err = np.abs(np.asarray(out) - np.asarray(ref))
    # oracle is fp64 vs fp64 dense: demand far below the fp32 bound
    assert np.all(err <= 1e-9 * (np.asarray(T) + 1.0)), float(err.max())


# --------------------------------------------------------- C1 golden + brute
def test_build_t4_golden(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    assert G.fwd_off.tolist() == g["fwd_off"]
    assert G.fwd_col.tolist() == g["fwd_col"]
    assert G.rev_eid.tolist() == g["rev_eid"]
    # symmetric graph: rev topology equals fwd topology ("one copy of the topology")
    assert G.rev_off.tolist() == g["fwd_off"]
    assert G.rev_col.tolist() == g["fwd_col"]
    assert np.diff(G.fwd_off).tolist() == g["deg"]


def test_build_d4_golden(golden):
    g = golden("d4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    for k in ["fwd_off", "fwd_col", "coo_to_eid", "rev_off", "rev_col", "rev_eid"]:
        assert getattr(G, k).tolist() == g[k], k
    assert np.diff(G.fwd_off).tolist() == g["d_in"]
    assert np.diff(G.rev_off).tolist() == g["d_out"]


def brute_build(V, src, dst):
    """Definition C1 by Python's sorted() on tuples (independent of the C qsort)."""
    E = len(src)
    order = sorted(range(E), key=lambda i: (int(dst[i]), int(src[i]), i))
    fwd_col = [int(src[i]) for i in order]
    fwd_off = [sum(1 for i in range(E) if dst[i] < v) for v in range(V + 1)]
    coo_to_eid = [0] * E
    for j, i in enumerate(order):
        coo_to_eid[i] = j
    sd = [(int(src[order[j]]), int(dst[order[j]]), j) for j in range(E)]
    rorder = sorted(range(E), key=lambda j: sd[j])
    rev_col = [sd[j][1] for j in rorder]
    rev_off = [sum(1 for i in range(E) if src[i] < u) for u in range(V + 1)]
    return fwd_off, fwd_col, coo_to_eid, rev_off, rev_col, list(rorder)


@pytest.mark.parametrize("seed", range(40))
def test_build_bruteforce(seed):
    V, src, dst = rand_graph(seed, Vmax=20, Emax=60)
    G = oracle.Graph(V, src, dst)
    fo, fc, c2e, ro, rc, re = brute_build(V, src, dst)
    assert G.fwd_off.tolist() == fo
    assert G.fwd_col.tolist() == fc
    assert G.coo_to_eid.tolist() == c2e
    assert G.rev_off.tolist() == ro
    assert G.rev_col.tolist() == rc
    assert G.rev_eid.tolist() == re


@pytest.mark.parametrize("seed", range(20))
def test_build_invariants(seed):
    V, src, dst = rand_graph(1000 + seed, Vmax=64, Emax=400)
    G = oracle.Graph(V, src, dst)
    E = len(src)
    assert sorted(G.rev_eid.tolist()) == list(range(E))
    assert sorted(G.coo_to_eid.tolist()) == list(range(E))
    row_of = np.repeat(np.arange(V), np.diff(G.fwd_off))
    assert np.array_equal(G.fwd_col[G.coo_to_eid], src)
    assert np.array_equal(row_of[G.coo_to_eid], dst)
    rrow = np.repeat(np.arange(V), np.diff(G.rev_off))
    assert np.array_equal(G.fwd_col[G.rev_eid], rrow)
    assert np.array_equal(row_of[G.rev_eid], G.rev_col)
    # the dense multiplicity matrix is the same from COO, fwd and rev
    A = dense_adj(V, src, dst)
    assert np.array_equal(dense_adj(V, G.fwd_col, row_of), A)
    assert np.array_equal(dense_adj(V, rrow, G.rev_col), A)


def test_symmetric_eid_involution():
    """on a symmetric simple graph, pairing slot (r->c) with (c->r) is an involution."""
    V = 200
    src, dst = datagen.chung_lu(V, 900, 0.5, 7)
    G = oracle.Graph(V, src, dst)
    assert np.array_equal(G.rev_off, G.fwd_off) and np.array_equal(G.rev_col, G.fwd_col)
    p = G.rev_eid.astype(np.int64)
    assert np.array_equal(p[p], np.arange(G.E))


def test_build_rejects_bad_ids():
    with pytest.raises(ValueError):
        oracle.Graph(3, [0, 3], [1, 1])
    with pytest.raises(ValueError):
        oracle.Graph(3, [0, -1], [1, 1])


def test_build_empty():
    G = oracle.Graph(5, np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert G.fwd_off.tolist() == [0] * 6 and G.rev_off.tolist() == [0] * 6
    G0 = oracle.Graph(0, np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert G0.fwd_off.tolist() == [0]


# ------------------------------------------------------------ C2/C3 scales
def test_scales_t4_and_clamp(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    sd, ss = G.scales(NORM_RIGHT)
    assert np.allclose(sd, 1.0 / np.array(g["deg"]), rtol=0, atol=1e-15) and np.all(ss == 1)
    # isolated vertex clamps to degree 1
    G5 = oracle.Graph(5, g["src"], g["dst"])
    sd, ss = G5.scales(NORM_BOTH)
    assert sd[4] == 1.0 and ss[4] == 1.0


# ------------------------------------------------------------------ C4 gspmm
def test_gspmm_t4_golden(golden):
    g = golden("t4.json")
    c = golden("t4_chain.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    X = np.array(g["X"], np.float32)[:, None]
    for rev in (False, True):
        out, T = G.gspmm(X, NORM_NONE, rev)
        assert np.allclose(out[:, 0], g["gspmm_none"], atol=1e-12)
        out, T = G.gspmm(X, NORM_BOTH, rev)
        assert np.allclose(out[:, 0], c["gspmm_both"], atol=1e-8)
    out, _ = G.gspmm(X, NORM_RIGHT, False)
    assert np.allclose(out[:, 0], g["gspmm_right_fwd"], atol=1e-12)
    out, _ = G.gspmm(X, NORM_RIGHT, True)
    assert np.allclose(out[:, 0], c["gspmm_right_rev"], atol=1e-12)


def test_gspmm_d4_golden(golden):
    g = golden("d4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    X = np.array(g["X"], np.float32)[:, None]
    for name, norm in [("none", NORM_NONE), ("right", NORM_RIGHT), ("both", NORM_BOTH)]:
        for rev, tag in [(False, "fwd"), (True, "rev")]:
            out, _ = G.gspmm(X, norm, rev)
            assert np.allclose(out[:, 0], g[f"gspmm_{name}_{tag}"], atol=1e-8), (name, tag)


@pytest.mark.parametrize("seed", range(200))
def test_gspmm_dense_bruteforce(seed):
    """BJ: brute-force dense matmul for graphs with <=64 vertices, all norms, both directions."""
    V, src, dst = rand_graph(seed)
    F = 1 + seed % 5
    X = datagen.uniform(seed, V, F)
    G = oracle.Graph(V, src, dst)
    for norm in (NORM_NONE, NORM_RIGHT, NORM_BOTH):
        M = dense_operator(V, src, dst, norm)
        out, T = G.gspmm(X, norm, False)
        check(out, T, M @ X.astype(np.float64))
        out, T = G.gspmm(X, norm, True)
        check(out, T, M.T @ X.astype(np.float64))


def test_gspmm_closed_form_symmetric():
    """BJ closed form D^-1/2 A D^-1/2 X on dense adjacency; symmetric => fwd == rev."""
    V = 60
    src, dst = datagen.chung_lu(V, 300, 0.4, 11)
    A = dense_adj(V, src, dst)
    assert np.array_equal(A, A.T)
    d = np.maximum(A.sum(1), 1)
    X = datagen.uniform(3, V, 7)
    ref = (d ** -0.5)[:, None] * (A @ ((d ** -0.5)[:, None] * X.astype(np.float64)))
    G = oracle.Graph(V, src, dst)
    f, T = G.gspmm(X, NORM_BOTH, False)
    r, _ = G.gspmm(X, NORM_BOTH, True)
    check(f, T, ref)
    assert np.allclose(f, r, atol=1e-13)


def test_gspmm_self_loop_identity():
    """self-loop-only graph is the identity (d = 1 everywhere)."""
    V = 9
    idx = np.arange(V, dtype=np.int64)
    G = oracle.Graph(V, idx, idx)
    X = datagen.uniform(5, V, 4)
    for norm in (NORM_NONE, NORM_RIGHT, NORM_BOTH):
        for rev in (False, True):
            out, _ = G.gspmm(X, norm, rev)
            assert np.array_equal(out, X.astype(np.float64))


@pytest.mark.parametrize("seed", range(30))
def test_gspmm_adjoint(seed):
    """<fwd(X), Y> == <X, rev(Y)> for every norm (rev is the adjoint)."""
    V, src, dst = rand_graph(500 + seed)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(seed, V, 3)
    Y = datagen.uniform(seed + 99, V, 3)
    for norm in (NORM_NONE, NORM_RIGHT, NORM_BOTH):
        a = np.sum(G.gspmm(X, norm, False)[0] * Y)
        b = np.sum(X * G.gspmm(Y, norm, True)[0])
        assert abs(a - b) <= 1e-10 * (1 + abs(a))


def test_gspmm_row_selection_and_ld():
    V, src, dst = rand_graph(77)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(1, V, 5, ld=8)
    full, T = G.gspmm(X, NORM_BOTH, False, F=5)
    rows = np.array([V - 1, 0, V // 2], np.int64)
    sel, Ts = G.gspmm(X, NORM_BOTH, False, rows=rows, F=5)
    assert np.array_equal(sel, full[rows]) and np.array_equal(Ts, T[rows])
    M = dense_operator(V, src, dst, NORM_BOTH)
    check(full, T, M @ X[:, :5].astype(np.float64))


# --------------------------------------------------------- C5 weighted gspmm
@pytest.mark.parametrize("seed", range(60))
def test_weighted_dense_bruteforce(seed):
    V, src, dst = rand_graph(2000 + seed)
    H = [1, 2, 4][seed % 3]
    Fh = 1 + seed % 3
    X = datagen.uniform(seed, V, H * Fh)
    E = len(src)
    w_coo = datagen.uniform(seed + 1, E, H) if E else np.zeros((0, H), np.float32)
    G = oracle.Graph(V, src, dst)
    w = np.zeros((E, H), np.float32)
    w[G.coo_to_eid] = w_coo                   # per-edge values travel with their edge ID
    out_f, Tf = G.gspmm_weighted(X, w, False)
    out_r, Tr = G.gspmm_weighted(X, w, True)
    for h in range(H):
        Mh = dense_adj(V, src, dst, w_coo[:, h].astype(np.float64))
        Xh = X[:, h * Fh:(h + 1) * Fh].astype(np.float64)
        check(out_f[:, h * Fh:(h + 1) * Fh], Tf[:, h * Fh:(h + 1) * Fh], Mh @ Xh)
        check(out_r[:, h * Fh:(h + 1) * Fh], Tr[:, h * Fh:(h + 1) * Fh], Mh.T @ Xh)


def test_weighted_unit_weights_equal_gspmm_none():
    """unit weights reduce gSpMMve to gSpMMv(sum)."""
    V, src, dst = rand_graph(31)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(2, V, 6)
    w = np.ones((G.E, 2), np.float32)
    for rev in (False, True):
        a = G.gspmm_weighted(X, w, rev)[0]
        b = G.gspmm(X, NORM_NONE, rev)[0]
        assert np.allclose(a, b, atol=1e-13)


def test_weighted_golden(golden):
    for name, gfile in [("t4", "t4.json"), ("d4", "d4.json")]:
        g = golden(gfile)
        c = golden("t4_chain.json") if name == "t4" else g
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        X = np.array(c["X"], np.float32)[:, None]
        Y = np.array(c["Y"], np.float32)[:, None]
        s, _ = G.gsddmm(X, Y, 1)
        assert np.allclose(s[:, 0], c["gsddmm_XY"], atol=1e-12)
        a = G.edge_softmax((s / 100.0).astype(np.float32))
        assert np.allclose(a[:, 0], c["edge_softmax_gsddmm_over_100"], atol=1e-8)
        f, _ = G.gspmm_weighted(X, a.astype(np.float32), False)
        r, _ = G.gspmm_weighted(X, a.astype(np.float32), True)
        assert np.allclose(f[:, 0], c["weighted_fwd_alpha_X"], atol=1e-6)
        assert np.allclose(r[:, 0], c["weighted_rev_alpha_X"], atol=1e-6)


# ------------------------------------------------------------------ C6 gsddmm
def test_gsddmm_t4_golden(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    X = np.array(g["X"], np.float32)[:, None]
    out, _ = G.gsddmm(X, np.ones((4, 1), np.float32), 1)
    assert out[:, 0].tolist() == g["gsddmm_X_rows_Y_ones"]


@pytest.mark.parametrize("seed", range(60))
def test_gsddmm_dense_bruteforce(seed):
    V, src, dst = rand_graph(3000 + seed)
    H = [1, 2, 8][seed % 3]
    Fh = 1 + seed % 4
    X = datagen.uniform(seed, V, H * Fh)
    Y = datagen.uniform(seed + 5, V, H * Fh)
    G = oracle.Graph(V, src, dst)
    out, T = G.gsddmm(X, Y, H)
    # per COO edge i: out[eid(i), h] = <X[dst_i, head h], Y[src_i, head h]>
    Xd = X[dst].astype(np.float64).reshape(len(src), H, Fh)
    Ys = Y[src].astype(np.float64).reshape(len(src), H, Fh)
    ref = np.einsum("ehf,ehf->eh", Xd, Ys)
    check(out[G.coo_to_eid], T[G.coo_to_eid], ref)


@pytest.mark.parametrize("seed", range(20))
def test_bilinear_identity(seed):
    """<gspmm_weighted(w, X), G> == <w, gsddmm(G, X)> (gSDDMMvv is the
    backward of gSpMMve w.r.t. the edge tensor)."""
    V, src, dst = rand_graph(4000 + seed)
    H, Fh = 2, 3
    Gr = oracle.Graph(V, src, dst)
    X = datagen.uniform(seed, V, H * Fh)
    Gm = datagen.uniform(seed + 1, V, H * Fh)
    w = datagen.uniform(seed + 2, Gr.E, H) if Gr.E else np.zeros((0, H), np.float32)
    a = np.sum(Gr.gspmm_weighted(X, w, False)[0] * Gm)
    b = np.sum(w.astype(np.float64) * Gr.gsddmm(Gm, X, H)[0])
    assert abs(a - b) <= 1e-10 * (1 + abs(a))


def test_gsddmm_row_selection_packs_edges():
    V, src, dst = rand_graph(88)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(1, V, 4)
    full, _ = G.gsddmm(X, X, 2)
    rows = np.array([3 % V, 0], np.int64)
    sel, _ = G.gsddmm(X, X, 2, rows=rows)
    assert np.array_equal(sel, full[G.row_edges(rows)])


# ------------------------------------------------------------- C7 softmax
@pytest.mark.parametrize("seed", range(40))
def test_softmax_characterisation(seed):
    V, src, dst = rand_graph(5000 + seed)
    G = oracle.Graph(V, src, dst)
    H = 1 + seed % 4
    e = datagen.uniform(seed, G.E, H, lo=-8, hi=8) if G.E else np.zeros((0, H), np.float32)
    a = G.edge_softmax(e)
    for v in range(V):
        s, t = G.fwd_off[v], G.fwd_off[v + 1]
        if s == t:
            continue
        blk = a[s:t]
        assert np.all(blk > 0)
        assert np.allclose(blk.sum(0), 1.0, atol=1e-13)
        ref = scipy.special.softmax(e[s:t].astype(np.float64), axis=0)
        assert np.allclose(blk, ref, atol=1e-14)
        # ratios fix the softmax uniquely: a_j / a_0 = exp(e_j - e_0)
        assert np.allclose(blk / blk[:1], np.exp(e[s:t].astype(np.float64) - e[s:s + 1]), rtol=1e-12)


def test_softmax_special_cases(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    a = G.edge_softmax(np.full((8, 1), 3.25, np.float32))
    assert np.allclose(a[:, 0], g["softmax_uniform_is_inverse_degree_per_slot"], atol=1e-15)
    e = np.zeros((8, 2), np.float32)
    e[4, 1] = 1e3                             # one dominating logit
    a = G.edge_softmax(e)
    assert a[4, 1] == pytest.approx(1.0) and a[5, 1] < 1e-300
    # shift invariance per row
    e = datagen.uniform(4, 8, 2)
    sh = e.copy()
    sh[4:7] += 5.0
    assert np.allclose(G.edge_softmax(e), G.edge_softmax(sh), atol=1e-6)


# ---------------------------------------------------------- C8 partition
def test_partition_golden(golden):
    for gf, cf in [("t4.json", "t4_chain.json"), ("d4.json", "d4.json")]:
        g, c = golden(gf), golden(cf)
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        for P, ref in c["partition_bounds"].items():
            assert G.partition_bounds(int(P)).tolist() == ref


@pytest.mark.parametrize("seed", range(30))
def test_partition_bruteforce(seed):
    V, src, dst = rand_graph(6000 + seed)
    G = oracle.Graph(V, src, dst)
    E = G.E
    for P in (1, 2, 3, 4, 8):
        b = G.partition_bounds(P)
        assert b[0] == 0 and b[-1] == V and np.all(np.diff(b) >= 0)
        for p in range(1, P):
            target = -(-p * E // P)
            cand = [v for v in range(V + 1) if G.fwd_off[v] >= target]
            assert b[p] == (min(cand) if cand else V)


@pytest.mark.parametrize("seed", range(20))
def test_partition_structure_concatenates_to_full(seed):
    """The padded partitions, run on the padded input, reproduce the full output."""
    V, src, dst = rand_graph(7000 + seed)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(seed, V, 3).astype(np.float64)
    M = dense_operator(V, src, dst, NORM_NONE)
    full = M @ X
    for P in (1, 2, 3, 4):
        parts = [G.partition_structure(P, p) for p in range(P)]
        R, b = parts[0][2], parts[0][3]
        Xpad = np.zeros((P * R, 3))
        for p in range(P):
            Xpad[p * R:p * R + b[p + 1] - b[p]] = X[b[p]:b[p + 1]]
        for p, (lo, lc, _, _) in enumerate(parts):
            assert lo.shape == (R + 1,) and lo[0] == 0
            assert np.all(lo[b[p + 1] - b[p]:] == lo[-1])          # padding rows empty
            loc = np.zeros((R, 3))
            for r in range(R):
                for j in range(lo[r], lo[r + 1]):
                    loc[r] += Xpad[lc[j]]
            assert np.allclose(loc[:b[p + 1] - b[p]], full[b[p]:b[p + 1]], atol=1e-12)


# ------------------------------------------------- C9 softmax backward (NEXT-1)
@pytest.mark.parametrize("seed", range(20))
def test_softmax_backward_directional_derivative(seed):
    """<dalpha, (softmax(e + eps d) - softmax(e - eps d)) / 2 eps> == <ds, d>: the
    backward is pinned to the (already pinned) forward by central differences."""
    V, src, dst = rand_graph(8000 + seed, Vmax=40, Emax=200)
    G = oracle.Graph(V, src, dst)
    if G.E == 0:
        return
    H = 1 + seed % 3
    e = datagen.uniform(seed, G.E, H, lo=-3, hi=3).astype(np.float64)
    g = datagen.uniform(seed + 1, G.E, H)
    d = datagen.uniform(seed + 2, G.E, H).astype(np.float64)
    a = G.edge_softmax(e.astype(np.float32))
    ds, _ = G.edge_softmax_backward(a.astype(np.float32), g)
    # forward on fp64-exact shifts: perturb in fp32-representable steps, use the fp64 oracle
    eps = 2.0 ** -12
    ap = G.edge_softmax((e + eps * d).astype(np.float32))
    am = G.edge_softmax((e - eps * d).astype(np.float32))
    dp = (e + eps * d).astype(np.float32).astype(np.float64) - (e - eps * d).astype(np.float32).astype(np.float64)
    lhs = np.sum(g.astype(np.float64) * (ap - am))
    rhs = np.sum(ds * dp)
    assert abs(lhs - rhs) <= 1e-5 * (1 + abs(rhs)), (lhs, rhs)


def test_softmax_backward_closed_forms(golden):
    g4 = golden("d4.json")
    G = oracle.Graph(g4["V"], g4["src"], g4["dst"])
    a = G.edge_softmax(datagen.uniform(3, G.E, 2))
    # uniform upstream gradient per row -> zero (softmax is shift invariant)
    ds, _ = G.edge_softmax_backward(a.astype(np.float32), np.full((G.E, 2), 0.75, np.float32))
    assert np.allclose(ds, 0, atol=1e-7)
    # single-edge rows (D4 rows 0 and 1) -> zero; every row sums to zero
    gr = datagen.uniform(4, G.E, 2)
    ds, _ = G.edge_softmax_backward(a.astype(np.float32), gr)
    assert np.allclose(ds[:2], 0, atol=1e-12)
    assert np.allclose(ds[2:7].sum(0), 0, atol=1e-6)
    # two-edge row closed form: ds1 = p (1 - p) (g1 - g2)
    G2 = oracle.Graph(2, [0, 1], [0, 0])
    al = np.array([[0.3], [0.7]], np.float32)
    gg = np.array([[2.0], [-1.0]], np.float32)
    ds, _ = G2.edge_softmax_backward(al, gg)
    p = np.float64(np.float32(0.3)); q = np.float64(np.float32(0.7))
    assert ds[0, 0] == pytest.approx(p * (2.0 - (p * 2.0 - q)), abs=1e-15)
    assert ds[0, 0] == pytest.approx(p * q * 3.0, rel=1e-6)


# --------------------------------------------------- C10 fused GAT (NEXT-2)
@pytest.mark.parametrize("seed", range(15))
def test_gat_forward_is_the_composition(seed):
    """C10 (fp64 end to end) == C5(C7(C6)) with the pinned components, up to the
    fp32 hand-off the component interfaces impose; softmax rows sum to 1."""
    V, src, dst = rand_graph(9000 + seed)
    G = oracle.Graph(V, src, dst)
    H = [1, 2, 4][seed % 3]
    Fh, Fvh = 1 + seed % 3, 2
    X = datagen.uniform(seed, V, H * Fh)
    Y = datagen.uniform(seed + 1, V, H * Fh)
    Vt = datagen.uniform(seed + 2, V, H * Fvh)
    a, out, T = G.gat_forward(X, Y, Vt, H)
    s, _ = G.gsddmm(X, Y, H)
    a2 = G.edge_softmax(s.astype(np.float32))
    assert np.allclose(a, a2, atol=2e-6)
    o2, T2 = G.gspmm_weighted(Vt, a2.astype(np.float32))
    assert np.all(np.abs(out - o2) <= 1e-5 * (T + 1))
    rows = np.repeat(np.arange(V), np.diff(G.fwd_off))
    sums = np.zeros((V, H))
    np.add.at(sums, rows, a)
    nz = np.diff(G.fwd_off) > 0
    assert np.allclose(sums[nz], 1.0, atol=1e-13)


# ----------------------------------------------- C11-C13 Table-1 surface (NEXT-3)
def coo_reduce(V, keys, vals, red):
    """Brute force: reduce vals grouped by keys (COO order, no CSR), empty -> 0."""
    F = vals.shape[1]
    out = np.zeros((V, F))
    for v in range(V):
        m = keys == v
        if m.any():
            blk = vals[m].astype(np.float64)
            out[v] = blk.sum(0) if red == oracle.RED_SUM else (blk.min(0) if red == oracle.RED_MIN else blk.max(0))
    return out


@pytest.mark.parametrize("seed", range(20))
def test_gspmm_reduce_bruteforce(seed):
    V, src, dst = rand_graph(10000 + seed)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(seed, V, 3)
    for red in (oracle.RED_SUM, oracle.RED_MIN, oracle.RED_MAX):
        out, T = G.gspmm_reduce(X, red, False)
        assert np.allclose(out, coo_reduce(V, dst, X[src], red), atol=1e-12)
        out, T = G.gspmm_reduce(X, red, True)
        assert np.allclose(out, coo_reduce(V, src, X[dst], red), atol=1e-12)
    s, _ = G.gspmm_reduce(X, oracle.RED_SUM)
    assert np.allclose(s, G.gspmm(X, NORM_NONE)[0], atol=1e-12)


@pytest.mark.parametrize("seed", range(20))
def test_gspmm_e_bruteforce(seed):
    V, src, dst = rand_graph(11000 + seed)
    G = oracle.Graph(V, src, dst)
    H = 1 + seed % 3
    w_coo = datagen.uniform(seed, G.E, H) if G.E else np.zeros((0, H), np.float32)
    w = np.zeros_like(w_coo)
    w[G.coo_to_eid] = w_coo
    for red in (oracle.RED_SUM, oracle.RED_MIN, oracle.RED_MAX):
        assert np.allclose(G.gspmm_e(w, red, False)[0], coo_reduce(V, dst, w_coo, red), atol=1e-12)
        assert np.allclose(G.gspmm_e(w, red, True)[0], coo_reduce(V, src, w_coo, red), atol=1e-12)


def test_gspmm_e_spec_examples(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    # all-ones sum -> degrees; max over T4 row 2 with We[j] = j -> 6
    assert G.gspmm_e(np.ones((8, 1), np.float32), oracle.RED_SUM)[0][:, 0].tolist() == g["deg"]
    assert G.gspmm_e(np.arange(8, dtype=np.float32)[:, None], oracle.RED_MAX)[0][2, 0] == 6.0
    G5 = oracle.Graph(5, g["src"], g["dst"])
    for red in (oracle.RED_SUM, oracle.RED_MIN, oracle.RED_MAX):   # empty row -> 0
        assert G5.gspmm_e(np.ones((8, 1), np.float32), red)[0][4, 0] == 0.0


@pytest.mark.parametrize("seed", range(10))
def test_gsddmm_ve_bruteforce(seed):
    V, src, dst = rand_graph(12000 + seed)
    G = oracle.Graph(V, src, dst)
    H = 1 + seed % 3
    X = datagen.uniform(seed, V, H, lo=0.5, hi=2.0)
    w = datagen.uniform(seed + 1, G.E, H) if G.E else np.zeros((0, H), np.float32)
    row_of = np.repeat(np.arange(V), np.diff(G.fwd_off))
    for op, f in [(oracle.OP_ADD, np.add), (oracle.OP_SUB, np.subtract), (oracle.OP_MUL, np.multiply),
                  (oracle.OP_DIV, np.divide)]:
        for side in (0, 1):
            vx = G.fwd_col if side else row_of
            ref = f(w.astype(np.float64), X[vx].astype(np.float64))
            assert np.allclose(G.gsddmm_ve(X, w, op, side), ref, atol=1e-12)


def test_gsddmm_ve_spec_examples(golden):
    g = golden("t4.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    w = datagen.uniform(1, 8, 1)
    # sub of zeros -> w; mul of ones on the column side -> gather X[col]
    assert np.array_equal(G.gsddmm_ve(np.zeros((4, 1), np.float32), w, oracle.OP_SUB, 0), w.astype(np.float64))
    X = np.array(g["X"], np.float32)[:, None]
    out = G.gsddmm_ve(X, np.ones((8, 1), np.float32), oracle.OP_MUL, 1)
    assert out[:, 0].tolist() == [X[c, 0] for c in g["fwd_col"]]


# ------------------------------------------- row-sampled COO oracle (NEXT-4)
@pytest.mark.parametrize("seed", range(10))
def test_rows_coo_matches_full_oracle(seed):
    """The COO-scan evaluation of C4 / C1 for selected rows equals the full
    oracle (itself pinned above) on the same graph."""
    V, src, dst = rand_graph(13000 + seed, Vmax=80, Emax=600)
    G = oracle.Graph(V, src, dst)
    X = datagen.uniform(seed, V, 4)
    rows = np.unique(np.random.default_rng(seed).integers(0, V, size=min(V, 9)))
    for norm in (NORM_NONE, NORM_RIGHT, NORM_BOTH):
        for rev in (False, True):
            ref, T = G.gspmm(X, norm, rev, rows=rows)
            out, T2 = oracle.gspmm_rows_coo(V, src, dst, X, norm, rows, rev)
            assert np.allclose(out, ref, atol=1e-12) and np.allclose(T, T2, atol=1e-12)
    for (first, pairs), v in zip(oracle.rows_coo(V, src, dst, rows), rows):
        assert first == G.fwd_off[v]
        assert np.array_equal(pairs[:, 0], G.fwd_col[G.fwd_off[v]:G.fwd_off[v + 1]])
        assert np.array_equal(G.coo_to_eid[pairs[:, 1]], np.arange(G.fwd_off[v], G.fwd_off[v + 1]))


# ------------------------------- C14 / C15 additive GAT attention (NEXT-3)
def test_gsddmm_add_leaky_t4_golden(golden):
    g, c = golden("t4.json"), golden("t4_additive.json")
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    el = np.array(c["el"], np.float32)[:, None]
    er = np.array(c["er"], np.float32)[:, None]
    assert np.allclose(G.gsddmm_add_leaky(el, er, c["slope"])[:, 0], c["scores"], rtol=1e-15, atol=1e-15)
    assert G.gsddmm_add_leaky(el, er, 1.0)[:, 0].tolist() == c["scores_slope1"]


@pytest.mark.parametrize("seed", range(15))
def test_gsddmm_add_leaky_bruteforce(seed):
    """Brute force from the COO list (per input edge i: lrelu(el[src_i] + er[dst_i]),
    placed at its edge ID); slope 1 == C13's u_add_v as two gSDDMMve calls."""
    V, src, dst = rand_graph(14000 + seed)
    G = oracle.Graph(V, src, dst)
    H = 1 + seed % 4
    el = datagen.uniform(seed, V, H, lo=-3, hi=3)
    er = datagen.uniform(seed + 1, V, H, lo=-3, hi=3)
    slope = [0.2, 0.01, 0.5][seed % 3]
    x = el[src].astype(np.float64) + er[dst].astype(np.float64)
    ref = np.zeros((G.E, H))
    ref[G.coo_to_eid] = np.where(x > 0, x, slope * x)
    assert np.array_equal(G.gsddmm_add_leaky(el, er, slope), ref)
    if G.E:
        zero = np.zeros((G.E, H), np.float32)
        dst_side = G.gsddmm_ve(er, zero, oracle.OP_ADD, 0).astype(np.float32)
        both = G.gsddmm_ve(el, dst_side, oracle.OP_ADD, 1)
        assert np.array_equal(G.gsddmm_add_leaky(el, er, 1.0), both)


@pytest.mark.parametrize("seed", range(12))
def test_gat_forward_additive_bruteforce(seed):
    """C15 against a per-destination brute force over the COO list (scores,
    scipy softmax, weighted sum of Vt[src]) and against the composition
    C5(C7(C14)) of pinned components; alpha rows sum to 1."""
    V, src, dst = rand_graph(15000 + seed)
    G = oracle.Graph(V, src, dst)
    H = [1, 2, 4][seed % 3]
    Fvh = 1 + seed % 3
    el = datagen.uniform(seed, V, H, lo=-4, hi=4)
    er = datagen.uniform(seed + 1, V, H, lo=-4, hi=4)
    Vt = datagen.uniform(seed + 2, V, H * Fvh)
    a, out, T = G.gat_forward_additive(el, er, Vt, 0.2)
    ref_a = np.zeros((G.E, H))
    ref_o = np.zeros((V, H * Fvh))
    for v in range(V):
        idx = np.nonzero(dst == v)[0]
        if idx.size == 0:
            continue
        x = el[src[idx]].astype(np.float64) + er[v].astype(np.float64)
        sc = np.where(x > 0, x, 0.2 * x)
        al = scipy.special.softmax(sc, axis=0)                    # [deg, H]
        ref_a[G.coo_to_eid[idx]] = al
        ref_o[v] = (np.repeat(al, Fvh, axis=1) * Vt[src[idx]].astype(np.float64)).sum(0)
    assert np.allclose(a, ref_a, atol=1e-13)
    check(out, T, ref_o)
    s = G.gsddmm_add_leaky(el, er, 0.2)
    a2 = G.edge_softmax(s.astype(np.float32))
    assert np.allclose(a, a2, atol=2e-6)
    o2, _ = G.gspmm_weighted(Vt, a2.astype(np.float32))
    assert np.all(np.abs(out - o2) <= 1e-5 * (T + 1))
