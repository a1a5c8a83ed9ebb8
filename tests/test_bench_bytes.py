"""bench.py's byte accounting on the BASELINE shapes: the
algorithmic bytes per launch match the survey's table, B_uniq counts each array
once, and the per-edge figure matches DESIGN.md §6 (CPU only)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

V, E, F, H = 232_965, 114_615_892, 64, 8   # Reddit-shaped (BJ configs)


def test_alg_bytes_reddit_matches_survey_table():
    # Reddit gspmm F=64 29.86 GB; GAT gsddmm / softmax / wspmm / wspmm-rev 33.53 / 7.34 / 33.53 / 33.99 GB
    assert bench.alg_bytes("gspmm_fwd", V, E, F, H) / 1e9 == pytest.approx(29.86, abs=0.01)
    assert bench.alg_bytes("gsddmm", V, E, F, H) / 1e9 == pytest.approx(33.53, abs=0.01)
    assert bench.alg_bytes("edge_softmax", V, E, F, H) / 1e9 == pytest.approx(7.34, abs=0.01)
    assert bench.alg_bytes("gspmm_weighted_fwd", V, E, F, H) / 1e9 == pytest.approx(33.53, abs=0.01)
    assert bench.alg_bytes("gspmm_weighted_rev", V, E, F, H) / 1e9 == pytest.approx(33.99, abs=0.01)
    # per edge at F = 64: 260.6 B
    assert bench.alg_bytes("gspmm_fwd", V, E, F, H) / E == pytest.approx(260.6, abs=0.1)


@pytest.mark.parametrize("op", ["gspmm_fwd", "gspmm_rev", "gspmm_weighted_fwd", "gspmm_weighted_rev", "gsddmm",
                                "edge_softmax", "gat_forward"])
def test_uniq_bytes_counts_each_array_once(op):
    u = bench.uniq_bytes(op, V, E, F, H, edge_scales=False)
    a = bench.alg_bytes(op, V, E, F, H)
    assert u <= a
    if op == "edge_softmax":          # nothing is gathered: every byte is read once anyway
        assert u == a
    elif op in ("gsddmm", "gat_forward"):   # Y == X (the bench's Z, Z): the 4EF gathers hit the table counted once
        assert a - u == 4 * E * F
    else:                             # the gathered table: 4EF per launch vs 4VF once
        assert a - u == 4 * E * F - 4 * V * F
    # the per-edge scale stream adds 4E when the graph carries it (gspmm only)
    d = bench.uniq_bytes(op, V, E, F, H, edge_scales=True) - u
    assert d == (4 * E if op in ("gspmm_fwd", "gspmm_rev") else 0)
