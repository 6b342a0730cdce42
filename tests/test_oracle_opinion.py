"""Pins for oracle.opinion (Listing 1)."""
import numpy as np
import pytest

import vg_inputs as vi
from oracle.opinion import step


def test_single_edge_example():
    # S:295 "me=0.5, you=0.6, threshold=0.2, strength=0.5, weight=1 -> 0.55"
    out, _ = step(np.array([0, 1, 1]), np.array([1]), np.array([1.0]), np.array([0.5, 0.6]),
                  0.2, 0.5)
    assert out[0] == pytest.approx(0.55, abs=1e-15) and out[1] == 0.6


def test_outside_confidence_unchanged():
    # S:296 "|difference| >= threshold -> opinion unchanged"
    out, _ = step(np.array([0, 1, 1]), np.array([1]), np.array([1.0]), np.array([0.1, 0.9]),
                  0.2, 0.5)
    assert out[0] == pytest.approx(0.1)


def test_consensus_fixed_point():
    # S:297 "complete graph, equal opinions -> fixed point"
    n = 6
    col = np.array([j for i in range(n) for j in range(n) if j != i])
    rp = np.arange(n + 1) * (n - 1)
    op = np.full(n, 0.37)
    out, _ = step(rp, col, np.full(len(col), 0.8), op, 0.5, 0.5)
    assert np.allclose(out, 0.37, atol=1e-15)


def test_closed_form_affine_fold():
    # The edge fold is a composition of affine maps: new = P x + sum_e w_e y_e prod_{e'>e}(1-w_e')
    g = vi.opinion_graph(40, 6, seed=3)
    out, _ = step(g["row_ptr"], g["col"], g["weight"], g["op"], 2.0, 0.7)   # all within
    op = g["op"].astype(np.float64)
    for i in range(40):
        es = range(g["row_ptr"][i], g["row_ptr"][i + 1])
        w = [0.7 * float(g["weight"][e]) for e in es]
        y = [op[g["col"][e]] for e in es]
        tot = op[i] * np.prod([1 - a for a in w])
        for k in range(len(w)):
            tot += w[k] * y[k] * np.prod([1 - a for a in w[k + 1:]])
        assert out[i] == pytest.approx(tot, abs=1e-14)


def test_contraction_and_consensus():
    # spread non-increasing with threshold >= 1 on a connected graph; complete
    # graph, threshold 1, strength*weight in (0,1): strictly decreasing until consensus.
    n = 8
    col = np.array([j for i in range(n) for j in range(n) if j != i])
    rp = np.arange(n + 1) * (n - 1)
    op = np.random.default_rng(0).random(n)
    spread = op.max() - op.min()
    for _ in range(200):
        op, _ = step(rp, col, np.full(len(col), 0.6), op, 1.0, 0.5)
        s = op.max() - op.min()
        assert s < spread or s < 1e-6
        spread = s
        if s < 1e-6:
            break
    assert spread < 1e-6


def test_band_recorded():
    out, bands = step(np.array([0, 1, 1]), np.array([1]), np.array([1.0]),
                      np.array([0.5, 0.7]), 0.2, 0.5)
    assert bands[0] == [0]
    alt, _ = step(np.array([0, 1, 1]), np.array([1]), np.array([1.0]), np.array([0.5, 0.7]),
                  0.2, 0.5, overrides={0: False})
    assert alt[0] != out[0]
