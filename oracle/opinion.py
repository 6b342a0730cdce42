"""Opinion-dynamics oracle (Listing 1) — TEST INFRASTRUCTURE.

Listing 1: a graph interaction `social_influence(me, you, edge)`: d = |me.opinion -
you.opinion|; if d < threshold: w = strength * edge.weight; me.new_opinion = (1 - w)
me.new_opinion + w you.opinion; then the self interaction `update_opinion`: opinion =
new_opinion.  S:292 fixes the order (edges sorted by (src, dst), new_opinion starting at the
current opinion) and S:103 "accumulating into src in edge order"; every read of `opinion`
sees the previous step.  Plain per-node, per-edge loops in fp64.
"""
from __future__ import annotations

import numpy as np

BAND = 1e-6


def step(row_ptr, col, weight, op, threshold, strength, rows=None, overrides=None):
    """New opinions for `rows` (default all).  overrides: {edge index: bool} forces the
    bounded-confidence decision of an edge (used for banded edges, |d - threshold| <= 1e-6).
    Returns (new [len(rows)], banded edge list per row)."""
    op = np.asarray(op, np.float64)
    w = np.asarray(weight, np.float64)
    rows = np.arange(len(op)) if rows is None else np.asarray(rows)
    out = np.empty(len(rows))
    bands = []
    for b, i in enumerate(rows):
        x = op[i]
        acc = x
        bl = []
        for e in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            y = op[int(col[e])]
            d = abs(x - y)
            within = d < threshold
            if abs(d - threshold) <= BAND:
                bl.append(e)
            if overrides and e in overrides:
                within = overrides[e]
            if within:
                ww = strength * w[e]
                acc = (1.0 - ww) * acc + ww * y
        out[b] = acc
        bands.append(bl)
    return out, bands
