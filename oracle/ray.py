"""Ray-disc vision oracle (reading A1-ray) — TEST INFRASTRUCTURE.

P:158 "a simple ray-casting model, segmenting their field of vision into a fixed number of
cells"; "an array of v values representing the distance to the nearest object at that
angle".  SPEC's reading: one ray per sector through the sector centre,
psi_k = -fov/2 + (k + 1/2) fov/v from the heading (CCW-positive, sector 0 the clockwise
edge: reading A3); neighbours are discs of radius d_r; view[c][k] = min over neighbours j of
channel c of the ray's entry distance t >= 0 (0 if the origin lies inside the disc,
S:170), clamped to d_v and divided by d_v; 1.0 if nothing is hit.  Only discs with
centre distance < d_v + d_r can be hit within d_v (candidate set).

Plain fp64: for every query row, every neighbour within d_v + d_r (brute force over all N,
torus minimal image), every ray: the quadratic |o + t u - c|^2 = r^2.
"""
from __future__ import annotations

import math

import numpy as np

from .env import minimal_image


def ray_disc(ux, uy, cx, cy, r):
    """Smallest t >= 0 with |t u - c| = r for unit u (origin at 0), or inf.

    b = u . c; h = r^2 - (|c|^2 - b^2); origin inside (|c| <= r) -> 0; h < 0 or b < 0 ->
    miss; else t = b - sqrt(h)."""
    b = ux * cx + uy * cy
    c2 = cx * cx + cy * cy
    h = r * r - (c2 - b * b)
    inside = c2 <= r * r
    hit = (h >= 0) & (b > 0)
    t = np.where(hit, b - np.sqrt(np.maximum(h, 0.0)), np.inf)
    return np.where(inside, 0.0, t), h


def ray_views(p, state_r, rows, dh_rel=5e-5, return_cond=False):
    """View [len(rows), channels * v] under the ray-disc reading, plus per-sector bounds
    [lo, hi] that the fp32 kernel must fall in (interval comparator):
    a near-grazing ray (|h| <= dh_rel r^2) may hit or miss and its t is ill-conditioned.

    ``return_cond`` also returns a mask of the *well-conditioned* sectors: every disc that
    may be hit is surely hit (no grazing disc) and the nearest one's sqrt sensitivity
    dh / (2 sqrt h) is <= 1e-6 d_v for every disc whose interval reaches the sector's upper
    bound, or nothing can be hit at all."""
    st = np.asarray(state_r, np.float64)
    n = st.shape[0]
    rows = np.asarray(rows)
    v = int(p.v)
    ch = 1 if p.env == "flock" else 2
    r = float(p.d_r)
    dv = float(p.d_v)
    fov = float(p.fov)
    w = fov / v
    psi = -fov / 2 + (np.arange(v) + 0.5) * w
    dh = dh_rel * r * r
    view = np.ones((len(rows), ch * v))
    cond = np.ones((len(rows), ch * v), dtype=bool)
    lo = np.ones((len(rows), ch * v))
    hi = np.ones((len(rows), ch * v))
    first_chaser = n - getattr(p, "n_chasers", 0) if p.env == "tag" else n
    for b, i in enumerate(rows):
        dx = minimal_image(p, st[i, 0], st[:, 0])
        dy = minimal_image(p, st[i, 1], st[:, 1])
        d = np.hypot(dx, dy)
        js = np.nonzero((d < dv + r) & (np.arange(n) != i))[0]
        if len(js) == 0:
            continue
        th = st[i, 2]
        ang = th + psi                                   # world-frame ray angles
        ux, uy = np.cos(ang)[None, :], np.sin(ang)[None, :]
        cx, cy = dx[js][:, None], dy[js][:, None]
        t, h = ray_disc(ux, uy, cx, cy, r)              # [J, v]
        tc = np.minimum(t / dv, 1.0)
        # tolerance of a sure hit: 1e-5 relative + the sqrt's sensitivity to h's fp32 error
        sq = np.sqrt(np.maximum(h, 0.0))
        err = 1e-5 * np.abs(t) + np.minimum(dh / (2 * np.maximum(sq, 1e-300)), math.sqrt(dh))
        err = np.where(t == 0.0, 0.0, err) / dv
        bpos = (ux * cx + uy * cy) > 0
        c2 = (cx * cx + cy * cy)
        sure = np.isfinite(t) & ((h >= dh) | (c2 <= r * r * (1 - 1e-6)))
        maybe = (bpos & (h >= -dh)) | (c2 <= r * r * (1 + 1e-6))
        tmay = np.where(maybe & ~np.isfinite(t), (ux * cx + uy * cy) / dv, tc)
        chan = np.zeros(len(js), int) if p.env == "flock" else (js >= first_chaser).astype(int)
        for c in range(ch):
            sel = chan == c
            if not sel.any():
                continue
            view[b, c * v:(c + 1) * v] = tc[sel].min(0)
            lo[b, c * v:(c + 1) * v] = np.minimum(np.where(maybe[sel], tmay[sel] - err[sel] - 1e-6, 1.0).min(0), 1.0)
            hi[b, c * v:(c + 1) * v] = np.minimum(np.where(sure[sel], tc[sel] + err[sel], 1.0).min(0), 1.0)
            # well conditioned: no grazing disc, and every disc whose interval reaches down
            # to the sector's hi has a small sqrt sensitivity
            sens = np.minimum(dh / (2 * np.maximum(sq[sel], 1e-300)), math.sqrt(dh)) / dv
            hic = hi[b, c * v:(c + 1) * v][None, :]
            relevant = sure[sel] & (tc[sel] - err[sel] - 1e-6 <= hic)
            near_ok = ~np.any(relevant & (sens > 1e-6), axis=0)
            cond[b, c * v:(c + 1) * v] = ~np.any(maybe[sel] & ~sure[sel], axis=0) & near_ok
    if return_cond:
        return view, np.clip(lo, 0.0, 1.0), hi, cond
    return view, np.clip(lo, 0.0, 1.0), hi
