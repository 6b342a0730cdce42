"""fp64 NumPy oracle of one Vogue environment step — TEST INFRASTRUCTURE (see __init__).

Every function cites the passage it follows: ``P:n`` = /root/reference/PAPER.md line n,
``S:n`` = SPEC.md line n (interfaces/defaults only), ``An`` = the reading of a gap listed in
SURVEY.md §8c and DESIGN.md §3.

Inputs are the fp32 state/actions/parameters, promoted exactly to fp64 (A12).  The only
place the oracle computes in fp32 on purpose is ``cell_ids``: the ABI *defines* the cell
id by an fp32 formula (A16), and the oracle evaluates exactly that formula with IEEE fp32
scalars, so the result is unique.
"""
from __future__ import annotations

import math

import numpy as np

FLOCK = "flock"
TAG = "tag"

#: Width of the "band" around every threshold, in the normalised coordinate that is
#: thresholded (A17): |d/d_v - 1|, |d/(2 d_r) - 1| and |u - k/v| with u the fraction of
#: the field of view.  Pairs inside a band may legitimately take either decision.
BAND = 1e-6


# ----------------------------------------------------------------------------- grid (A16)
def grid_size(p) -> int:
    """Cells per axis G (A16): the largest integer with L/G >= d_v (1 + 2^-12).

    S:45 / S:77 require cell size >= query radius; the 2^-12 margin absorbs the fp32
    rounding of the cell-id formula.  ``p.grid`` > 0 overrides (must still satisfy it).
    """
    if getattr(p, "grid", 0):
        return int(p.grid)
    need = float(p.d_v) * (1.0 + 2.0 ** -12)
    g = int(math.floor(float(p.width) / need))
    while g > 0 and float(p.width) / g < need:
        g -= 1
    return g


def cell_ids(p, state32: np.ndarray) -> np.ndarray:
    """Per-agent cell id cy*G + cx (A16; "floor(x_i/cell_size)").

    The ABI fixes cx = min(G-1, floor(RN32(x * RN32(G/L)))), evaluated here with IEEE fp32
    NumPy scalars (exactly rounded), so GPU and oracle must agree bit for bit.
    """
    g = grid_size(p)
    gs = np.float32(g) / np.float32(p.width)              # RN32(G/L)
    st = np.asarray(state32, dtype=np.float32)
    cx = np.floor(st[..., 0] * gs).astype(np.int64)        # fp32 product, then floor
    cy = np.floor(st[..., 1] * gs).astype(np.int64)
    cx = np.minimum(cx, g - 1)
    cy = np.minimum(cy, g - 1)
    return (cy * g + cx).astype(np.uint32)


def bins(p, state32: np.ndarray) -> dict:
    """SpatialGrid: textbook stable counting sort by cell, per replica.

    Returns cell_id [R,N], cell_start [R*G^2 + 1] (global offsets into the flat [R*N]
    arrays), perm [R,N] (local agent ids, ascending within each cell), and
    sorted [R,N,4] = state[perm] (tag: 4th column = type, 0 runner / 1 chaser).
    """
    st = np.asarray(state32, dtype=np.float32).reshape(p.n_replicas, p.n_agents, 4)
    g = grid_size(p)
    cid = cell_ids(p, st)
    counts = np.stack([np.bincount(cid[r], minlength=g * g) for r in range(p.n_replicas)])
    cell_start = np.concatenate([[0], np.cumsum(counts.reshape(-1))]).astype(np.uint32)
    perm = np.stack([np.argsort(cid[r], kind="stable") for r in range(p.n_replicas)])
    perm = perm.astype(np.uint32)
    srt = np.take_along_axis(st, perm[..., None].astype(np.int64), axis=1).copy()
    if p.env == TAG:
        srt[..., 3] = (perm >= p.n_agents - p.n_chasers).astype(np.float32)
    return {"cell_id": cid, "cell_start": cell_start, "perm": perm, "sorted": srt}


# ------------------------------------------------------------------------ integrate (a1)
def integrate(p, state: np.ndarray, actions: np.ndarray) -> np.ndarray:
    """One simultaneous update of heading, speed and position (fp64).

    Flock: a = (accelerate, rotate), clamped to the action box
    (S:257).  theta' = (theta + a_1) mod 2 pi; s' = clamp(s + a_0, s_min, s_max)
    (reading A7 of P:171's garbled min/max); p' = (p + s' (cos theta', sin theta')) mod L
    (torus, A9), in the order rotate -> accelerate -> move (A8).
    Tag: a = (rotate, move); move clamped to [0, s_max(type)], no
    persistent speed (4th column passed through).
    """
    st = np.asarray(state, dtype=np.float64).reshape(p.n_replicas, p.n_agents, 4)
    a = np.asarray(actions, dtype=np.float64).reshape(p.n_replicas, p.n_agents, 2)
    L = float(p.width)
    out = st.copy()
    two_pi = 2.0 * math.pi
    if p.env == FLOCK:
        acc = np.clip(a[..., 0], -p.a_max, p.a_max)
        turn = np.clip(a[..., 1], -p.theta_max, p.theta_max)
        th = np.mod(st[..., 2] + turn, two_pi)
        speed = np.minimum(np.maximum(st[..., 3] + acc, p.s_min), p.s_max)
        dist = speed
        out[..., 3] = speed
    else:
        turn = np.clip(a[..., 0], -p.theta_max, p.theta_max)
        th = np.mod(st[..., 2] + turn, two_pi)
        smax = np.full(p.n_agents, float(p.s_max))
        smax[p.n_agents - p.n_chasers:] = p.s_max_chaser
        dist = np.clip(a[..., 1], 0.0, smax[None, :])
    th = np.where(th >= two_pi, th - two_pi, th)
    x = np.mod(st[..., 0] + dist * np.cos(th), L)
    y = np.mod(st[..., 1] + dist * np.sin(th), L)
    out[..., 0] = np.where(x >= L, x - L, x)
    out[..., 1] = np.where(y >= L, y - L, y)
    out[..., 2] = th
    return out


# ------------------------------------------------------------------ pair geometry (a3-a5)
def minimal_image(p, xi, xj):
    """Torus minimal-image displacement xj - xi (A9, A11), fp64."""
    d = np.asarray(xj, np.float64) - np.asarray(xi, np.float64)
    L = float(p.width)
    return d - L * np.rint(d / L)


def reward_f(p, d, contact):
    """Flock reward contribution f(d) (Eq. 1 and Fig. 4; A5).

    f = -c_collide for a contact (d <= 2 d_r, A6); otherwise a closeness bonus rising
    linearly from 0 at 2 d_r to c_near at d_peak, then falling linearly to 0 at d_v.
    """
    d = np.asarray(d, np.float64)
    two_dr = 2.0 * float(p.d_r)
    rise = p.c_near * (d - two_dr) / (p.d_peak - two_dr)
    fall = p.c_near * (p.d_v - d) / (p.d_v - p.d_peak)
    bonus = np.where(d <= p.d_peak, rise, fall)
    bonus = np.where(d <= two_dr, 0.0, bonus)
    return np.where(contact, -float(p.c_collide), bonus)


def _pairs(p, st, rows):
    """All (row, j) pairs with torus distance within d_v (1 + 2 BAND), j != row.

    Plain brute force over all N agents for each query row (the definition of "spatial
    proximity").  Returns flat arrays over those pairs.
    """
    x, y = st[:, 0], st[:, 1]
    rb, jb, dxb, dyb, db = [], [], [], [], []
    block = max(1, min(256, (1 << 22) // max(1, st.shape[0])))
    lim = float(p.d_v) * (1.0 + 2.0 * BAND)
    for s0 in range(0, len(rows), block):
        rr = rows[s0:s0 + block]
        dx = minimal_image(p, x[rr][:, None], x[None, :])
        dy = minimal_image(p, y[rr][:, None], y[None, :])
        d = np.hypot(dx, dy)
        near = d <= lim
        near[np.arange(len(rr)), rr] = False              # j != i (A13)
        b, j = np.nonzero(near)
        rb.append(b + s0)
        jb.append(j)
        dxb.append(dx[b, j])
        dyb.append(dy[b, j])
        db.append(d[b, j])
    cat = (lambda a, dt: np.concatenate(a).astype(dt) if a else np.zeros(0, dt))
    return (cat(rb, np.int64), cat(jb, np.int64), cat(dxb, np.float64),
            cat(dyb, np.float64), cat(db, np.float64))


def sense_rows(p, state_r: np.ndarray, rows, overrides: dict | None = None) -> dict:
    """Observation, reward and counts for query rows ``rows`` of ONE replica.

    Definition (v sectors, distance to the nearest neighbour per sector;
    P:171 flock obs = 128-sector view + speed; P:194 tag obs = two 64-sector colour
    channels; Eq. 1 reward; readings A1-A6, A13, A24):

    * neighbours: j != i with torus distance d_ij < d_v (Eq. 1, strict, A6);
    * contact: d_ij <= 2 d_r (A6, inclusive);
    * bearing phi = atan2(h x d, h . d) in (-pi, pi], h = (cos theta_i, sin theta_i);
      visible iff -fov/2 <= phi < fov/2 (A3); sector k = floor((phi + fov/2)/fov * v);
    * obs[ch(j) v + k] = min d_ij / d_v over visible j, 1.0 if none (A2); flock
      obs[v] = s_i / s_max (A24);
    * reward: flock sum_j f(d_ij) over neighbours (Eq. 1, all directions, A4); tag
      chaser +r_touch per runner within 2 d_r, runner -r_touch per chaser within 2 d_r
      plus w * sum f(d) over runner neighbours (A15).

    ``overrides`` maps (row position, j) -> (in_radius, contact, sector) to force the
    decision of a pair (sector -1 = not visible); the comparator uses it to evaluate the
    alternative outcomes of banded pairs (A17, A19).

    Returns arrays over the rows plus ``bands``: for each row position a list of
    (j, [alternative decisions]) for pairs within BAND of a threshold.
    """
    st = np.asarray(state_r, dtype=np.float64)
    n = st.shape[0]
    rows = np.asarray(rows, dtype=np.int64)
    nr = len(rows)
    v, ch = int(p.v), (1 if p.env == FLOCK else 2)
    L = float(p.width)
    del L
    fov = float(p.fov)

    b, j, dx, dy, d = _pairs(p, st, rows)
    th = st[rows[b], 2]
    hx, hy = np.cos(th), np.sin(th)
    fwd = hx * dx + hy * dy
    left = hx * dy - hy * dx
    # atan2(0, 0) = 0 (A13): a coincident agent is dead ahead.  Set explicitly: at d = 0,
    # h . d and h x d are signed zeros, which IEEE atan2 maps to +-pi when cos(theta) < 0.
    phi = np.where(d == 0.0, 0.0, np.arctan2(left, fwd))
    u = (phi + fov / 2.0) / fov

    in_r = d < p.d_v
    contact = d <= 2.0 * p.d_r
    vis = (phi >= -fov / 2.0) & (phi < fov / 2.0)
    k = np.clip(np.floor(u * v), 0, v - 1).astype(np.int64)
    ksec = np.where(vis, k, -1)

    # ---- bands (A17): alternatives for pairs within BAND of a threshold
    rband = np.abs(d / p.d_v - 1.0) <= BAND
    cband = np.abs(d / (2.0 * p.d_r) - 1.0) <= BAND
    kb = np.rint(u * v)
    sband = (np.abs(u - kb / v) <= BAND) & (kb >= 0) & (kb <= v)
    bands: list[list] = [[] for _ in range(nr)]
    for t in np.nonzero(rband | cband | sband)[0]:
        r_opts = [True, False] if rband[t] else [bool(in_r[t])]
        c_opts = [True, False] if cband[t] else [bool(contact[t])]
        if sband[t]:
            kk = int(kb[t])
            k_opts = [kk - 1 if kk >= 1 else -1, kk if kk <= v - 1 else -1]
        else:
            k_opts = [int(ksec[t])]
        alts = [(ro, co, ko) for ro in r_opts for co in c_opts for ko in k_opts]
        if len(alts) > 1:
            bands[int(b[t])].append((int(j[t]), alts))

    if overrides:
        index = {(int(bb), int(jj)): t for t, (bb, jj) in enumerate(zip(b, j))}
        in_r, contact, ksec = in_r.copy(), contact.copy(), ksec.copy()
        for key, (ro, co, ko) in overrides.items():
            t = index[key]
            in_r[t], contact[t], ksec[t] = ro, co, ko

    contact = contact & in_r
    ksec = np.where(in_r, ksec, -1)

    # ---- conditioning of the reward terms (for the comparator's derived fp32 bound,
    # DESIGN.md §5): per row, over the in-radius non-contact terms (weight w_prox for
    # tag runner pairs), sum_j |f'(d_j)| d_j (sensitivity to a relative distance error)
    # and sum_j (|k| d_j + |b|) over both lines of f = min(rise, fall) (A5; magnitudes
    # of the line evaluation, i.e. sensitivity to relative coefficient errors).
    two_dr = 2.0 * float(p.d_r)
    k_rise = p.c_near / (p.d_peak - two_dr)
    k_fall = p.c_near / (p.d_v - p.d_peak)
    slope = np.where(d <= p.d_peak, k_rise, k_fall)
    lines = k_rise * d + k_rise * two_dr + k_fall * d + k_fall * p.d_v
    f_term = in_r & ~contact

    # ---- counts
    n_neigh = np.bincount(b[in_r], minlength=nr).astype(np.uint32)
    n_touch = np.zeros(nr, np.uint32)
    if p.env == FLOCK:
        n_collide = np.bincount(b[contact], minlength=nr).astype(np.uint32)
        terms = np.where(in_r, reward_f(p, d, contact), 0.0)
        reward = np.bincount(b, weights=terms, minlength=nr)
        sum_abs = np.bincount(b, weights=np.abs(terms), minlength=nr)
        wt = f_term.astype(np.float64)
        chan = np.zeros_like(j)
    else:
        first_chaser = n - p.n_chasers
        tj = (j >= first_chaser).astype(np.int64)            # 0 runner, 1 chaser
        tq = (rows[b] >= first_chaser).astype(np.int64)
        same = tj == tq
        n_collide = np.bincount(b[contact & same], minlength=nr).astype(np.uint32)
        n_touch = np.bincount(b[contact & ~same], minlength=nr).astype(np.uint32)
        prox = np.where(in_r & (tq == 0) & (tj == 0),
                        p.w_prox * reward_f(p, d, contact), 0.0)
        row_is_chaser = rows >= first_chaser
        touch = p.r_touch * n_touch.astype(np.float64)
        reward = np.where(row_is_chaser, touch,
                          -touch + np.bincount(b, weights=prox, minlength=nr))
        sum_abs = touch + np.bincount(b, weights=np.abs(prox), minlength=nr)
        wt = np.where(f_term & (tq == 0) & (tj == 0), float(p.w_prox), 0.0)
        chan = tj
    n_terms = np.bincount(b, weights=(wt > 0).astype(np.float64), minlength=nr)
    slope_d = np.bincount(b, weights=wt * slope * d, minlength=nr)
    line_abs = np.bincount(b, weights=wt * lines, minlength=nr)

    # ---- observation (per-sector nearest distance)
    view = np.ones((nr, ch * v), dtype=np.float64)
    occ = np.zeros((nr, ch * v), dtype=bool)
    sel = ksec >= 0
    col = chan[sel] * v + ksec[sel]
    np.minimum.at(view, (b[sel], col), d[sel] / p.d_v)
    occ[b[sel], col] = True
    if p.env == FLOCK:
        obs = np.concatenate([view, (st[rows, 3] / p.s_max)[:, None]], axis=1)
    else:
        obs = view
    words = (ch * v + 31) // 32
    occ_bits = np.zeros((nr, words), dtype=np.uint64)
    for w in range(words):
        seg = occ[:, 32 * w:32 * (w + 1)]
        occ_bits[:, w] = (seg.astype(np.uint64) << np.arange(seg.shape[1], dtype=np.uint64)).sum(1)
    return {
        "obs": obs, "reward": reward, "sum_abs": sum_abs, "n_terms": n_terms,
        "slope_d": slope_d, "line_abs": line_abs, "n_neigh": n_neigh,
        "n_collide": n_collide, "n_touch": n_touch,
        "sector_occ": occ_bits.astype(np.uint32), "bands": bands,
    }


def sense(p, state: np.ndarray, replicas=None, rows=None, workers: int = 1) -> dict:
    """``sense_rows`` over every replica (or the listed ones) and every row (or ``rows``).

    ``workers`` > 1 splits independent query-row blocks over a process pool (rows are
    independent: each reads the same snapshot).
    """
    st = np.asarray(state, dtype=np.float64).reshape(p.n_replicas, p.n_agents, 4)
    reps = range(p.n_replicas) if replicas is None else replicas
    rws = np.arange(p.n_agents) if rows is None else np.asarray(rows)
    outs = []
    for r in reps:
        if workers > 1 and len(rws) > 256:
            import multiprocessing as mp
            chunks = np.array_split(rws, max(workers, len(rws) // 256))
            with mp.get_context("fork").Pool(workers) as pool:
                parts = pool.starmap(sense_rows, [(p, st[r], c) for c in chunks])
            outs.append(_concat(parts))
        else:
            outs.append(sense_rows(p, st[r], rws))
    res = {k: np.stack([o[k] for o in outs]) for k in outs[0] if k != "bands"}
    res["bands"] = [o["bands"] for o in outs]
    return res


def _concat(parts):
    res = {k: np.concatenate([q[k] for q in parts]) for k in parts[0] if k != "bands"}
    res["bands"] = [bb for q in parts for bb in q["bands"]]
    return res


def step(p, state: np.ndarray, actions: np.ndarray, workers: int = 1) -> dict:
    """One full environment update: integrate, then sense the new snapshot (A8)."""
    new = integrate(p, state, actions)
    out = sense(p, new, workers=workers)
    out["state"] = new
    return out
