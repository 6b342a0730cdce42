"""Comparison contract between the CUDA path and the oracle.

* integer outputs (cell ids, bins, counts, sector occupancy): bit-exact, except that a row
  whose mismatch is explained by a *banded* pair (within 1e-6 of the radius, the contact
  distance or a sector boundary, A17) may equal the oracle re-evaluated with that pair's
  alternative decision;
* observation view entries: |gpu - ref| <= 1e-5 ref (1.0 exactly when the sector is empty);
* flock speed entry: |gpu - ref| <= 1e-5 ref;
* reward: |gpu - ref| <= max(1e-5 sum_j |term_j|, B) — relative to the sum of absolute
  terms (robust to cancellation), or, where that is below what fp32 can deliver (a row
  whose neighbours sit near f = 0, e.g. just inside d_v), the kernel's derived worst-case
  fp32 error B of the same row (``reward_bound``);
* integrate: torus |dp| <= 1e-5 L, circular |dtheta| <= 1e-5 2 pi, |ds| <= 1e-5 s_max.
Rows with more than 4 banded pairs are "don't care" (counted, asserted rare).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

import oracle

REL = 1e-5
U = 2.0 ** -24          # fp32 unit roundoff
#: relative error of the kernel's distance d: dx, dy rounded (u each), dy^2
#: and the fma rounded (d^2 within 5u -> d within 2.5u), MUFU sqrt.approx assumed <= 2^-22
#: (4u); 8u leaves margin.
EPS_D = 8 * U
#: relative error of one line evaluation k d + b of f (A5): k, b each within 3u of their
#: fp64 values (derive(): a subtraction, a division, a product), the fma rounds once (u).
EPS_LINE = 4 * U


def reward_bound(ref, b):
    """Derived worst-case |gpu - ref| of row b's reward: per f-term
    |f'(d)| EPS_D d + EPS_LINE (|k_rise| d + |b_rise| + |k_fall| d + |b_fall|) + 2^-33
    (fixed-point rounding, A16b), plus 2u sum|term| (tag's RN32(w f) per term and the
    final RN32 of the int64 sum).  The oracle supplies the per-row sums."""
    return (EPS_D * ref["slope_d"][b] + EPS_LINE * ref["line_abs"][b]
            + ref["n_terms"][b] * 2.0 ** -33 + 2 * U * ref["sum_abs"][b])


def reward_tol(ref, b):
    return max(REL * ref["sum_abs"][b], reward_bound(ref, b))


def torus_err(a, b, period):
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    return np.minimum(d, period - d)


def check_integrate(p, gpu_state, ref_state):
    """Return max errors; assert within the integrate tolerance."""
    g = np.asarray(gpu_state, np.float64).reshape(-1, 4)
    r = np.asarray(ref_state, np.float64).reshape(-1, 4)
    ep = max(torus_err(g[:, 0], r[:, 0], p.width).max(initial=0),
             torus_err(g[:, 1], r[:, 1], p.width).max(initial=0))
    et = torus_err(g[:, 2], r[:, 2], 2 * math.pi).max(initial=0)
    es = np.abs(g[:, 3] - r[:, 3]).max(initial=0)
    assert ep <= REL * p.width, f"position error {ep}"
    assert et <= REL * 2 * math.pi, f"heading error {et}"
    assert es <= REL * p.s_max, f"speed error {es}"
    assert np.all((g[:, :2] >= 0) & (g[:, :2] < p.width))
    assert np.all((g[:, 2] >= 0) & (g[:, 2] < np.float32(2 * math.pi)))
    return {"pos": ep, "heading": et, "speed": es}


def check_bins(p, gpu_bins, state32):
    """Bit-exact comparison of the binning (A16: the oracle evaluates the fp32 formula)."""
    ref = oracle.bins(p, state32)
    for k in ("cell_id", "cell_start", "perm"):
        g = np.asarray(gpu_bins[k]).astype(np.int64).reshape(ref[k].shape)
        assert np.array_equal(g, ref[k].astype(np.int64)), f"bins.{k} differs"
    gs = np.asarray(gpu_bins["sorted"], np.float32).reshape(ref["sorted"].shape)
    assert np.array_equal(gs.view(np.uint32), ref["sorted"].view(np.uint32)), "bins.sorted differs"


def _row_ok(p, ref, b, g, why=None):
    """Does GPU row g (dict of arrays) satisfy the contract against oracle row b of ref?"""
    for k in ("n_neigh", "n_collide", "n_touch"):
        if k in g and int(g[k]) != int(ref[k][b]):
            return _why(why, f"{k}: gpu {int(g[k])} ref {int(ref[k][b])}")
    if "sector_occ" in g and not np.array_equal(np.asarray(g["sector_occ"]).astype(np.uint32),
                                                ref["sector_occ"][b]):
        return _why(why, "sector_occ")
    if "obs" in g:
        go = np.asarray(g["obs"], np.float64)
        ro = ref["obs"][b]
        nv = (1 if p.env == "flock" else 2) * p.v
        empty = ro[:nv] == 1.0
        if not np.all(go[:nv][empty] == 1.0):
            return _why(why, "obs: empty sector not 1.0")
        if np.any(go[:nv][~empty] >= 1.0):
            return _why(why, "obs: occupied sector reads 1.0")
        err = np.abs(go[:nv][~empty] - ro[:nv][~empty])
        if np.any(err > REL * ro[:nv][~empty]):
            return _why(why, f"obs: rel err {np.max(err / ro[:nv][~empty])}")
        if p.env == "flock" and abs(go[nv] - ro[nv]) > REL * ro[nv]:
            return _why(why, "obs: speed entry")
    if "reward" in g:
        tol = reward_tol(ref, b)
        if abs(float(g["reward"]) - ref["reward"][b]) > tol:
            return _why(why, f"reward: gpu {float(g['reward'])} ref {ref['reward'][b]} tol {tol}")
    return True


def _why(why, msg):
    if why is not None:
        why.append(msg)
    return False


def check_sense(p, state_r, gpu: dict, rows=None, max_flags=4, workers=1):
    """Compare GPU outputs of one replica (arrays indexed by agent id) with the oracle on
    ``rows`` (default: all).  Returns statistics; raises AssertionError on a violation.
    ``workers`` > 1 evaluates the oracle rows on a process pool (oracle.sense; pinned
    against workers = 1 by tests/test_oracle_sense.py)."""
    n = np.asarray(state_r).shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows)
    if workers > 1:
        q = p.replace(n_replicas=1)
        full = oracle.sense(q, np.asarray(state_r)[None], rows=rows, workers=workers)
        ref = {k: v[0] for k, v in full.items() if k != "bands"}
        ref["bands"] = full["bands"][0]
    else:
        ref = oracle.sense_rows(p, state_r, rows)
    stats = {"rows": len(rows), "banded_pairs": 0, "banded_rows": 0, "alt_rows": 0,
             "dont_care": 0, "max_obs_rel": 0.0, "max_reward_err": 0.0,
             "max_reward_err_over_tol": 0.0, "bound_rows": 0}
    failures = []
    for b, i in enumerate(rows):
        g = {k: np.asarray(v)[i] for k, v in gpu.items()}
        nb = len(ref["bands"][b])
        stats["banded_pairs"] += nb
        stats["banded_rows"] += nb > 0
        if _row_ok(p, ref, b, g):
            if "obs" in g:
                ro = ref["obs"][b]
                occ = ro < 1.0
                if occ.any():
                    rel = np.abs(np.asarray(g["obs"], np.float64)[occ] - ro[occ]) / ro[occ].clip(1e-30)
                    stats["max_obs_rel"] = max(stats["max_obs_rel"], float(np.max(rel)))
            if "reward" in g:
                e = abs(float(g["reward"]) - ref["reward"][b])
                tol = reward_tol(ref, b)
                stats["max_reward_err"] = max(stats["max_reward_err"], e)
                if tol > 0:
                    stats["max_reward_err_over_tol"] = max(stats["max_reward_err_over_tol"], e / tol)
                stats["bound_rows"] += int(reward_bound(ref, b) > REL * ref["sum_abs"][b])
            continue
        if nb == 0:
            why = []
            _row_ok(p, ref, b, g, why)
            failures.append((int(i), why))
            continue
        if nb > max_flags:
            stats["dont_care"] += 1
            continue
        js = [j for j, _ in ref["bands"][b]]
        alts = [a for _, a in ref["bands"][b]]
        ok = False
        for combo in itertools.product(*alts):
            ov = {(0, j): a for j, a in zip(js, combo)}
            alt = oracle.sense_rows(p, state_r, [i], overrides=ov)
            if _row_ok(p, alt, 0, g):
                ok = True
                break
        if ok:
            stats["alt_rows"] += 1
        else:
            why = []
            _row_ok(p, ref, b, g, why)
            failures.append((int(i), ["banded, no alternative matches"] + why))
    assert not failures, f"{len(failures)} rows violate the contract, e.g. {failures[:5]}"
    assert stats["dont_care"] <= max(1, 1e-4 * len(rows)), stats
    return stats
