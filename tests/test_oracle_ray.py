"""Pins for oracle.ray: closed forms, bisection root finder,
monotonicity, limit cases.  No GPU."""
import math

import numpy as np
import pytest

import vg_inputs as vi
from oracle.ray import ray_disc, ray_views


def test_head_on_hit():
    # S:173 "origin (0,0), dir (1,0), disc center (5,0) radius 1 -> 4"
    t, _ = ray_disc(np.array(1.0), np.array(0.0), np.array(5.0), np.array(0.0), 1.0)
    assert t == 4.0


def test_perpendicular_miss_and_behind():
    # S:174 "disc center (0,5) radius 1, dir (1,0) -> absent"; a disc behind is missed too
    t, _ = ray_disc(np.array(1.0), np.array(0.0), np.array(0.0), np.array(5.0), 1.0)
    assert np.isinf(t)
    t, _ = ray_disc(np.array(1.0), np.array(0.0), np.array(-5.0), np.array(0.0), 1.0)
    assert np.isinf(t)


def test_origin_inside_is_zero():
    # S:170 "origin inside the disc returns 0"
    t, _ = ray_disc(np.array(0.0), np.array(1.0), np.array(0.3), np.array(0.2), 1.0)
    assert t == 0.0


def test_bisection_root_finder():
    # S:175 "random configurations -> matches bisection root-finder on |o + t d - c| - r"
    rng = np.random.default_rng(0)
    for _ in range(300):
        a = rng.uniform(-math.pi, math.pi)
        ux, uy = math.cos(a), math.sin(a)
        cx, cy = rng.uniform(-6, 6, 2)
        r = rng.uniform(0.1, 2.0)
        t, _ = ray_disc(np.array(ux), np.array(uy), np.array(cx), np.array(cy), r)
        f = lambda s: math.hypot(s * ux - cx, s * uy - cy) - r  # noqa: E731
        if f(0) <= 0:
            assert t == 0.0
            continue
        s_star = ux * cx + uy * cy                       # closest approach along the ray
        if s_star <= 0 or f(s_star) > 0:
            assert np.isinf(t)
            continue
        lo, hi = 0.0, s_star                              # f(lo) > 0 >= f(hi)
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            lo, hi = (mid, hi) if f(mid) > 0 else (lo, mid)
        assert float(t) == pytest.approx(hi, abs=1e-9)


def test_dead_ahead_central_sectors():
    # a neighbour dead ahead at d < d_v, v even -> the two central sectors read
    # (d - correction)/d_v < d/d_v; rays off the disc read 1.0.
    p = vi.flock_params(2)
    st = np.array([[50, 50, 0.0, 0.275], [53, 50, 0.0, 0.275]])
    view, lo, hi = ray_views(p, st, [0])
    c = view[0]
    assert c[63] == c[64] < 0.3 and c[63] > (3 - 0.25) / 10 - 1e-12
    hits = np.nonzero(c < 1)[0]
    assert list(hits) == list(range(64 - len(hits) // 2, 64 + len(hits) // 2))
    # half-width of the hit range: asin(d_r/d) / sector width sectors each side
    alpha = math.asin(0.25 / 3)
    assert abs(len(hits) - 2 * alpha / (p.fov / 128)) <= 2


def test_isolated_and_far():
    # S:182 "isolated agent -> all entries 1.0"
    p = vi.flock_params(2)
    view, _, _ = ray_views(p, np.array([[10, 10, 0, 0.2], [60, 60, 0, 0.2]]), [0])
    assert np.all(view == 1.0)


def test_monotone_as_neighbour_approaches():
    # S:187 "moving a lone neighbour radially closer along a sector ray never increases it"
    p = vi.flock_params(2)
    prev = None
    for dd in np.linspace(9.5, 0.6, 25):
        view, _, _ = ray_views(p, np.array([[50, 50, 0.0, 0.2], [50 + dd, 50, 0, 0.2]]), [0])
        cur = view[0]
        if prev is not None:
            assert np.all(cur <= prev + 1e-12)
        prev = cur


def test_bounds_bracket_the_value():
    p = vi.flock_params(800)
    st = vi.init_state(p, seed=3)[0].astype(np.float64)
    view, lo, hi = ray_views(p, st, np.arange(100))
    assert np.all(lo <= view + 1e-15) and np.all(view <= hi + 1e-15)


def test_interval_narrow_where_well_conditioned():
    # The comparator's [lo, hi] must not be loose: on sectors with no grazing
    # disc and a well-conditioned nearest hit, hi - lo <= 2 (1e-5 view + 1e-6) + 1e-6; those
    # sectors are the bulk of the hits.
    import vg_inputs as vi
    from oracle.ray import ray_views
    p = vi.flock_params(3000).replace(vision="ray")
    st = vi.init_state(p, seed=4)[0].astype(np.float64)
    view, lo, hi, cond = ray_views(p, st, np.arange(200), return_cond=True)
    assert np.all((lo <= view + 1e-12) & (view <= hi + 1e-12))
    assert np.all((hi - lo)[cond] <= 2e-5 * view[cond] + 3e-6 + 1e-9)
    hit = view < 1.0
    assert (cond & hit).sum() >= 0.7 * hit.sum()
