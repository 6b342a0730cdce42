"""Pins for oracle.integrate (a1, a1') — closed forms and SPEC examples, no GPU."""
import math

import numpy as np
import pytest

import oracle
import vg_inputs as vi


def _one(p, x, y, th, s):
    return np.array([[[x, y, th, s]]], dtype=np.float32)


def _act(a0, a1):
    return np.array([[[a0, a1]]], dtype=np.float32)


def test_speed_upper_clamp():
    # S:252 "s_t=s_max, a_t=a_max -> s_max"
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 10, 10, 0, p.s_max), _act(p.a_max, 0))
    assert out[0, 0, 3] == pytest.approx(p.s_max, abs=0)


def test_speed_lower_clamp():
    # S:253 "s_t=s_min, a_t=-a_max -> s_min"
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 10, 10, 0, p.s_min), _act(-p.a_max, 0))
    assert out[0, 0, 3] == pytest.approx(p.s_min, abs=0)


def test_speed_interior():
    # S:254 "s_t=0.5, a_t=0.1, bounds [0.1, 1.0] -> 0.6"; the paper's garbled
    # min(s_min, max(s + a, s_max)) would give 0.1 — reading A7 rejects it.
    p = vi.flock_params(1, s_min=0.1, s_max=1.0, a_max=0.2)
    out = oracle.integrate(p, _one(p, 10, 10, 0, 0.5), _act(0.1, 0))
    assert out[0, 0, 3] == pytest.approx(0.6, abs=1e-7)


def test_move_uses_new_speed_and_heading():
    # A8: rotate -> accelerate -> move with the NEW heading and speed.
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 50, 50, 0.0, 0.3), _act(0.1, 0.2))
    th = float(np.float32(0.2))
    s = float(np.float32(0.3)) + float(np.float32(0.1))
    assert out[0, 0, 2] == pytest.approx(th, abs=1e-12)
    assert out[0, 0, 3] == pytest.approx(s, abs=1e-12)
    assert out[0, 0, 0] == pytest.approx(50 + s * math.cos(th), abs=1e-9)
    assert out[0, 0, 1] == pytest.approx(50 + s * math.sin(th), abs=1e-9)


def test_heading_wrap_negative():
    # S:117 "heading written -0.1 -> reads back 2 pi - 0.1"
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 10, 10, 0.0, 0.3), _act(0, -0.1))
    assert out[0, 0, 2] == pytest.approx(2 * math.pi - float(np.float32(0.1)), abs=1e-12)


def test_heading_63_turns():
    # S:90 "heading += 0.1 over 63 commits from 0 -> 6.3 mod 2 pi = 0.01681 (1e-9)"
    p = vi.flock_params(1)
    st = _one(p, 10, 10, 0.0, 0.3)
    turn = 0.1
    cur = st.astype(np.float64)
    for _ in range(63):
        cur = oracle.integrate(p, cur, np.array([[[0.0, turn]]]))
    assert cur[0, 0, 2] == pytest.approx(6.3 - 2 * math.pi, abs=1e-9)
    assert cur[0, 0, 2] == pytest.approx(0.01681469, abs=1e-8)


def test_position_wrap():
    # S:116 "position written to (101, 5) -> reads back (1, 5)": 100.8 + 0.5 wraps to 0.8
    # (x = 99.9, heading 0, speed 0.5 -> 100.4 -> 0.4).
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 99.9, 5.0, 0.0, 0.5), _act(0.0, 0.0))
    assert out[0, 0, 0] == pytest.approx(float(np.float32(99.9)) + 0.5 - 100.0, abs=1e-12)
    assert out[0, 0, 1] == pytest.approx(5.0, abs=1e-12)
    # negative side
    out = oracle.integrate(p, _one(p, 0.2, 5.0, math.pi, 0.5), _act(0.0, 0.0))
    th = float(np.float32(math.pi))
    assert out[0, 0, 0] == pytest.approx(100.0 + float(np.float32(0.2)) + 0.5 * math.cos(th), abs=1e-9)


def test_straight_line_closed_form():
    # a = 0 => p_k = p_0 + k s (cos th, sin th) mod L.
    p = vi.flock_params(50)
    st = vi.init_state(p, seed=3).astype(np.float64)
    x0 = st.copy()
    zero = np.zeros((1, 50, 2))
    for _ in range(40):
        st = oracle.integrate(p, st, zero)
    s = x0[0, :, 3]
    ex = np.mod(x0[0, :, 0] + 40 * s * np.cos(x0[0, :, 2]), p.width)
    ey = np.mod(x0[0, :, 1] + 40 * s * np.sin(x0[0, :, 2]), p.width)
    dx = oracle.minimal_image(p, ex, st[0, :, 0])
    dy = oracle.minimal_image(p, ey, st[0, :, 1])
    assert np.max(np.abs(dx)) < 1e-9 and np.max(np.abs(dy)) < 1e-9


def test_action_clamped_not_rejected():
    # out-of-box actions are clipped to the box.
    p = vi.flock_params(1)
    out = oracle.integrate(p, _one(p, 10, 10, 1.0, 0.3), _act(10.0, -10.0))
    assert out[0, 0, 3] == pytest.approx(min(0.3 + p.a_max, p.s_max), abs=1e-7)
    assert out[0, 0, 2] == pytest.approx(float(np.float32(1.0)) - p.theta_max, abs=1e-12)


def test_tag_move_clamp_per_type():
    # P:194 "moves them along the heading, in the range [0, s_max]"; chasers 0.75 s_max
    p = vi.tag_params(2, n_chasers=1)
    st = np.array([[[10, 10, 0, 0], [20, 20, 0, 0]]], dtype=np.float32)
    out = oracle.integrate(p, st, np.array([[[0, 10.0], [0, 10.0]]], np.float32))
    assert out[0, 0, 0] == pytest.approx(10 + p.s_max, abs=1e-9)          # runner
    assert out[0, 1, 0] == pytest.approx(20 + p.s_max_chaser, abs=1e-9)   # chaser
    out = oracle.integrate(p, st, np.array([[[0, -10.0], [0.1, -3.0]]], np.float32))
    assert out[0, 0, 0] == 10 and out[0, 1, 0] == 20                        # no backwards move
    assert out[0, 1, 2] == pytest.approx(float(np.float32(0.1)), abs=1e-12)
    assert np.all(out[..., 3] == 0)                                          # passthrough


def test_bounds_invariants_random():
    # speed within [s_min, s_max], positions within [0, L), heading in [0, 2 pi).
    p = vi.flock_params(300)
    st = vi.init_state(p, seed=1).astype(np.float64)
    for t in range(20):
        a = vi.actions(p, seed=1, step=t) * 3.0   # also exercises clamping
        st = oracle.integrate(p, st, a)
        assert np.all((st[..., 3] >= p.s_min) & (st[..., 3] <= p.s_max))
        assert np.all((st[..., :2] >= 0) & (st[..., :2] < p.width))
        assert np.all((st[..., 2] >= 0) & (st[..., 2] < 2 * math.pi))
