"""Pins for the comparison contract itself and for the oracle paths only the GPU tests and
the bench use (no GPU):

* the derived reward bound (tests/vg_parity.py ``reward_bound``) holds for
  an fp32 emulation of the kernel's per-pair reward arithmetic (worst-case MUFU sqrt error
  injected), and it is tighter than the round-1 floor on sparse rows;
* ``oracle.sense(workers > 1)`` (process pool over row blocks) equals ``workers = 1``;
* ``oracle.step`` (integrate, then sense the new snapshot: reading A8 of P:190) on a
  hand-placed two-agent world with closed-form positions, bearing and reward.
"""
import math

import numpy as np
import pytest

import oracle
import vg_inputs as vi
import vg_parity as parity

F32 = np.float32


def _fma32(a, b, c):
    # fp32 fma: a*b is exact in fp64 (24 + 24 bits), one fp64 addition, one fp32 rounding
    # (the fp64 sum's own rounding is ~2^-29 relative to the result: far below 2^-24).
    return F32(np.float64(a) * np.float64(b) + np.float64(c))


def _kernel_terms(p, qx, qy, cx, cy, sqrt_err):
    """fp32 emulation of K4's per-pair reward term in 2^-32 fixed-point units (A5, A16b):
    dx, dy (one rounding each), d^2 = fma(dx, dx, dy*dy), d = sqrt(d^2) (1 + sqrt_err),
    f = min(fma(k_r, d, b_r), fma(-k_f, d, b_f)) with derive()'s fp32 coefficients."""
    two_dr = F32(2) * F32(p.d_r)
    k_r = F32(F32(p.c_near) / F32(F32(p.d_peak) - two_dr))
    b_r = F32(-k_r * two_dr)
    k_f = F32(F32(p.c_near) / F32(F32(p.d_v) - F32(p.d_peak)))
    b_f = F32(k_f * F32(p.d_v))
    s = F32(4294967296.0)
    out = []
    for x0, y0, x1, y1, e in zip(qx, qy, cx, cy, sqrt_err):
        dx, dy = F32(x1 - x0), F32(y1 - y0)
        d2 = _fma32(dx, dx, F32(dy * dy))
        d = F32(np.sqrt(np.float64(d2)) * (1.0 + e))
        f = min(_fma32(k_r * s, d, b_r * s), _fma32(-k_f * s, d, b_f * s))
        out.append(float(np.rint(np.float64(f))) * 2.0 ** -32)
    return np.array(out)


def test_reward_bound_covers_fp32_emulation():
    p = vi.flock_params(2)
    rng = np.random.default_rng(3)
    n = 20000
    qx = rng.uniform(10, 90, n).astype(F32)
    qy = rng.uniform(10, 90, n).astype(F32)
    d = rng.uniform(2 * p.d_r * 1.001, p.d_v * 0.99999, n)
    a = rng.uniform(0, 2 * math.pi, n)
    cx = (qx + d * np.cos(a)).astype(F32)
    cy = (qy + d * np.sin(a)).astype(F32)
    err = rng.choice([-1.0, 1.0], n) * 2.0 ** -22           # worst-case MUFU sqrt error
    got = _kernel_terms(p, qx, qy, cx, cy, err)
    worst = 0.0
    for i in range(n):
        st = np.array([[qx[i], qy[i], 0.0, 0.3], [cx[i], cy[i], 0.0, 0.3]], np.float64)
        ref = oracle.sense_rows(p, st, [0])
        if ref["n_collide"][0] or ref["n_neigh"][0] != 1 or ref["bands"][0]:
            continue
        e = abs(got[i] - ref["reward"][0])
        b = parity.reward_bound(ref, 0) - 2 * parity.U * ref["sum_abs"][0]   # per term
        assert e <= b, (i, e, b)
        worst = max(worst, e / b)
        if i > 3000:
            break
    assert worst > 0.05          # the bound is not vacuous (observed ~0.2-0.5)


def test_reward_bound_tighter_than_round1_floor():
    # Sparse C1 rows (sum |f| ~ 1): the derived bound replaces the old 1e-5 (sum|f| + c_near)
    p = vi.workload("c1")
    st = vi.init_state(p, seed=0)[0].astype(np.float64)
    ref = oracle.sense_rows(p, st, np.arange(p.n_agents))
    for b in range(p.n_agents):
        old = parity.REL * (ref["sum_abs"][b] + p.c_near)
        assert parity.reward_tol(ref, b) < old
        assert parity.reward_bound(ref, b) < 2e-6 * max(1, ref["n_terms"][b])


def test_sense_workers_equals_serial():
    p = vi.flock_params(3000)
    st = vi.init_state(p, seed=21)
    rows = np.random.default_rng(0).choice(p.n_agents, 700, replace=False)
    a = oracle.sense(p, st, rows=rows, workers=1)
    b = oracle.sense(p, st, rows=rows, workers=3)
    for k in a:
        if k == "bands":
            assert a[k] == b[k]
        else:
            assert np.array_equal(a[k], b[k]), k


def test_step_two_agents_closed_form():
    # Agent 0 at (50, 50) heading 0, speed 0.3; agent 1 at (50.3, 52) heading pi/2, speed
    # 0.2; zero actions.  After the move (A8): (50.3, 50) and (50.3, 52.2): d = 2.2, agent 1
    # at bearing +90 deg from agent 0 (sector 110, module docstring of test_oracle_sense),
    # agent 0 straight behind agent 1 (blind spot); both rewards f(2.2) = 0.5 * 1.7 / 4.75.
    p = vi.flock_params(2)
    st = np.array([[[50.0, 50.0, 0.0, 0.3], [50.3, 52.0, math.pi / 2, 0.2]]])
    act = np.zeros((1, 2, 2))
    for workers in (1, 2):
        out = oracle.step(p, st, act, workers=workers)
        assert out["state"][0, 0, :2] == pytest.approx([50.3, 50.0], abs=1e-12)
        assert out["state"][0, 1, :2] == pytest.approx([50.3, 52.2], abs=1e-12)
        f = 0.5 * (2.2 - 0.5) / (5.25 - 0.5)
        assert out["reward"][0] == pytest.approx([f, f], rel=1e-6)
        assert list(out["n_neigh"][0]) == [1, 1]
        view0 = out["obs"][0, 0, :128]
        assert np.nonzero(view0 < 1)[0].tolist() == [110]
        assert view0[110] == pytest.approx(0.22, rel=1e-6)
        assert np.all(out["obs"][0, 1, :128] == 1.0)
        assert out["obs"][0, 0, 128] == pytest.approx(0.3 / 0.5, rel=1e-6)
