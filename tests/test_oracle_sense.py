"""Pins for oracle.sense_rows (a3-a5): hand-placed worlds with closed-form observations and
rewards, library neighbour search, exact integer arithmetic, invariants and closed-form
expectations.  No GPU.

Hand values used below (reading A3: fov = 250 deg centred on the heading, CCW-positive
bearing, sector k covers u in [k/v, (k+1)/v) with u = (phi + fov/2)/fov; A5: f from S:219):
  * neighbour at bearing +90 deg: u = (90 + 125)/250 = 0.86  -> k = floor(110.08) = 110
  * neighbour at bearing -90 deg: u = 35/250 = 0.14           -> k = floor(17.92) = 17
  * bearing +124 deg: u = 0.996 -> k = 127;  -124 deg: u = 0.004 -> k = 0;  +-126 deg: blind
  * f(0.25) = -1, f(0.5) = -1 (contact inclusive), f(2.875) = 0.5 * 2.375/4.75 = 0.25,
    f(5.25) = 0.5, f(7.625) = 0.5 * 2.375/4.75 = 0.25, f(5) = 0.5 * 4.5/4.75
"""
import math

import numpy as np
import pytest

import oracle
import vg_inputs as vi

DEG = math.pi / 180.0


def world(p, agents):
    st = np.array([agents], dtype=np.float64)
    return p.replace(n_agents=st.shape[1]), st


def sense_all(p, st):
    return oracle.sense_rows(p, st[0], np.arange(st.shape[1]))


def test_lone_agent():
    # S:244 "n=1 -> view all ones, speed element = 0.5 (s_min + s_max)/s_max"
    p = vi.flock_params(1)
    p, st = world(p, [[50, 50, 1.0, 0.5 * (p.s_min + p.s_max)]])
    o = sense_all(p, st)
    assert np.all(o["obs"][0, :128] == 1.0)
    assert o["obs"][0, 128] == pytest.approx(0.5 * (p.s_min + p.s_max) / p.s_max, rel=1e-12)
    assert o["n_neigh"][0] == 0 and o["reward"][0] == 0 and np.all(o["sector_occ"] == 0)


def test_left_and_right_neighbours():
    p, st = world(vi.flock_params(2), [[50, 50, 0.0, 0.275], [50, 55, 0.0, 0.275]])
    o = sense_all(p, st)
    # agent 0 sees agent 1 at +90 deg (left), agent 1 sees agent 0 at -90 deg (right)
    for i, k in [(0, 110), (1, 17)]:
        view = o["obs"][i, :128]
        assert view[k] == pytest.approx(0.5, abs=1e-15)
        assert np.sum(view < 1.0) == 1
        assert o["sector_occ"][i, k // 32] == (1 << (k % 32))
        assert o["n_neigh"][i] == 1
        assert o["reward"][i] == pytest.approx(0.5 * 4.5 / 4.75, rel=1e-12)
        assert o["n_collide"][i] == 0


def test_blind_spot_and_fov_edges():
    p = vi.flock_params(2)
    for bearing, expect in [(124, 127), (-124, 0), (126, None), (-126, None), (180, None),
                            (0.5, 64), (-0.5, 63)]:
        b = bearing * DEG
        p2, st = world(p, [[50, 50, 0.3, 0.275],
                           [50 + 4 * math.cos(0.3 + b), 50 + 4 * math.sin(0.3 + b), 0, 0.275]])
        o = oracle.sense_rows(p2, st[0], [0])
        view = o["obs"][0, :128]
        assert o["n_neigh"][0] == 1                       # reward/neighbours ignore the fov (A4)
        assert o["reward"][0] == pytest.approx(0.5 * 3.5 / 4.75, rel=1e-9)
        if expect is None:
            assert np.all(view == 1.0)
        else:
            assert view[expect] == pytest.approx(0.4, rel=1e-12)
            assert np.sum(view < 1) == 1


def test_every_sector_centre():
    # A neighbour placed at the centre of sector k reads d/d_v in sector k only, k = 0..v-1.
    p = vi.flock_params(2)
    th0 = 0.7
    w = p.fov / p.v
    for k in range(p.v):
        beta = -p.fov / 2 + (k + 0.5) * w
        p2, st = world(p, [[50, 50, th0, 0.275],
                           [50 + 3 * math.cos(th0 + beta), 50 + 3 * math.sin(th0 + beta), 0, 0.3]])
        o = oracle.sense_rows(p2, st[0], [0])
        view = o["obs"][0, :128]
        assert view[k] == pytest.approx(0.3, rel=1e-12)
        assert np.sum(view < 1) == 1
        bits = o["sector_occ"][0]
        assert bits[k // 32] == (1 << (k % 32)) and bits.sum() == bits[k // 32]


@pytest.mark.parametrize("d,f,contact", [(0.25, -1.0, 1), (0.5, -1.0, 1), (2.875, 0.25, 0),
                                         (5.25, 0.5, 0), (7.625, 0.25, 0),
                                         (9.99, 0.5 * 0.01 / 4.75, 0), (10.0, 0.0, 0)])
def test_two_agent_reward(d, f, contact):
    # f(d_r) = -c_collide, f(d_peak) = c_near, d = d_v excluded (strict)
    p, st = world(vi.flock_params(2), [[20, 30, 0, 0.275], [20 + d, 30, 2.0, 0.275]])
    o = sense_all(p, st)
    for i in range(2):
        assert o["reward"][i] == pytest.approx(f, abs=1e-12)
        assert o["n_collide"][i] == contact
        assert o["n_neigh"][i] == (1 if d < 10 else 0)


def test_reward_f_points():
    p = vi.flock_params(2)
    d = np.array([0.0, 0.25, 0.5, 0.5000001, 2.875, 5.25, 7.625, 9.9999999])
    c = d <= 0.5
    f = oracle.reward_f(p, d, c)
    assert np.allclose(f, [-1, -1, -1, 0, 0.25, 0.5, 0.25, 0], atol=1e-6)


def test_wrap_neighbour():
    p, st = world(vi.flock_params(2), [[0.5, 50, math.pi / 2, 0.275], [99.5, 50, 0, 0.275]])
    o = sense_all(p, st)
    assert o["n_neigh"][0] == 1
    assert o["reward"][0] == pytest.approx(0.5 * 0.5 / 4.75, rel=1e-9)
    # agent 0 faces +y; agent 1 is at displacement (-1, 0): bearing +90 deg -> sector 110
    assert o["obs"][0, 110] == pytest.approx(0.1, rel=1e-9)


def test_dead_ahead_is_banded():
    # A3/A13: dead ahead sits exactly on the boundary beta_{v/2}: sector v/2, banded.
    p, st = world(vi.flock_params(2), [[50, 50, 0.0, 0.275], [53, 50, 0, 0.275]])
    o = oracle.sense_rows(p, st[0], [0])
    assert o["obs"][0, 64] == pytest.approx(0.3, rel=1e-12)
    (j, alts), = o["bands"][0]
    assert j == 1 and sorted(a[2] for a in alts) == [63, 64]
    # forcing the alternative moves the value to sector 63
    o2 = oracle.sense_rows(p, st[0], [0], overrides={(0, 1): (True, False, 63)})
    assert o2["obs"][0, 63] == pytest.approx(0.3, rel=1e-12) and o2["obs"][0, 64] == 1.0


@pytest.mark.parametrize("heading", [0.0, 1.0, 2.5, 3.2, 4.2572885, 5.9])
def test_coincident_agent_dead_ahead_any_heading(heading):
    # A13: a coincident other agent (d = 0) is dead ahead, phi = 0, whatever the heading —
    # including headings with cos < 0, where h . d and h x d are signed zeros that IEEE
    # atan2 would map to +-pi (behind, outside the field of view).
    p, st = world(vi.flock_params(2), [[50, 50, heading, 0.275], [50, 50, 1.0, 0.275]])
    o = oracle.sense_rows(p, st[0], [0])
    assert o["obs"][0, 64] == 0.0 and o["n_collide"][0] == 1 and o["n_neigh"][0] == 1
    (j, alts), = o["bands"][0]
    assert j == 1 and sorted(a[2] for a in alts) == [63, 64]


def test_neighbours_match_kdtree():
    # Library routine: scipy cKDTree with periodic boxsize (uses <=; compare off-band).
    from scipy.spatial import cKDTree
    p = vi.flock_params(1500)
    st = vi.init_state(p, seed=11).astype(np.float64)
    o = sense_all(p, st)
    pos = st[0, :, :2]
    tree = cKDTree(pos, boxsize=p.width)
    pairs = tree.query_pairs(p.d_v, output_type="ndarray")
    cnt = np.bincount(pairs.ravel(), minlength=p.n_agents)
    assert np.array_equal(cnt, o["n_neigh"])
    close = tree.query_pairs(2 * p.d_r, output_type="ndarray")
    assert np.array_equal(np.bincount(close.ravel(), minlength=p.n_agents), o["n_collide"])
    # reward sum rule: sum_i r_i = 2 sum_{i<j} f(d_ij) (S:300 pair symmetry)
    sdm = tree.sparse_distance_matrix(tree, p.d_v, output_type="ndarray")
    sdm = sdm[sdm["i"] < sdm["j"]]
    dd = sdm["v"]
    tot = 2 * oracle.reward_f(p, dd, dd <= 2 * p.d_r).sum()
    assert o["reward"].sum() == pytest.approx(tot, rel=1e-12)
    assert o["n_neigh"].sum() % 2 == 0


def test_dyadic_world_exact_thresholds():
    # Coordinates on a 2^-8 lattice: compare every decision with exact integer arithmetic.
    p = vi.flock_params(400, width=128.0, d_v=8.0)
    rng = np.random.default_rng(4)
    q = rng.integers(0, 128 * 256, size=(400, 2))
    # force some pairs exactly at d = d_v and d = 2 d_r
    q[1] = q[0] + [8 * 256, 0]
    q[3] = q[2] + [0, 128]
    q %= 128 * 256
    st = np.zeros((1, 400, 4))
    st[0, :, :2] = q / 256.0
    st[0, :, 3] = 0.275
    o = sense_all(p, st)
    M = 128 * 256
    dq = q[None, :, :] - q[:, None, :]
    dq = (dq + M // 2) % M - M // 2                      # exact minimal image on the lattice
    d2 = (dq ** 2).sum(-1)
    np.fill_diagonal(d2, 1 << 60)
    assert np.array_equal(o["n_neigh"], (d2 < (8 * 256) ** 2).sum(1))
    assert np.array_equal(o["n_collide"], (d2 <= 128 ** 2).sum(1))
    assert d2[0, 1] == (8 * 256) ** 2 and d2[2, 3] == 128 ** 2   # both exactly on a threshold
    assert o["n_collide"][2] >= 1


def test_periodic_translation_invariance():
    # Torus (A9): translating every position by the same vector (mod L) changes nothing an
    # agent senses.  On a 2^-8 lattice the translated coordinates are exact, so every output
    # is identical, including pairs that now wrap across the seam and pairs exactly on
    # the thresholds.
    p = vi.flock_params(600, width=128.0, d_v=8.0)
    rng = np.random.default_rng(12)
    q = rng.integers(0, 128 * 256, size=(600, 2))
    q[1] = q[0] + [8 * 256, 0]                            # on the radius
    q[3] = q[2] + [0, 128]                                # on the contact distance
    q %= 128 * 256
    st = np.zeros((1, 600, 4))
    st[0, :, 2] = rng.integers(0, 6 * 256, 600) / 256.0   # headings on the lattice too
    st[0, :, 3] = 0.275
    outs = []
    for shift in ([0, 0], [64 * 256 + 17, 3 * 256 + 5], [127 * 256, 100 * 256 + 255]):
        st[0, :, :2] = ((q + np.array(shift)) % (128 * 256)) / 256.0
        outs.append(sense_all(p, st))
    for o in outs[1:]:
        for k in ("n_neigh", "n_collide", "sector_occ"):
            assert np.array_equal(o[k], outs[0][k]), k
        assert np.array_equal(o["obs"], outs[0]["obs"])
        assert np.allclose(o["reward"], outs[0]["reward"], rtol=0, atol=1e-12)


def _rot90(p, st):
    x, y, th = st[0, :, 0], st[0, :, 1], st[0, :, 2]
    out = st.copy()
    out[0, :, 0] = np.mod(p.width - y, p.width)
    out[0, :, 1] = x
    out[0, :, 2] = np.mod(th + math.pi / 2, 2 * math.pi)
    return out


def _unbanded_rows(o):
    return np.array([len(b) == 0 for b in o["bands"]])


def test_rotation_equivariance():
    # rotating positions and headings by 90 deg leaves every agent's view unchanged.
    p = vi.flock_params(800)
    st = vi.init_state(p, seed=3).astype(np.float64)
    o1, o2 = sense_all(p, st), sense_all(p, _rot90(p, st))
    ok = _unbanded_rows(o1) & _unbanded_rows(o2)
    assert ok.mean() > 0.9
    assert np.allclose(o1["obs"][ok], o2["obs"][ok], rtol=1e-9, atol=0)
    assert np.array_equal(o1["n_neigh"], o2["n_neigh"])
    assert np.allclose(o1["reward"], o2["reward"], rtol=1e-9, atol=1e-12)


def test_mirror_reverses_sectors():
    # Mirror (x, y, th) -> (x, L - y, -th): bearing phi -> -phi, sector k -> v-1-k.
    p = vi.flock_params(800)
    st = vi.init_state(p, seed=8).astype(np.float64)
    m = st.copy()
    m[0, :, 1] = np.mod(p.width - st[0, :, 1], p.width)
    m[0, :, 2] = np.mod(-st[0, :, 2], 2 * math.pi)
    o1, o2 = sense_all(p, st), sense_all(p, m)
    ok = _unbanded_rows(o1) & _unbanded_rows(o2)
    assert np.allclose(o1["obs"][ok, :128], o2["obs"][ok, 127::-1], rtol=1e-9, atol=0)


def test_closed_form_expectations_c2():
    # SURVEY §8d sanity table at C2 density (iid uniform positions on the torus):
    # E[n_neigh] = (N-1) pi d_v^2 / L^2 = 157.05, E[n_collide] = (N-1) pi (2 d_r)^2 / L^2,
    # E[reward] = (N-1)/L^2 * integral_0^{d_v} f(d) 2 pi d dd = 38.77,
    # P(sector occupied) = 1 - (1 - (fov/v) d_v^2 / (2 L^2))^(N-1) = 0.5735.
    from scipy.integrate import quad
    p = vi.workload("c2")
    st = vi.init_state(p, seed=0).astype(np.float64)
    o = sense_all(p, st)
    n, L2 = p.n_agents, p.width ** 2
    integral = quad(lambda d: oracle.reward_f(p, d, d <= 2 * p.d_r) * 2 * math.pi * d,
                    0, p.d_v, points=[0.5, 5.25], limit=200)[0]
    assert integral == pytest.approx(77.558, abs=2e-3)
    assert o["n_neigh"].mean() == pytest.approx((n - 1) * math.pi * p.d_v ** 2 / L2, rel=0.01)
    assert o["reward"].mean() == pytest.approx((n - 1) / L2 * integral, rel=0.03)
    assert o["n_collide"].mean() == pytest.approx((n - 1) * math.pi * 0.25 / L2, rel=0.15)
    occ = np.unpackbits(o["sector_occ"].view(np.uint8), bitorder="little").mean()
    pocc = 1 - (1 - (p.fov / p.v) * p.d_v ** 2 / (2 * L2)) ** (n - 1)
    assert pocc == pytest.approx(0.5735, abs=1e-3)
    assert occ == pytest.approx(pocc, abs=0.01)


# ------------------------------------------------------------------------------- tag
def test_tag_coincident_touch():
    # S:286 "runner and chaser coincident -> chaser +r_touch, runner -r_touch"
    p, st = world(vi.tag_params(2, n_chasers=1), [[50, 50, 0, 0], [50, 50, 1, 0]])
    o = sense_all(p, st)
    assert o["reward"][0] == pytest.approx(-1.0) and o["reward"][1] == pytest.approx(1.0)
    assert list(o["n_touch"]) == [1, 1] and list(o["n_collide"]) == [0, 0]
    # d = 0: phi = atan2(0, 0) = 0 -> dead ahead, sector v/2 = 32 of the other type's channel
    assert o["obs"][0, 64 + 32] == 0.0 and np.sum(o["obs"][0] < 1) == 1
    assert o["obs"][1, 32] == 0.0 and np.sum(o["obs"][1] < 1) == 1


def test_tag_far_apart_and_isolated():
    # S:277 far apart -> other-type channel all ones; S:287 all isolated -> all rewards 0
    p, st = world(vi.tag_params(2, n_chasers=1), [[10, 10, 0, 0], [60, 60, 1, 0]])
    o = sense_all(p, st)
    assert np.all(o["obs"] == 1.0) and np.all(o["reward"] == 0)


def test_tag_runner_proximity_only_from_runners():
    p = vi.tag_params(3, n_chasers=1)
    p, st = world(p, [[50, 50, 0, 0], [55.25, 50, 0, 0], [50, 55.25, 0, 0]])
    o = sense_all(p, st)
    # runners 0 and 1 at 5.25 (f = 0.5, weight 0.1); chaser 2 gives no proximity reward;
    # runners 0-1 ... agent 1 to chaser distance = sqrt(2)*5.25 > 7: no touch.
    assert o["reward"][0] == pytest.approx(p.w_prox * 0.5, rel=1e-7)
    assert o["reward"][1] == pytest.approx(p.w_prox * 0.5, rel=1e-7)
    assert o["reward"][2] == 0.0
    # channels: runner 0 sees runner 1 (ch 0, dead ahead k=32) and chaser 2 (ch 1, +90 deg)
    u = (90 * DEG + p.fov / 2) / p.fov
    assert o["obs"][0, 32] == pytest.approx(0.525) and o["obs"][0, 64 + int(u * 64)] == pytest.approx(0.525)


def test_tag_channel_separation_and_zero_sum():
    # S:279 delete-and-recompute: runners' channel 0 is unaffected by deleting all chasers;
    # S:303 zero-sum touches at w = 0.
    p = vi.tag_params(600, n_chasers=60, width=40.0, d_v=4.0, w_prox=0.0)
    st = vi.init_state(p, seed=2).astype(np.float64)
    o = sense_all(p, st)
    q = p.replace(n_agents=540, n_chasers=0)
    o2 = oracle.sense_rows(q, st[0, :540], np.arange(540))
    assert np.array_equal(o["obs"][:540, :64], o2["obs"][:, :64])
    assert np.all(o2["obs"][:, 64:] == 1.0)
    chaser = np.arange(600) >= 540
    assert o["reward"][chaser].sum() == pytest.approx(-o["reward"][~chaser].sum())
    assert o["n_touch"][chaser].sum() == o["n_touch"][~chaser].sum() > 0
