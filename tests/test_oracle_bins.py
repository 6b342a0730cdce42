"""Pins for oracle.grid_size / cell_ids / bins (a2) — SPEC examples, textbook sort, no GPU."""

import numpy as np

import oracle
import vg_inputs as vi


def test_grid_size_readings():
    # A16: largest G with L/G >= d_v (1 + 2^-12): 9 at L=100, d_v=10 (not 10); 141 at
    # C5's L = 1414.2136, which the C5 workload overrides with G = 136 (8 | G).
    assert oracle.grid_size(vi.flock_params(10)) == 9
    assert oracle.grid_size(vi.workload("c5").replace(grid=0)) == 141
    assert oracle.grid_size(vi.workload("c5")) == 136
    p = vi.flock_params(10, width=128.0, d_v=8.0)
    assert oracle.grid_size(p) == 15
    p = vi.flock_params(10)
    assert p.width / 9 >= p.d_v * (1 + 2 ** -12) > p.width / 10
    p = vi.workload("c5")
    assert p.width / 136 >= p.d_v * (1 + 2 ** -12) > p.width / 142


def test_single_agent_cell():
    # S:61 "1 agent at (0,0), cell_size=10, world 100x100 -> single cell (0,0)=[0]"
    p = vi.flock_params(1, d_v=9.0, grid=10)
    st = np.array([[[0, 0, 0, 0.275]]], np.float32)
    b = oracle.bins(p, st)
    assert b["cell_id"][0, 0] == 0
    assert list(b["perm"][0]) == [0]
    assert b["cell_start"][0] == 0 and b["cell_start"][1] == 1 and b["cell_start"][-1] == 1


def test_two_agents_cells():
    # S:62 "agents at (1,1) and (11,1), cell_size=10 -> cells (0,0)=[0], (1,0)=[1]"
    p = vi.flock_params(2, d_v=9.0, grid=10)
    st = np.array([[[1, 1, 0, 0.275], [11, 1, 0, 0.275]]], np.float32)
    b = oracle.bins(p, st)
    assert list(b["cell_id"][0]) == [0, 1]          # (cx, cy) = (0,0), (1,0) -> cy*G + cx
    # and with cy: (1, 11) -> cell (0,1) = 10
    st2 = np.array([[[1, 11, 0, 0.275]]], np.float32)
    assert oracle.bins(p.replace(n_agents=1), st2)["cell_id"][0, 0] == 10


def test_bins_are_a_stable_permutation():
    # S:63 "union of all cell lists is a permutation"; S:44 exactly one cell; S:46 ascending.
    p = vi.flock_params(2000, n_replicas=3)
    st = vi.init_state(p, seed=5)
    b = oracle.bins(p, st)
    g = oracle.grid_size(p)
    cs = b["cell_start"].astype(np.int64)
    assert cs[0] == 0 and cs[-1] == p.total_agents
    assert np.all(np.diff(cs) >= 0)
    for r in range(3):
        perm = b["perm"][r].astype(np.int64)
        assert sorted(perm.tolist()) == list(range(p.n_agents))
        cid = b["cell_id"][r].astype(np.int64)
        for c in range(g * g):
            lo, hi = cs[r * g * g + c] - r * p.n_agents, cs[r * g * g + c + 1] - r * p.n_agents
            members = perm[lo:hi]
            assert np.all(cid[members] == c)
            assert np.all(np.diff(members) > 0)
        assert np.array_equal(b["sorted"][r], st[r][perm])


def test_fp32_cell_formula_vs_exact_floor():
    # A16 cross-check: RN32(x * RN32(G/L)) differs from exact floor(x G / L) only within
    # a 1e-6 G band of a cell edge.
    p = vi.workload("c5").replace(n_agents=200000)
    st = vi.init_state(p, seed=2)
    g = oracle.grid_size(p)
    cid = oracle.bins(p, st)["cell_id"][0].astype(np.int64)
    x = st[0, :, 0].astype(np.float64)
    y = st[0, :, 1].astype(np.float64)
    ex = np.minimum(np.floor(x * g / p.width), g - 1) + g * np.minimum(np.floor(y * g / p.width), g - 1)
    bad = np.nonzero(ex != cid)[0]
    for i in bad:
        fx, fy = x[i] * g / p.width, y[i] * g / p.width
        near = min(abs(fx - round(fx)), abs(fy - round(fy)))
        assert near <= 1e-6 * g


def test_neighbours_lie_in_3x3_stencil():
    # Cell size >= d_v: every pair with d < d_v is within one cell (mod G).
    for p in [vi.flock_params(3000), vi.workload("c5").replace(n_agents=300000)]:
        st = vi.init_state(p, seed=9)[0]
        g = oracle.grid_size(p)
        cid = oracle.cell_ids(p, st[None])[0].astype(np.int64)
        cx, cy = cid % g, cid // g
        from scipy.spatial import cKDTree
        pairs = cKDTree(st[:, :2].astype(np.float64), boxsize=p.width).query_pairs(
            p.d_v, output_type="ndarray")
        ddx = np.abs(cx[pairs[:, 0]] - cx[pairs[:, 1]])
        ddy = np.abs(cy[pairs[:, 0]] - cy[pairs[:, 1]])
        assert np.all((ddx <= 1) | (ddx == g - 1))
        assert np.all((ddy <= 1) | (ddy == g - 1))


def test_tag_sorted_type_column():
    p = vi.tag_params(50, n_chasers=5)
    st = vi.init_state(p, seed=1)
    b = oracle.bins(p, st)
    assert np.array_equal(b["sorted"][0, :, 3], (b["perm"][0] >= 45).astype(np.float32))
