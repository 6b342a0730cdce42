"""GPU parity of K8 (GAE, NEXT #3) and K9 (opinion dynamics, NEXT #4) vs the oracles.

GAE tolerance (derived): the kernel evaluates delta with 2 roundings and the recursion with
one fused multiply-add per step, so |dA_k| <= 2^-22 (t - k + 3) S_k with
S_k = sum_l (gamma lambda)^l (|r| + gamma |V'| + |V|)_{k+l}.
Opinion tolerance: each edge update rounds 3 times on values in [0, 1]: 2^-22 (deg + 1);
an edge whose |d - threshold| <= 1e-6 may take either decision (band, as for the env)."""
import numpy as np
import pytest

import vg_inputs as vi
from oracle.gae import gae as gae_ref
from oracle import opinion as opo

pytestmark = pytest.mark.gpu


def _gae_check(n, t, g, l, seed):
    import torch
    from paper_2207_03945_b200 import rl
    rng = np.random.default_rng(seed)
    r = rng.normal(size=(t, n)).astype(np.float32)
    v = rng.normal(size=(t + 1, n)).astype(np.float32)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    adv = torch.empty((t, n), device="cuda")
    ret = torch.empty((t, n), device="cuda")
    rl.gae(dev(r), dev(v), adv, ret, g, l)
    torch.cuda.synchronize()
    cols = np.arange(n) if n <= 4096 else rng.choice(n, 2048, replace=False)
    # the kernel uses fp32 gamma and gl = RN32(gamma * lambda); the oracle gets the same values
    gl = float(np.float32(np.float32(g) * np.float32(l)))
    g32 = float(np.float32(g))
    ref = gae_ref(r[:, cols], v[:, cols], g32, gl / g32 if g32 else 0.0)
    a = np.abs(r[:, cols]).astype(np.float64) + float(np.float32(g)) * np.abs(v[1:, cols]) + np.abs(v[:-1, cols])
    S = np.zeros_like(a)
    acc = np.zeros(len(cols))
    for k in range(t - 1, -1, -1):
        acc = a[k] + gl * acc
        S[k] = acc
    tol = 2.0 ** -22 * (t - np.arange(t)[:, None] + 3) * S
    da = np.abs(adv.cpu().numpy()[:, cols] - ref["adv"])
    dr = np.abs(ret.cpu().numpy()[:, cols] - ref["ret"])
    assert np.all(da <= tol), da.max()
    assert np.all(dr <= tol + 2.0 ** -23 * np.abs(v[:-1, cols])), dr.max()


@pytest.mark.parametrize("n,t", [(1, 1), (1000, 128), (257, 7), (3000, 33)])
def test_gae_parity(cuda, n, t):
    _gae_check(n, t, 0.99, 0.95, n + t)


def test_gae_full_size(cuda):
    # bench size: 10^6 agents x 128 steps, sampled agents against the oracle
    _gae_check(1_000_000, 128, 0.99, 0.95, 7)


def test_gae_edge_params(cuda):
    _gae_check(500, 20, 1.0, 1.0, 1)
    _gae_check(500, 20, 0.9, 0.0, 2)


def _opinion_check(g, thr, strength, rows=None):
    import torch
    from paper_2207_03945_b200 import rl
    d = {k: torch.from_numpy(v).cuda() for k, v in g.items()}
    out = torch.empty_like(d["op"])
    rl.opinion_step(d["row_ptr"], d["col"], d["weight"], d["op"], out, thr, strength)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    n = len(g["op"])
    rows = np.arange(n) if rows is None else rows
    ref, bands = opo.step(g["row_ptr"], g["col"], g["weight"], g["op"], float(np.float32(thr)),
                          float(np.float32(strength)), rows=rows)
    deg = (g["row_ptr"][rows + 1] - g["row_ptr"][rows]).astype(np.float64)
    tol = 2.0 ** -22 * (deg + 1)
    bad = np.nonzero(np.abs(got[rows] - ref) > tol)[0]
    for b in bad:                                  # a banded edge may take either decision
        ok = False
        for e in bands[b]:
            for alt in (True, False):
                r2, _ = opo.step(g["row_ptr"], g["col"], g["weight"], g["op"],
                                 float(np.float32(thr)), float(np.float32(strength)),
                                 rows=[rows[b]], overrides={e: alt})
                ok |= abs(got[rows[b]] - r2[0]) <= tol[b]
        assert ok, (rows[b], got[rows[b]], ref[b])
    return len(bad)


@pytest.mark.parametrize("n,deg", [(1, 0), (2, 1), (3000, 16), (500, 64)])
def test_opinion_parity(cuda, n, deg):
    g = vi.opinion_graph(n, deg, seed=n)
    _opinion_check(g, 0.3, 0.5)


def test_opinion_full_size_sampled(cuda):
    g = vi.opinion_graph_fast(1_000_000, 16, seed=1)
    rows = np.random.default_rng(0).choice(1_000_000, 3000, replace=False)
    _opinion_check(g, 0.3, 0.5, rows)


def test_opinion_consensus_dynamics(cuda):
    # complete graph, threshold 1 -> spread shrinks to consensus on the GPU too
    import torch
    from paper_2207_03945_b200 import rl
    n = 32
    col = np.array([j for i in range(n) for j in range(n) if j != i], np.int32)
    rp = (np.arange(n + 1) * (n - 1)).astype(np.int32)
    w = np.full(len(col), 0.3, np.float32)
    op = torch.from_numpy(np.random.default_rng(3).random(n).astype(np.float32)).cuda()
    t = {k: torch.from_numpy(v).cuda() for k, v in (("rp", rp), ("col", col), ("w", w))}
    nxt = torch.empty_like(op)
    spread = float(op.max() - op.min())
    for _ in range(100):
        rl.opinion_step(t["rp"], t["col"], t["w"], op, nxt, 1.0, 0.5)
        op, nxt = nxt, op
        s = float(op.max() - op.min())
        assert s <= spread
        spread = s
    assert spread < 1e-5


@pytest.mark.parametrize("bad", ["dangling_col", "negative_col", "row_ptr_decreasing",
                                 "row_ptr_past_end"])
def test_opinion_invalid_graph_raises(cuda, bad):
    # a dangling index is an invariant violation -> VG_ESTATE naming the node; the
    # invalid edge is never read (no out-of-bounds access), valid nodes are still updated.
    import torch
    from paper_2207_03945_b200 import rl
    from paper_2207_03945_b200._lib import VgError
    g = vi.opinion_graph(64, 4, seed=2)
    rp, col = g["row_ptr"].copy(), g["col"].copy()
    if bad == "dangling_col":
        col[int(rp[10])] = 64
    elif bad == "negative_col":
        col[int(rp[10])] = -5
    elif bad == "row_ptr_decreasing":
        rp[11] = rp[10] - 1
    else:
        rp[11] = len(col) + 7
        rp[12:] = len(col) + 7
    d = {k: torch.from_numpy(v).cuda() for k, v in
         (("rp", rp), ("col", col), ("w", g["weight"]), ("op", g["op"]))}
    nxt = torch.empty_like(d["op"])
    with pytest.raises(VgError, match="VG_ESTATE.*node 10"):
        rl.opinion_step(d["rp"], d["col"], d["w"], d["op"], nxt, 0.3, 0.5)
    # the record is cleared: a valid graph afterwards passes
    v = {k: torch.from_numpy(x).cuda() for k, x in
         (("rp", g["row_ptr"]), ("col", g["col"]), ("w", g["weight"]))}
    rl.opinion_step(v["rp"], v["col"], v["w"], d["op"], nxt, 0.3, 0.5)
