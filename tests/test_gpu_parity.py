"""GPU parity: the CUDA path (through the C ABI, via the ctypes binding) against the fp64
oracle on the same seeded inputs, one step at a time (SURVEY.md §8c protocol): the oracle
integrates the GPU's fp32 state of step t and senses the GPU's fp32 state of step t+1, so
fp32/fp64 drift never compounds."""
import math

import numpy as np
import pytest

import oracle
import vg_inputs as vi
import vg_parity as parity

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def dev(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def outs_np(out, r):
    d = {}
    for k in ("obs", "reward", "n_neigh", "n_collide", "n_touch", "sector_occ"):
        t = getattr(out, k)
        if t is not None:
            a = host(t[r])
            d[k] = a.view(np.uint32) if a.dtype == np.int32 else a
    return d


def make_world(p):
    import paper_2207_03945_b200 as vg
    return vg.World(p)


def _workers():
    import os
    return max(1, min(32, len(os.sched_getaffinity(0))))


def run_and_check(p, state0, n_steps, replicas=None, rows=None, seed=0, check_bins=True,
                  workers=1):
    """Step the GPU world n_steps with seeded actions; check every step against the oracle."""
    torch = _torch()
    w = make_world(p)
    out = w.alloc_outputs()
    st = dev(state0)
    stats = []
    reps = range(p.n_replicas) if replicas is None else replicas
    for t in range(n_steps):
        prev = host(st)
        act = vi.actions(p, seed=seed, step=t)
        w.step(st, dev(act), out)
        torch.cuda.synchronize()
        assert w.sync_errors() == -1
        cur = host(st)
        ref_state = oracle.integrate(p, prev, act)
        parity.check_integrate(p, cur, ref_state)
        if check_bins:
            bins = {k: host(v) for k, v in w.get_bins().items()}
            parity.check_bins(p, bins, cur)
        for r in reps:
            stats.append(parity.check_sense(p, cur[r], outs_np(out, r), rows=rows,
                                            workers=workers))
    w.close()
    return stats


def test_c1_100_steps(cuda):
    # configs[0]: flock, 100 agents, 100 steps with seeded random actions — every row, step.
    p = vi.workload("c1")
    stats = run_and_check(p, vi.init_state(p, seed=0), 100)
    assert sum(s["rows"] for s in stats) == 100 * 100


def test_c2_flock_5000(cuda):
    # configs[1], every row, 10 steps (SURVEY.md §8c parity depth)
    p = vi.workload("c2")
    stats = run_and_check(p, vi.init_state(p, seed=0), 10, workers=_workers())
    assert sum(s["rows"] for s in stats) == 10 * p.n_agents
    print(stats[-1])


def test_c3_tag_10000(cuda):
    # configs[2] (tag, 9,000 runners + 1,000 chasers), every row, 10 steps
    p = vi.workload("c3")
    stats = run_and_check(p, vi.init_state(p, seed=0), 10, workers=_workers())
    assert sum(s["rows"] for s in stats) == 10 * p.n_agents
    print(stats[-1])


def test_c4_full_size_sampled_replicas(cuda):
    # configs[3] at its full size (the bench launch configuration), replicas {0,1,511,1023},
    # every row of each, 3 steps.
    p = vi.workload("c4")
    st0 = vi.init_state(p, seed=0)
    run_and_check(p, st0, 3, replicas=[0, 1, 511, 1023], workers=_workers())


def test_64bit_output_indexing(cuda):
    # 3,500 replicas x 5,000 agents: rows x obs_dim > 2^31, so K4 takes its NULL-checked
    # 64-bit-index path; first, middle and last replicas against the oracle.
    p = vi.workload("c4").replace(n_replicas=3500)
    assert p.total_agents * 130 > 2 ** 31
    run_and_check(p, vi.init_state(p, seed=5), 1, replicas=[0, 1750, 3499], check_bins=False)


def test_c5_full_size_sampled_rows(cuda):
    # configs[4]: 1M-agent world in the bench's launch configuration, 3 steps; each step:
    # integrate and bins bit-exact in full, sensing on 4,096 sampled rows against all N
    # (SURVEY.md §8c), plus size-independent properties (sum rule, closed-form expectations).
    torch = _torch()
    p = vi.workload("c5")
    w = make_world(p)
    out = w.alloc_outputs()
    st = dev(vi.init_state(p, seed=0))
    for t in range(3):
        prev = host(st)
        act = vi.actions(p, seed=0, step=t)
        w.step(st, dev(act), out)
        torch.cuda.synchronize()
        assert w.sync_errors() == -1
        cur = host(st)
        parity.check_integrate(p, cur, oracle.integrate(p, prev, act))
        parity.check_bins(p, {k: host(v) for k, v in w.get_bins().items()}, cur)
        rows = np.random.default_rng(1 + t).choice(p.n_agents, 4096, replace=False)
        s = parity.check_sense(p, cur[0], outs_np(out, 0), rows=rows, workers=_workers())
        print(t, s)
    nn = host(out.n_neigh).astype(np.int64)
    assert nn.sum() % 2 == 0
    e = (p.n_agents - 1) * math.pi * p.d_v ** 2 / p.width ** 2
    assert nn.mean() == pytest.approx(e, rel=5e-3)
    occ = np.unpackbits(host(out.sector_occ).view(np.uint8), bitorder="little").mean()
    pocc = 1 - (1 - (p.fov / p.v) * p.d_v ** 2 / (2 * p.width ** 2)) ** (p.n_agents - 1)
    assert occ == pytest.approx(pocc, abs=3e-3)
    w.close()


@pytest.mark.parametrize("fov,v", [(2 * math.pi, 128), (0.5, 128), (1.0, 7), (4.36, 64),
                                   (4.36, 1), (2 * math.pi, 1)])
def test_sector_model_variants(cuda, fov, v):
    # fov = 2 pi (the seam at phi = pi), narrow sectors (atan2 path: sector-table bins would
    # hold two boundaries), few wide sectors, tag-like v = 64: every sector decision agrees
    # with the oracle up to the bands.
    p = vi.flock_params(2500, width=70.0, d_v=7.0, fov=np.float32(fov), v=v)
    run_and_check(p, vi.init_state(p, seed=11), 2)


def test_default_constants_path(cuda):
    # K4's sector pass has an instance with the paper's default constants compiled in; the
    # benchmark worlds must take it (their derived fp32 constants are bitwise the compiled
    # ones) and any other parameter set must not.  Parity of both instances is covered by
    # the tests above (defaults: c1-c5, edge cases; generic: sector variants, d_v = 3, ...).
    for p in [vi.workload(n) for n in ("c1", "c2", "c3", "c4", "c5")] + \
            [vi.workload("c2").replace(vision="ray"), vi.workload("c3").replace(vision="ray")]:
        w = make_world(p)
        assert w.sense_defaults, p
        w.close()
    for p in (vi.flock_params(2000, v=64), vi.flock_params(2000, d_v=12.0),
              vi.tag_params(2000, w_prox=0.2),
              vi.flock_params(2000, d_r=0.3).replace(vision="ray")):
        w = make_world(p)
        assert not w.sense_defaults, p
        w.close()


@pytest.mark.parametrize("name,vision", [("c2", "sector"), ("c3", "sector"), ("c2", "ray"),
                                         ("c3", "ray")])
def test_default_constants_bitwise_generic(cuda, name, vision, monkeypatch):
    # The default-constant instance and the generic one (VG_SENSE_GENERIC=1) must give
    # bitwise-identical outputs on the same state: the constants are the same fp32 values.
    torch = _torch()
    p = vi.workload(name).replace(vision=vision)
    st = dev(vi.init_state(p, seed=23))
    res = []
    for gen in ("0", "1"):
        monkeypatch.setenv("VG_SENSE_GENERIC", gen)
        w = make_world(p)
        assert w.sense_defaults == (gen == "0")
        out = w.alloc_outputs()
        w.bin(st)
        w.sense(out)
        torch.cuda.synchronize()
        res.append({k: host(getattr(out, k)).copy() for k in
                    ("obs", "reward", "n_neigh", "n_collide", "n_touch", "sector_occ")
                    if getattr(out, k) is not None})
        w.close()
    for k in res[0]:
        assert np.array_equal(res[0][k].view(np.uint8), res[1][k].view(np.uint8)), k


@pytest.mark.parametrize("case", ["gather_replicas", "gather_tag_replicas", "cta_sort",
                                  "warp_sort", "gather_tag_dense", "cta_sort_dense",
                                  "fused_replicas", "staged_replicas", "staged_tag_replicas"])
def test_binning_paths(cuda, case):
    # Each K2-K3b variant against the oracle's bins (bit-exact) and sense outputs:
    # K3g (per-cell gather, several replicas), K3b' (one CTA per cell: few cells, N above
    # K3g's limit) and K3b (one warp per cell: many cells).  kernels_per_step names the path.
    rows = None
    if case == "gather_replicas":
        p, kps = vi.flock_params(3000, n_replicas=4), 3
    elif case == "gather_tag_replicas":
        p, kps = vi.tag_params(2000, n_replicas=3), 3
    elif case == "cta_sort":
        p, kps = vi.flock_params(20000), 5
        rows = np.arange(0, 20000, 41)
    elif case == "warp_sort":
        p, kps = vi.flock_params(20000, width=400.0, d_v=10.0), 5
        rows = np.arange(0, 20000, 41)
    elif case == "gather_tag_dense":         # cells above 1,024 members: K3g's fallback
        p, kps = vi.tag_params(4000), 3
        rows = np.arange(0, 4000, 7)
    elif case == "cta_sort_dense":           # N > 16,384 with dense cells: K3b''s fallback
        p, kps = vi.flock_params(17000), 5
        rows = np.arange(0, 17000, 53)
    elif case == "fused_replicas":           # K1-K3b fused, one CTA per replica (< n_sm replicas)
        p, kps = vi.flock_params(2500, n_replicas=100), 2
    else:                                    # the persistent TMA-staged fused bin (>= n_sm replicas)
        mk = vi.flock_params if case == "staged_replicas" else vi.tag_params
        p, kps = mk(1500, n_replicas=300), 2
    st0 = vi.clustered_state(p, seed=5, n_clusters=3, sigma=1.5) if case.endswith("dense") \
        else vi.init_state(p, seed=17)
    w = make_world(p)
    assert w.kernels_per_step == kps
    if case.endswith("dense"):
        w.bin(dev(st0))
        cs = host(w.get_bins()["cell_start"]).astype(np.int64)
        assert np.diff(cs).max() > 1024                  # the fallback path really runs
    w.close()
    reps = [0, 1, p.n_replicas // 2, p.n_replicas - 1] if p.n_replicas > 4 else None
    run_and_check(p, st0, 2, rows=rows, replicas=reps)


def test_staged_fused_bin_equals_per_replica_kernel(cuda, monkeypatch):
    # the persistent staged fused bins (MODE 1: one 1024-thread CTA per SM with TMA input;
    # MODE 2: two 512-thread CTAs per SM) and the one-CTA-per-replica kernel (VG_RB_STAGED=0):
    # bitwise the same bins and outputs on a c4-shaped world
    torch = _torch()
    p = vi.workload("c4").replace(n_replicas=400)
    st0 = vi.init_state(p, seed=8)
    act = vi.actions(p, seed=8, step=0)
    res = []
    for staged in ("1", "2", "0"):
        monkeypatch.setenv("VG_RB_STAGED", staged)
        w = make_world(p)
        out = w.alloc_outputs()
        st = dev(st0)
        w.step(st, dev(act), out)
        torch.cuda.synchronize()
        assert w.sync_errors() == -1
        bins = {k: host(v).copy() for k, v in w.get_bins().items()}
        res.append((host(st), bins, {k: host(getattr(out, k)) for k in ("obs", "reward", "n_neigh")}))
        w.close()
    for other in res[1:]:
        assert np.array_equal(res[0][0].view(np.uint32), other[0].view(np.uint32))
        for k in res[0][1]:
            assert np.array_equal(res[0][1][k].view(np.uint8), other[1][k].view(np.uint8)), k
        for k in res[0][2]:
            assert np.array_equal(res[0][2][k].view(np.uint8), other[2][k].view(np.uint8)), k


@pytest.mark.parametrize("grid", [9, 0])
def test_large_cells_small_radius(cuda, grid):
    # d_v = 3 in cells of 11.1 (grid 9: a run is ~11 radii long, the windows cut most of it)
    # and the auto grid (G = 33); sub-bin windows and chord narrowing at other ratios.
    p = vi.flock_params(4000, width=100.0, d_v=3.0, grid=grid)
    run_and_check(p, vi.init_state(p, seed=13), 2)


def test_long_run_stability(cuda):
    # 300 steps of the 10^6-agent world through the cached graph with fresh random actions
    # each step: no device error, state stays in its domain, and the last step still
    # matches the oracle on sampled rows (no slow corruption, no rare race).
    torch = _torch()
    p = vi.workload("c5")
    w = make_world(p)
    out = w.alloc_outputs()
    st = dev(vi.init_state(p, seed=4))
    g = torch.Generator(device="cuda").manual_seed(7)
    lo = torch.tensor([-0.1, -0.2], device="cuda")
    for t in range(300):
        a = (torch.rand((1, p.n_agents, 2), device="cuda", generator=g) * 2 - 1) * -lo
        w.step(st, a, out)
    torch.cuda.synchronize()
    assert w.sync_errors() == -1
    cur = host(st)
    assert (cur[0, :, :2] >= 0).all() and (cur[0, :, :2] < p.width).all()
    assert (cur[0, :, 2] >= 0).all() and (cur[0, :, 2] < 2 * math.pi).all()
    assert (cur[0, :, 3] >= p.s_min).all() and (cur[0, :, 3] <= p.s_max).all()
    rows = np.random.default_rng(9).choice(p.n_agents, 64, replace=False)
    parity.check_sense(p, cur[0], outs_np(out, 0), rows=rows)
    w.close()


def test_c5_clustered_sampled_rows(cuda):
    # The stress state at full size: cells with ~2000 agents are split into many K4 work
    # items (chunk_q = 64); rows sampled from the densest cells and at random.
    torch = _torch()
    p = vi.workload("c5")
    w = make_world(p)
    out = w.alloc_outputs()
    st0 = vi.clustered_state(p, seed=2)
    w.bin(dev(st0))
    w.sense(out)
    torch.cuda.synchronize()
    bins = {k: host(v) for k, v in w.get_bins().items()}
    parity.check_bins(p, bins, st0)
    counts = np.diff(bins["cell_start"].astype(np.int64))
    dense = np.argsort(counts)[-4:]                       # the four densest cells
    rng = np.random.default_rng(3)
    rows = [int(bins["perm"][0][bins["cell_start"][c] + rng.integers(0, counts[c])])
            for c in dense for _ in range(6)]
    rows += list(rng.choice(p.n_agents, 24, replace=False))
    parity.check_sense(p, st0[0], outs_np(out, 0), rows=np.array(rows))
    assert counts.max() > 8 * 128                         # really split over many items
    w.close()


@pytest.mark.parametrize("case", ["lone", "pair", "sparse", "g3", "many_replicas",
                                  "clustered", "tag_no_chasers", "tag_all_chasers"])
def test_edge_cases(cuda, case):
    if case == "lone":
        p = vi.flock_params(1)
    elif case == "pair":
        p = vi.flock_params(2, width=30.0)
    elif case == "sparse":
        p = vi.flock_params(37, width=400.0, d_v=10.0)        # mostly empty cells
    elif case == "g3":
        p = vi.flock_params(300, width=30.1, d_v=10.0)        # G = 3, the minimum
    elif case == "many_replicas":
        p = vi.flock_params(7, n_replicas=3000, width=40.0)
    elif case == "clustered":
        p = vi.flock_params(4000)
    elif case == "tag_no_chasers":
        p = vi.tag_params(500, n_chasers=0, width=60.0)
    else:
        p = vi.tag_params(500, n_chasers=500, width=60.0)
    st0 = vi.clustered_state(p, seed=3, n_clusters=3, sigma=1.5) if case == "clustered" \
        else vi.init_state(p, seed=5)
    if case == "g3":
        assert oracle.grid_size(p) == 3
    reps = [0, 1, 2999] if case == "many_replicas" else None
    run_and_check(p, st0, 3, replicas=reps)


@pytest.mark.parametrize("env", ["flock", "tag"])
def test_coincident_agents(cuda, env):
    # Agents at exactly the same position (A13: d = 0, phi = atan2(0, 0) = 0, a contact):
    # exact duplicates, a triple, and a pair one ulp apart.  The flock sector pass keeps
    # every (dx, dy) = (+0, +0) entry out of the sector minima with the self pair and
    # restores a coincident other agent at the emit (K4 8-byte ring entries).
    torch = _torch()
    p = vi.flock_params(600, width=60.0) if env == "flock" else vi.tag_params(600, width=60.0)
    st = vi.init_state(p, seed=8)
    st[0, 10:20, :2] = st[0, 0:10, :2]
    st[0, 20:23, :2] = st[0, 30, :2]
    st[0, 40, :2] = st[0, 41, :2]
    st[0, 40, 0] = np.nextafter(st[0, 41, 0], np.float32(np.inf))
    w = make_world(p)
    out = w.alloc_outputs()
    w.bin(dev(st))
    w.sense(out)
    torch.cuda.synchronize()
    assert w.sync_errors() == -1
    parity.check_sense(p, st[0], outs_np(out, 0))
    contacts = host(out.n_collide)[0].astype(np.int64)
    if env == "tag":
        contacts += host(out.n_touch)[0]
    assert (contacts[list(range(23)) + [30]] >= 1).all()
    w.close()


def test_dyadic_world_bit_exact_thresholds(cuda):
    # On a 2^-8 lattice with L = 128 every difference and d^2 is exact in fp32 and fp64:
    # radius and contact decisions must agree exactly, even for pairs exactly on them.
    torch = _torch()
    p = vi.flock_params(400, width=128.0, d_v=8.0)
    rng = np.random.default_rng(4)
    q = rng.integers(0, 128 * 256, size=(400, 2))
    q[1] = q[0] + [8 * 256, 0]
    q[3] = q[2] + [0, 128]
    q[5] = (q[4] + [127 * 256 + 200, 0]) % (128 * 256)        # wrapped pair
    q %= 128 * 256
    st = np.zeros((1, 400, 4), np.float32)
    st[0, :, :2] = q / 256.0
    st[0, :, 2] = (rng.random(400) * 6.0).astype(np.float32)
    st[0, :, 3] = 0.275
    w = make_world(p)
    out = w.alloc_outputs()
    x = dev(st)
    w.bin(x)
    w.sense(out)
    torch.cuda.synchronize()
    ref = oracle.sense_rows(p, st[0], np.arange(400))
    assert np.array_equal(host(out.n_neigh)[0], ref["n_neigh"])
    assert np.array_equal(host(out.n_collide)[0], ref["n_collide"])
    parity.check_sense(p, st[0], outs_np(out, 0))
    w.close()


@pytest.mark.parametrize("vision", ["sector", "ray"])
def test_window_rim_neighbours(cuda, vision):
    # K4 cuts each stencil run to a candidate window: neighbours on the rim
    # of the view disc, at wrap edges and in the adjacent rows must all still be found.
    torch = _torch()
    p = vi.flock_params(3000, width=100.0, d_v=10.0, vision=vision)
    st = vi.rim_state(p, 60, seed=9, radius=p.d_v + (p.d_r if vision == "ray" else 0.0))
    w = make_world(p)
    out = w.alloc_outputs()
    w.bin(dev(st))
    w.sense(out)
    torch.cuda.synchronize()
    rows = np.arange(60 * 17)                       # the queries and their rim neighbours
    if vision == "ray":
        import test_gpu_ray as tr
        tr._check(p, outs_np(out, 0), st[0], rows)
    else:
        parity.check_sense(p, st[0], outs_np(out, 0), rows=rows)
    if vision == "sector":
        assert (host(out.n_neigh)[0][:60] >= 16).all()   # every ring member is in range
    w.close()


@pytest.mark.parametrize("env", ["flock", "tag"])
def test_periodic_translation_bitwise(cuda, env):
    # Torus (A9) on a 2^-8 lattice: translating every agent by the same vector (mod L) moves
    # agents across cells, runs and the wrap seam, but every difference stays exact — all
    # outputs must be bit-identical per agent (and match the oracle).
    torch = _torch()
    n = 6000
    p = (vi.flock_params(n, width=128.0, d_v=8.0) if env == "flock"
         else vi.tag_params(n, width=128.0, d_v=8.0))
    rng = np.random.default_rng(21)
    q = rng.integers(0, 128 * 256, size=(n, 2))
    st = np.zeros((1, n, 4), np.float32)
    st[0, :, 2] = rng.integers(0, 6 * 256, n) / 256.0
    st[0, :, 3] = 0.275 if env == "flock" else 0.0
    w = make_world(p)
    res = []
    for shift in ([0, 0], [64 * 256 + 17, 3 * 256 + 5], [127 * 256 + 255, 100 * 256 + 1]):
        st[0, :, :2] = ((q + np.array(shift)) % (128 * 256)) / 256.0
        out = w.alloc_outputs()
        w.bin(dev(st))
        w.sense(out)
        torch.cuda.synchronize()
        res.append({k: host(getattr(out, k)).copy() for k in
                    ("obs", "reward", "n_neigh", "n_collide", "n_touch", "sector_occ")
                    if getattr(out, k) is not None})
        if shift == [0, 0]:
            parity.check_sense(p, st[0].copy(), outs_np(out, 0), rows=np.arange(0, n, 7))
    for r in res[1:]:
        for k, v in r.items():
            assert np.array_equal(v.view(np.uint32), res[0][k].view(np.uint32)), k
    w.close()


def test_reward_kernel_matches_sense(cuda):
    torch = _torch()
    for p in (vi.workload("c2"), vi.tag_params(3000, width=60.0)):
        w = make_world(p)
        a, b = w.alloc_outputs(), w.alloc_outputs()
        st = dev(vi.init_state(p, seed=2))
        w.bin(st)
        w.sense(a)
        w.reward(b)
        torch.cuda.synchronize()
        for k in ("reward", "n_neigh", "n_collide", "n_touch"):
            if getattr(a, k) is not None:
                assert torch.equal(getattr(a, k), getattr(b, k)), k
        w.close()


@pytest.mark.parametrize("which", ["no_obs", "no_occ", "only_obs", "no_counts"])
def test_partial_outputs_equal_full(cuda, which):
    # K4 has a fast path when every output is present and a NULL-checked path otherwise:
    # any subset of outputs must equal the same outputs of a full run bit for bit.
    torch = _torch()
    for p in (vi.workload("c2"), vi.tag_params(3000, width=60.0)):
        w = make_world(p)
        st = dev(vi.init_state(p, seed=6))
        full = w.alloc_outputs()
        kw = {"no_obs": dict(obs=False), "no_occ": dict(sector_occ=False),
              "only_obs": dict(reward=False, counts=False, sector_occ=False),
              "no_counts": dict(counts=False)}[which]
        part = w.alloc_outputs(**kw)
        w.bin(st)
        w.sense(full)
        w.sense(part)
        torch.cuda.synchronize()
        for k in ("obs", "reward", "n_neigh", "n_collide", "n_touch", "sector_occ"):
            a, b = getattr(part, k), getattr(full, k)
            if a is not None and b is not None:
                assert torch.equal(a.view(torch.int32), b.view(torch.int32)), (which, k)
        w.close()


def test_unaligned_occupancy_rows_equal_aligned(cuda):
    # K4 writes the four occupancy words of a row as one 16-byte store when the caller's
    # tensor is 16-byte aligned, and word by word otherwise: both give the same words.
    torch = _torch()
    for p in (vi.workload("c2"), vi.tag_params(3000, width=60.0)):
        w = make_world(p)
        st = dev(vi.init_state(p, seed=6))
        full = w.alloc_outputs()
        odd = w.alloc_outputs()
        n = p.n_replicas * p.n_agents * w.occ_words
        raw = torch.empty(n + 1, dtype=torch.int32, device="cuda")
        odd.sector_occ = raw[1:].view(p.n_replicas, p.n_agents, w.occ_words)   # 4-byte offset
        assert odd.sector_occ.data_ptr() % 16 != 0
        w.bin(st)
        w.sense(full)
        w.sense(odd)
        torch.cuda.synchronize()
        for k in ("obs", "reward", "n_neigh", "n_collide", "sector_occ"):
            assert torch.equal(getattr(odd, k).view(torch.int32), getattr(full, k).view(torch.int32)), k
        w.close()


def test_integrate_then_bin_sense_equals_step(cuda):
    torch = _torch()
    p = vi.workload("c2")
    w = make_world(p)
    s1, s2 = dev(vi.init_state(p, seed=1)), dev(vi.init_state(p, seed=1))
    act = dev(vi.actions(p, seed=1, step=0))
    o1, o2 = w.alloc_outputs(), w.alloc_outputs()
    w.step(s1, act, o1)
    w.integrate(s2, act)
    w.bin(s2)
    w.sense(o2)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2)
    for k in ("obs", "reward", "n_neigh", "n_collide", "sector_occ"):
        assert torch.equal(getattr(o1, k), getattr(o2, k)), k
    w.close()


def test_determinism_bitwise(cuda):
    torch = _torch()
    p = vi.workload("c2")
    res = []
    for _ in range(2):
        w = make_world(p)
        st = dev(vi.init_state(p, seed=0))
        out = w.alloc_outputs()
        for t in range(5):
            w.step(st, dev(vi.actions(p, seed=0, step=t)), out)
        torch.cuda.synchronize()
        res.append((st.clone(), out.obs.clone(), out.reward.clone(), out.sector_occ.clone()))
        w.close()
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_step_host_matches_step(cuda):
    torch = _torch()
    p = vi.workload("c2")
    w = make_world(p)
    s1, s2 = dev(vi.init_state(p, seed=1)), dev(vi.init_state(p, seed=1))
    o1, o2 = w.alloc_outputs(), w.alloc_outputs()
    act = vi.actions(p, seed=1, step=0)
    act_h = torch.from_numpy(act).pin_memory()
    rew_h = torch.empty((1, p.n_agents), dtype=torch.float32).pin_memory()
    w.step(s1, dev(act), o1)
    w.step_host(s2, act_h, o2, rew_h)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(o1.obs, o2.obs)
    assert torch.equal(o1.reward.cpu(), rew_h)
    w.close()


def test_cuda_graph_capture(cuda):
    torch = _torch()
    p = vi.workload("c2")
    w = make_world(p)
    st = dev(vi.init_state(p, seed=0))
    ref_st = st.clone()
    act = dev(vi.actions(p, seed=0, step=0))
    out, ref = w.alloc_outputs(), w.alloc_outputs()
    w.step(ref_st, act, ref)          # eager reference
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            w.step(st, act, out)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(st, ref_st) and torch.equal(out.obs, ref.obs)
    assert torch.equal(out.reward, ref.reward)
    w.close()


def test_free_running_drift_c1(cuda):
    # Open-loop actions: positions do not depend on observations, so the oracle's own fp64
    # trajectory stays within the integrate tolerance of the fp32 GPU one for 100 steps.
    torch = _torch()
    p = vi.workload("c1")
    w = make_world(p)
    st = dev(vi.init_state(p, seed=0))
    ref = vi.init_state(p, seed=0).astype(np.float64)
    out = w.alloc_outputs()
    for t in range(100):
        act = vi.actions(p, seed=0, step=t)
        w.step(st, dev(act), out)
        ref = oracle.integrate(p, ref, act)
    torch.cuda.synchronize()
    parity.check_integrate(p, host(st), ref)
    w.close()


@pytest.mark.parametrize("what", ["nan_action", "pos_out_of_range", "bad_heading"])
def test_device_errors(cuda, what):
    import paper_2207_03945_b200 as vg
    torch = _torch()
    p = vi.workload("c2")
    w = make_world(p)
    st = vi.init_state(p, seed=0)
    act = vi.actions(p, seed=0, step=0)
    bad = 1234
    if what == "nan_action":
        act[0, bad, 1] = np.nan
    elif what == "pos_out_of_range":
        st[0, bad, 0] = p.width
    else:
        st[0, bad, 2] = -0.5
    x = dev(st)
    w.step(x, dev(act), w.alloc_outputs())
    with pytest.raises(vg.VgError) as ei:
        w.sync_errors()
    assert ei.value.bad_agent == bad and "VG_ESTATE" in str(ei.value)
    assert w.sync_errors() == -1                      # cleared
    w.close()
    torch.cuda.synchronize()


def test_out_of_box_actions_are_clamped(cuda):
    torch = _torch()
    p = vi.workload("c2")
    w = make_world(p)
    st = dev(vi.init_state(p, seed=0))
    prev = host(st)
    act = vi.actions(p, seed=0, step=0) * 25.0
    w.integrate(st, dev(act))
    torch.cuda.synchronize()
    parity.check_integrate(p, host(st), oracle.integrate(p, prev, act))
    w.close()


@pytest.mark.parametrize("env", ["flock", "tag"])
def test_sense_columns_partition_equals_sense(cuda, env):
    # vg_sense_columns over a partition of the grid columns (the replicated-state scheme,
    # DESIGN.md §7b) writes every row exactly as vg_sense does; a range writes only the rows
    # of agents binned in its columns.
    torch = _torch()
    p = (vi.flock_params(20000, width=200.0, d_v=10.0) if env == "flock"
         else vi.tag_params(20000, width=200.0, d_v=10.0))
    w = make_world(p)
    st = dev(vi.init_state(p, seed=12))
    w.bin(st)
    full = w.alloc_outputs()
    w.sense(full)
    part = w.alloc_outputs()
    for k in ("obs", "reward", "n_neigh", "n_collide", "sector_occ", "n_touch"):
        t = getattr(part, k)
        if t is not None:
            t.view(torch.int32).fill_(-7)
    G = w.grid
    cuts = [0, 5, 11, G]
    w.sense_columns(part, cuts[0], cuts[1])
    torch.cuda.synchronize()
    cx = np.floor(host(st)[0, :, 0].astype(np.float32) * np.float32(np.float32(G) / np.float32(p.width)))
    first = np.minimum(cx, G - 1) < cuts[1]
    got = host(part.n_neigh)[0].view(np.int32)
    assert np.all(got[~first] == -7) and np.all(got[first] != -7)
    for a, b in zip(cuts[1:-1], cuts[2:]):
        w.sense_columns(part, a, b)
    torch.cuda.synchronize()
    for k in ("obs", "reward", "n_neigh", "n_collide", "sector_occ", "n_touch"):
        if getattr(full, k) is not None:
            assert torch.equal(getattr(part, k).view(torch.int32), getattr(full, k).view(torch.int32)), k
    w.close()
