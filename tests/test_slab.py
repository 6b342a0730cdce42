"""Slab mode (one world split over P ranks by x-slabs).

CPU (gloo, world_size 2 and 3): the host-side plan and the message exchange pairing —
the same exchange_dist code that runs over NCCL on a GPU box.
GPU (-m gpu): P slab worlds in one process (loopback exchange) must give results bitwise
identical, per agent id, to the single-world path — the P-invariance test.
"""
import os
import socket

import numpy as np
import pytest

import vg_inputs as vi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, nbytes, q):
    import torch
    import torch.distributed as dist
    from paper_2207_03945_b200 import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G = 4 * world
        pl = slab.plan(G, world, rank)
        plans = [None] * world
        dist.all_gather_object(plans, pl)
        msgs = {k: torch.zeros(nbytes, dtype=torch.uint8) for k in
                ("send_left", "send_right", "recv_left", "recv_right")}
        msgs["send_left"].fill_(10 * rank + 1)
        msgs["send_right"].fill_(10 * rank + 2)
        slab.exchange_dist(msgs, pl["left"], pl["right"])
        q.put((rank, plans, int(msgs["recv_left"][0]), int(msgs["recv_right"][0]),
               bool((msgs["recv_left"] == msgs["recv_left"][0]).all()),
               bool((msgs["recv_right"] == msgs["recv_right"][0]).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_pairing(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, 4096, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    G = 4 * world
    for rank, plans, got_l, got_r, uni_l, uni_r in res:
        # columns partition [0, G) and neighbours are symmetric
        cols = sorted(c for pl in plans for c in range(pl["lo"], pl["hi"]))
        assert cols == list(range(G))
        me = plans[rank]
        assert plans[me["left"]]["right"] == rank and plans[me["right"]]["left"] == rank
        # recv_left holds the left rank's send_right; recv_right the right rank's send_left
        assert got_l == 10 * me["left"] + 2 and got_r == 10 * me["right"] + 1
        assert uni_l and uni_r


def test_plan_validation():
    from paper_2207_03945_b200 import slab, VgError
    assert slab.plan(136, 8, 7) == {"lo": 119, "hi": 136, "left": 6, "right": 0}
    with pytest.raises(VgError):
        slab.plan(136, 5, 0)          # 5 does not divide 136
    with pytest.raises(VgError):
        slab.plan(8, 8, 0)            # < 2 columns per rank


def test_slab_config_validation():
    import ctypes
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import _lib
    p = vi.workload("c5")
    for kw, needle in [({"rank": 0, "world_size": 1}, "world_size"),
                       ({"rank": 3, "world_size": 3}, "rank"),
                       ({"rank": 0, "world_size": 5}, "grid")]:
        c = vg.config_from_params(p, kw)
        h = ctypes.c_void_p()
        assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL
        assert needle in _lib.lib.vg_last_error().decode()
    c = vg.config_from_params(p.replace(n_replicas=2), {"rank": 0, "world_size": 2})
    h = ctypes.c_void_p()
    assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL


# ------------------------------------------------------------------------------ GPU
def _compare_group(p, P, steps, state0, seed=0, halo=0, interior=True):
    import torch
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200.slab import SlabGroup
    dev = torch.device("cuda", 0)
    rep = vg.World(p, device=dev)
    grp = SlabGroup(p, P, device=dev, halo_capacity=halo)
    st = torch.from_numpy(state0).to(dev)
    out_r = rep.alloc_outputs()
    outs = [w.alloc_outputs() for w in grp.worlds]
    rep.bin(st)
    rep.sense(out_r)
    grp.load(st)
    grp.sense(outs)
    keys = ["obs", "reward", "n_neigh", "n_collide", "sector_occ"] + (["n_touch"] if p.env == "tag" else [])

    def check(tag):
        torch.cuda.synchronize()
        seen = torch.zeros(p.n_agents, dtype=torch.int32, device=dev)
        for w, o in zip(grp.worlds, outs):
            assert w.sync_errors() == -1
            n = w.slab_own_count()
            ids = o.agent_id[0, :n].long()
            seen[ids] += 1
            for k in keys:
                a = getattr(o, k)[0, :n]
                b = getattr(out_r, k)[0][ids]
                assert torch.equal(a.view(torch.int32), b.view(torch.int32)), f"{tag}: {k} differs (P={P})"
            oid, ost = w.slab_owned()            # (cell, id) order; output rows: sense order
            assert torch.equal(torch.sort(oid.long()).values, torch.sort(ids).values)
            cols = 4 if p.env == "flock" else 3
            assert torch.equal(ost[:, :cols], st[0][oid.long()][:, :cols]), f"{tag}: state differs"
        assert torch.equal(seen, torch.ones_like(seen)), "every agent owned exactly once"

    check("load")
    for t in range(steps):
        act = torch.from_numpy(vi.actions(p, seed=seed, step=t)).to(dev)
        rows = []
        for w, o in zip(grp.worlds, outs):
            a = torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device=dev)
            n = w.slab_own_count()
            a[0, :n] = act[0][o.agent_id[0, :n].long()]
            rows.append(a)
        rep.step(st, act, out_r)
        grp.step(rows, outs, interior=interior)
        check(f"step {t}")
    grp.close()
    rep.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_slab_bit_identical_flock(cuda, P):
    p = vi.flock_params(20000, width=200.0, d_v=10.0, grid=16)
    _compare_group(p, P, 4, vi.init_state(p, seed=3))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_slab_finish_runs_interior_phase(cuda, P):
    # vg_slab_finish without a vg_slab_interior call runs the interior phase itself
    p = vi.flock_params(20000, width=200.0, d_v=10.0, grid=16)
    _compare_group(p, P, 2, vi.init_state(p, seed=9), interior=False)


@pytest.mark.gpu
def test_slab_call_order_and_step_without_comm(cuda):
    import torch
    import paper_2207_03945_b200 as vg
    p = vi.flock_params(4000, width=170.0, d_v=10.0, grid=16)
    w = vg.World(p, slab={"rank": 0, "world_size": 2})
    out = w.alloc_outputs()
    w.slab_load(torch.from_numpy(vi.init_state(p, seed=1)).cuda())
    w.slab_sense(out)
    with pytest.raises(vg.VgError, match="VG_EINVAL.*slab_begin first"):
        w.slab_interior(out)
    with pytest.raises(vg.VgError, match="VG_EINVAL.*slab_begin first"):
        w.slab_finish(out)
    a = torch.zeros((1, p.n_agents, 2), device="cuda")
    with pytest.raises(vg.VgError, match="VG_EINVAL.*communicator"):
        w.slab_step(a, out)
    w.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_slab_window_rim(cuda, P):
    # K4 windows run along columns in slab mode: rim neighbours (vi.rim_state) at slab and
    # wrap edges must give the single-world result bit for bit.
    p = vi.flock_params(6000, width=170.0, d_v=10.0, grid=16)
    _compare_group(p, P, 2, vi.rim_state(p, 150, seed=5, radius=p.d_v))


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["flock", "tag"])
def test_slab_bit_identical_ray(cuda, env):
    # the ray-disc vision variant (NEXT #2) through the slab path: windows of radius
    # d_v + d_r along the columns, ghost columns, migrants — bit-identical to one world.
    mk = vi.flock_params if env == "flock" else vi.tag_params
    p = mk(12000, width=176.0, d_v=10.0, grid=16).replace(vision="ray")
    _compare_group(p, 4, 2, vi.init_state(p, seed=8))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_slab_bit_identical_tag(cuda, P):
    p = vi.tag_params(12000, width=120.0, d_v=10.0, grid=9 if P == 3 else 8)
    _compare_group(p, P, 3, vi.init_state(p, seed=4))


@pytest.mark.gpu
def test_slab_clustered_and_overflow(cuda):
    import torch
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200.slab import SlabGroup
    p = vi.flock_params(6000, width=120.0, d_v=10.0, grid=8)
    st0 = vi.clustered_state(p, seed=2, n_clusters=4, sigma=6.0)
    _compare_group(p, 4, 3, st0)
    # a tiny halo capacity must be reported, not silently dropped
    grp = SlabGroup(p, 2, halo_capacity=8)
    grp.load(torch.from_numpy(st0).cuda())
    outs = [w.alloc_outputs() for w in grp.worlds]
    grp.sense(outs)
    rows = [torch.zeros((1, p.n_agents, 2), device="cuda") for _ in range(2)]
    grp.step(rows, outs)
    torch.cuda.synchronize()
    with pytest.raises(vg.VgError, match="VG_EOVERFLOW"):
        for w in grp.worlds:
            w.sync_errors()
    grp.close()


@pytest.mark.gpu
def test_slab_c5_full_size(cuda):
    # configs[4] (10^6 agents, G = 136) at P = 8 slabs: bit-identical to one world.
    p = vi.workload("c5")
    _compare_group(p, 8, 2, vi.init_state(p, seed=0))


# ------------------------------------------------- multi-process slab step (one GPU)
def _mp_slab_worker(rank, world, port, params, steps, seed, q):
    """One slab rank in its own process: gloo process group, messages staged through
    pinned host tensors (slab.HostStaging), begin -> interior -> exchange -> finish."""
    import torch
    import torch.distributed as dist
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        p = params
        w = vg.World(p, device=dev, slab={"rank": rank, "world_size": world})
        out = w.alloc_outputs()
        stg = slab.HostStaging(w)
        w.slab_load(torch.from_numpy(vi.init_state(p, seed=seed)).to(dev))
        w.slab_sense(out)
        res = []
        for t in range(steps):
            act = torch.from_numpy(vi.actions(p, seed=seed, step=t)).to(dev)
            n = w.slab_own_count()
            a = torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device=dev)
            a[0, :n] = act[0][out.agent_id[0, :n].long()]
            slab.slab_step_dist(w, a, out, staging=stg)
            torch.cuda.synchronize()
            assert w.sync_errors() == -1
            n = w.slab_own_count()
            keys = ["obs", "reward", "n_neigh", "n_collide", "sector_occ", "agent_id"]
            res.append({k: getattr(out, k)[0, :n].cpu().numpy().copy() for k in keys})
        q.put((rank, res))
        w.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_slab_multiprocess_host_staging(cuda, P):
    # P ranks as P processes on the one GPU, exchanging the halo through host memory (gloo;
    # no kernel waits on another process): every agent's outputs bitwise equal to one world.
    import torch
    import torch.multiprocessing as mp
    import paper_2207_03945_b200 as vg
    p = vi.flock_params(12000, width=170.0, d_v=10.0, grid=16)
    steps, seed = 3, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mp_slab_worker, args=(r, P, port, p, steps, seed, q))
             for r in range(P)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=300) for _ in range(P))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    rep = vg.World(p)
    out = rep.alloc_outputs()
    st = torch.from_numpy(vi.init_state(p, seed=seed)).cuda()
    for t in range(steps):
        rep.step(st, torch.from_numpy(vi.actions(p, seed=seed, step=t)).cuda(), out)
        torch.cuda.synchronize()
        seen = np.zeros(p.n_agents, np.int64)
        for r in range(P):
            g = got[r][t]
            ids = g["agent_id"].astype(np.int64)
            seen[ids] += 1
            for k in ("obs", "reward", "n_neigh", "n_collide", "sector_occ"):
                ref = getattr(out, k)[0].cpu().numpy()[ids]
                assert np.array_equal(g[k].view(np.uint32), ref.view(np.uint32)), (t, r, k)
        assert np.all(seen == 1)
    rep.close()
