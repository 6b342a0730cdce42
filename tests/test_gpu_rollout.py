"""vg_rollout (the paper's experience-collection loop, Fig. 5 / P:198-205) equals the same
sequence of individual ABI calls bit for bit, and captures into one CUDA graph."""
import numpy as np
import pytest

import vg_inputs as vi
from oracle.gae import gae as gae_ref

pytestmark = pytest.mark.gpu


def _setup(p, t):
    import torch
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import rl
    from paper_2207_03945_b200.policy import Policy, action_box
    w = vg.World(p)
    pol = Policy(w.obs_dim, *action_box(p))
    pol.set_weights(vi.policy_weights(w.obs_dim, seed=2, log_std=-0.7))
    buf = rl.TrajectoryBuffer(p.total_agents, t, w.obs_dim)
    st = torch.from_numpy(vi.init_state(p, seed=3)).cuda()
    out0 = vg.Outputs(obs=buf.obs[0].view(p.n_replicas, p.n_agents, -1))
    w.bin(st)
    w.sense(out0)
    return w, pol, buf, st


@pytest.mark.parametrize("env", ["flock", "tag"])
def test_rollout_equals_manual_loop(cuda, env):
    import torch
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import rl
    p = vi.flock_params(3000, n_replicas=2) if env == "flock" else vi.tag_params(3000)
    t = 6
    w, pol, buf, st = _setup(p, t)
    st_manual = st.clone()
    obs0 = buf.obs[0].clone()
    rl.rollout(w, pol, st, buf, seed=9, step0=100, gamma=0.99, lam=0.95)
    torch.cuda.synchronize()
    # the same calls one by one
    M = p.total_agents
    obs = obs0
    vals, acts, logps, rews = [], [], [], []
    for k in range(t):
        po = {"mean": None, "value": torch.empty(M, device="cuda"),
              "action": torch.empty(M, 2, device="cuda"), "logp": torch.empty(M, device="cuda")}
        pol.forward(obs.contiguous(), po, seed=9, step=100 + k)
        out = w.alloc_outputs(counts=False, sector_occ=False)
        w.step(st_manual, po["action"].view(p.n_replicas, p.n_agents, 2), out)
        vals.append(po["value"]); acts.append(po["action"]); logps.append(po["logp"])
        rews.append(out.reward.view(-1))
        obs = out.obs.view(M, -1)
    pv = {"mean": None, "value": torch.empty(M, device="cuda"), "action": None, "logp": None}
    pol.forward(obs.contiguous(), pv, seed=9, step=100 + t)
    torch.cuda.synchronize()
    assert torch.equal(st, st_manual)
    for k in range(t):
        assert torch.equal(buf.action[k], acts[k]) and torch.equal(buf.logp[k], logps[k])
        assert torch.equal(buf.value[k], vals[k]) and torch.equal(buf.reward[k], rews[k])
    assert torch.equal(buf.value[t], pv["value"]) and torch.equal(buf.obs[t], obs)
    # GAE of the buffer vs the oracle's direct sum
    ref = gae_ref(buf.reward.cpu().numpy(), buf.value.cpu().numpy(),
                  float(np.float32(0.99)), float(np.float32(np.float32(0.99) * np.float32(0.95))) / float(np.float32(0.99)))
    assert np.allclose(buf.adv.cpu().numpy(), ref["adv"], atol=1e-4, rtol=1e-5)
    w.close(); pol.close()


def test_rollout_graph_capture(cuda):
    import torch
    from paper_2207_03945_b200 import rl
    p = vi.workload("c2")
    t = 4
    w, pol, buf, st = _setup(p, t)
    st_eager, obs0 = st.clone(), buf.obs[0].clone()
    rl.rollout(w, pol, st_eager, buf, seed=1)
    torch.cuda.synchronize()
    eager = {k: getattr(buf, k).clone() for k in ("obs", "action", "reward", "value", "adv")}
    buf.obs[0].copy_(obs0)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            rl.rollout(w, pol, st, buf, seed=1)
    buf.obs[0].copy_(obs0)
    st_copy = st  # graph was only captured; state untouched so far
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(st_copy, st_eager)
    for k, v in eager.items():
        assert torch.equal(getattr(buf, k), v), k
    w.close(); pol.close()


def test_rollout_tag_per_type_policies(cuda):
    # "In the tag environment, the runner and chaser types share independent
    # policies" — runners act with one weight set, chasers with another; each row's value,
    # action and log-prob equal the single-policy forward of its own type's weights (the
    # same calls one by one, bit for bit), and differ from the other type's.
    import torch
    from paper_2207_03945_b200 import rl
    from paper_2207_03945_b200.policy import Policy, action_box
    p = vi.tag_params(3000, n_replicas=2)
    t = 3
    w, pol, buf, st = _setup(p, t)
    pc = Policy(w.obs_dim, *action_box(p))
    pc.set_weights(vi.policy_weights(w.obs_dim, seed=5, log_std=-1.3))
    st_manual, obs0 = st.clone(), buf.obs[0].clone()
    rl.rollout(w, pol, st, buf, seed=4, step0=7, policy_chaser=pc)
    torch.cuda.synchronize()
    M, N, nc = p.total_agents, p.n_agents, p.n_chasers
    chaser = (torch.arange(M, device="cuda") % N) >= N - nc
    obs = obs0
    for k in range(t):
        outs = []
        for pl in (pol, pc):
            po = {"mean": None, "value": torch.empty(M, device="cuda"),
                  "action": torch.empty(M, 2, device="cuda"), "logp": torch.empty(M, device="cuda")}
            pl.forward(obs.contiguous(), po, seed=4, step=7 + k)
            outs.append(po)
        for key, dst in (("value", buf.value[k]), ("action", buf.action[k]), ("logp", buf.logp[k])):
            ref = torch.where(chaser.view(-1, *([1] * (outs[0][key].dim() - 1))),
                              outs[1][key], outs[0][key])
            assert torch.equal(dst, ref), (k, key)
            assert not torch.equal(outs[0][key][chaser], outs[1][key][chaser])
        act = buf.action[k].view(p.n_replicas, N, 2)
        o = w.alloc_outputs(counts=False, sector_occ=False)
        w.step(st_manual, act.contiguous(), o)
        obs = o.obs.view(M, -1)
    torch.cuda.synchronize()
    assert torch.equal(st, st_manual)
    w.close(); pol.close(); pc.close()


def test_rollout_chaser_policy_needs_tag(cuda):
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import rl
    p = vi.flock_params(500)
    w, pol, buf, st = _setup(p, 2)
    with pytest.raises(vg.VgError, match="VG_EINVAL.*tag"):
        rl.rollout(w, pol, st, buf, policy_chaser=pol)
    w.close(); pol.close()
