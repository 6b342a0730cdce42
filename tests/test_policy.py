"""K7 shared-policy forward on tcgen05 vs the fp64 oracle (oracle/policy.py).

Two checks:
1. against the fp64 oracle, within a worst-case bound propagated per row from the kernel's
   arithmetic: operands rounded to fp16 (rel 2^-11, abs 2^-25 near zero), fp32
   accumulation (K 2^-24 of sum |w x|), tanh by the hardware tanh.approx.f32 (abs error
   <= 7.84e-6 measured over 2^22 points of [-12, 12] by tools/probes/tanh_probe.cu; 1e-5
   taken), Lipschitz-1 tanh; all three layers on the tensor cores (fp16 operands, fp32
   accumulate);
2. against an emulation of the kernel's quantization (fp16 operands, weights and hidden
   activations, otherwise exact) within 2e-4 absolute — tight enough that any layout or
   indexing error (O(0.1)) fails.
Actions/log-probs: the same Philox bits on both sides, fp32 Box-Muller (~1e-6 relative)."""

import numpy as np
import pytest

import vg_inputs as vi
from oracle import policy as pol

U16, A16, U32 = 2.0 ** -11, 2.0 ** -25, 2.0 ** -24
TANH_ABS = 1e-5
EMU_TOL = 2e-4


def _emulate(w, x):
    """fp16-quantized operands and hidden activations, fp64 everywhere else."""
    q = lambda a: np.asarray(a, np.float32).astype(np.float16).astype(np.float64)  # noqa: E731
    f = {k: np.asarray(v, np.float64) for k, v in w.items()}
    xq = q(x)
    h = q(np.tanh(xq @ q(f["W1"]).T + f["b1"]))
    h = q(np.tanh(h @ q(f["W2"]).T + f["b2"]))          # layer 3 also runs on the tensor cores
    g = q(np.tanh(xq @ q(f["V1"]).T + f["c1"]))
    g = q(np.tanh(g @ q(f["V2"]).T + f["c2"]))
    return h @ q(f["W3"]).T + f["b3"], (g @ q(f["V3"]).T + f["c3"])[:, 0]


def _bound(w, x):
    """Per-row error bounds of (mean[2], value) for the kernel's arithmetic."""
    f = {k: np.asarray(v, np.float64) for k, v in w.items()}
    ex = U16 * np.abs(x) + A16

    def layer(W, b, inp, e_in):
        aW = np.abs(W)
        eW = U16 * aW + A16
        z = inp @ W.T + b
        e = e_in @ aW.T + (np.abs(inp) + e_in) @ eW.T \
            + inp.shape[1] * U32 * (np.abs(inp) @ aW.T) + U32 * np.abs(b)
        h = np.tanh(z)
        eh = e + TANH_ABS                                   # tanh Lipschitz 1 + approx error
        return h, eh

    out = {}
    for pre, (W1, b1, W2, b2, W3, b3) in {"a": ("W1", "b1", "W2", "b2", "W3", "b3"),
                                           "c": ("V1", "c1", "V2", "c2", "V3", "c3")}.items():
        h1, e1 = layer(f[W1], f[b1], x, ex)
        e1q = e1 + U16 * np.abs(h1) + A16                   # h1 rounded to fp16 for layer 2
        h2, e2 = layer(f[W2], f[b2], h1, e1q)
        e2q = e2 + U16 * np.abs(h2) + A16                   # h2 rounded to fp16 for layer 3
        aW3 = np.abs(f[W3])
        eo = e2q @ aW3.T + (np.abs(h2) + e2q) @ (U16 * aW3 + A16).T \
            + 64 * U32 * (np.abs(h2) @ aW3.T) + U32 * np.abs(f[b3])
        out[pre] = eo
    return out["a"], out["c"][:, 0]


def _run(obs_np, w, box, seed=5, step=3):
    import torch
    from paper_2207_03945_b200.policy import Policy
    dev = torch.device("cuda", 0)
    pl = Policy(obs_np.shape[1], box[0], box[1], device=dev)
    pl.set_weights(w)
    obs = torch.from_numpy(np.ascontiguousarray(obs_np, dtype=np.float32)).to(dev)
    out = pl.alloc(obs_np.shape[0])
    pl.forward(obs, out, seed=seed, step=step)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    pl.close()
    return res


def _check(obs_np, w, box, seed=5, step=3):
    g = _run(obs_np, w, box, seed, step)
    ref = pol.forward(w, obs_np)
    ea, ev = _bound(w, obs_np.astype(np.float64))
    dm = np.abs(g["mean"] - ref["mean"])
    dv = np.abs(g["value"] - ref["value"])
    assert np.all(dm <= ea), f"mean err {dm.max()} vs bound {ea.min()}"
    assert np.all(dv <= ev), f"value err {dv.max()}"
    em, evv = _emulate(w, obs_np.astype(np.float64))
    assert np.abs(g["mean"] - em).max() <= EMU_TOL, np.abs(g["mean"] - em).max()
    assert np.abs(g["value"] - evv).max() <= EMU_TOL, np.abs(g["value"] - evv).max()
    s = pol.sample(w, g["mean"].astype(np.float64), np.arange(obs_np.shape[0]), seed, step,
                   np.array(box[0]), np.array(box[1]))      # noise on the GPU's own mean
    sig = np.exp(np.clip(np.asarray(w["log_std"], np.float64), -5.0, 2.0))
    tol_a = 1e-5 * (np.abs(s["eps"]) + 1) * sig + 1e-6
    assert np.all(np.abs(g["action"] - s["action"]) <= tol_a)
    assert np.all(np.abs(g["logp"] - s["logp"]) <= 1e-5 * (1 + (s["eps"] ** 2).sum(-1)))
    lo, hi = np.array(box[0]), np.array(box[1])
    assert np.all((g["action"] >= lo.astype(np.float32)) & (g["action"] <= hi.astype(np.float32)))
    return (float(dm.max()), float(np.median(dm)), float(ea.min()),
            float(np.abs(g["mean"] - em).max()))


@pytest.mark.gpu
@pytest.mark.parametrize("rows", [1, 127, 128, 129, 1000, 4099])
def test_policy_random_obs(cuda, rows):
    p = vi.workload("c2")
    w = vi.policy_weights(p.obs_dim, seed=1)
    rng = np.random.default_rng(rows)
    obs = rng.random((rows, p.obs_dim)).astype(np.float32)
    obs[rng.random(obs.shape) < 0.4] = 1.0                  # empty sectors read 1.0
    print(_check(obs, w, ((-p.a_max, -p.theta_max), (p.a_max, p.theta_max))))


@pytest.mark.gpu
@pytest.mark.parametrize("log_std", [(-30.0, 10.0), (3.0, -6.0)])
def test_policy_log_std_clamped(cuda, log_std):
    # log_std clamped to [-5, 2] in the sample scale and the log-prob (the oracle
    # clamps too, pinned by test_oracle_policy.test_sample_rules)
    p = vi.workload("c2")
    w = vi.policy_weights(p.obs_dim, seed=1)
    w["log_std"] = np.array(log_std, np.float32)
    obs = np.random.default_rng(0).random((300, p.obs_dim)).astype(np.float32)
    _check(obs, w, ((-50.0, -50.0), (50.0, 50.0)))
    g = _run(obs, w, ((-50.0, -50.0), (50.0, 50.0)))
    assert np.all(np.isfinite(g["action"])) and np.all(np.isfinite(g["logp"]))


@pytest.mark.gpu
def test_policy_on_env_observations(cuda):
    # The real pipeline: obs from vg_step (flock C2 and tag C3), then the policy.
    import torch
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200.policy import action_box
    for p in (vi.workload("c2"), vi.workload("c3")):
        world = vg.World(p)
        out = world.alloc_outputs()
        st = torch.from_numpy(vi.init_state(p, seed=2)).cuda()
        world.step(st, torch.from_numpy(vi.actions(p, seed=2)).cuda(), out)
        torch.cuda.synchronize()
        obs = out.obs[0].cpu().numpy()
        w = vi.policy_weights(p.obs_dim, seed=4, log_std=-0.5)
        _check(obs, w, action_box(p), seed=11, step=1)
        world.close()


@pytest.mark.gpu
def test_policy_full_size_c5_sampled(cuda):
    # 10^6 rows (bench launch size): sampled rows against the oracle, all rows finite/in-box.
    import torch
    from paper_2207_03945_b200.policy import Policy
    p = vi.workload("c5")
    w = vi.policy_weights(p.obs_dim, seed=7)
    rng = np.random.default_rng(0)
    obs = torch.rand((p.n_agents, p.obs_dim), device="cuda")
    pl = Policy(p.obs_dim, (-p.a_max, -p.theta_max), (p.a_max, p.theta_max))
    pl.set_weights(w)
    out = pl.alloc(p.n_agents)
    pl.forward(obs, out, seed=9, step=2)
    torch.cuda.synchronize()
    rows = rng.choice(p.n_agents, 2000, replace=False)
    x = obs[rows].cpu().numpy().astype(np.float64)
    ref = pol.forward(w, x)
    ea, ev = _bound(w, x)
    assert np.all(np.abs(out["mean"][rows].cpu().numpy() - ref["mean"]) <= ea)
    assert np.all(np.abs(out["value"][rows].cpu().numpy() - ref["value"]) <= ev)
    em, evv = _emulate(w, x)
    assert np.abs(out["mean"][rows].cpu().numpy() - em).max() <= EMU_TOL
    assert np.abs(out["value"][rows].cpu().numpy() - evv).max() <= EMU_TOL
    assert torch.isfinite(out["action"]).all() and torch.isfinite(out["logp"]).all()
    pl.close()


def test_policy_config_validation():
    import ctypes
    from paper_2207_03945_b200 import _lib
    cfg = _lib.VgPolicyConfig()
    cfg.obs_dim = 200
    h = ctypes.c_void_p()
    assert _lib.lib.vg_policy_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.VG_EINVAL
    assert "obs_dim" in _lib.lib.vg_last_error().decode()


@pytest.mark.gpu
def test_policy_row_class_writes_only_its_rows(cuda):
    # vg_policy_forward_class: period 700, split 500 -> rows with (r mod 700) >= 500 are
    # class 1; a class-1 call writes exactly those rows, with the values of the full call.
    import torch
    from paper_2207_03945_b200.policy import Policy
    p = vi.workload("c3")
    w = vi.policy_weights(p.obs_dim, seed=3)
    rows = 2100
    obs = torch.rand((rows, p.obs_dim), device="cuda")
    pl = Policy(p.obs_dim, (-1.0, 0.0), (1.0, 1.0))
    pl.set_weights(w)
    full = pl.alloc(rows)
    pl.forward(obs, full, seed=2, step=5)
    part = {k: (torch.full_like(v, 7.0) if v is not None else None) for k, v in pl.alloc(rows).items()}
    pl.forward(obs, part, seed=2, step=5, row_class=(700, 500, 1))
    torch.cuda.synchronize()
    cls1 = (torch.arange(rows, device="cuda") % 700) >= 500
    for k in ("mean", "value", "action", "logp"):
        assert torch.equal(part[k][cls1], full[k][cls1]), k
        assert bool((part[k][~cls1] == 7.0).all()), k
    pl.close()
