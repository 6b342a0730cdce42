"""GAE over the on-device trajectory buffer and the opinion
dynamics graph interaction of Listing 1 (NEXT #4).  Argument marshalling only."""
from __future__ import annotations

import torch

from . import _lib
from ._lib import check


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _f32(t: torch.Tensor, name: str, shape=None):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and
            t.is_contiguous()):
        raise ValueError(f"{name}: contiguous float32 CUDA tensor required")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")


class TrajectoryBuffer:
    """Time-major rollout storage for n agents x t steps: obs [t+1][n][obs_dim]
    (obs[t] seeds the next rollout), action [t][n][2], logp, reward [t][n], value [t+1][n]
    (bootstrap row), adv, ret.  vg_step / vg_policy_forward write straight into step k's
    slices (no copies)."""

    def __init__(self, n: int, t: int, obs_dim: int, device=None):
        d = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=d)  # noqa: E731
        self.n, self.t = n, t
        self.obs = z(t + 1, n, obs_dim)
        self.action = z(t, n, 2)
        self.logp = z(t, n)
        self.reward = z(t, n)
        self.value = z(t + 1, n)
        self.adv = z(t, n)
        self.ret = z(t, n)

    def compute_gae(self, gamma: float = 0.99, lam: float = 0.95) -> None:
        gae(self.reward, self.value, self.adv, self.ret, gamma, lam)


def gae(reward, value, adv, ret, gamma: float = 0.99, lam: float = 0.95) -> None:
    t, n = reward.shape
    _f32(reward, "reward")
    _f32(value, "value", (t + 1, n))
    _f32(adv, "adv", (t, n))
    _f32(ret, "ret", (t, n))
    check(_lib.lib.vg_gae(reward.data_ptr(), value.data_ptr(), n, t, gamma, lam,
                          adv.data_ptr(), ret.data_ptr(), _stream(reward)))


def opinion_step(row_ptr, col, weight, op_in, op_out, threshold: float, strength: float,
                 check_errors: bool = True) -> None:
    """vg_opinion_step; with ``check_errors`` (default) also vg_opinion_sync_errors, which
    synchronizes the stream and raises VG_ESTATE on an invalid row or dangling edge."""
    n = op_in.numel()
    for x, nm in ((row_ptr, "row_ptr"), (col, "col")):
        if not (x.is_cuda and x.dtype == torch.int32 and x.is_contiguous()):
            raise ValueError(f"{nm}: contiguous int32 CUDA tensor required")
    _f32(weight, "weight")
    _f32(op_in, "op_in")
    _f32(op_out, "op_out", (n,))
    if row_ptr.numel() != n + 1:
        raise ValueError("row_ptr: n + 1 entries required")
    if weight.numel() != col.numel():
        raise ValueError(f"weight: {weight.numel()} entries, col has {col.numel()}")
    if not (row_ptr.device == col.device == weight.device == op_in.device == op_out.device):
        raise ValueError("opinion_step: all tensors must be on one device")
    check(_lib.lib.vg_opinion_step(row_ptr.data_ptr(), col.data_ptr(), weight.data_ptr(), n,
                                   col.numel(), op_in.data_ptr(), op_out.data_ptr(), threshold,
                                   strength, _stream(op_in)))
    if check_errors:
        import ctypes
        bad = ctypes.c_int64(-1)
        check(_lib.lib.vg_opinion_sync_errors(_stream(op_in), ctypes.byref(bad)))


def rollout(world, policy, state: torch.Tensor, buf: TrajectoryBuffer, seed: int = 0,
            step0: int = 0, gamma: float = 0.99, lam: float = 0.95,
            policy_chaser=None) -> None:
    """vg_rollout: t steps of the paper's experience-collection loop (Fig. 5) on device.
    buf.obs[0] must hold the current observation (e.g. from world.bin + world.sense).
    Tag worlds: ``policy_chaser`` gives the chasers their own policy, ``policy``
    then drives the runners."""
    import ctypes
    world._check_tensor(state, "state", (world.R, world.N, 4))
    if buf.obs.device != state.device:
        raise ValueError(f"trajectory buffer on {buf.obs.device}, state on {state.device}")
    for pl in (policy, policy_chaser):
        if pl is not None and getattr(pl, "device", state.device) != state.device:
            raise ValueError(f"policy on {pl.device}, state on {state.device}")
    b = _lib.VgRolloutBuffers(buf.obs.data_ptr(), buf.action.data_ptr(), buf.logp.data_ptr(),
                              buf.reward.data_ptr(), buf.value.data_ptr(), buf.adv.data_ptr(),
                              buf.ret.data_ptr())
    if buf.n != world.R * world.N or buf.obs.shape[2] != world.obs_dim:
        raise ValueError("trajectory buffer does not match the world")
    check(_lib.lib.vg_rollout(world._h, policy._h,
                              policy_chaser._h if policy_chaser is not None else None,
                              state.data_ptr(), ctypes.byref(b), buf.t,
                              ctypes.c_uint64(seed), ctypes.c_uint64(step0), gamma, lam,
                              _stream(state)))
