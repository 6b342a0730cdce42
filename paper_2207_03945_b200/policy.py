"""Shared-policy forward on the tensor cores (include/vg.h
vg_policy_*): actor-critic MLP obs -> 64 -> 64 -> (mean[2], value) with tanh (
S:329-333) over all agents, then a = clip(mean + exp(log_std) eps, box) with Philox noise
(S:355-372).  Argument marshalling only."""
from __future__ import annotations

import ctypes
from ctypes import byref, c_void_p

import torch

from . import _lib
from ._lib import check

WEIGHT_ORDER = ("W1", "b1", "W2", "b2", "W3", "b3", "log_std", "V1", "c1", "V2", "c2", "V3", "c3")


def action_box(params) -> tuple:
    """(lo, hi) of the action box of an EnvParams-like object."""
    if params.env == "flock":
        return (-params.a_max, -params.theta_max), (params.a_max, params.theta_max)
    return (-params.theta_max, 0.0), (params.theta_max, max(params.s_max, params.s_max_chaser))


class Policy:
    def __init__(self, obs_dim: int, act_lo, act_hi, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        cfg = _lib.VgPolicyConfig()
        cfg.obs_dim = int(obs_dim)
        for d in range(2):
            cfg.act_lo[d] = float(act_lo[d])
            cfg.act_hi[d] = float(act_hi[d])
        self.obs_dim = int(obs_dim)
        self._h = c_void_p()
        with torch.cuda.device(self.device):
            check(_lib.lib.vg_policy_create(byref(cfg), byref(self._h)))
        self._w = None

    def set_weights(self, weights: dict) -> None:
        """weights: name -> fp32 array/tensor in nn.Linear layout (WEIGHT_ORDER)."""
        ts = [torch.as_tensor(weights[k], dtype=torch.float32).to(self.device).contiguous()
              for k in WEIGHT_ORDER]
        self._w = ts                                        # keep alive until packed
        arr = (c_void_p * 13)(*[t.data_ptr() for t in ts])
        check(_lib.lib.vg_policy_set_weights(self._h, arr,
                                             torch.cuda.current_stream(self.device).cuda_stream))

    def alloc(self, rows: int, sample: bool = True) -> dict:
        z = lambda *s: torch.empty(s, dtype=torch.float32, device=self.device)  # noqa: E731
        return {"mean": z(rows, 2), "value": z(rows), "action": z(rows, 2) if sample else None,
                "logp": z(rows) if sample else None}

    def forward(self, obs: torch.Tensor, out: dict, seed: int = 0, step: int = 0,
                row_class: tuple | None = None) -> None:
        """vg_policy_forward; ``row_class`` = (period, split, cls) writes only the rows r
        with ((r mod period) >= split) == cls (vg_policy_forward_class: per-type policies)."""
        rows = obs.numel() // self.obs_dim
        if obs.dtype != torch.float32 or obs.device != self.device or not obs.is_contiguous() \
                or obs.numel() != rows * self.obs_dim:
            raise ValueError("obs: contiguous float32 CUDA tensor [rows, obs_dim] required")
        o = _lib.VgPolicyOutputs()
        for k in ("mean", "value", "action", "logp"):
            t = out.get(k)
            if t is not None and (t.dtype != torch.float32 or t.device != self.device or
                                  t.numel() < rows * (2 if k in ("mean", "action") else 1)):
                raise ValueError(f"{k}: float32 CUDA tensor with enough rows required")
            setattr(o, k, None if t is None else t.data_ptr())
        period, split, cls = row_class if row_class is not None else (0, 0, 0)
        check(_lib.lib.vg_policy_forward_class(self._h, obs.data_ptr(), rows, int(period),
                                               int(split), int(cls), byref(o),
                                               ctypes.c_uint64(seed), ctypes.c_uint64(step),
                                               torch.cuda.current_stream(self.device).cuda_stream))

    def close(self) -> None:
        if self._h:
            _lib.lib.vg_policy_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
