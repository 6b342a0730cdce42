"""paper_2207_03945_b200 — B200-native batched environment step of the Vogue MARL
environments (arxiv 2207.03945): flock and tag.

``World`` wraps one libvg world (include/vg.h) over caller-owned torch CUDA tensors:

    w = World(params)                     # params: vg_inputs.EnvParams-like object
    out = w.alloc_outputs()
    w.step(state, actions, out)           # integrate -> bin -> sense + reward

Tensors: state float32 [R, N, 4] (x, y, theta, s), actions float32 [R, N, 2], all on the
world's CUDA device, contiguous.  Calls are asynchronous on the current torch stream and
CUDA-graph capturable.  PyTorch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes
import dataclasses
from ctypes import byref, c_int64, c_void_p

import torch

from . import _lib
from ._lib import VgError, check  # noqa: F401

__all__ = ["World", "Outputs", "VgError", "config_from_params"]

_ENV = {"flock": _lib.ENV_FLOCK, "tag": _lib.ENV_TAG}


def config_from_params(p, slab: dict | None = None) -> _lib.VgConfig:
    """Build a vg_config from an EnvParams-like object (same field names).  ``slab`` =
    {"rank": g, "world_size": P, "halo_capacity": 0} selects slab mode (one world split
    over P ranks by x-slabs)."""
    c = _lib.VgConfig()
    c.env = _ENV[p.env]
    c.vision = {"sector": 0, "ray": 1}[getattr(p, "vision", "sector")]
    c.shard = 1 if slab else 0
    if slab:
        c.rank = int(slab["rank"])
        c.world_size = int(slab["world_size"])
        c.halo_capacity = int(slab.get("halo_capacity", 0))
        nid = slab.get("nccl_unique_id")       # bytes (vg_nccl_unique_id): world owns a comm
        if nid is not None:
            if len(nid) != 128:
                raise ValueError("nccl_unique_id: 128 bytes required")
            c._nccl_id_buf = ctypes.create_string_buffer(bytes(nid), 128)   # kept alive
            c.nccl_unique_id = ctypes.cast(c._nccl_id_buf, ctypes.c_void_p)
    c.n_agents = int(p.n_agents)
    c.n_replicas = int(p.n_replicas)
    for f in ("width", "d_v", "d_r", "fov", "s_min", "s_max", "a_max", "theta_max",
              "c_collide", "c_near", "d_peak", "r_touch", "w_prox", "s_max_chaser"):
        setattr(c, f, float(getattr(p, f)))
    c.v = int(p.v)
    c.grid = int(getattr(p, "grid", 0))
    c.n_chasers = int(getattr(p, "n_chasers", 0))
    return c


@dataclasses.dataclass
class Outputs:
    """Caller-owned output tensors (vg_outputs); None = not written."""
    obs: torch.Tensor | None = None
    reward: torch.Tensor | None = None
    n_neigh: torch.Tensor | None = None
    n_collide: torch.Tensor | None = None
    n_touch: torch.Tensor | None = None
    sector_occ: torch.Tensor | None = None
    agent_id: torch.Tensor | None = None      # slab mode: global id of each row


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class _CudaArray:
    """Borrowed device buffer exposed through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}
        self._owner = owner


def nccl_unique_id() -> bytes:
    """vg_nccl_unique_id: 128 bytes naming a new NCCL communicator (make on one rank,
    broadcast, pass to every rank's World(slab={..., "nccl_unique_id": id}))."""
    buf = ctypes.create_string_buffer(128)
    check(_lib.lib.vg_nccl_unique_id(buf, 128))
    return buf.raw


class World:
    def __init__(self, params, device: int | torch.device | None = None,
                 slab: dict | None = None):
        self.params = params
        self.slab = dict(slab) if slab else None
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        if dev.type != "cuda":
            raise ValueError("World needs a CUDA device (there is no CPU path)")
        self.device = dev
        self._cfg = config_from_params(params, slab)
        self._h = c_void_p()
        with torch.cuda.device(dev):
            torch.cuda.init()
            check(_lib.lib.vg_world_create(byref(self._cfg), byref(self._h)))
        info = _lib.VgWorldInfo()
        check(_lib.lib.vg_world_query(self._h, byref(info)))
        self.grid = info.grid
        self.cell_size = info.cell_size
        self.n_cells = info.n_cells
        self.obs_dim = info.obs_dim
        self.channels = info.channels
        self.occ_words = info.occ_words
        self.scratch_bytes = info.scratch_bytes
        self.kernels_per_step = info.kernels_per_step
        self.sense_defaults = bool(info.sense_defaults)
        self.R, self.N = int(params.n_replicas), int(params.n_agents)
        self.is_tag = params.env == "tag"
        if self.slab:
            io = _lib.VgSlabIo()
            check(_lib.lib.vg_slab_get_io(self._h, byref(io)))
            self.slab_io = io
            mk = lambda p: torch.as_tensor(  # noqa: E731
                _CudaArray(p, (io.message_bytes,), "|u1", self), device=self.device)
            self.messages = {"send_left": mk(io.send_left), "send_right": mk(io.send_right),
                             "recv_left": mk(io.recv_left), "recv_right": mk(io.recv_right)}

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if self._h:
            _lib.lib.vg_world_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ helpers
    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _check_tensor(self, t: torch.Tensor, name: str, shape, dtype=torch.float32):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name}: expected a torch.Tensor")
        if t.device != self.device:
            raise ValueError(f"{name}: on {t.device}, world is on {self.device}")
        if t.dtype != dtype:
            raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")

    def _outs(self, out: Outputs) -> _lib.VgOutputs:
        R, N = self.R, self.N
        spec = {"obs": ((R, N, self.obs_dim), torch.float32),
                "reward": ((R, N), torch.float32),
                "n_neigh": ((R, N), torch.int32), "n_collide": ((R, N), torch.int32),
                "n_touch": ((R, N), torch.int32),
                "sector_occ": ((R, N, self.occ_words), torch.int32),
                "agent_id": ((R, N), torch.int32)}
        o = _lib.VgOutputs()
        for name, (shape, dt) in spec.items():
            t = getattr(out, name)
            if t is not None:
                if dt == torch.int32 and t.dtype == torch.uint32:
                    dt = torch.uint32
                self._check_tensor(t, name, shape, dt)
            setattr(o, name, _ptr(t))
        return o

    def alloc_outputs(self, obs=True, reward=True, counts=True, sector_occ=True) -> Outputs:
        R, N, d = self.R, self.N, self.device
        z = lambda *s, dt=torch.float32: torch.empty(s, dtype=dt, device=d)  # noqa: E731
        return Outputs(
            obs=z(R, N, self.obs_dim) if obs else None,
            reward=z(R, N) if reward else None,
            n_neigh=z(R, N, dt=torch.int32) if counts else None,
            n_collide=z(R, N, dt=torch.int32) if counts else None,
            n_touch=z(R, N, dt=torch.int32) if (counts and self.is_tag) else None,
            sector_occ=z(R, N, self.occ_words, dt=torch.int32) if sector_occ else None,
            agent_id=z(R, N, dt=torch.int32) if self.slab else None,
        )

    # ------------------------------------------------------------------ the ABI
    def bin(self, state: torch.Tensor) -> None:
        self._check_tensor(state, "state", (self.R, self.N, 4))
        check(_lib.lib.vg_bin(self._h, state.data_ptr(), self._stream()))

    def sense(self, out: Outputs) -> None:
        o = self._outs(out)
        check(_lib.lib.vg_sense(self._h, byref(o), self._stream()))

    def reward(self, out: Outputs) -> None:
        o = self._outs(out)
        check(_lib.lib.vg_reward(self._h, byref(o), self._stream()))

    def integrate(self, state: torch.Tensor, actions: torch.Tensor) -> None:
        self._check_tensor(state, "state", (self.R, self.N, 4))
        self._check_tensor(actions, "actions", (self.R, self.N, 2))
        check(_lib.lib.vg_integrate(self._h, state.data_ptr(), actions.data_ptr(),
                                    self._stream()))

    def step(self, state: torch.Tensor, actions: torch.Tensor, out: Outputs) -> None:
        self._check_tensor(state, "state", (self.R, self.N, 4))
        self._check_tensor(actions, "actions", (self.R, self.N, 2))
        o = self._outs(out)
        check(_lib.lib.vg_step(self._h, state.data_ptr(), actions.data_ptr(), byref(o),
                               self._stream()))

    def step_host(self, state: torch.Tensor, actions_host: torch.Tensor, out: Outputs,
                  reward_host: torch.Tensor | None) -> None:
        """vg_step_host: actions from (pinned) host memory, reward copied back to host."""
        self._check_tensor(state, "state", (self.R, self.N, 4))
        if actions_host.device.type != "cpu" or actions_host.dtype != torch.float32 or \
                tuple(actions_host.shape) != (self.R, self.N, 2) or not actions_host.is_contiguous():
            raise ValueError("actions_host: contiguous float32 CPU tensor [R, N, 2] required")
        if reward_host is not None and (reward_host.device.type != "cpu" or
                                        reward_host.dtype != torch.float32 or
                                        tuple(reward_host.shape) != (self.R, self.N) or
                                        not reward_host.is_contiguous()):
            # vg_step_host writes exactly 4 R N bytes at data_ptr(): anything else would be
            # a host heap overrun or land on the wrong elements
            raise ValueError("reward_host: contiguous float32 CPU tensor [R, N] required")
        o = self._outs(out)
        check(_lib.lib.vg_step_host(self._h, state.data_ptr(), actions_host.data_ptr(),
                                    byref(o), _ptr(reward_host), self._stream()))

    def get_bins(self) -> dict:
        """Zero-copy views of the last binning (valid until the next bin/step).  Slab mode:
        the local set (owned + ghosts) on the column-major local grid; perm = global ids."""
        ptrs = [c_void_p() for _ in range(4)]
        check(_lib.lib.vg_get_bins(self._h, *[byref(p) for p in ptrs]))
        R, N = self.R, self.N
        if self.slab:
            R, N = 1, self.N + 2 * ((self.slab_io.message_bytes - 16) // 20)
        mk = lambda p, shape, ts: torch.as_tensor(  # noqa: E731
            _CudaArray(p.value, shape, ts, self), device=self.device)
        return {"cell_id": mk(ptrs[0], (R, N), "<i4"),
                "cell_start": mk(ptrs[1], (self.n_cells + 1,), "<i4"),
                "perm": mk(ptrs[2], (R, N), "<i4"),
                "sorted": mk(ptrs[3], (R, N, 4), "<f4")}

    # ------------------------------------------------------------------ slab mode
    def slab_load(self, state_global: torch.Tensor) -> None:
        """Take this rank's owned + ghost agents from the full state [1, N, 4] and bin them."""
        self._check_tensor(state_global, "state_global", (1, self.N, 4))
        check(_lib.lib.vg_slab_load(self._h, state_global.data_ptr(), self._stream()))

    def slab_sense(self, out: Outputs) -> None:
        o = self._outs(out)
        check(_lib.lib.vg_slab_sense(self._h, byref(o), self._stream()))

    def slab_begin(self, actions: torch.Tensor) -> None:
        """Integrate the owned rows with actions[row] (rows of the last output) and route."""
        self._check_tensor(actions, "actions", (1, self.N, 2))
        check(_lib.lib.vg_slab_begin(self._h, actions.data_ptr(), self._stream()))

    def sense_columns(self, out: Outputs, col_lo: int, col_hi: int) -> None:
        """vg_sense_columns: sense only the cells of grid columns [col_lo, col_hi) (R = 1)."""
        o = self._outs(out)
        check(_lib.lib.vg_sense_columns(self._h, byref(o), int(col_lo), int(col_hi),
                                        self._stream()))

    def slab_interior(self, out: Outputs) -> None:
        """vg_slab_interior: bin + sense the interior columns (no halo needed)."""
        o = self._outs(out)
        check(_lib.lib.vg_slab_interior(self._h, byref(o), self._stream()))

    def slab_finish(self, out: Outputs) -> None:
        o = self._outs(out)
        check(_lib.lib.vg_slab_finish(self._h, byref(o), self._stream()))

    def slab_step(self, actions: torch.Tensor, out: Outputs) -> None:
        """vg_slab_step: one step with the world's own NCCL halo exchange, overlapped with
        the interior phase (needs slab={"nccl_unique_id": ...} at creation)."""
        self._check_tensor(actions, "actions", (1, self.N, 2))
        o = self._outs(out)
        check(_lib.lib.vg_slab_step(self._h, actions.data_ptr(), byref(o), self._stream()))

    def slab_owned(self) -> tuple:
        """(global ids [n_own], state records [n_own, 4]) of the owned agents in (cell, id)
        order (vg_get_bins; owned = the first n_own records, memory columns 0..W-1); output
        rows use the sense order — map them by outs.agent_id."""
        n = self.slab_own_count()
        b = self.get_bins()
        return b["perm"][0, :n].clone(), b["sorted"][0, :n].clone()

    def slab_own_count(self) -> int:
        n = c_int64(0)
        check(_lib.lib.vg_slab_own_count(self._h, self._stream(), byref(n)))
        return n.value

    def profile_begin(self, max_steps: int) -> None:
        """Record per-phase CUDA events for the next max_steps vg_step calls."""
        check(_lib.lib.vg_profile_begin(self._h, int(max_steps)))

    def profile_end(self) -> tuple[dict, int]:
        """Synchronize; return ({phase: total ms}, steps recorded)."""
        ms = (ctypes.c_double * _lib.N_PHASES)()
        n = ctypes.c_int32(0)
        check(_lib.lib.vg_profile_end(self._h, self._stream(), ms, byref(n)))
        return dict(zip(_lib.PHASES, list(ms))), n.value

    def sync_errors(self) -> int:
        """Synchronize; return -1 if clean, else raise VgError(VG_ESTATE) with the index."""
        bad = c_int64(-1)
        st = _lib.lib.vg_sync_errors(self._h, self._stream(), byref(bad))
        if st == _lib.VG_ESTATE:
            err = VgError(st, _lib.lib.vg_last_error().decode())
            err.bad_agent = bad.value
            raise err
        check(st)
        return bad.value

