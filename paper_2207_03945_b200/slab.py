"""Slab mode plumbing: one world split over P ranks by
x-slabs of cell columns, with a one-column halo exchanged every step.

The device work (integrate + route, unpack, binning, sensing) is in libvg; this module
only moves the four fixed-size messages between ranks:

* ``exchange_dist`` — one process per GPU: torch.distributed point-to-point (NCCL over
  NVLink on the GPU box; gloo in the CPU tests), send_left -> left rank's recv_right and
  send_right -> right rank's recv_left.  For P = 2 both neighbours are the same rank: the
  receives are posted in the order (from right, from left) so that they pair with the
  peer's sends (to left, to right) in issue order.
* ``SlabGroup`` — P slab worlds in ONE process on one device, exchanged with
  vg_slab_exchange_loopback (device copies; no kernel waits on another).  Used by the
  single-GPU tests of the partition / migration / ghost logic.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import check


def plan(grid: int, world_size: int, rank: int) -> dict:
    """lo, hi (owned global cell columns), left, right (neighbour ranks) — host only."""
    out = (ctypes.c_int32 * 4)()
    check(_lib.lib.vg_slab_plan(grid, world_size, rank, out))
    return {"lo": out[0], "hi": out[1], "left": out[2], "right": out[3]}


def exchange_dist(messages: dict, left: int, right: int, group=None) -> None:
    """Halo exchange with torch.distributed P2P (async ops, waited on the current stream)."""
    import torch.distributed as dist
    ops = [dist.P2POp(dist.isend, messages["send_left"], left, group),
           dist.P2POp(dist.isend, messages["send_right"], right, group),
           dist.P2POp(dist.irecv, messages["recv_right"], right, group),
           dist.P2POp(dist.irecv, messages["recv_left"], left, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def slab_step_dist(world, actions: torch.Tensor, out, group=None) -> None:
    """One environment step of this rank's slab: begin -> exchange -> finish."""
    world.slab_begin(actions)
    exchange_dist(world.messages, world.slab_io.left_rank, world.slab_io.right_rank, group)
    world.slab_finish(out)


class SlabGroup:
    """P slab worlds of one environment in one process (single device, loopback exchange)."""

    def __init__(self, params, world_size: int, device=None, halo_capacity: int = 0):
        from . import World
        self.worlds = [World(params, device=device,
                             slab={"rank": g, "world_size": world_size,
                                   "halo_capacity": halo_capacity})
                       for g in range(world_size)]
        self._arr = (ctypes.c_void_p * world_size)(*[w._h.value for w in self.worlds])

    def load(self, state_global: torch.Tensor) -> None:
        for w in self.worlds:
            w.slab_load(state_global)

    def sense(self, outs) -> None:
        for w, o in zip(self.worlds, outs):
            w.slab_sense(o)

    def step(self, actions: list, outs: list) -> None:
        for w, a in zip(self.worlds, actions):
            w.slab_begin(a)
        w0 = self.worlds[0]
        check(_lib.lib.vg_slab_exchange_loopback(self._arr, len(self.worlds), w0._stream()))
        for w, o in zip(self.worlds, outs):
            w.slab_finish(o)

    def close(self) -> None:
        for w in self.worlds:
            w.close()
