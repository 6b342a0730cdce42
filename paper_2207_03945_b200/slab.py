"""Slab mode plumbing: one world split over P ranks by
x-slabs of cell columns, with a one-column halo exchanged every step.

The device work (integrate + route, interior and boundary binning and sensing) and, with
``World.slab_step``, the halo exchange itself (the world's own NCCL communicator on its
comm stream, overlapped with the interior phase) are in libvg.  This module covers the
other ways to move the four fixed-size messages:

* ``slab_step_dist`` — one process per rank over torch.distributed P2P: NCCL on device
  buffers (the exchange runs on NCCL's stream while the interior phase runs), or
  ``staging="host"`` (gloo: the messages go through pinned host tensors — the CPU tests and
  the multi-process test on one GPU).  send_left -> left rank's recv_right, send_right ->
  right rank's recv_left; for P = 2 both neighbours are the same rank: the receives are
  posted in the order (from right, from left) to pair with the peer's (to left, to right).
* ``SlabGroup`` — P slab worlds in ONE process on one device, exchanged with
  vg_slab_exchange_loopback (device copies; no kernel waits on another).  Used by the
  single-GPU tests of the partition / migration / ghost / phase logic.
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


def exchange_post(messages: dict, left: int, right: int, group=None) -> list:
    """Post the halo exchange with torch.distributed P2P; returns the requests."""
    import torch.distributed as dist
    ops = [dist.P2POp(dist.isend, messages["send_left"], left, group),
           dist.P2POp(dist.isend, messages["send_right"], right, group),
           dist.P2POp(dist.irecv, messages["recv_right"], right, group),
           dist.P2POp(dist.irecv, messages["recv_left"], left, group)]
    return dist.batch_isend_irecv(ops)


def exchange_dist(messages: dict, left: int, right: int, group=None) -> None:
    """Halo exchange with torch.distributed P2P (async ops, waited on the current stream)."""
    for req in exchange_post(messages, left, right, group):
        req.wait()


class HostStaging:
    """Pinned host copies of a world's four messages, for transports without device
    buffers (gloo)."""

    def __init__(self, world):
        nb = int(world.slab_io.message_bytes)
        self.host = {k: torch.empty(nb, dtype=torch.uint8).pin_memory() for k in
                     ("send_left", "send_right", "recv_left", "recv_right")}


def slab_step_dist(world, actions: torch.Tensor, out, group=None, staging=None) -> None:
    """One step of this rank's slab: begin -> (exchange || interior) -> finish.

    Device buffers (NCCL): the P2P ops run on NCCL's stream after the begin kernels; the
    interior phase is enqueued before waiting on them, so it overlaps the transfer.
    ``staging`` (a HostStaging): send buffers -> host, exchange (gloo), host -> receive
    buffers, with the interior phase enqueued before the host blocks on the copies."""
    io = world.slab_io
    world.slab_begin(actions)
    if staging is None:
        reqs = exchange_post(world.messages, io.left_rank, io.right_rank, group)
        world.slab_interior(out)
        for r in reqs:
            r.wait()
    else:
        h, m = staging.host, world.messages
        h["send_left"].copy_(m["send_left"], non_blocking=True)
        h["send_right"].copy_(m["send_right"], non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        world.slab_interior(out)
        done.synchronize()
        exchange_dist(h, io.left_rank, io.right_rank, group)
        m["recv_left"].copy_(h["recv_left"], non_blocking=True)
        m["recv_right"].copy_(h["recv_right"], non_blocking=True)
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

    def step(self, actions: list, outs: list, interior: bool = True) -> None:
        """begin (all) -> interior (all) -> exchange -> finish (all), the order of a
        distributed step; ``interior=False`` leaves the interior phase to finish."""
        for w, a in zip(self.worlds, actions):
            w.slab_begin(a)
        if interior:
            for w, o in zip(self.worlds, outs):
                w.slab_interior(o)
        w0 = self.worlds[0]
        check(_lib.lib.vg_slab_exchange_loopback(self._arr, len(self.worlds), w0._stream()))
        for w, o in zip(self.worlds, outs):
            w.slab_finish(o)

    def close(self) -> None:
        for w in self.worlds:
            w.close()
