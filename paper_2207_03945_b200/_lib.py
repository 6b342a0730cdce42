"""ctypes binding of libvg (include/vg.h).  Argument marshalling only — every step of the
environment update runs in the CUDA kernels of libvg.so.  There is no fallback: if the
library is missing or fails to load, importing this module raises."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int32, c_int64, c_void_p

_PKG = os.path.dirname(os.path.abspath(__file__))
# VG_LIB_VARIANT=<name> loads build/variants/libvg_<name>.so (tuning experiments built by
# tools/build_variants.py); unset = the in-tree libvg.so.
LIB_PATH = (os.path.join(os.path.dirname(_PKG), "build", "variants",
                         f"libvg_{os.environ['VG_LIB_VARIANT']}.so")
            if os.environ.get("VG_LIB_VARIANT") else os.path.join(_PKG, "libvg.so"))

VG_OK, VG_EINVAL, VG_ESTATE, VG_ECUDA, VG_ENCCL, VG_EOVERFLOW, VG_ENOMEM = range(7)
N_PHASES = 5
PHASES = ["integrate_bin", "scan_cells", "scatter", "cell_sort", "sense"]
STATUS_NAMES = ["VG_OK", "VG_EINVAL", "VG_ESTATE", "VG_ECUDA", "VG_ENCCL", "VG_EOVERFLOW",
                "VG_ENOMEM"]
ENV_FLOCK, ENV_TAG = 0, 1


class VgConfig(ctypes.Structure):
    _fields_ = [
        ("env", c_int32), ("vision", c_int32), ("shard", c_int32),
        ("n_agents", c_int32), ("n_replicas", c_int32),
        ("width", c_float), ("d_v", c_float), ("d_r", c_float), ("fov", c_float),
        ("v", c_int32), ("grid", c_int32),
        ("s_min", c_float), ("s_max", c_float), ("a_max", c_float), ("theta_max", c_float),
        ("c_collide", c_float), ("c_near", c_float), ("d_peak", c_float),
        ("n_chasers", c_int32), ("r_touch", c_float), ("w_prox", c_float),
        ("s_max_chaser", c_float),
        ("rank", c_int32), ("world_size", c_int32), ("halo_capacity", c_int32),
        ("nccl_unique_id", c_void_p),
    ]


class VgOutputs(ctypes.Structure):
    _fields_ = [
        ("obs", c_void_p), ("reward", c_void_p), ("n_neigh", c_void_p),
        ("n_collide", c_void_p), ("n_touch", c_void_p), ("sector_occ", c_void_p),
        ("agent_id", c_void_p),
    ]


class VgSlabIo(ctypes.Structure):
    _fields_ = [
        ("send_left", c_void_p), ("send_right", c_void_p),
        ("recv_left", c_void_p), ("recv_right", c_void_p),
        ("message_bytes", c_int64), ("left_rank", c_int32), ("right_rank", c_int32),
        ("lo", c_int32), ("hi", c_int32), ("capacity_rows", c_int64),
    ]


class VgPolicyConfig(ctypes.Structure):
    _fields_ = [("obs_dim", c_int32), ("act_lo", c_float * 2), ("act_hi", c_float * 2)]


class VgPolicyOutputs(ctypes.Structure):
    _fields_ = [("mean", c_void_p), ("value", c_void_p), ("action", c_void_p), ("logp", c_void_p)]


class VgRolloutBuffers(ctypes.Structure):
    _fields_ = [("obs", c_void_p), ("action", c_void_p), ("logp", c_void_p),
                ("reward", c_void_p), ("value", c_void_p), ("adv", c_void_p), ("ret", c_void_p)]


class VgWorldInfo(ctypes.Structure):
    _fields_ = [
        ("grid", c_int32), ("cell_size", c_float), ("n_cells", c_int32),
        ("obs_dim", c_int32), ("channels", c_int32), ("occ_words", c_int32),
        ("total_agents", c_int64), ("scratch_bytes", c_int64), ("kernels_per_step", c_int32),
        ("sense_defaults", c_int32),
    ]


#: Every symbol include/vg.h declares, with (restype, argtypes).
SIGNATURES = {
    "vg_abi_version": (c_int32, []),
    "vg_last_error": (c_char_p, []),
    "vg_world_create": (c_int32, [POINTER(VgConfig), POINTER(c_void_p)]),
    "vg_world_destroy": (None, [c_void_p]),
    "vg_world_query": (c_int32, [c_void_p, POINTER(VgWorldInfo)]),
    "vg_bin": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "vg_sense": (c_int32, [c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_reward": (c_int32, [c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_integrate": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "vg_step": (c_int32, [c_void_p, c_void_p, c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_step_host": (c_int32, [c_void_p, c_void_p, c_void_p, POINTER(VgOutputs), c_void_p,
                               c_void_p]),
    "vg_get_bins": (c_int32, [c_void_p, POINTER(c_void_p), POINTER(c_void_p),
                              POINTER(c_void_p), POINTER(c_void_p)]),
    "vg_sync_errors": (c_int32, [c_void_p, c_void_p, POINTER(c_int64)]),
    "vg_slab_plan": (c_int32, [c_int32, c_int32, c_int32, POINTER(c_int32)]),
    "vg_slab_load": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "vg_slab_sense": (c_int32, [c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_slab_begin": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "vg_slab_get_io": (c_int32, [c_void_p, POINTER(VgSlabIo)]),
    "vg_slab_exchange_loopback": (c_int32, [POINTER(c_void_p), c_int32, c_void_p]),
    "vg_sense_columns": (c_int32, [c_void_p, POINTER(VgOutputs), c_int32, c_int32, c_void_p]),
    "vg_slab_interior": (c_int32, [c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_slab_finish": (c_int32, [c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_slab_step": (c_int32, [c_void_p, c_void_p, POINTER(VgOutputs), c_void_p]),
    "vg_nccl_unique_id": (c_int32, [c_void_p, c_int32]),
    "vg_slab_own_count": (c_int32, [c_void_p, c_void_p, POINTER(c_int64)]),
    "vg_policy_create": (c_int32, [POINTER(VgPolicyConfig), POINTER(c_void_p)]),
    "vg_policy_destroy": (None, [c_void_p]),
    "vg_policy_set_weights": (c_int32, [c_void_p, POINTER(c_void_p), c_void_p]),
    "vg_policy_forward": (c_int32, [c_void_p, c_void_p, c_int64, POINTER(VgPolicyOutputs),
                                    ctypes.c_uint64, ctypes.c_uint64, c_void_p]),
    "vg_rollout": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(VgRolloutBuffers),
                             c_int32, ctypes.c_uint64, ctypes.c_uint64, c_float, c_float,
                             c_void_p]),
    "vg_policy_forward_class": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                          POINTER(VgPolicyOutputs), ctypes.c_uint64,
                                          ctypes.c_uint64, c_void_p]),
    "vg_gae": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_float, c_float, c_void_p,
                         c_void_p, c_void_p]),
    "vg_opinion_step": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p,
                                  c_void_p, c_float, c_float, c_void_p]),
    "vg_opinion_sync_errors": (c_int32, [c_void_p, POINTER(c_int64)]),
    "vg_profile_begin": (c_int32, [c_void_p, c_int32]),
    "vg_profile_end": (c_int32, [c_void_p, c_void_p, POINTER(ctypes.c_double),
                                 POINTER(c_int32)]),
}


class VgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libvg.so not found at {LIB_PATH}; build it with "
            "`python -m paper_2207_03945_b200._build` (nvcc, sm_100a). There is no fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != VG_OK:
        raise VgError(status, lib.vg_last_error().decode())
