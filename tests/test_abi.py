"""The C-ABI library loads and exports every symbol include/vg.h declares; configuration
validation (synchronous, no device needed) rejects invalid fields by name.  No GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import vg_inputs as vi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2207_03945_b200 import _lib
    declared = _declared()
    assert "vg_step" in declared and "vg_world_create" in declared
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vg_\w+)", nm))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert s in _lib.SIGNATURES, f"binding lacks {s}"
        getattr(_lib.lib, s)


def test_abi_version():
    from paper_2207_03945_b200 import _lib
    assert _lib.lib.vg_abi_version() == 3


def test_struct_layout_matches_header():
    # The ctypes mirror must have the C layout: compile a tiny C program printing sizeof /
    # offsetof with gcc and compare.
    from paper_2207_03945_b200 import _lib
    prog = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "vg.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu\n", sizeof(vg_config), offsetof(vg_config, nccl_unique_id),
             offsetof(vg_config, n_chasers), sizeof(vg_outputs), sizeof(vg_world_info),
             offsetof(vg_world_info, total_agents));
      return 0;
    }"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = list(map(int, subprocess.run([exe], capture_output=True, text=True,
                                           check=True).stdout.split()))
    exp = [ctypes.sizeof(_lib.VgConfig), _lib.VgConfig.nccl_unique_id.offset,
           _lib.VgConfig.n_chasers.offset, ctypes.sizeof(_lib.VgOutputs),
           ctypes.sizeof(_lib.VgWorldInfo), _lib.VgWorldInfo.total_agents.offset]
    assert got == exp


@pytest.mark.parametrize("field,value,needle", [
    ("n_agents", 0, "n_agents"), ("d_v", 60.0, "d_v"), ("d_r", 6.0, "d_r"),
    ("fov", 7.0, "fov"), ("v", 129, "v:"), ("theta_max", 4.0, "theta_max"),
    ("s_min", 0.6, "s_min"), ("a_max", 0.0, "a_max"), ("grid", 10, "grid"),
    ("grid", 2, "grid"), ("d_peak", 0.4, "d_peak"), ("c_collide", -1.0, "c_collide"),
    # (N - 1) x max per-pair reward must fit the 2^-32 fixed-point sum (< 2^31, A16b)
    ("c_collide", 5e5, "fixed-point"), ("c_near", 5e5, "fixed-point"),
])
def test_config_validation_names_field(field, value, needle):
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import _lib
    c = vg.config_from_params(vi.workload("c2"))
    setattr(c, field, value)
    h = ctypes.c_void_p()
    st = _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h))
    assert st == _lib.VG_EINVAL
    assert needle in _lib.lib.vg_last_error().decode()
    assert not h.value


def test_tag_validation():
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import _lib
    c = vg.config_from_params(vi.workload("c3"))
    c.n_chasers = 10001
    h = ctypes.c_void_p()
    assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL
    assert "n_chasers" in _lib.lib.vg_last_error().decode()
    c = vg.config_from_params(vi.workload("c3"))
    c.v = 65                                   # 2 channels x 65 > 128 slots
    assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL


def test_unbuilt_modes_rejected():
    import paper_2207_03945_b200 as vg
    from paper_2207_03945_b200 import _lib
    c = vg.config_from_params(vi.workload("c2"))
    c.vision = 2
    h = ctypes.c_void_p()
    assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL
    assert "vision" in _lib.lib.vg_last_error().decode()
    # ray vision needs cell size >= (d_v + d_r)(1 + 2^-12)
    c = vg.config_from_params(vi.flock_params(100, width=100.0, d_v=10.0, grid=9, d_r=1.2,
                                              vision="ray"))
    assert _lib.lib.vg_world_create(ctypes.byref(c), ctypes.byref(h)) == _lib.VG_EINVAL
    assert "ray vision" in _lib.lib.vg_last_error().decode()


def test_null_arguments():
    from paper_2207_03945_b200 import _lib
    assert _lib.lib.vg_opinion_step(None, None, None, 4, 0, None, None, 0.1, 0.1,
                                    None) == _lib.VG_EINVAL
    assert _lib.lib.vg_world_create(None, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_bin(None, None, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_step(None, None, None, None, None) == _lib.VG_EINVAL


def test_nccl_unique_id_host_only():
    # vg_nccl_unique_id loads libnccl at run time (no GPU needed): 128 bytes, fresh each call;
    # a short buffer is VG_EINVAL.  If libnccl cannot be loaded the call reports VG_ENCCL.
    from paper_2207_03945_b200 import _lib
    import paper_2207_03945_b200 as vg
    buf = ctypes.create_string_buffer(64)
    assert _lib.lib.vg_nccl_unique_id(buf, 64) == _lib.VG_EINVAL
    try:
        a, b = vg.nccl_unique_id(), vg.nccl_unique_id()
    except vg.VgError as e:
        assert "VG_ENCCL" in str(e)
        return
    assert len(a) == 128 and a != b


def test_new_entry_points_reject_null():
    from paper_2207_03945_b200 import _lib
    assert _lib.lib.vg_sense_columns(None, None, 0, 1, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_slab_step(None, None, None, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_slab_interior(None, None, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_policy_forward_class(None, None, 0, 0, 0, 0, None, 0, 0, None) == _lib.VG_EINVAL
    assert _lib.lib.vg_rollout(None, None, None, None, None, 1, 0, 0, 0.9, 0.9, None) == _lib.VG_EINVAL
