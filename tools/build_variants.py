"""Build tuning variants of libvg.so with -D overrides into build/variants/ (git-ignored).

Usage: python tools/build_variants.py name:-DX=1,-DY=2 [name2:...]
Load one with VG_LIB_VARIANT=name (paper_2207_03945_b200/_lib.py)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2207_03945_b200"))
import _build  # noqa: E402

out = os.path.join(ROOT, "build", "variants")
os.makedirs(out, exist_ok=True)
procs = []
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *[d for d in defs.split(",") if d],
           "-I", os.path.join(ROOT, "include"), "-I", _build.CSRC, *_build.SOURCES,
           "-o", os.path.join(out, f"libvg_{name}.so")]
    procs.append((name, subprocess.Popen(cmd)))
for name, p in procs:
    assert p.wait() == 0, name
    print("built", name)
