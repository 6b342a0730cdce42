"""Where does a small world's step time go?  Per-step CUDA events for c1 / c2 under
different L2 states before each step (measurement study; not the bench contract):
  write   256 MiB fill before each step (bench.py's flush: L2 full of dirty lines)
  wread   the fill, then a 256 MiB read (L2 full of clean lines)
  none    no flush (warm L2)
  batch   100 steps between one event pair (warm, back to back)
Usage: python tools/small_step_probe.py [c1 c2 ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import vg_inputs as vi  # noqa: E402
import paper_2207_03945_b200 as vg  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rd = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for cfg in (sys.argv[1:] or ["c1", "c2"]):
    p = vi.workload(cfg)
    w = vg.World(p)
    out = w.alloc_outputs()
    st = torch.from_numpy(vi.init_state(p)).to(dev)
    acts = [torch.from_numpy(vi.actions(p, step=k)).to(dev) for k in range(4)]
    for k in range(10):
        w.step(st, acts[k % 4], out)
    torch.cuda.synchronize()
    res = {}
    for mode in ("write", "wread", "none"):
        K = 40
        e0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        torch.cuda._sleep(10_000_000)
        for k in range(K):
            if mode != "none":
                flush.fill_(k & 0xFF)
            if mode == "wread":
                rd.sum()
            e0[k].record()
            w.step(st, acts[k % 4], out)
            e1[k].record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in zip(e0, e1))
        res[mode] = round(ts[K // 2], 2)
    K = 100
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(10_000_000)
    a.record()
    for k in range(K):
        w.step(st, acts[k % 4], out)
    b.record()
    torch.cuda.synchronize()
    res["batch"] = round(a.elapsed_time(b) * 1e3 / K, 2)
    print(cfg, "median us per step:", res, flush=True)
    w.close()
