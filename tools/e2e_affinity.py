"""H2D / D2H bandwidth of pinned buffers with and without the process bound to the GPU's
local CPUs (NVML cpu affinity), and the NUMA layout of the box."""
import os
import subprocess
import sys

import torch

mode = sys.argv[1] if len(sys.argv) > 1 else "none"
if mode == "nvml":
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    pynvml.nvmlDeviceSetCpuAffinity(h)
print(mode, "cpus", len(os.sched_getaffinity(0)), sorted(os.sched_getaffinity(0))[:4], "...")
a = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
r = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
dr = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    d.copy_(a, non_blocking=True); r.copy_(dr, non_blocking=True)
torch.cuda.synchronize()
import time
ts = []
for _ in range(30):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(); d.copy_(a, non_blocking=True); e1.record(); r.copy_(dr, non_blocking=True); e2.record()
    e2.synchronize()
    ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
ts.sort()
h2d, d2h = ts[15]
print(mode, f"h2d {8.388608 / h2d:.1f} GB/s  d2h {4.194304 / d2h:.1f} GB/s")
