"""Single-GPU estimate of the slab-mode (c5 split over P ranks) per-rank step: P slab
worlds stepped with the loopback exchange on one device (kernels of all P ranks serialised,
so GPU time / P ~ one rank's kernels), plus the host enqueue time of one rank's
begin + interior + finish calls.  NCCL transfer time is not included (one GPU)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import vg_inputs as vi  # noqa: E402
from paper_2207_03945_b200.slab import SlabGroup  # noqa: E402

res = {}
p = vi.workload("c5")
st = torch.from_numpy(vi.init_state(p, seed=0)).cuda()
for P in (2, 4, 8):
    grp = SlabGroup(p, P)
    outs = [w.alloc_outputs() for w in grp.worlds]
    grp.load(st)
    grp.sense(outs)
    acts = []
    for w, o in zip(grp.worlds, outs):
        a = torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device="cuda")
        acts.append(a)
    for _ in range(3):
        grp.step(acts, outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 10
    e0.record()
    for _ in range(K):
        grp.step(acts, outs)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / K
    w = grp.worlds[0]
    t0 = time.perf_counter()
    for _ in range(K):
        w.slab_begin(acts[0])
        w.slab_interior(outs[0])
        w.slab_finish(outs[0])
    host_ms = (time.perf_counter() - t0) * 1e3 / K
    torch.cuda.synchronize()
    res[P] = {"group_gpu_ms": gpu_ms, "per_rank_gpu_ms": gpu_ms / P, "host_enqueue_ms": host_ms,
              "est_agent_steps_per_s": p.n_agents / (max(gpu_ms / P, host_ms) / 1e3)}
    print(P, res[P], flush=True)
    grp.close()
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "slab_timing.json"), "w"), indent=1)
