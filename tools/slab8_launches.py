"""c5 split into P = 8 slab worlds in one process (loopback exchange), a few steps: for an
ncu launch list of one slab step's kernels (tools/gpu_* scripts)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import vg_inputs as vi  # noqa: E402
from paper_2207_03945_b200.slab import SlabGroup  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = vi.workload("c5")
st = torch.from_numpy(vi.init_state(p, seed=0)).cuda()
grp = SlabGroup(p, P)
outs = [w.alloc_outputs() for w in grp.worlds]
grp.load(st)
grp.sense(outs)
acts = [torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device="cuda") for _ in range(P)]
for _ in range(3):
    grp.step(acts, outs)
torch.cuda.synchronize()
grp.close()
print("ok")
