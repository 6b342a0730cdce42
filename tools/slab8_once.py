"""Run the c5 world split into 8 slabs (loopback exchange) for a few steps — the command profiled by ncu for the slab launch list."""
import sys, os, torch
sys.path[:0] = ["/root/repo"]
import vg_inputs as vi
from paper_2207_03945_b200.slab import SlabGroup
p = vi.workload("c5")
st = torch.from_numpy(vi.init_state(p, seed=0)).cuda()
grp = SlabGroup(p, 8)
outs = [w.alloc_outputs() for w in grp.worlds]
grp.load(st); grp.sense(outs)
acts = [torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device="cuda") for _ in range(8)]
for _ in range(3): grp.step(acts, outs)
torch.cuda.synchronize()
