"""ncu target: the c5 world as 8 slab worlds on one GPU, stepped 4 times (per-kernel launch list of slab mode)."""
import sys, torch
import os; sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import vg_inputs as vi
from paper_2207_03945_b200.slab import SlabGroup
p = vi.workload("c5")
st = torch.from_numpy(vi.init_state(p, seed=0)).cuda()
grp = SlabGroup(p, 8)
outs = [w.alloc_outputs() for w in grp.worlds]
grp.load(st); grp.sense(outs)
acts = [torch.zeros((1, p.n_agents, 2), dtype=torch.float32, device="cuda") for _ in range(8)]
for _ in range(4):
    grp.step(acts, outs)
torch.cuda.synchronize()
