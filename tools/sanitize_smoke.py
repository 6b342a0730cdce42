"""Small workloads through every kernel (every binning path included): a plain smoke run,
and the input for compute-sanitizer (memcheck / racecheck / synccheck, one tool per
process) where the pool allows it (it is closed on this round's pool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import vg_inputs as vi  # noqa: E402
import paper_2207_03945_b200 as vg  # noqa: E402
from paper_2207_03945_b200 import rl  # noqa: E402
from paper_2207_03945_b200.policy import Policy, action_box  # noqa: E402
from paper_2207_03945_b200.slab import SlabGroup  # noqa: E402

os.environ.setdefault("VG_NO_GRAPH", "0")
# fused replica bin (first three), K3g gather (one and two replicas), K3b' (few cells,
# N > 16,384; and dense clustered cells: its merge-sort fallback), K3b (many cells)
for p, clustered in ((vi.flock_params(300, width=40.0), False),
                     (vi.tag_params(400, width=40.0), False),
                     (vi.flock_params(7, n_replicas=5, width=40.0), False),
                     (vi.flock_params(3000, width=40.0), False),
                     (vi.tag_params(2000, n_replicas=2, width=40.0), False),
                     (vi.flock_params(20000), False),
                     (vi.flock_params(20000), True),        # 16 clusters of ~1250
                     (vi.flock_params(4000, width=400.0, d_v=10.0), False)):
    w = vg.World(p)
    out = w.alloc_outputs()
    st0 = vi.clustered_state(p, seed=1, n_clusters=16, sigma=1.0) if clustered \
        else vi.init_state(p, seed=1)
    st = torch.from_numpy(st0).cuda()
    for t in range(2):
        w.step(st, torch.from_numpy(vi.actions(p, seed=1, step=t)).cuda(), out)
    w.reward(out)
    torch.cuda.synchronize()
    w.sync_errors()
    pl = Policy(w.obs_dim, *action_box(p))
    pl.set_weights(vi.policy_weights(w.obs_dim))
    po = pl.alloc(p.total_agents)
    pl.forward(out.obs.view(-1, w.obs_dim), po, seed=1, step=0)
    torch.cuda.synchronize()
    pl.close()
    w.close()
p = vi.flock_params(2000, width=120.0, d_v=10.0, grid=8)
g = SlabGroup(p, 2)
g.load(torch.from_numpy(vi.init_state(p, seed=2)).cuda())
outs = [w.alloc_outputs() for w in g.worlds]
g.sense(outs)
g.step([torch.zeros((1, p.n_agents, 2), device="cuda") for _ in range(2)], outs)
torch.cuda.synchronize()
g.close()
r = torch.randn(9, 300, device="cuda")
v = torch.randn(10, 300, device="cuda")
rl.gae(r, v, torch.empty_like(r), torch.empty_like(r))
og = {k: torch.from_numpy(a).cuda() for k, a in vi.opinion_graph(200, 8).items()}
rl.opinion_step(og["row_ptr"], og["col"], og["weight"], og["op"], torch.empty_like(og["op"]), 0.3, 0.5)
torch.cuda.synchronize()
print("sanitize smoke ok")
