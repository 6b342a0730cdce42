"""Parity statistics at C2, C3, C4 (sampled replicas) and C5 (sampled rows): banded pairs,
rows resolved by a banded alternative, max errors — for DESIGN.md §5."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import vg_inputs as vi  # noqa: E402
import vg_parity as parity  # noqa: E402
import paper_2207_03945_b200 as vg  # noqa: E402

res = {}
WORKERS = max(1, min(32, len(os.sched_getaffinity(0))))
for name, reps, rows, steps in (("c2", [0], None, 10), ("c3", [0], None, 10),
                                ("c4", [0, 1, 511, 1023], None, 3), ("c5", [0], 4096, 3)):
    p = vi.workload(name)
    w = vg.World(p)
    out = w.alloc_outputs()
    st = torch.from_numpy(vi.init_state(p, seed=11)).cuda()
    agg = {"rows": 0, "banded_pairs": 0, "banded_rows": 0, "alt_rows": 0, "dont_care": 0,
           "max_obs_rel": 0.0, "max_reward_err": 0.0, "max_reward_err_over_tol": 0.0,
           "bound_rows": 0, "steps": steps}
    for t in range(steps):
        w.step(st, torch.from_numpy(vi.actions(p, seed=11, step=t)).cuda(), out)
        torch.cuda.synchronize()
        cur = st.cpu().numpy()
        rws = None if rows is None else np.random.default_rng(t + 1).choice(p.n_agents, rows, replace=False)
        for r in reps:
            g = {k: getattr(out, k)[r].cpu().numpy() for k in
                 ("obs", "reward", "n_neigh", "n_collide", "n_touch", "sector_occ")
                 if getattr(out, k) is not None}
            g = {k: (a.view(np.uint32) if a.dtype == np.int32 else a) for k, a in g.items()}
            s = parity.check_sense(p, cur[r], g, rows=rws, workers=WORKERS)
            for k in s:
                agg[k] = max(agg[k], s[k]) if k.startswith("max") else agg[k] + s[k]
    res[name] = agg
    w.close()
    print(name, agg, flush=True)
json.dump(res, open(os.path.join(ROOT, "profiles", "parity_stats.json"), "w"), indent=1, default=float)
