"""Sense time of a 10^6-agent flock world vs a tag world of the same density (tag reads float4 candidates and 2 channels)."""
import sys, torch
sys.path[:0] = ["/root/repo"]
import vg_inputs as vi, paper_2207_03945_b200 as vg
for env in ("flock", "tag"):
    mk = vi.flock_params if env == "flock" else vi.tag_params
    kw = {} if env == "flock" else {"n_chasers": 100_000}
    p = mk(1_000_000, width=vi.C5_WIDTH, d_v=10.0, grid=136, **kw)
    w = vg.World(p); out = w.alloc_outputs()
    st = torch.from_numpy(vi.init_state(p, seed=0)).cuda()
    w.bin(st)
    for _ in range(3): w.sense(out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): w.sense(out)
    e1.record(); torch.cuda.synchronize()
    print(env, "sense ms", e0.elapsed_time(e1) / 10, "n_neigh", out.n_neigh.float().mean().item())
    w.close()
