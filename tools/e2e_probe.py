"""Where the end-to-end (vg_step_host) time goes at c5: pinned H2D of the actions, the
device step, D2H of the reward, and the whole call + sync, each timed alone (CUDA events
and wall clock, medians of 30)."""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import vg_inputs as vi  # noqa: E402
import paper_2207_03945_b200 as vg  # noqa: E402

p = vi.workload(sys.argv[1] if len(sys.argv) > 1 else "c5")
dev = torch.device("cuda", 0)
w = vg.World(p, device=dev)
out = w.alloc_outputs()
st = torch.from_numpy(vi.init_state(p, seed=0)).to(dev)
a_h = torch.from_numpy(vi.actions(p, seed=0, step=0)).pin_memory()
a_d = a_h.to(dev)
r_h = torch.empty(tuple(out.reward.shape), dtype=torch.float32).pin_memory()
s = torch.cuda.current_stream(dev)


def ev(fn, n=30):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def wall(fn, n=30):
    ts = []
    for _ in range(3):
        fn()
        s.synchronize()
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        s.synchronize()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


res = {
    "h2d_actions_us": ev(lambda: a_d.copy_(a_h, non_blocking=True)),
    "d2h_reward_us": ev(lambda: r_h.copy_(out.reward, non_blocking=True)),
    "step_device_us": ev(lambda: w.step(st, a_d, out)),
    "step_host_events_us": ev(lambda: w.step_host(st, a_h, out, r_h)),
    "step_host_wall_us": wall(lambda: w.step_host(st, a_h, out, r_h)),
    "step_device_wall_us": wall(lambda: w.step(st, a_d, out)),
    "empty_sync_wall_us": wall(lambda: None),
}
res["h2d_GBps"] = a_h.numel() * 4 / res["h2d_actions_us"] / 1e3
res["d2h_GBps"] = r_h.numel() * 4 / res["d2h_reward_us"] / 1e3
print({k: round(v, 1) for k, v in res.items()})
