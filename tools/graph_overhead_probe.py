"""Platform probe: device time per replay of a CUDA graph of k tiny kernels (torch add_ on
a 1-element tensor), replayed back to back; and k eager launches.  Separates graph-node
latency from our kernels' own time for launch-bound small worlds.
Usage: python tools/graph_overhead_probe.py"""
import torch

x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
for k in (1, 2, 3, 5, 8):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(k):
                x.add_(1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(200):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    gt = a.elapsed_time(b) * 1e3 / 200
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(200):
        for _ in range(k):
            x.add_(1)
    b.record()
    torch.cuda.synchronize()
    et = a.elapsed_time(b) * 1e3 / 200
    print(f"k={k}: graph replay {gt:.2f} us, eager {et:.2f} us", flush=True)
