"""Per-node cost of dependent kernels in a CUDA graph on this GPU (launch-latency floor)."""
import torch

x = torch.zeros(1024, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for n in (32, 320):
        g = torch.cuda.CUDAGraph()
        x.add_(1)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1)
        for _ in range(5):
            g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            g.replay()
        e1.record(s)
        s.synchronize()
        print(f"{n} tiny dependent kernels per graph: {1000 * e0.elapsed_time(e1) / 20 / n:.2f} us per kernel")
