"""Back-to-back device time per launch of the optimiser kernels at the TD3 parameter counts (the
latency regime): Adam / Polyak over the configs[1] actor (124 822) and twin critic (2 x 72 193)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_17496_b200 as pk
torch.cuda.set_device(0)
for n in (124_822, 144_386, 1_079_000, 5_080_603):
    f = dict(dtype=torch.float32, device="cuda")
    p, g, m, v = torch.randn(n, **f), torch.randn(n, **f) * 1e-3, torch.zeros(n, **f), torch.zeros(n, **f)
    t = torch.zeros(2, dtype=torch.int64, device="cuda")
    tg = p.clone()
    res = {}
    for name, fn in (("adam", lambda: pk.adam(p, g, m, v, t, 1e-4)), ("polyak", lambda: pk.polyak(tg, p, 0.005))):
        for _ in range(10): fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) * 1000 / 20, 2)
    print(n, res)
