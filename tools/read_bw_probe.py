import torch, statistics, json, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
dev = torch.device('cuda', 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
res = {}
for mb in (51, 400):
    R = 8
    xs = [torch.randint(-100, 100, ((mb << 20) // 8,), dtype=torch.int64, device=dev) for _ in range(R)]
    outs = [torch.empty((), dtype=torch.int64, device=dev) for _ in range(R)]
    def run():
        for i in range(R):
            torch.sum(xs[i], dim=0, out=outs[i])
    run()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    ts = []
    for _ in range(10):
        bench.l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) / R)
    us = statistics.median(ts) * 1e3
    res[f"torch_sum_{mb}MB"] = {"us": round(us, 2), "GBs": round((mb << 20) / (us * 1e-6) / 1e9, 1)}
    del xs
print(json.dumps(res))
