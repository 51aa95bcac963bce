import torch, time, json
dev = torch.device("cuda", 0)
res = {}
for mb in (6, 61):
    h = torch.empty(mb << 20, dtype=torch.int8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.int8, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        res[f"{name}_{mb}MB_GBs"] = round((mb << 20) / (min(ts) * 1e-3) / 1e9, 1)
# concurrent h2d 61MB + d2h 44MB on two streams
h1 = torch.empty(61 << 20, dtype=torch.int8).pin_memory(); d1 = torch.empty(61 << 20, dtype=torch.int8, device=dev)
h2 = torch.empty(44 << 20, dtype=torch.int8).pin_memory(); d2 = torch.empty(44 << 20, dtype=torch.int8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
res["concurrent_61in_44out_ms"] = round(min(ts) * 1e3, 3)
print(json.dumps(res))

# write-combined pinned host memory (cudaHostAllocWriteCombined) for the H2D side
try:
    import ctypes
    import numpy as np
    from cuda.bindings import runtime as rt
    nbytes = 61 << 20
    err, ptr = rt.cudaHostAlloc(nbytes, rt.cudaHostAllocWriteCombined)
    assert err == rt.cudaError_t.cudaSuccess, err
    arr = np.ctypeslib.as_array((ctypes.c_int8 * nbytes).from_address(int(ptr)))
    hwc = torch.from_numpy(arr)
    d = torch.empty(nbytes, dtype=torch.int8, device=dev)
    hreg = torch.empty(nbytes, dtype=torch.int8).pin_memory()
    out = {}
    for name, h in (("pinned", hreg), ("write_combined", hwc)):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); d.copy_(h, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        out[f"h2d_61MB_{name}_GBs"] = round(nbytes / (min(ts) * 1e-3) / 1e9, 1)
    out["wc_is_pinned"] = bool(hwc.is_pinned())
    print(json.dumps(out))
except Exception as exc:  # noqa: BLE001
    print(json.dumps({"write_combined": f"unavailable: {exc}"}))
