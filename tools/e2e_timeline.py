"""Timeline of bench.py's e2e step (pinned H2D -> pack -> FIC conv -> finalize ->
D2H per layer, three streams): CUDA events after every copy / layer, printed
relative to the step start, to see where the step exceeds its PCIe floor."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402

dev = torch.device("cuda", 0)
rb = bench.BATCH
layers = []
for li, (name, c, h, w, k, st) in enumerate(bench.RESNET50_3X3):
    ls = api.layer_shape(rb, c, h, w, k, 3, 3, st, st, 1, 1)
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
    pl = api.ConvPlan(ls, f, abi.CHECK_FIC)
    layers.append({"name": name, "ls": ls, "plan": pl, "packed": pl.packed_buffer(),
                   "ep": pl.epilog_params(0.05, torch.linspace(-2.0, 2.0, k).tolist(), True),
                   "hin": x.cpu().pin_memory(), "din": torch.empty_like(x),
                   "dout": torch.empty(ls.output_dims(), dtype=torch.int8, device=dev),
                   "hout": torch.empty(ls.output_dims(), dtype=torch.int8).pin_memory()})
groups = int(os.environ.get("E2E_GROUPS", "0"))  # >0: copies per group of consecutive layers
if groups:
    os.environ["E2E_ONE_PINNED"] = "1"
if os.environ.get("E2E_ONE_PINNED"):  # carve every host buffer from one pinned block per direction
    tot_in = sum(L["hin"].numel() for L in layers)
    tot_out = sum(L["hout"].numel() for L in layers)
    big_in = torch.empty(tot_in, dtype=torch.int8).pin_memory()
    big_out = torch.empty(tot_out, dtype=torch.int8).pin_memory()
    oi = oo = 0
    for L in layers:
        v = big_in[oi:oi + L["hin"].numel()].view(L["hin"].shape)
        v.copy_(L["hin"])
        L["hin"] = v
        oi += v.numel()
        L["hout"] = big_out[oo:oo + L["hout"].numel()].view(L["hout"].shape)
        oo += L["hout"].numel()
    # matching contiguous device blocks
    dbig_in = torch.empty(tot_in, dtype=torch.int8, device=dev)
    dbig_out = torch.empty(tot_out, dtype=torch.int8, device=dev)
    oi = oo = 0
    for L in layers:
        L["din"] = dbig_in[oi:oi + L["hin"].numel()].view(L["hin"].shape)
        L["in_off"] = oi
        oi += L["hin"].numel()
        L["dout"] = dbig_out[oo:oo + L["hout"].numel()].view(L["hout"].shape)
        L["out_off"] = oo
        oo += L["hout"].numel()
oc_dev = torch.empty(216 * len(layers), dtype=torch.uint8, device=dev)
oc_host = torch.empty(216 * len(layers), dtype=torch.uint8).pin_memory()
order = sys.argv[1].split(",") if len(sys.argv) > 1 else None
idx = [int(i) for i in order] if order else list(range(len(layers)))
s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
sp = C.c_void_p(s_cmp.cuda_stream)


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def step_grouped(marks):
    cur = torch.cuda.current_stream()
    for st_ in (s_in, s_cmp, s_out):
        st_.wait_stream(cur)
    n = len(layers)
    bounds = [round(i * n / groups) for i in range(groups + 1)]
    for gi in range(groups):
        ls_ = list(range(bounds[gi], bounds[gi + 1]))
        a, b = layers[ls_[0]], layers[ls_[-1]]
        i0, i1 = a["in_off"], b["in_off"] + b["hin"].numel()
        o0, o1 = a["out_off"], b["out_off"] + b["hout"].numel()
        with torch.cuda.stream(s_in):
            dbig_in[i0:i1].copy_(big_in[i0:i1], non_blocking=True)
        s_cmp.wait_stream(s_in)
        for i in ls_:
            L = layers[i]
            L["plan"].pack(L["din"], L["packed"], stream=sp)
            L["plan"].run(L["packed"], L["dout"], abi.OUT_I8_NCHW, ep=L["ep"], stream=sp)
            abi.call("abed_conv_plan_finalize", L["plan"].handle, oc_dev[i * 216:].data_ptr(), sp)
        s_out.wait_stream(s_cmp)
        with torch.cuda.stream(s_out):
            big_out[o0:o1].copy_(dbig_out[o0:o1], non_blocking=True)
    with torch.cuda.stream(s_out):
        s_out.wait_stream(s_cmp)
        oc_host.copy_(oc_dev, non_blocking=True)
    for st_ in (s_in, s_cmp, s_out):
        cur.wait_stream(st_)


def step(marks):
    if groups:
        return step_grouped(marks)
    cur = torch.cuda.current_stream()
    for st_ in (s_in, s_cmp, s_out):
        st_.wait_stream(cur)
    for i in idx:
        L = layers[i]
        with torch.cuda.stream(s_in):
            L["din"].copy_(L["hin"], non_blocking=True)
            marks.append((f"h2d {L['name']} {L['hin'].numel() >> 10} KB", ev(s_in)))
        s_cmp.wait_stream(s_in)
        marks.append((f"cmp-start {L['name']}", ev(s_cmp)))
        L["plan"].pack(L["din"], L["packed"], stream=sp)
        marks.append((f"pack {L['name']}", ev(s_cmp)))
        L["plan"].run(L["packed"], L["dout"], abi.OUT_I8_NCHW, ep=L["ep"], stream=sp)
        marks.append((f"conv {L['name']}", ev(s_cmp)))
        abi.call("abed_conv_plan_finalize", L["plan"].handle, oc_dev[i * 216:].data_ptr(), sp)
        marks.append((f"cmp {L['name']}", ev(s_cmp)))
        s_out.wait_stream(s_cmp)
        with torch.cuda.stream(s_out):
            L["hout"].copy_(L["dout"], non_blocking=True)
            marks.append((f"d2h {L['name']} {L['hout'].numel() >> 10} KB", ev(s_out)))
    with torch.cuda.stream(s_out):
        s_out.wait_stream(s_cmp)
        oc_host.copy_(oc_dev, non_blocking=True)
    for st_ in (s_in, s_cmp, s_out):
        cur.wait_stream(st_)


for _ in range(3):
    step([])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step([])
ts = []
for _ in range(10):
    e0 = ev(torch.cuda.current_stream())
    g.replay()
    e1 = ev(torch.cuda.current_stream())
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"graph_step_ms_min": round(min(ts), 3), "graph_step_ms_mean": round(sum(ts) / len(ts), 3)}))
marks = []
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
bench.l2_flush(flush)
e0 = ev(torch.cuda.current_stream())
step(marks)
e1 = ev(torch.cuda.current_stream())
torch.cuda.synchronize()
for name, e in marks:
    print(f"{e0.elapsed_time(e) * 1e3:9.1f} us  {name}")
print(json.dumps({"step_ms": round(e0.elapsed_time(e1), 3)}))
