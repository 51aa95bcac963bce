"""Early perf probe: per-layer time of the fused conv (unprotected / FC / FIC) on cfg2 shapes."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_04984_b200 import abi

LAYERS = [  # ResNet-50 3x3 convs, batch 32
    ("l1", (32, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)),
    ("l2.0", (32, 128, 56, 56, 128, 3, 3, 2, 2, 1, 1)),
    ("l2", (32, 128, 28, 28, 128, 3, 3, 1, 1, 1, 1)),
    ("l3.0", (32, 256, 28, 28, 256, 3, 3, 2, 2, 1, 1)),
    ("l3", (32, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1)),
    ("l4.0", (32, 512, 14, 14, 512, 3, 3, 2, 2, 1, 1)),
    ("l4", (32, 512, 7, 7, 512, 3, 3, 1, 1, 1, 1)),
]


def bench(ls, checks, iters=50, out_mode=abi.OUT_I8_PACKED, force_bn=0):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, device="cuda", generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, device="cuda", generator=g)
    plan = C.c_void_p()
    abi.call("abed_conv_plan_create", C.byref(ls), f.data_ptr(), checks, force_bn, C.byref(plan))
    info = abi.PlanInfo()
    abi.call("abed_conv_plan_info", plan, C.byref(info))
    packed = torch.empty(info.packed_input_bytes, dtype=torch.int8, device="cuda")
    abi.call("abed_pack_input", plan, x.data_ptr(), packed.data_ptr(), None)
    out = torch.zeros(ls.n * ls.k * ls.p * ls.q * 4 + (1 << 20), dtype=torch.int8, device="cuda")
    od = torch.zeros(512, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def step():
        abi.call("abed_conv_plan_run", plan, packed.data_ptr(), None, out_mode, out.data_ptr(), None, -1, 0, st)
        if checks:
            abi.call("abed_conv_plan_finalize", plan, od.data_ptr(), st)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    abi.call("abed_conv_plan_destroy", plan)
    return ms, info


only = sys.argv[1:]
for name, dims in LAYERS:
    if only and name not in only:
        continue
    ls = abi.layer_shape(*dims)
    ops = 2 * ls.n * ls.k * ls.p * ls.q * ls.c * ls.r * ls.s
    row = [name]
    for checks in (0, abi.CHECK_FC, abi.CHECK_FIC):
        ms, info = bench(ls, checks)
        row.append(f"ck{checks}: {ms*1e3:7.1f}us {ops/ms/1e9:7.1f}TOPS bn={info.block_n} nt={info.n_tiles} mt={info.m_tiles} res={info.b_resident} gps={info.gps}")
    print(" | ".join(row), flush=True)
