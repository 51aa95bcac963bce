"""Attribute one bench layer's kernel time with the conv kernel's timing-experiment
flags (abed_debug_set_conv_trace flags; results are NOT valid outputs).  The flags
exist only in a diagnostics build: rm -rf build && ABED_NVCC_EXTRA=-DABED_CONV_DEBUG=1
python -c "from paper_2006_04984_b200 import _build; _build.build()".  Flags:
  0 normal, 1 epilogue skips the TMEM->register->store work, 16 skips only the
  requantise math, 8 MMA-only (epilogue / commits of all but the last 2 units
  skipped).  Per flag: graph of R back-to-back launches after an L2 flush, CUDA
  events / R.

    python tools/epi_probe.py --layer 0 --batch 1024 --checks 0 --flags 0,1,16,8
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--checks", type=int, default=0)
    ap.add_argument("--flags", default="0,1,16,8")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--finalize", action="store_true", help="finalize after every run (inside the timed graph)")
    ap.add_argument("--reuse", action="store_true",
                    help="FIC: keep the first run's input checksum (no in-kernel input pass)")
    a = ap.parse_args()
    name, c, h, w, k, st = RESNET50_3X3[a.layer]
    ls = api.layer_shape(a.batch, c, h, w, k, 3, 3, st, st, 1, 1)
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(1000 + a.layer, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(1000 + a.layer, 2)).view(ls.filter_dims())
    plan = api.ConvPlan(ls, f, a.checks)
    packed = plan.pack(x)
    out = torch.zeros(ls.n * ((k + 15) // 16 * 16) * (ls.p + 1) * (ls.q + 1) + (1 << 16), dtype=torch.int8,
                      device="cuda")
    ep = plan.epilog_params(0.05, torch.linspace(-2.0, 2.0, k).tolist(), True)
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for fl in [int(v) for v in a.flags.split(",")]:
        abi.call("abed_debug_set_conv_trace", plan.handle, None, fl)
        with torch.cuda.stream(stream):
            plan.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            if a.checks:
                plan.finalize()
            if a.reuse:
                abi.call("abed_conv_plan_set_reuse_input_checksum", plan.handle, 1)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(a.reps):
                plan.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
                if a.finalize and a.checks:
                    plan.finalize()
        ts = []
        for i in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) * 1e3 / a.reps)
        res[fl] = round(statistics.mean(ts), 2)
    ops = 2.0 * ls.n * ls.k * ls.p * ls.q * ls.c * 9
    print(name, "batch", a.batch, "checks", a.checks, "reuse" if a.reuse else "", {f"flags{k_}": v for k_, v in res.items()},
          "TOPS@flags0", round(ops / (res[min(res)] * 1e-6) / 1e12, 1) if 0 in res else None)


if __name__ == "__main__":
    main()
