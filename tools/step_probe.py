"""Diagnostics: the 16-layer FIC step with and without its verdict launch (and the
unprotected step), captured like bench.py (PDL chain, L2 flush before each step,
CUDA events) -- separates the per-pass verdict cost from the kernels'.

    python tools/step_probe.py [--batch 32]
"""
import argparse
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
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    layers = []
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        ls = api.layer_shape(a.batch, c, h, w, k, 3, 3, st, st, 1, 1)
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(1000 + li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(1000 + li, 2)).view(ls.filter_dims())
        L = {"fic": api.ConvPlan(ls, f, abi.CHECK_FIC), "unp": api.ConvPlan(ls, f, 0)}
        L["packed"] = L["unp"].pack(x)
        L["out"] = torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + (1 << 16), dtype=torch.int8, device="cuda")
        bias = torch.linspace(-2.0, 2.0, k).tolist()
        L["ep"] = {v: L[v].epilog_params(0.05, bias, True) for v in ("fic", "unp")}
        layers.append(L)
    ps = api.PlanSet([L["fic"] for L in layers])
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step(v, fin):
        for L in layers:
            L[v].run(L["packed"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"][v])
        if fin:
            ps.finalize()

    graphs = {}
    for key, (v, fin) in {"unprotected": ("unp", False), "fic_no_verdict": ("fic", False),
                          "fic": ("fic", True)}.items():
        with torch.cuda.stream(stream):
            step(v, fin)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(v, fin)
        graphs[key] = g
    res = {}
    for key, g in graphs.items():
        ts = []
        for i in range(a.steps + 3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        res[key] = round(statistics.mean(ts), 2)
    print({k: v for k, v in res.items()}, "us per step;",
          "verdict", round(res["fic"] - res["fic_no_verdict"], 2), "us;",
          "FIC kernels vs unprotected", round(100 * (res["fic_no_verdict"] / res["unprotected"] - 1), 2), "%")


if __name__ == "__main__":
    main()
