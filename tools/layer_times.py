"""Per-layer kernel time (graph of R back-to-back launches after an L2 flush,
CUDA events / R) for several variants of the bench layers (diagnostics).

    python tools/layer_times.py [--only name,...]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import BATCH, RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402

R = 10


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    variants = [("unprotected", 0, 0, 0), ("fic", abi.CHECK_FIC, 0, 0), ("fic-reuse-rhs", abi.CHECK_FIC, 1, 0),
                ("fic-reuse-novd", abi.CHECK_FIC, 1, 32), ("fic-reuse-nosum", abi.CHECK_FIC, 1, 64),
                ("fic-reuse-none", abi.CHECK_FIC, 1, 96), ("fc", abi.CHECK_FC, 0, 0), ("fic-staged", abi.CHECK_FIC, 0, -1)]
    print(f"{'layer':15s} " + " ".join(f"{v[0]:>15s}" for v in variants) + "   (us per launch)")
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        if only and name not in only:
            continue
        ls = api.layer_shape(BATCH, c, h, w, k, 3, 3, st, st, 1, 1)
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
        row = []
        for vname, checks, reuse, dbg in variants:
            pl = api.ConvPlan(ls, f, checks)
            if dbg < 0:
                pl.set_input_checksum_source(abi.RHS_STAGED)
                dbg = 0
            packed = pl.pack(x)
            out = torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + 65536, dtype=torch.int8, device="cuda")
            ep = pl.epilog_params(0.05, torch.linspace(-2, 2, k), True)
            with torch.cuda.stream(stream):
                pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            torch.cuda.synchronize()
            abi.call("abed_conv_plan_set_reuse_input_checksum", pl.handle, reuse)
            abi.call("abed_debug_set_conv_trace", pl.handle, None, dbg)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(R):
                    pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            ts = []
            for i in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                if i:
                    ts.append(e0.elapsed_time(e1) * 1e3 / R)
            row.append(statistics.median(ts))
        print(f"{name:15s} " + " ".join(f"{t:15.2f}" for t in row))


if __name__ == "__main__":
    main()
