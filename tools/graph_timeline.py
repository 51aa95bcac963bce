"""Timeline of the bench step graph (16 ResNet-50 3x3 layers) from per-CTA
globaltimer stamps: per layer, first CTA start / last CTA exit, kernel span and
the gap to the previous layer (diagnostics).

    python tools/graph_timeline.py [--variant unprotected|fic|fc]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import BATCH, RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="unprotected")
    a = ap.parse_args()
    checks = {"unprotected": 0, "fc": abi.CHECK_FC, "fic": abi.CHECK_FIC}[a.variant]
    layers = []
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        ls = api.layer_shape(BATCH, c, h, w, k, 3, 3, st, st, 1, 1)
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
        pl = api.ConvPlan(ls, f, checks)
        out = torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + 65536, dtype=torch.int8, device="cuda")
        tr = torch.zeros(1024 * 24, dtype=torch.int64, device="cuda")
        layers.append((name, pl, pl.pack(x), out, pl.epilog_params(0.05, torch.linspace(-2, 2, k), True), tr))
    stream = torch.cuda.Stream()

    def step():
        for name, pl, packed, out, ep, tr in layers:
            pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)

    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    for name, pl, packed, out, ep, tr in layers:
        abi.call("abed_debug_set_conv_trace", pl.handle, C.c_void_p(tr.data_ptr()), 0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        flush.zero_()
        g.replay()
    torch.cuda.synchronize()
    for *_, tr in layers:
        tr.zero_()
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph step {e0.elapsed_time(e1) * 1e3:.1f} us ({a.variant})")
    t0 = None
    prev_end = None
    busy = 0.0
    for name, pl, packed, out, ep, tr in layers:
        rows = [r for r in tr.view(-1, 24).cpu().tolist() if r[1] != 0]
        start = min(r[0] for r in rows)
        end = max(r[14] for r in rows)
        if t0 is None:
            t0 = start
        gap = (start - prev_end) / 1e3 if prev_end is not None else 0.0
        span = (end - start) / 1e3
        busy += span
        rel = [r[16] for r in rows if r[16]]
        first = [r[17] for r in rows if r[17]]
        lastmma = [r[18] for r in rows if r[18]]
        epi = [r[19] for r in rows if r[19]]
        extra = ""
        if prev_end is not None and rel:
            import statistics as st
            extra = (f"  | release-prevend {(min(rel) - prev_end) / 1e3:5.2f}  first-ready(med) "
                     f"{(st.median(first) - min(rel)) / 1e3:5.2f}  last-mma(max) {(max(lastmma) - min(rel)) / 1e3:5.2f}"
                     f"  epi-done(max) {(max(epi) - min(rel)) / 1e3:5.2f}  exit(max) {(end - min(rel)) / 1e3:5.2f}")
        print(f"{name:15s} start {(start - t0) / 1e3:7.2f} us  end {(end - t0) / 1e3:7.2f} us  span {span:6.2f} us  "
              f"gap-from-prev-end {gap:6.2f} us  ctas {len(rows)}{extra}")
        prev_end = end
    print(f"sum of kernel spans {busy:.1f} us")


if __name__ == "__main__":
    main()
