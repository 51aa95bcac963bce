"""Per-layer time of the MobileNetV2 INT8 block chain (bench.py
measure_mobilenetv2_int8 layers, batch 32): unprotected / FIC (FR input pass) /
FIC with the input checksum reused (no input pass) -- each layer's launch as a
graph of R back-to-back runs after an L2 flush; us per launch (diagnostics)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import BATCH, MBV2_BLOCKS  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402

R = 5


def timed(fn, stream, flush):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(R):
            fn()
    ts = []
    for i in range(4):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return statistics.median(ts)


def main():
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    print(f"{'layer':28s} {'unprotected':>12s} {'fic':>12s} {'fic-reuse':>12s}")
    seed = 900
    tot = [0.0, 0.0, 0.0]
    for bi, (ci, hw, t, co, st) in enumerate(MBV2_BLOCKS):
        e = ci * t
        ho = (hw + 2 - 3) // st + 1
        shapes = [("pw", api.layer_shape(BATCH, ci, hw, hw, e, 1, 1, 1, 1, 0, 0)),
                  ("dw", api.layer_shape(BATCH, e, hw, hw, e, 3, 3, st, st, 1, 1)),
                  ("pw", api.layer_shape(BATCH, e, ho, ho, co, 1, 1, 1, 1, 0, 0))]
        plans = []
        for kind, ls in shapes:
            seed += 1
            if kind == "pw":
                f = api.fill_random_i8(ls.k * ls.c, api.derive_seed(seed, 2)).view(ls.filter_dims())
                mk = lambda ch, ls=ls, f=f: api.ConvPlan(ls, f, ch)  # noqa: E731
            else:
                f = api.fill_random_i8(ls.c * 9, api.derive_seed(seed, 2)).view(ls.c, 1, 3, 3)
                mk = lambda ch, ls=ls, f=f: api.ConvPlanDW(ls, f, ch)  # noqa: E731
            plans.append((kind, ls, mk(0), mk(abi.CHECK_FIC), mk(abi.CHECK_FIC)))
        for li, (kind, ls, pu, pf, pr) in enumerate(plans):
            x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(seed + li, 1)).view(ls.input_dims())
            xin = pu.pack(x)
            nxt = plans[li + 1][2] if li + 1 < len(plans) else None
            out = nxt.packed_buffer() if nxt else torch.zeros(
                ls.n * ((ls.k + 15) // 16 * 16) * (ls.p + 1) * (ls.q + 1) + (1 << 16), dtype=torch.int8, device="cuda")
            row = []
            for pl in (pu, pf, pr):
                ep = pl.epilog_params(0.02, None, True)
                with torch.cuda.stream(stream):
                    pl.run(xin, out, abi.OUT_I8_PACKED, ep=ep, next_plan=nxt)
                torch.cuda.synchronize()
                if pl is pr:
                    abi.call("abed_conv_plan_set_reuse_input_checksum", pl.handle, 1)
                with torch.cuda.stream(stream):
                    row.append(timed(lambda: pl.run(xin, out, abi.OUT_I8_PACKED, ep=ep, next_plan=nxt), stream, flush))
            tot = [a + b for a, b in zip(tot, row)]
            name = f"b{bi} {kind} {ls.c}->{ls.k} {ls.h}x{ls.w} s{ls.stride_h}"
            print(f"{name:28s} " + " ".join(f"{v:12.2f}" for v in row), flush=True)
    print(f"{'total':28s} " + " ".join(f"{v:12.2f}" for v in tot))


if __name__ == "__main__":
    main()
