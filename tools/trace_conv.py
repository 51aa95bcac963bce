"""Per-CTA clock timeline of the conv kernel for the bench layers (diagnostics).

    python tools/trace_conv.py [--variant unprotected|fc|fic] [--only name,...]

Prints, per layer: event-timed kernel duration, and the median / max over CTAs of
setup, first-stage-ready, last-MMA-issue, epilogue-done (cycles from CTA entry),
summed MMA-warp waits on operand stages and epilogue waits on accumulators, and the
spread of CTA start times (globaltimer).
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import BATCH, RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="unprotected")
    ap.add_argument("--only", default="")
    ap.add_argument("--dbg", type=int, default=0, help="debug flags (bit 0: epilogue skips its work)")
    ap.add_argument("--fresh-rhs", action="store_true", help="FIC: recompute the input checksum every run")
    ap.add_argument("--batch", type=int, default=BATCH)
    a = ap.parse_args()
    checks = {"unprotected": 0, "fc": abi.CHECK_FC, "fic": abi.CHECK_FIC}[a.variant]
    only = set(a.only.split(",")) if a.only else None
    trace = torch.zeros(1024 * 24, dtype=torch.int64, device="cuda")
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        if only and name not in only:
            continue
        ls = api.layer_shape(a.batch, c, h, w, k, 3, 3, st, st, 1, 1)
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
        pl = api.ConvPlan(ls, f, checks)
        packed = pl.pack(x)
        out = torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + 65536, dtype=torch.int8, device="cuda")
        ep = pl.epilog_params(0.05, torch.linspace(-2, 2, k), True)
        abi.call("abed_conv_plan_set_reuse_input_checksum", pl.handle, 0 if a.fresh_rhs else 1)
        for _ in range(3):
            pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep, stream=C.c_void_p(cur.cuda_stream))
            e1.record(cur)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        trace.zero_()
        abi.call("abed_debug_set_conv_trace", pl.handle, C.c_void_p(trace.data_ptr()), a.dbg)
        pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
        torch.cuda.synchronize()
        abi.call("abed_debug_set_conv_trace", pl.handle, None, 0)
        t = trace.view(-1, 24).cpu()
        rows = [r for r in t.tolist() if r[1] != 0]
        i = pl.info
        g0 = min(r[0] for r in rows)

        def med(j):
            v = [r[j] for r in rows]
            return f"{statistics.median(v):>7.0f}/{max(v):>7.0f}"

        starts = [(r[0] - g0) / 1e3 for r in rows]
        print(f"{name:15s} bn={i.block_n:3d} nt={i.n_tiles} mt={i.m_tiles:3d} gps={i.gps} res={i.b_resident} "
              f"ctas={len(rows)} units(max)={max(r[6] for r in rows)} event_us={min(ts):6.2f} | "
              f"setup {med(2)} 1st-copy {med(8)} 1st-ready {med(3)} last-mma {med(4)} prod-done {med(7)} "
              f"epi-done {med(5)} | mma-wait {med(9)} epi-wait {med(10)} last-acc {med(11)} epi-proc {med(12)} mma-tempty-wait {med(13)} rhs-done {med(15)} | "
              f"start spread {max(starts):.2f}us")


if __name__ == "__main__":
    main()
