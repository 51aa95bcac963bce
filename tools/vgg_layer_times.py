"""Per-layer time of the VGG-16 FP16 block (bench.py measure_vgg16_fp16 layers,
batch 64): unprotected / FIC / FIC with the input checksum reused (no FR pass) /
FC.  One graph of R launches per (layer, variant) after an L2 flush; us per launch."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import VGG16_3X3, VGG_BATCH  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402

R = 5


def main():
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    variants = [("unprotected", 0, 0), ("fic", abi.CHECK_FIC, 0), ("fic-reuse", abi.CHECK_FIC, 1), ("fc", abi.CHECK_FC, 0)]
    print(f"{'layer':10s} " + " ".join(f"{v[0]:>12s}" for v in variants) + "   (us per launch)")
    tot = [0.0] * len(variants)
    for name, c, hw, k in VGG16_3X3:
        ls = api.layer_shape(VGG_BATCH, c, hw, hw, k, 3, 3, 1, 1, 1, 1)
        x = torch.empty(ls.input_dims(), dtype=torch.float32, device="cuda").uniform_(-1, 1, generator=gen)
        f = torch.empty(ls.filter_dims(), dtype=torch.float32, device="cuda").uniform_(-1, 1, generator=gen) * 0.05
        out = torch.zeros((VGG_BATCH * ((k + 15) // 16 * 16) * (ls.p + 1) * (ls.q + 1) + (1 << 16)) * 2,
                          dtype=torch.int8, device="cuda")
        row = []
        packed = None
        for vname, checks, reuse in variants:
            pl = api.ConvPlanH(ls, f, abi.F16, checks, 1e30, 1e30)
            if packed is None:
                packed = pl.pack(x)
            ep = pl.epilog_params(1.0, None, True)
            with torch.cuda.stream(stream):
                pl.run(packed, out, abi.OUT_H_PACKED, ep=ep)
            torch.cuda.synchronize()
            abi.call("abed_conv_plan_set_reuse_input_checksum", pl.handle, reuse)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(R):
                    pl.run(packed, out, abi.OUT_H_PACKED, ep=ep)
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
            row.append(statistics.median(ts))
            del pl
        del x
        tot = [a + b for a, b in zip(tot, row)]
        print(f"{name:10s} " + " ".join(f"{t:12.2f}" for t in row), flush=True)
    print(f"{'total':10s} " + " ".join(f"{t:12.2f}" for t in tot))


if __name__ == "__main__":
    main()
