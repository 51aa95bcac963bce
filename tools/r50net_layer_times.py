"""Per-layer time of the whole-network ResNet-50 INT8 block (bench.py
resnet50_chains, batch 32): unprotected / FIC (FR) / FIC with the input checksum
reused (no input pass).  Distinct layer shapes only, each as a graph of R
back-to-back launches after an L2 flush; us per launch (diagnostics)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import BATCH, resnet50_chains  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402

R = 10


def main():
    stream = torch.cuda.Stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    seen = {}
    for chain in resnet50_chains(BATCH):
        for ls in chain:
            key = (ls.c, ls.h, ls.k, ls.r, ls.stride_h)
            seen[key] = seen.get(key, (ls, 0))[0], seen.get(key, (ls, 0))[1] + 1
    print(f"{'layer (c h k r s) x count':30s} {'unprotected':>12s} {'fic':>12s} {'fic-reuse':>12s} {'info':>s}")
    tot = [0.0, 0.0, 0.0]
    for li, ((c, h, k, r, st), (ls, cnt)) in enumerate(seen.items()):
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
        row = []
        info = ""
        for checks, reuse in ((0, 0), (abi.CHECK_FIC, 0), (abi.CHECK_FIC, 1)):
            pl = api.ConvPlan(ls, f, checks)
            packed = pl.pack(x)
            out = torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + 65536, dtype=torch.int8, device="cuda")
            ep = pl.epilog_params(0.05, torch.linspace(-2, 2, k), True)
            with torch.cuda.stream(stream):
                pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            torch.cuda.synchronize()
            abi.call("abed_conv_plan_set_reuse_input_checksum", pl.handle, reuse)
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
            if checks == 0:
                inf = pl.info
                info = f"bn={inf.block_n} nt={inf.n_tiles} mt={inf.m_tiles}"
        tot = [a + b * cnt for a, b in zip(tot, row)]
        name = f"{c} {h} {k} {r}x{r} s{st} x{cnt}"
        print(f"{name:30s} " + " ".join(f"{v:12.2f}" for v in row) + "  " + info, flush=True)
    print(f"{'total (x count)':30s} " + " ".join(f"{v:12.2f}" for v in tot))


if __name__ == "__main__":
    main()
