"""One eager pass of the bench workload (16 ResNet-50 3x3 layers, batch 32) for
ncu: `--variant fic|fc|unprotected`, `--layers l1,l3` to restrict.  Also prints a
cuBLAS INT8 GEMM rate (torch._int_mm, 8192^3) as a measured int8 reference.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py --variant fic
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import BATCH, RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="fic")
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--int-mm", action="store_true")
    a = ap.parse_args()
    checks = {"unprotected": 0, "fc": abi.CHECK_FC, "fic": abi.CHECK_FIC}[a.variant]
    only = set(a.only.split(",")) if a.only else None
    layers = []
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        if only and name not in only:
            continue
        ls = api.layer_shape(BATCH, c, h, w, k, 3, 3, st, st, 1, 1)
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(li, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(li, 2)).view(ls.filter_dims())
        pl = api.ConvPlan(ls, f, checks)
        layers.append((name, pl, pl.pack(x), torch.zeros(ls.n * k * (ls.p + 1) * (ls.q + 1) + 65536, dtype=torch.int8,
                                                         device="cuda"), pl.epilog_params(0.05, torch.linspace(-2, 2, k), True)))
    torch.cuda.synchronize()
    for name, pl, *_ in layers:
        i = pl.info
        print(f"{name}: block_n={i.block_n} n_tiles={i.n_tiles} m_tiles={i.m_tiles} gps={i.gps} "
              f"b_resident={i.b_resident} n_phase={i.n_phase} Hl={i.Hl} Wl={i.Wl} smem={i.smem_bytes}")
    for _ in range(a.reps):
        for name, pl, packed, out, ep in layers:
            pl.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            if checks:
                pl.finalize()
    torch.cuda.synchronize()
    if a.int_mm:
        m = 8192
        A = torch.randint(-128, 127, (m, m), dtype=torch.int8, device="cuda")
        B = torch.randint(-128, 127, (m, m), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(A, B)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 10
        for _ in range(n):
            torch._int_mm(A, B)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        print(f"cuBLAS int8 GEMM 8192^3: {2 * m ** 3 / dt / 1e12:.1f} TOPS")


if __name__ == "__main__":
    main()
