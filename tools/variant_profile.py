"""One bench layer in one plan variant, run back to back (an ncu target).

    python tools/variant_profile.py --layer 0 --checks 8 [--iters 20] [--batch 32]

checks: ABED_CHECK_* bits (1 FC, 2 FIC, 4 IC, 8 ICBatch); the run is exactly what
bench.py times for that variant (OUT_I8_PACKED, bias linspace(-2,2), scale 0.05,
ReLU) plus the plan's finalize.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import RESNET50_3X3  # noqa: E402
from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--checks", type=int, default=abi.CHECK_FIC)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=32)
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
    for _ in range(a.iters):
        plan.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
        if a.checks:
            plan.finalize()
    torch.cuda.synchronize()
    print(name, [o.status for o in plan.outcomes()] if a.checks else "")


if __name__ == "__main__":
    main()
