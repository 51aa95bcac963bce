"""Runs the ABFT GEMM plan once per mode (online operands) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/abft_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_04984_b200 import api  # noqa: E402

m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (25088, 1152, 128)))
a = api.fill_random_i8(m * k, api.derive_seed(91, 1)).view(m, k)
b = api.fill_random_i8(k * n, api.derive_seed(91, 2)).view(k, n)
c = torch.empty((m, n), dtype=torch.int32, device="cuda")
ca = torch.empty((m + 1, n + 1), dtype=torch.int64, device="cuda")
plan = api.AbftPlan(m, n, k)
for mode in (api.ABFT_PLAIN, api.ABFT_FUSED_ROW, api.ABFT_CHECKED):
    plan.run(a, b, c, ca, mode)
    torch.cuda.synchronize()
    plan.run(a, None, c, ca, mode)
    torch.cuda.synchronize()
print("verdicts", [o.status for o in plan.verdicts()])
