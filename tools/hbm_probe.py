"""The HBM-bound kernels of bench.py's hbm_kernels block, run a few times each
(an ncu target): K6 filter checksum, K7 batch checksum, pack_input."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2006_04984_b200 import abi, api  # noqa: E402

n, c, h, w, k = 256, 64, 56, 56, 64
x = api.fill_random_i8(n * c * h * w, api.derive_seed(77, 1)).view(n, c, h, w)
f4 = api.fill_random_i8(512 * 512 * 9, api.derive_seed(77, 2)).view(512, 512, 3, 3)
ls = api.layer_shape(n, c, h, w, k, 3, 3, 1, 1, 1, 1)
f1 = api.fill_random_i8(k * c * 9, api.derive_seed(77, 3)).view(k, c, 3, 3)
plan = api.ConvPlan(ls, f1, 0)
packed = plan.packed_buffer()
sums_f = torch.empty((1, 512, 3, 3), dtype=torch.int32, device="cuda")
sums_x = torch.empty((1, c, h, w), dtype=torch.int32, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for _ in range(3):
    if which in ("all", "k6"):
        abi.call("abed_gen_filter_checksum", f4.data_ptr(), api._dims(f4), sums_f.data_ptr(), st)
    if which in ("all", "k7"):
        abi.call("abed_ic_batch_checksum", x.data_ptr(), api._dims(x), sums_x.data_ptr(), st)
    if which in ("all", "pack"):
        abi.call("abed_pack_input", plan.handle, x.data_ptr(), packed.data_ptr(), st)
torch.cuda.synchronize()
print("ok")
