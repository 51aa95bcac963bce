"""The HBM-bound kernels once each on ResNet-50 layer1 tensors at batch 32, for
ncu (gpu__time_duration, dram bytes); batch = argv[1] (default 32): gen_filter_checksum (512x512x3x3 filters),
ic_batch_checksum, gen_input_checksum, epilog (i32 -> i8, ReLU), pack_input.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/hbm.csv python tools/profile_hbm.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2006_04984_b200 import abi, api  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    c, h, w, k = 64, 56, 56, 64
    x = api.fill_random_i8(n * c * h * w, api.derive_seed(77, 1)).view(n, c, h, w)
    f4 = api.fill_random_i8(512 * 512 * 9, api.derive_seed(77, 2)).view(512, 512, 3, 3)
    ls = api.layer_shape(n, c, h, w, k, 3, 3, 1, 1, 1, 1)
    acc = torch.randint(-40000, 40000, (n, k, h, w), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        api.gen_filter_checksum(f4)
        api.ic_batch_checksum(x)
        api.gen_input_checksum(x, ls)
        api.epilog(acc, 0.05, torch.linspace(-2, 2, k), True)
        f1 = api.fill_random_i8(k * c * 9, api.derive_seed(77, 3)).view(k, c, 3, 3)
        api.ConvPlan(ls, f1, 0).pack(x)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
