"""bench.py's hbm_kernels block alone (K6 filter checksum, K7 batch checksum,
pack_input), printed as one JSON line: run it under different tuning
environment variables (ABED_COLSUM_MAX_CLUSTER) to compare launch shapes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
r = bench.measure_hbm_kernels(dev, stream, flush, bench.measured_peaks())
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("ABED_")},
                  **{k: (v["us"], v["frac_of_hbm"]) for k, v in r["kernels"].items()}}))
