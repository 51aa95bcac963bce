"""Generates tests/golden/golden.json from the REFERENCE implementation itself
(oracle/_ref/libabed_ref*.so, compiled from /root/reference/proj/include by
oracle/Makefile).  Run here, where the reference tree exists:

    make -C oracle && python tests/golden/make_golden.py

The fixture stores, per case, the exact scalars and a sha256 of every output
tensor (raw little-endian bytes), so tests can pin the C oracle and the GPU
library against the reference without the reference being present.
Data convention: input = SplitMix64(derive_seed(seed, 1)), filters =
SplitMix64(derive_seed(seed, 2)) (abed_main.cpp:143-165 make_data_tensor).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle  # noqa: E402

OUT = os.path.join(HERE, "golden.json")

# (n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w), seed
CONV_CASES = [
    ((1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1), 7),      # cfg1 (BASELINE configs[0]); CLI seed 7 (cli_test.cpp:48)
    ((2, 4, 8, 8, 3, 3, 3, 2, 2, 1, 1), 21),          # convolution_test.cpp:42-48 shape
    ((1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1), 3),         # faults_test.cpp:12 small_shape
    ((2, 32, 9, 11, 16, 3, 3, 1, 1, 1, 1), 5),
    ((3, 16, 10, 10, 24, 3, 3, 1, 1, 1, 1), 6),
    ((2, 64, 16, 16, 128, 3, 3, 2, 2, 1, 1), 8),      # stride-2 (ResNet layerN.0 pattern)
    ((2, 128, 14, 14, 256, 3, 3, 1, 1, 1, 1), 9),
    ((2, 256, 7, 7, 512, 3, 3, 1, 1, 1, 1), 10),
    ((2, 64, 16, 16, 64, 1, 1, 1, 1, 0, 0), 11),      # pointwise
    ((1, 16, 10, 10, 32, 5, 5, 1, 1, 2, 2), 12),
    ((2, 3, 7, 9, 5, 3, 3, 1, 2, 0, 1), 13),          # ragged: odd strides/pads, C and K not multiples of 16
    ((1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0), 14),          # degenerate minimum (checksum_test.cpp:401)
    ((4, 3, 6, 6, 2, 3, 3, 1, 1, 1, 1), 15),          # checksum_test.cpp:360 IcBatch shape
    ((32, 64, 14, 14, 64, 3, 3, 1, 1, 1, 1), 16),     # batch 32 (ICBatch digits > 1 plane)
]

CAMPAIGN_CFG1 = (1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs,
            "lhs_f": o.lhs_f, "rhs_f": o.rhs_f}


def data(ref, ls, seed):
    x = ref.random_i8(ls.n * ls.c * ls.h * ls.w, ref.derive_seed(seed, 1)).reshape(ls.input_dims())
    f = ref.random_i8(ls.k * ls.c * ls.r * ls.s, ref.derive_seed(seed, 2)).reshape(ls.filter_dims())
    return x, f


def conv_case(ref, dims, seed):
    ls = ref.layer_shape(*dims)
    x, f = data(ref, ls, seed)
    conv = ref.conv_i8(x, f, ls)
    nkpq = conv.size
    bias = np.linspace(-3.0, 3.0, ls.k).astype(np.float32)
    case = {"dims": list(dims), "seed": seed, "conv_sha": sha(conv), "conv_sum": int(conv.astype(np.int64).sum()),
            "conv_first": conv.ravel()[:8].tolist(),
            "epilog_relu_sha": sha(ref.epilog(conv, 0.05, np.zeros(ls.k, np.float32))),
            "epilog_bias_sha": sha(ref.epilog(conv, 0.0123, bias)),
            "epilog_ident_sha": sha(ref.epilog(conv, 0.0123, bias, relu=False)),
            "epilog_f32_sha": sha(ref.epilog(conv, 0.0123, bias, relu=False, out_f32=True))}
    fc = ref.gen_filter_checksum(f)
    planes = ref.decompose_checksum_filters(fc)
    extra = ref.recombine_extra_fmaps(ref.conv_checksum_planes(x, ls, planes))
    ic = ref.gen_input_checksum(x, ls)
    batch = ref.ic_batch_checksum(x)
    bext = ref.conv_batch_checksum(batch, f, ls)
    case.update({"fc_sha": sha(fc), "planes_sha": sha(planes), "extra_sha": sha(extra), "ic_sha": sha(ic),
                 "fic_dot": ref.fic_dot(fc, ic), "batch_sha": sha(batch), "batch_extra_sha": sha(bext)})
    case["verify_pass"] = {"fc": outcome(ref.fc_verify(conv, extra)), "ic": outcome(ref.ic_verify_k(conv, f, ic)),
                           "icbatch": outcome(ref.ic_batch_verify(conv, bext)),
                           "fic": outcome(ref.fic_verify(conv, ref.fic_dot(fc, ic)))}
    # one flipped ConvOut element (faults.hpp:230-233 semantics)
    key, bit = (nkpq * 5) // 7, 9
    bad = conv.copy().ravel()
    bad.view(np.uint32)[key] ^= np.uint32(1 << bit)
    bad = bad.reshape(conv.shape)
    case["flip"] = {"key": key, "bit": bit}
    case["verify_flip"] = {"fc": outcome(ref.fc_verify(bad, extra)), "ic": outcome(ref.ic_verify_k(bad, f, ic)),
                           "icbatch": outcome(ref.ic_batch_verify(bad, bext)),
                           "fic": outcome(ref.fic_verify(bad, ref.fic_dot(fc, ic)))}
    case["plan"] = {k: getattr(ref.plan_precision(ls), k) for k, _ in ref.plan_precision(ls)._fields_}
    if ls.n * ls.k * ls.p * ls.q < 2_000_000:
        out, cs, nic = ref.fused_conv_epilog(x, f, ls, 0.02, bias, checksum=True,
                                             next_ls=ref.layer_shape(ls.n, ls.k, ls.p, ls.q, 2, 3, 3, 1, 1, 1, 1))
        case["fused"] = {"out_sha": sha(out), "checksum": cs, "next_ic_sha": sha(nic)}
    return case


def float_cases(ref):
    res = []
    for dims, seed, integers in [((1, 3, 6, 6, 4, 3, 3, 1, 1, 1, 1), 91, False), ((1, 2, 6, 6, 3, 3, 3, 1, 1, 1, 1), 90, True),
                                 ((2, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1), 92, False)]:
        ls = ref.layer_shape(*dims)
        if integers:
            x = ref.random_i8(ls.n * ls.c * ls.h * ls.w, seed).astype(np.float32).reshape(ls.input_dims())
            f = ref.random_i8(ls.k * ls.c * ls.r * ls.s, seed + 1).astype(np.float32).reshape(ls.filter_dims())
        else:
            x = ref.random_f32(ls.n * ls.c * ls.h * ls.w, ref.derive_seed(seed, 1)).reshape(ls.input_dims())
            f = ref.random_f32(ls.k * ls.c * ls.r * ls.s, ref.derive_seed(seed, 2)).reshape(ls.filter_dims())
        conv = ref.conv_f32(x, f, ls)
        fs = ref.filter_checksum_f64(f)
        ins = ref.input_checksum_f64(x, ls)
        res.append({"dims": list(dims), "seed": seed, "integers": integers, "x_sha": sha(x), "f_sha": sha(f),
                    "conv_sha": sha(conv), "fs_sha": sha(fs), "is_sha": sha(ins)})
    return res


def trial_cases(ref):
    res = []
    ls = ref.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    ones_x = np.ones(ls.input_dims(), np.int8)
    ones_f = np.ones(ls.filter_dims(), np.int8)
    xr, fr = data(ref, ls, 4242)
    for name, x, f in [("ones", ones_x, ones_f), ("random", xr, fr)]:
        for scheme in (0, 1, 3):
            for target in (0, 1, 2):
                for seed in (1, 2, 3, 99):
                    o = ref.run_trial(ls, x, f, scheme, target, seed=seed)
                    res.append({"data": name, "scheme": scheme, "target": target, "seed": seed,
                                "classification": o.classification, "flat_index": o.flat_index, "bit": o.bit,
                                "differs": o.final_output_differs, "verify": outcome(o.verify)})
    return res


def campaigns(ref):
    res = []
    cfg1 = ref.layer_shape(*CAMPAIGN_CFG1)
    # acceptance_main.cpp:134-179 (criterion 2): ones, scale 0.05, seeds 0xC2+i
    plan = [(0, 1), (0, 2), (0, 0), (3, 0), (3, 1), (3, 2)]
    for i, (scheme, target) in enumerate(plan):
        t0 = time.time()
        r = ref.run_campaign(cfg1, scheme, target, 1000, 0xC2 + i, mode=0, scale=0.05)
        res.append({"dims": list(CAMPAIGN_CFG1), "scheme": scheme, "target": target, "trials": 1000, "root_seed": 0xC2 + i,
                    "mode": 0, "counts": [r.detected, r.detected_benign, r.sdc, r.masked]})
        print(f"campaign {scheme}/{target}: {res[-1]['counts']} ({time.time() - t0:.1f}s)", flush=True)
    small = ref.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    for scheme in (0, 1, 3):
        for target in (0, 1, 2):
            for mode in (0, 1):
                r = ref.run_campaign(small, scheme, target, 200, 4242 + 10 * scheme + target, mode=mode, scale=0.05)
                res.append({"dims": [1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1], "scheme": scheme, "target": target, "trials": 200,
                            "root_seed": 4242 + 10 * scheme + target, "mode": mode,
                            "counts": [r.detected, r.detected_benign, r.sdc, r.masked]})
    return res


def main():
    ref = Oracle("ref")
    t0 = time.time()
    out = {"generator": "tests/golden/make_golden.py", "reference": ref.lib_path,
           "conv": [conv_case(ref, d, s) for d, s in CONV_CASES]}
    print(f"conv cases {time.time() - t0:.1f}s", flush=True)
    out["float"] = float_cases(ref)
    out["trials"] = trial_cases(ref)
    out["campaigns"] = campaigns(ref)
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
