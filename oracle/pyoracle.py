"""TEST INFRASTRUCTURE ONLY: numpy front end over the C oracle (liboracle.so)
and the reference build (_ref/libabed_ref*.so).

`Oracle("ora")` and `Oracle("ref")` expose the same methods, so every test can
run a computation through the restatement and through the reference itself and
compare.  Nothing in the product imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

import sys  # noqa: E402

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
from paper_2006_04984_b200.abi import (CampaignConfig, CampaignReport, Dims4, LayerShape,  # noqa: E402
                                       PrecisionPlan, TrialOutcome, VerifyOutcome)

P = C.c_void_p


def _cpu_has(flag: str) -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return flag in f.read()
    except OSError:
        return False


def build_oracle() -> None:
    """make -C oracle liboracle.so (+ _ref when the reference tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if os.path.isdir("/root/reference/proj/include/abed"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_lib_path() -> str | None:
    native = os.path.join(HERE, "_ref", "libabed_ref.so")
    v3 = os.path.join(HERE, "_ref", "libabed_ref_v3.so")
    if _cpu_has("avx512_vnni") and _cpu_has("avx512bw") and os.path.exists(native):
        return native
    return v3 if os.path.exists(v3) else None


def ref_available() -> bool:
    return ref_lib_path() is not None


def ref_kind() -> str:
    p = ref_lib_path()
    return "native-vnni" if p and p.endswith("libabed_ref.so") else "x86-64-v3"


def round_f16(a: np.ndarray) -> np.ndarray:
    """f32 -> IEEE binary16 (round to nearest even) -> f32."""
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """f32 -> bfloat16 (round to nearest even, finite inputs) -> f32."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(P)


def dims(t) -> Dims4:
    d = list(t) + [1] * (4 - len(t))
    return Dims4(*d)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


class Oracle:
    def __init__(self, which: str = "ora"):
        self.which = which
        if which == "ora":
            path = os.path.join(HERE, "liboracle.so")
            if not os.path.exists(path):
                build_oracle()
            self.lib = C.CDLL(path)
            self.p = "ora_"
        else:
            path = ref_lib_path()
            if path is None:
                raise RuntimeError("reference build (oracle/_ref) not available")
            self.lib = C.CDLL(path)
            self.p = "ref_"
        self.lib_path = path

    def _f(self, name, restype=C.c_int):
        fn = getattr(self.lib, self.p + name)
        fn.restype = restype
        return fn

    def _chk(self, code):
        if code != 0:
            raise OracleError(code)

    # ---------------------------------------------------------------- rng
    def derive_seed(self, root, index):
        fn = self._f("derive_seed", C.c_uint64)
        fn.argtypes = [C.c_uint64, C.c_uint64]
        return fn(root, index)

    def random_i8(self, n, seed):
        """n elements of a fresh SplitMix64(seed) stream (fill_random_i8, rng.hpp:46)."""
        out = np.empty(n, np.int8)
        if self.which == "ref":
            fn = self._f("fill_random_i8", None)
            fn.argtypes = [P, C.c_int64, C.c_uint64]
            fn(ptr(out), n, seed)
        else:
            st = C.c_uint64(seed)
            fn = self._f("fill_random_i8", None)
            fn.argtypes = [P, C.c_int64, P]
            fn(ptr(out), n, C.byref(st))
        return out

    def random_f32(self, n, seed, lo=-1.0, hi=1.0):
        out = np.empty(n, np.float32)
        if self.which == "ref":
            fn = self._f("fill_random_f32", None)
            fn.argtypes = [P, C.c_int64, C.c_uint64, C.c_float, C.c_float]
            fn(ptr(out), n, seed, lo, hi)
        else:
            st = C.c_uint64(seed)
            fn = self._f("fill_random_f32", None)
            fn.argtypes = [P, C.c_int64, P, C.c_float, C.c_float]
            fn(ptr(out), n, C.byref(st), lo, hi)
        return out

    # ------------------------------------------------------------- shapes
    def layer_shape(self, n, c, h, w, k, r, s, stride_h=1, stride_w=1, pad_h=0, pad_w=0):
        out = LayerShape()
        fn = self._f("layer_shape_make")
        fn.argtypes = [C.c_int64] * 11 + [C.POINTER(LayerShape)]
        self._chk(fn(n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w, C.byref(out)))
        return out

    # ---------------------------------------------------------------- conv
    def conv_i8(self, x, f, ls):
        out = np.empty(ls.output_dims(), np.int32)
        fn = self._f("conv_i8" if self.which == "ora" else "conv_fast_i8")
        fn.argtypes = [P, P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.int8)), ptr(np.ascontiguousarray(f, np.int8)), C.byref(ls), ptr(out)))
        return out

    def conv_f32(self, x, f, ls):
        out = np.empty(ls.output_dims(), np.float32)
        fn = self._f("conv_f32" if self.which == "ora" else "conv_direct_f32")
        fn.argtypes = [P, P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.float32)), ptr(np.ascontiguousarray(f, np.float32)), C.byref(ls), ptr(out)))
        return out

    def dwconv_i8(self, x, f, ls):
        """Depthwise conv_reference (one filter per channel), int32."""
        out = np.empty(ls.output_dims(), np.int32)
        fn = self._f("dwconv_i8")
        fn.argtypes = [P, P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.int8)), ptr(np.ascontiguousarray(f, np.int8)), C.byref(ls), ptr(out)))
        return out

    def conv_f64(self, x, f, ls):
        """conv_reference with f64 accumulation (float mode on tensor cores: the
        value an fp16/bf16 x f32-accumulate conv approximates)."""
        out = np.empty(ls.output_dims(), np.float64)
        fn = self._f("conv_f64")
        fn.argtypes = [P, P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.float32)), ptr(np.ascontiguousarray(f, np.float32)), C.byref(ls), ptr(out)))
        return out

    def epilog(self, convout, scale, bias, relu=True, out_f32=False):
        convout = np.ascontiguousarray(convout, np.int32)
        bias = np.ascontiguousarray(bias, np.float32)
        out = np.empty(convout.shape, np.float32 if out_f32 else np.int8)
        fn = self._f("epilog")
        fn.argtypes = [P, Dims4, C.c_float, P, C.c_int64, C.c_int, C.c_int, P]
        self._chk(fn(ptr(convout), dims(convout.shape), scale, ptr(bias), bias.size, 0 if relu else 1,
                     3 if out_f32 else 0, ptr(out)))
        return out

    # ----------------------------------------------------------- checksums
    def gen_filter_checksum(self, f):
        f = np.ascontiguousarray(f, np.int8)
        out = np.empty((1,) + f.shape[1:], np.int32)
        fn = self._f("gen_filter_checksum")
        fn.argtypes = [P, Dims4, P]
        self._chk(fn(ptr(f), dims(f.shape), ptr(out)))
        return out

    def decompose_checksum_filters(self, sums):
        sums = np.ascontiguousarray(sums, np.int32)
        out = np.empty((4,) + sums.shape, np.int8)
        fn = self._f("decompose_checksum_filters", C.c_int if self.which == "ref" else None)
        fn.argtypes = [P, C.c_int64, P]
        fn(ptr(sums), sums.size, ptr(out))
        return out

    def conv_checksum_planes(self, x, ls, planes):
        out = np.empty((4, ls.n, 1, ls.p, ls.q), np.int32)
        fn = self._f("conv_checksum_planes")
        fn.argtypes = [P, C.POINTER(LayerShape), P, P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.int8)), C.byref(ls), ptr(np.ascontiguousarray(planes, np.int8)), ptr(out)))
        return out

    def recombine_extra_fmaps(self, extra):
        extra = np.ascontiguousarray(extra, np.int32)
        out = np.empty(extra.shape[1:], np.int64)
        fn = self._f("recombine_extra_fmaps", C.c_int if self.which == "ref" else None)
        fn.argtypes = [P, C.c_int64, P]
        fn(ptr(extra), out.size, ptr(out))
        return out

    def fc_verify(self, convout, extra, original_k=-1):
        convout = np.ascontiguousarray(convout, np.int32)
        o = VerifyOutcome()
        fn = self._f("fc_verify")
        fn.argtypes = [P, Dims4, P, C.c_int64, C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(convout), dims(convout.shape), ptr(np.ascontiguousarray(extra, np.int64)), original_k, C.byref(o)))
        return o

    def gen_input_checksum(self, x, ls):
        out = np.empty((1, ls.c, ls.r, ls.s), np.int32)
        fn = self._f("gen_input_checksum")
        fn.argtypes = [P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.int8)), C.byref(ls), ptr(out)))
        return out

    def fic_dot(self, fc, ic):
        fc = np.ascontiguousarray(fc, np.int32)
        ic = np.ascontiguousarray(ic, np.int32)
        if self.which == "ref":
            r = C.c_int64()
            fn = self._f("fic_dot")
            fn.argtypes = [P, P, C.c_int64, C.POINTER(C.c_int64)]
            self._chk(fn(ptr(fc), ptr(ic), fc.size, C.byref(r)))
            return r.value
        fn = self._f("fic_dot", C.c_int64)
        fn.argtypes = [P, P, C.c_int64]
        return fn(ptr(fc), ptr(ic), fc.size)

    def fic_verify(self, convout, expected, forced32=False):
        convout = np.ascontiguousarray(convout, np.int32)
        o = VerifyOutcome()
        if self.which == "ref":
            fn = self._f("fic_verify")
            fn.argtypes = [P, C.c_int64, C.c_int64, C.c_int, C.POINTER(VerifyOutcome)]
            self._chk(fn(ptr(convout), convout.size, expected, 1 if forced32 else 0, C.byref(o)))
        else:
            fn = self._f("fic_verify_forced32" if forced32 else "fic_verify", None)
            fn.argtypes = [P, C.c_int64, C.c_int64, C.POINTER(VerifyOutcome)]
            fn(ptr(convout), convout.size, expected, C.byref(o))
        return o

    # ------------------------------------------------------------ ABFT GEMM
    def abft_gemm(self, a, b):
        """abft_gemm (abft_gemm.hpp:102-152): (c i32 m x n, c_aug i64 (m+1) x (n+1), row, col)."""
        a = np.ascontiguousarray(a, np.int8)
        b = np.ascontiguousarray(b, np.int8)
        m, k = a.shape
        kb, n = b.shape
        c = np.empty((m, n), np.int32)
        ca = np.empty((m + 1, n + 1), np.int64)
        row, col = VerifyOutcome(), VerifyOutcome()
        fn = self._f("abft_gemm")
        fn.argtypes = [P, C.c_int64, C.c_int64, P, C.c_int64, C.c_int64, P, P, C.POINTER(VerifyOutcome),
                       C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(a), m, k, ptr(b), kb, n, ptr(c), ptr(ca), C.byref(row), C.byref(col)))
        return c, ca, row, col

    def abft_check(self, c_aug):
        """abft_check (abft_gemm.hpp:70-96) -> (row, col)."""
        ca = np.ascontiguousarray(c_aug, np.int64)
        row, col = VerifyOutcome(), VerifyOutcome()
        fn = self._f("abft_check")
        fn.argtypes = [P, C.c_int64, C.c_int64, C.POINTER(VerifyOutcome), C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(ca), ca.shape[0], ca.shape[1], C.byref(row), C.byref(col)))
        return row, col

    def abft_costs(self, m, n, k, single_pass=False):
        """abft_costs (abft_gemm.hpp:41-55), reference build only: 5 x [ops, read, write, moved]."""
        out = np.zeros(20, np.int64)
        fn = self._f("abft_costs", None)
        fn.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, P]
        fn(m, n, k, 1 if single_pass else 0, ptr(out))
        return out.reshape(5, 4)

    def ic_verify_k(self, convout, f, ic):
        convout = np.ascontiguousarray(convout, np.int32)
        f = np.ascontiguousarray(f, np.int8)
        o = VerifyOutcome()
        fn = self._f("ic_verify_k")
        fn.argtypes = [P, Dims4, P, Dims4, P, C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(convout), dims(convout.shape), ptr(f), dims(f.shape), ptr(np.ascontiguousarray(ic, np.int32)), C.byref(o)))
        return o

    def ic_batch_checksum(self, x):
        x = np.ascontiguousarray(x, np.int8)
        out = np.empty((1,) + x.shape[1:], np.int32)
        fn = self._f("ic_batch_checksum", C.c_int if self.which == "ref" else None)
        fn.argtypes = [P, Dims4, P]
        fn(ptr(x), dims(x.shape), ptr(out))
        return out

    def conv_batch_checksum(self, batch, f, ls):
        out = np.empty((1, ls.k, ls.p, ls.q), np.int64)
        fn = self._f("conv_batch_checksum")
        fn.argtypes = [P, P, C.POINTER(LayerShape), P]
        self._chk(fn(ptr(np.ascontiguousarray(batch, np.int32)), ptr(np.ascontiguousarray(f, np.int8)), C.byref(ls), ptr(out)))
        return out

    def ic_batch_verify(self, convout, extra):
        convout = np.ascontiguousarray(convout, np.int32)
        o = VerifyOutcome()
        fn = self._f("ic_batch_verify")
        fn.argtypes = [P, Dims4, P, C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(convout), dims(convout.shape), ptr(np.ascontiguousarray(extra, np.int64)), C.byref(o)))
        return o

    def plan_precision(self, ls, bits=8):
        p = PrecisionPlan()
        fn = self._f("plan_precision")
        fn.argtypes = [C.POINTER(LayerShape), C.c_int, C.POINTER(PrecisionPlan)]
        self._chk(fn(C.byref(ls), bits, C.byref(p)))
        return p

    def filter_checksum_f64(self, f):
        f = np.ascontiguousarray(f, np.float32)
        out = np.empty(f.shape[1] * f.shape[2] * f.shape[3], np.float64)
        fn = self._f("filter_checksum_f64", C.c_int if self.which == "ref" else None)
        fn.argtypes = [P, Dims4, P]
        fn(ptr(f), dims(f.shape), ptr(out))
        return out

    def input_checksum_f64(self, x, ls):
        out = np.empty(ls.c * ls.r * ls.s, np.float64)
        fn = self._f("input_checksum_f64", C.c_int if self.which == "ref" else None)
        fn.argtypes = [P, C.POINTER(LayerShape), P]
        fn(ptr(np.ascontiguousarray(x, np.float32)), C.byref(ls), ptr(out))
        return out

    def fc_verify_f32(self, convout, extra, tau):
        """checksum.hpp:541-565 (C restatement: the 'ora' build)."""
        assert self.which == "ora", "fc_verify_f32 is bound from the C restatement"
        convout = np.ascontiguousarray(convout, np.float32)
        o = VerifyOutcome()
        fn = self._f("fc_verify_f32")
        fn.argtypes = [P, Dims4, P, C.c_double, C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(convout), dims(convout.shape), ptr(np.ascontiguousarray(extra, np.float32)), tau, C.byref(o)))
        return o

    def fic_verify_f32(self, convout, expected, tau):
        """checksum.hpp:537-539 (C restatement: the 'ora' build)."""
        assert self.which == "ora", "fic_verify_f32 is bound from the C restatement"
        convout = np.ascontiguousarray(convout, np.float32)
        o = VerifyOutcome()
        fn = self._f("fic_verify_f32")
        fn.argtypes = [P, C.c_int64, C.c_double, C.c_double, C.POINTER(VerifyOutcome)]
        self._chk(fn(ptr(convout), convout.size, expected, tau, C.byref(o)))
        return o

    def fic_dot_f64(self, a, b):
        """checksum.hpp:530-535 (acc = fma(a, b, acc), the reference's contracted loop)."""
        fn = self._f("fic_dot_f64", C.c_double)
        fn.argtypes = [P, P, C.c_int64]
        a = np.ascontiguousarray(a, np.float64)
        return fn(ptr(a), ptr(np.ascontiguousarray(b, np.float64)), a.size)

    def fused_conv_epilog(self, x, f, ls, scale, bias, relu=True, out_f32=False, checksum=False, next_ls=None):
        out = np.empty(ls.output_dims(), np.float32 if out_f32 else np.int8)
        cs = C.c_int64()
        nic = np.empty((1, next_ls.c, next_ls.r, next_ls.s), np.int32) if next_ls is not None else None
        fn = self._f("fused_conv_epilog")
        fn.argtypes = [P, P, C.POINTER(LayerShape), C.c_float, P, C.c_int, C.c_int, P, P, P, P]
        self._chk(fn(ptr(np.ascontiguousarray(x, np.int8)), ptr(np.ascontiguousarray(f, np.int8)), C.byref(ls), scale,
                     ptr(np.ascontiguousarray(bias, np.float32)), 0 if relu else 1, 3 if out_f32 else 0, ptr(out),
                     C.byref(cs) if checksum else None, C.byref(next_ls) if next_ls is not None else None,
                     ptr(nic) if nic is not None else None))
        return out, (cs.value if checksum else None), nic

    def run_trial(self, ls, x, f, scheme, target, scale=0.05, bias=None, relu=True, out_f32=False, seed=1):
        o = TrialOutcome()
        b = np.ascontiguousarray(bias if bias is not None else np.zeros(0), np.float32)
        fn = self._f("run_trial")
        fn.argtypes = [C.POINTER(LayerShape), P, P, C.c_int, C.c_int, C.c_float, P, C.c_int64, C.c_int, C.c_int,
                       C.c_uint64, C.POINTER(TrialOutcome)]
        self._chk(fn(C.byref(ls), ptr(np.ascontiguousarray(x, np.int8)), ptr(np.ascontiguousarray(f, np.int8)), scheme,
                     target, scale, ptr(b) if b.size else None, b.size, 0 if relu else 1, 3 if out_f32 else 0, seed,
                     C.byref(o)))
        return o

    def run_campaign(self, ls, scheme, target, trials, root_seed, mode=0, scale=0.05, jobs=0, begin=0, end=None):
        cfg = CampaignConfig(shape=ls, scheme=scheme, target=target, trials=trials, root_seed=root_seed, mode=mode,
                             scale=scale, bias_host=None, bias_len=0, activation=0, output_kind=0, jobs=jobs)
        rep = CampaignReport()
        if self.which == "ref":
            fn = self._f("run_campaign")
            fn.argtypes = [C.POINTER(CampaignConfig), C.POINTER(CampaignReport)]
            self._chk(fn(C.byref(cfg), C.byref(rep)))
        else:
            fn = self._f("run_campaign")
            fn.argtypes = [C.POINTER(CampaignConfig), C.c_int64, C.c_int64, C.POINTER(CampaignReport)]
            self._chk(fn(C.byref(cfg), begin, trials if end is None else end, C.byref(rep)))
        return rep

    def time_layer(self, ls, scheme, threads, x, f):
        """Reference only: seconds for conv_fast_i8 + scheme check + epilog over the batch."""
        fn = self._f("time_layer", C.c_double)
        fn.argtypes = [C.POINTER(LayerShape), C.c_int, C.c_int, P, P]
        return fn(C.byref(ls), scheme, threads, ptr(np.ascontiguousarray(x, np.int8)), ptr(np.ascontiguousarray(f, np.int8)))
