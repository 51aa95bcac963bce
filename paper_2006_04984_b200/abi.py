"""ctypes view of the C ABI in include/abed_b200.h.

This module only loads the in-tree libabed_b200.so and declares its structs and
signatures.  There is deliberately no fallback: if the library is missing or
no sm_100 device is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libabed_b200.so")

# status codes / enums (abed_b200.h)
OK, ERR_INVALID_ARGUMENT, ERR_OUT_OF_RANGE, ERR_RUNTIME, ERR_CUDA, ERR_NO_DEVICE = range(6)
I8, I32, I64, F32 = 0, 1, 2, 3
RELU, IDENTITY = 0, 1
FC, IC, ICBATCH, FIC = 0, 1, 2, 3
TARGET_INPUT, TARGET_FILTER, TARGET_CONVOUT = 0, 1, 2
DETECTED, SDC, MASKED, DETECTED_BENIGN = 0, 1, 2, 3
DATA_ONES, DATA_RANDOM_I8 = 0, 1
CHECK_FC, CHECK_FIC, CHECK_IC, CHECK_ICBATCH = 1, 2, 4, 8
# FIC input-checksum source (abed_conv_plan_set_input_checksum_source)
RHS_STAGED, RHS_REREAD = 0, 1
OUT_NONE, OUT_I32_NCHW, OUT_I8_NCHW, OUT_F32_NCHW, OUT_I8_PACKED, OUT_I8_COMPARE, OUT_H_PACKED, OUT_H_COMPARE = range(8)
F16, BF16 = 4, 5  # float mode on tensor cores: 16-bit operand storage kinds


class Dims4(C.Structure):
    _fields_ = [("d0", C.c_int64), ("d1", C.c_int64), ("d2", C.c_int64), ("d3", C.c_int64)]


class LayerShape(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("n", "c", "h", "w", "k", "r", "s", "stride_h", "stride_w", "pad_h", "pad_w", "p", "q")]

    def crs(self):
        return self.c * self.r * self.s

    def npq(self):
        return self.n * self.p * self.q

    def nkpq(self):
        return self.n * self.k * self.p * self.q

    def input_dims(self):
        return (self.n, self.c, self.h, self.w)

    def filter_dims(self):
        return (self.k, self.c, self.r, self.s)

    def output_dims(self):
        return (self.n, self.k, self.p, self.q)

    def astuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_)

    def __eq__(self, other):
        return isinstance(other, LayerShape) and self.astuple() == other.astuple()

    def __repr__(self):
        return "LayerShape(%s)" % ", ".join(f"{f}={getattr(self, f)}" for f, _ in self._fields_)


class EpilogParams(C.Structure):
    _fields_ = [("scale", C.c_float), ("bias", C.c_void_p), ("bias_len", C.c_int64),
                ("activation", C.c_int32), ("output_kind", C.c_int32)]


class VerifyOutcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("has_locus", C.c_int32), ("locus", C.c_int64 * 3),
                ("lhs", C.c_int64), ("rhs", C.c_int64), ("lhs_f", C.c_double), ("rhs_f", C.c_double),
                ("error_count", C.c_int64)]

    def passed(self):
        return self.status == 0

    def locus_tuple(self):
        return tuple(self.locus) if self.has_locus else None


class PrecisionPlan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("operand_bits", "bits_output_fmap", "bits_reduced_fc", "bits_reduced_fic",
                 "bits_filter_checksum", "bits_input_checksum", "output_fmap_kind", "reduced_fc_kind",
                 "reduced_fic_kind", "filter_checksum_kind", "input_checksum_kind")]


class CampaignConfig(C.Structure):
    _fields_ = [("shape", LayerShape), ("scheme", C.c_int32), ("target", C.c_int32), ("trials", C.c_int64),
                ("root_seed", C.c_uint64), ("mode", C.c_int32), ("scale", C.c_float),
                ("bias_host", C.c_void_p), ("bias_len", C.c_int64), ("activation", C.c_int32),
                ("output_kind", C.c_int32), ("jobs", C.c_int32)]


class CampaignReport(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("target", C.c_int32), ("trials", C.c_int64), ("detected", C.c_int64),
                ("detected_benign", C.c_int64), ("sdc", C.c_int64), ("masked", C.c_int64), ("seed", C.c_uint64)]

    def astuple(self):
        return (self.detected, self.detected_benign, self.sdc, self.masked)


class TrialOutcome(C.Structure):
    _fields_ = [("classification", C.c_int32), ("target", C.c_int32), ("flat_index", C.c_int64),
                ("bit", C.c_int32), ("final_output_differs", C.c_int32), ("verify", VerifyOutcome)]


class PlanInfo(C.Structure):
    _fields_ = [("packed_input_bytes", C.c_int64), ("block_n", C.c_int32), ("n_tiles", C.c_int32),
                ("m_tiles", C.c_int32), ("gps", C.c_int32), ("b_resident", C.c_int32), ("n_phase", C.c_int32),
                ("Hl", C.c_int32), ("Wl", C.c_int32), ("smem_bytes", C.c_int64)]


P = C.c_void_p
i64, i32, u64 = C.c_int64, C.c_int32, C.c_uint64
SHP = C.POINTER(LayerShape)
OUTC = C.POINTER(VerifyOutcome)

# name -> (restype, argtypes)
SIGNATURES = {
    "abed_last_error": (C.c_char_p, []),
    "abed_device_check": (C.c_int, []),
    "abed_version": (C.c_int, []),
    "abed_malloc": (C.c_int, [C.POINTER(P), C.c_size_t]),
    "abed_free": (C.c_int, [P]),
    "abed_memcpy_h2d": (C.c_int, [P, P, C.c_size_t]),
    "abed_memcpy_d2h": (C.c_int, [P, P, C.c_size_t]),
    "abed_memset": (C.c_int, [P, C.c_int, C.c_size_t]),
    "abed_synchronize": (C.c_int, []),
    "abed_layer_shape_make": (C.c_int, [i64] * 11 + [SHP]),
    "abed_fill_random_i8": (C.c_int, [P, i64, u64, u64, P]),
    "abed_fill_random_extreme": (C.c_int, [P, i64, u64, u64, P]),
    "abed_derive_seed": (u64, [u64, u64]),
    "abed_abft_gemm_i8": (C.c_int, [P, i64, i64, P, i64, i64, P, P, OUTC, OUTC]),
    "abed_abft_check": (C.c_int, [P, i64, i64, OUTC, OUTC]),
    "abed_abft_plan_create": (C.c_int, [i64, i64, i64, C.POINTER(P)]),
    "abed_abft_plan_destroy": (C.c_int, [P]),
    "abed_abft_plan_run": (C.c_int, [P, P, P, P, P, P, i32, P]),
    "abed_conv_i8": (C.c_int, [P, P, SHP, P, P]),
    "abed_conv_f32": (C.c_int, [P, P, SHP, P, P]),
    "abed_epilog": (C.c_int, [P, Dims4, C.POINTER(EpilogParams), P, P]),
    "abed_gen_filter_checksum": (C.c_int, [P, Dims4, P, P]),
    "abed_decompose_checksum_filters": (C.c_int, [P, i64, P, P]),
    "abed_conv_checksum_planes": (C.c_int, [P, SHP, P, P, P]),
    "abed_recombine_extra_fmaps": (C.c_int, [P, i64, P, P]),
    "abed_conv_filter_checksum": (C.c_int, [P, SHP, P, P, P]),
    "abed_fc_verify": (C.c_int, [P, Dims4, P, i64, OUTC]),
    "abed_gen_input_checksum": (C.c_int, [P, SHP, P, P]),
    "abed_reduce_all_i64": (C.c_int, [P, i64, C.POINTER(i64)]),
    "abed_reduce_all_wrap32": (C.c_int, [P, i64, C.POINTER(i32)]),
    "abed_fic_dot": (C.c_int, [P, P, i64, C.POINTER(i64)]),
    "abed_fic_verify": (C.c_int, [P, i64, i64, OUTC]),
    "abed_fic_verify_forced32": (C.c_int, [P, i64, i64, OUTC]),
    "abed_ic_verify_k": (C.c_int, [P, Dims4, P, Dims4, P, OUTC]),
    "abed_ic_batch_checksum": (C.c_int, [P, Dims4, P, P]),
    "abed_conv_batch_checksum": (C.c_int, [P, P, SHP, P, P]),
    "abed_ic_batch_verify": (C.c_int, [P, Dims4, P, OUTC]),
    "abed_plan_precision": (C.c_int, [SHP, i32, C.POINTER(PrecisionPlan)]),
    "abed_float_verify": (C.c_int, [C.c_double, C.c_double, C.c_double, OUTC]),
    "abed_filter_checksum_f64": (C.c_int, [P, Dims4, P, P]),
    "abed_input_checksum_f64": (C.c_int, [P, SHP, P, P]),
    "abed_reduce_all_f64": (C.c_int, [P, i64, C.POINTER(C.c_double)]),
    "abed_fic_dot_f64": (C.c_int, [P, P, i64, C.POINTER(C.c_double)]),
    "abed_fic_verify_f32": (C.c_int, [P, i64, C.c_double, C.c_double, OUTC]),
    "abed_fc_verify_f32": (C.c_int, [P, Dims4, P, C.c_double, OUTC]),
    "abed_ic_verify_k_f32": (C.c_int, [P, Dims4, P, Dims4, P, C.c_double, OUTC]),
    "abed_fused_conv_epilog": (C.c_int, [P, P, SHP, C.POINTER(EpilogParams), P, C.POINTER(i64), SHP, P, P]),
    "abed_flip_bit": (C.c_int, [P, i32, i64, i64, i32, P]),
    "abed_run_trial": (C.c_int, [SHP, P, P, i32, i32, C.c_float, P, i64, i32, i32, u64,
                                 C.POINTER(TrialOutcome)]),
    "abed_run_campaign": (C.c_int, [C.POINTER(CampaignConfig), i64, i64, C.POINTER(CampaignReport)]),
    "abed_run_campaign_batched": (C.c_int, [C.POINTER(CampaignConfig), i64, i64, C.POINTER(CampaignReport)]),
    "abed_campaign_create": (C.c_int, [C.POINTER(CampaignConfig), C.POINTER(P)]),
    "abed_campaign_run": (C.c_int, [P, i64, i64, P, P]),
    "abed_campaign_report_of": (C.c_int, [P, C.POINTER(i64), i64, C.POINTER(CampaignReport)]),
    "abed_campaign_destroy": (C.c_int, [P]),
    "abed_campaign_create_shard": (C.c_int, [C.POINTER(CampaignConfig), i64, i64, C.POINTER(P)]),
    "abed_campaign_run_records": (C.c_int, [P, i64, i64, P, P]),
    "abed_campaign_classify": (C.c_int, [P, P, i64, P, P]),
    "abed_conv_plan_create": (C.c_int, [SHP, P, i32, i32, C.POINTER(P)]),
    "abed_conv_plan_destroy": (C.c_int, [P]),
    "abed_conv_plan_info": (C.c_int, [P, C.POINTER(PlanInfo)]),
    "abed_pack_input": (C.c_int, [P, P, P, P]),
    "abed_conv_plan_run": (C.c_int, [P, P, C.POINTER(EpilogParams), i32, P, P, i64, i32, P]),
    "abed_conv_plan_finalize": (C.c_int, [P, P, P]),
    "abed_conv_plan_compare_count": (C.c_int, [P, C.POINTER(i64)]),
    "abed_debug_set_conv_trace": (C.c_int, [P, P, i32]),
    "abed_conv_plan_create_h": (C.c_int, [SHP, P, i32, i32, C.c_double, C.c_double, i32, C.POINTER(P)]),
    "abed_pack_input_h": (C.c_int, [P, P, P, P]),
    "abed_conv_plan_set_tau": (C.c_int, [P, C.c_double, C.c_double]),
    "abed_conv_plan_finalize_many": (C.c_int, [P, i32, P, P]),
    "abed_conv_plan_create_dw": (C.c_int, [SHP, P, i32, C.POINTER(P)]),
    "abed_conv_plan_set_af_input": (C.c_int, [P, i32]),
    "abed_conv_plan_set_reuse_input_checksum": (C.c_int, [P, i32]),
    "abed_conv_plan_set_paired_finalize": (C.c_int, [P, i32]),
    "abed_conv_plan_set_input_checksum_source": (C.c_int, [P, i32]),
    "abed_probe_mma_i8_peak": (C.c_int, [i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "abed_verdict_records": (C.c_int, [P, i32, P, i64, P, P]),
    "abed_verdict_combine": (C.c_int, [P, i32, i32, P, P, P]),
    "abed_verdict_records_host": (C.c_int, [P, i32, P, i64, P]),
    "abed_verdict_combine_host": (C.c_int, [P, i32, i32, P, P]),
}

_lib = None


class AbedError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(AbedError, ValueError):
    pass


class OutOfRange(AbedError, IndexError):
    pass


def load(path: str = LIB_PATH):
    """Loads the in-tree library (built by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libabed_b200.so not built at {path}; run __graft_entry__.build()")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(lib, name):
                continue  # tests/test_abi_symbols.py asserts the full export list
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(code: int):
    if code == OK:
        return
    msg = load().abed_last_error().decode(errors="replace")
    if code == ERR_INVALID_ARGUMENT:
        raise InvalidArgument(code, msg)
    if code == ERR_OUT_OF_RANGE:
        raise OutOfRange(code, msg)
    raise AbedError(code, msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args))


def layer_shape(n, c, h, w, k, r, s, stride_h=1, stride_w=1, pad_h=0, pad_w=0) -> LayerShape:
    out = LayerShape()
    call("abed_layer_shape_make", n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w, C.byref(out))
    return out
