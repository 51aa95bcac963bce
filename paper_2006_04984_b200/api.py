"""Python mirror of the reference's `abed::` API over the C ABI.

Same names and argument meaning as /root/reference/proj/include/abed/*.hpp,
operating on torch CUDA tensors in the reference layouts (NCHW int8 input, KCRS
int8 filters, NKPQ int32 ConvOut).  Errors are raised like the reference's
exceptions: abi.InvalidArgument (std::invalid_argument, also a ValueError),
abi.OutOfRange (std::out_of_range, also an IndexError).  Every call runs on the
GPU through libabed_b200.so; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import abi
from .abi import LayerShape, VerifyOutcome, call

I8, I32, I64, F32 = abi.I8, abi.I32, abi.I64, abi.F32
KIND = {torch.int8: I8, torch.int32: I32, torch.int64: I64, torch.float32: F32}


def _p(t: torch.Tensor):
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _keep_alive(t, stream):
    """A temporary read by a kernel on a caller-supplied stream: tell the caching
    allocator, so its memory is not reused before that stream has consumed it."""
    if t is None or stream is None:
        return
    raw = stream.value if isinstance(stream, C.c_void_p) else getattr(stream, "cuda_stream", stream)
    if raw is None or raw == torch.cuda.current_stream().cuda_stream:
        return
    t.record_stream(torch.cuda.ExternalStream(int(raw)))


def _dims(t: torch.Tensor) -> abi.Dims4:
    d = list(t.shape) + [1] * (4 - t.dim())
    return abi.Dims4(*d)


def _empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device="cuda")


class LayerShapeT(LayerShape):
    pass


def layer_shape(n, c, h, w, k, r, s, stride_h=1, stride_w=1, pad_h=0, pad_w=0) -> LayerShape:
    """tensor.hpp:178 LayerShape::make"""
    return abi.layer_shape(n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w)


# ------------------------------------------------------------------ L0
def fill_random_i8(n: int, seed: int, offset: int = 0) -> torch.Tensor:
    """rng.hpp:46 on a fresh SplitMix64(seed) stream advanced by `offset` draws."""
    t = _empty((n,), torch.int8)
    call("abed_fill_random_i8", _p(t), n, seed, offset, _stream())
    return t


def derive_seed(root: int, index: int) -> int:
    return abi.load().abed_derive_seed(root, index)


# ------------------------------------------------------------------ L1
def conv_direct(x: torch.Tensor, f: torch.Tensor, ls: LayerShape) -> torch.Tensor:
    """convolution.hpp:237 conv_direct == :224 detail::conv_fast_i8 (tcgen05)."""
    _check_conv(x, f, ls, torch.int8)
    out = _empty(ls.output_dims(), torch.int32)
    call("abed_conv_i8", _p(x), _p(f), C.byref(ls), _p(out), _stream())
    return out


conv_fast_i8 = conv_direct


def conv_direct_f32(x, f, ls):
    _check_conv(x, f, ls, torch.float32)
    out = _empty(ls.output_dims(), torch.float32)
    call("abed_conv_f32", _p(x), _p(f), C.byref(ls), _p(out), _stream())
    return out


def _check_conv(x, f, ls, dtype):
    # convolution.hpp:67-73
    if x.dtype != dtype or tuple(x.shape) != ls.input_dims():
        raise abi.InvalidArgument(abi.ERR_INVALID_ARGUMENT, "conv: input tensor does not match shape")
    if f.dtype != dtype or tuple(f.shape) != ls.filter_dims():
        raise abi.InvalidArgument(abi.ERR_INVALID_ARGUMENT, "conv: filter tensor does not match shape")


def epilog(convout: torch.Tensor, scale: float, bias, relu: bool = True, output_kind: int = I8) -> torch.Tensor:
    """convolution.hpp:353 epilog"""
    bias_t = torch.as_tensor(bias, dtype=torch.float32).reshape(-1).cuda()
    ep = abi.EpilogParams(scale, bias_t.data_ptr(), bias_t.numel(), abi.RELU if relu else abi.IDENTITY, output_kind)
    out = _empty(tuple(convout.shape), torch.int8 if output_kind == I8 else torch.float32)
    call("abed_epilog", _p(convout), _dims(convout), C.byref(ep), _p(out), _stream())
    return out


# ------------------------------------------------------------------ L2
def gen_filter_checksum(f: torch.Tensor) -> torch.Tensor:
    out = _empty((1,) + tuple(f.shape[1:]), torch.int32)
    call("abed_gen_filter_checksum", _p(f), _dims(f), _p(out), _stream())
    return out


def decompose_checksum_filters(sums: torch.Tensor) -> torch.Tensor:
    out = _empty((4,) + tuple(sums.shape), torch.int8)
    call("abed_decompose_checksum_filters", _p(sums), sums.numel(), _p(out), _stream())
    return out


def conv_checksum_planes(x, ls, planes):
    out = _empty((4, ls.n, 1, ls.p, ls.q), torch.int32)
    call("abed_conv_checksum_planes", _p(x), C.byref(ls), _p(planes), _p(out), _stream())
    return out


def recombine_extra_fmaps(extra):
    out = _empty(tuple(extra.shape[1:]), torch.int64)
    call("abed_recombine_extra_fmaps", _p(extra), out.numel(), _p(out), _stream())
    return out


def conv_filter_checksum(x, ls, sums):
    out = _empty((ls.n, 1, ls.p, ls.q), torch.int64)
    call("abed_conv_filter_checksum", _p(x), C.byref(ls), _p(sums), _p(out), _stream())
    return out


def _sync():
    torch.cuda.current_stream().synchronize()


def fc_verify(convout, extra, original_k=-1) -> VerifyOutcome:
    _sync()
    o = VerifyOutcome()
    call("abed_fc_verify", _p(convout), _dims(convout), _p(extra), original_k, C.byref(o))
    return o


def gen_input_checksum(x, ls):
    out = _empty((1, ls.c, ls.r, ls.s), torch.int32)
    call("abed_gen_input_checksum", _p(x), C.byref(ls), _p(out), _stream())
    return out


def reduce_all_i64(convout) -> int:
    _sync()
    r = C.c_int64()
    call("abed_reduce_all_i64", _p(convout), convout.numel(), C.byref(r))
    return r.value


def fic_dot(fc, ic) -> int:
    _sync()
    r = C.c_int64()
    call("abed_fic_dot", _p(fc), _p(ic), fc.numel(), C.byref(r))
    return r.value


def fic_verify(convout, expected: int) -> VerifyOutcome:
    _sync()
    o = VerifyOutcome()
    call("abed_fic_verify", _p(convout), convout.numel(), expected, C.byref(o))
    return o


def fic_verify_forced32(convout, expected: int) -> VerifyOutcome:
    _sync()
    o = VerifyOutcome()
    call("abed_fic_verify_forced32", _p(convout), convout.numel(), expected, C.byref(o))
    return o


def ic_verify_k(convout, f, ic) -> VerifyOutcome:
    _sync()
    o = VerifyOutcome()
    call("abed_ic_verify_k", _p(convout), _dims(convout), _p(f), _dims(f), _p(ic), C.byref(o))
    return o


def ic_batch_checksum(x):
    out = _empty((1,) + tuple(x.shape[1:]), torch.int32)
    call("abed_ic_batch_checksum", _p(x), _dims(x), _p(out), _stream())
    return out


def conv_batch_checksum(batch, f, ls):
    out = _empty((1, ls.k, ls.p, ls.q), torch.int64)
    call("abed_conv_batch_checksum", _p(batch), _p(f), C.byref(ls), _p(out), _stream())
    return out


def ic_batch_verify(convout, extra) -> VerifyOutcome:
    _sync()
    o = VerifyOutcome()
    call("abed_ic_batch_verify", _p(convout), _dims(convout), _p(extra), C.byref(o))
    return o


def plan_precision(ls, operand_bits=8):
    p = abi.PrecisionPlan()
    call("abed_plan_precision", C.byref(ls), operand_bits, C.byref(p))
    return p


def fused_conv_epilog(x, f, ls, scale, bias, relu=True, output_kind=I8, output_checksum=False, next_layer=None):
    """checksum.hpp:616 fused_conv_epilog -> (output, output_checksum | None, next_input_checksum | None)"""
    bias_t = torch.as_tensor(bias, dtype=torch.float32).reshape(-1).cuda()
    ep = abi.EpilogParams(scale, bias_t.data_ptr(), bias_t.numel(), abi.RELU if relu else abi.IDENTITY, output_kind)
    out = _empty(ls.output_dims(), torch.int8 if output_kind == I8 else torch.float32)
    cs = C.c_int64()
    nic = _empty((1, next_layer.c, next_layer.r, next_layer.s), torch.int32) if next_layer is not None else None
    call("abed_fused_conv_epilog", _p(x), _p(f), C.byref(ls), C.byref(ep), _p(out),
         C.byref(cs) if output_checksum else None, C.byref(next_layer) if next_layer is not None else None,
         _p(nic) if nic is not None else None, _stream())
    return out, (cs.value if output_checksum else None), nic


# float mode
def float_verify(lhs, rhs, tau):
    o = VerifyOutcome()
    call("abed_float_verify", lhs, rhs, tau, C.byref(o))
    return o


def filter_checksum_f64(f):
    out = _empty((f.shape[1] * f.shape[2] * f.shape[3],), torch.float64)
    call("abed_filter_checksum_f64", _p(f), _dims(f), _p(out), _stream())
    return out


def input_checksum_f64(x, ls):
    out = _empty((ls.c * ls.r * ls.s,), torch.float64)
    call("abed_input_checksum_f64", _p(x), C.byref(ls), _p(out), _stream())
    return out


def reduce_all_f64(c):
    _sync()
    r = C.c_double()
    call("abed_reduce_all_f64", _p(c), c.numel(), C.byref(r))
    return r.value


def fic_dot_f64(a, b):
    _sync()
    r = C.c_double()
    call("abed_fic_dot_f64", _p(a), _p(b), a.numel(), C.byref(r))
    return r.value


def fic_verify_f32(c, expected, tau):
    _sync()
    o = VerifyOutcome()
    call("abed_fic_verify_f32", _p(c), c.numel(), expected, tau, C.byref(o))
    return o


def fc_verify_f32(c, extra, tau):
    _sync()
    o = VerifyOutcome()
    call("abed_fc_verify_f32", _p(c), _dims(c), _p(extra), tau, C.byref(o))
    return o


def ic_verify_k_f32(c, f, ic, tau):
    _sync()
    o = VerifyOutcome()
    call("abed_ic_verify_k_f32", _p(c), _dims(c), _p(f), _dims(f), _p(ic), tau, C.byref(o))
    return o


# ------------------------------------------------------------------ L3 faults
def flip_bit_(t: torch.Tensor, flat_index: int, bit: int) -> torch.Tensor:
    """faults.hpp:53 flip_bit_inplace"""
    call("abed_flip_bit", _p(t), KIND[t.dtype], t.numel(), flat_index, bit, _stream())
    return t


def flip_bit(t: torch.Tensor, flat_index: int, bit: int) -> torch.Tensor:
    return flip_bit_(t.clone(), flat_index, bit)


def run_trial(ls, x, f, scheme, target, scale=0.05, bias=None, relu=True, output_kind=I8, seed=1):
    o = abi.TrialOutcome()
    b = (C.c_float * len(bias))(*bias) if bias is not None else None
    call("abed_run_trial", C.byref(ls), _p(x), _p(f), scheme, target, scale, b, 0 if bias is None else len(bias),
         abi.RELU if relu else abi.IDENTITY, output_kind, seed, C.byref(o))
    return o


def campaign_config(ls, scheme, target, trials=1000, root_seed=1, mode=abi.DATA_ONES, scale=0.05, bias=None,
                    relu=True, output_kind=I8):
    """faults.hpp:77-86 CampaignConfig (the bias array rides on the returned config)."""
    b = (C.c_float * len(bias))(*bias) if bias is not None else None
    cfg = abi.CampaignConfig(shape=ls, scheme=scheme, target=target, trials=trials, root_seed=root_seed, mode=mode,
                             scale=scale, bias_host=C.cast(b, C.c_void_p) if b is not None else None,
                             bias_len=0 if bias is None else len(bias), activation=abi.RELU if relu else abi.IDENTITY,
                             output_kind=output_kind, jobs=0)
    cfg._bias_keepalive = b
    return cfg


def run_campaign(ls, scheme, target, trials=1000, root_seed=1, mode=abi.DATA_ONES, scale=0.05, bias=None, relu=True,
                 output_kind=I8, begin=0, end=None, batched=False):
    """faults.hpp:276 run_campaign over trials [begin, end).  batched=False re-runs
    the fused protected conv per trial; batched=True evaluates every trial in one
    trial-parallel launch (abed_run_campaign_batched); the reports are identical."""
    cfg = campaign_config(ls, scheme, target, trials, root_seed, mode, scale, bias, relu, output_kind)
    rep = abi.CampaignReport()
    call("abed_run_campaign_batched" if batched else "abed_run_campaign", C.byref(cfg), begin,
         trials if end is None else end, C.byref(rep))
    return rep


class Campaign:
    """Device-resident trial-parallel campaign (abed_campaign_*): run(begin, end)
    adds the classification counts of those trials into a device int64[4]
    (detected, sdc, masked, detected_benign) with one launch."""

    def __init__(self, ls, scheme, target, trials=1000, root_seed=1, mode=abi.DATA_ONES, scale=0.05, bias=None,
                 relu=True, output_kind=I8, images=None):
        """images=(begin, end): this process's batch shard (per-trial records instead of counts)."""
        self.cfg = campaign_config(ls, scheme, target, trials, root_seed, mode, scale, bias, relu, output_kind)
        self.handle = C.c_void_p()
        if images is None:
            call("abed_campaign_create", C.byref(self.cfg), C.byref(self.handle))
        else:
            call("abed_campaign_create_shard", C.byref(self.cfg), images[0], images[1], C.byref(self.handle))

    def run(self, counts: torch.Tensor, begin=0, end=None, stream=None):
        call("abed_campaign_run", self.handle, begin, self.cfg.trials if end is None else end, _p(counts),
             stream or _stream())

    def run_records(self, records: torch.Tensor, begin=0, end=None, stream=None):
        """records: int64 [end - begin, 3] per-trial {check failed, output differs, sum delta} of this shard."""
        call("abed_campaign_run_records", self.handle, begin, self.cfg.trials if end is None else end, _p(records),
             stream or _stream())

    def classify(self, records: torch.Tensor, counts: torch.Tensor, stream=None):
        """counts (int64 [4]) += classification of the (shard-summed) records."""
        call("abed_campaign_classify", self.handle, _p(records), records.shape[0], _p(counts), stream or _stream())

    def report(self, counts, trials):
        h = (C.c_int64 * 4)(*[int(v) for v in counts.cpu().tolist()])
        rep = abi.CampaignReport()
        call("abed_campaign_report_of", self.handle, h, trials, C.byref(rep))
        return rep

    def __del__(self):
        try:
            if self.handle:
                call("abed_campaign_destroy", self.handle)
        except Exception:
            pass


# ------------------------------------------------------------------ protected conv plan (hot path)
# ---------------------------------------------------------------- ABFT GEMM
ABFT_CHECKED, ABFT_PLAIN, ABFT_FUSED_ROW = 0, 1, 2


def abft_gemm(a, b):
    """abft_gemm (abft_gemm.hpp:102-152): row/column-checksum ABFT for an int8 GEMM
    on the tcgen05 GEMM.  a: m x k, b: k x n int8 CUDA tensors (row-major).
    Returns (c int32 m x n, c_aug int64 (m+1) x (n+1), row_check, col_check)."""
    if a.dtype != torch.int8 or b.dtype != torch.int8:
        raise abi.InvalidArgument(abi.ERR_INVALID_ARGUMENT, "abft_gemm: operands must be i8")
    m, k = a.shape
    kb, n = b.shape
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    ca = torch.empty((m + 1, n + 1), dtype=torch.int64, device=a.device)
    row, col = VerifyOutcome(), VerifyOutcome()
    _sync()
    call("abed_abft_gemm_i8", _p(a), m, k, _p(b), kb, n, _p(c), _p(ca), C.byref(row), C.byref(col))
    return c, ca, row, col


def abft_check(c_aug):
    """abft_check (abft_gemm.hpp:70-96) on an int64 (m+1) x (n+1) CUDA tensor -> (row, col)."""
    row, col = VerifyOutcome(), VerifyOutcome()
    _sync()
    call("abed_abft_check", _p(c_aug), c_aug.shape[0], c_aug.shape[1], C.byref(row), C.byref(col))
    return row, col


class AbftPlan:
    """Allocation-free ABFT GEMM runs on the current stream (timing, graphs).
    mode ABFT_CHECKED: the reference's online tasks (2)-(6); ABFT_PLAIN: the same
    GEMM without checksums; ABFT_FUSED_ROW: row check fused into the GEMM epilogue."""

    def __init__(self, m, n, k):
        self.m, self.n, self.k = m, n, k
        h = C.c_void_p()
        call("abed_abft_plan_create", m, n, k, C.byref(h))
        self.h = h
        self.outcomes = torch.zeros(2 * C.sizeof(VerifyOutcome), dtype=torch.uint8, device="cuda")

    def run(self, a, b, c=None, c_aug=None, mode=ABFT_CHECKED):
        call("abed_abft_plan_run", self.h, _p(a), _p(b) if b is not None else None, _p(c) if c is not None else None,
             _p(c_aug) if c_aug is not None else None, _p(self.outcomes), mode, _stream())

    def verdicts(self):
        raw = self.outcomes.cpu().numpy().tobytes()
        sz = C.sizeof(VerifyOutcome)
        return VerifyOutcome.from_buffer_copy(raw[:sz]), VerifyOutcome.from_buffer_copy(raw[sz:])

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and abi is not None and abi._lib is not None:
            abi._lib.abed_abft_plan_destroy(h)
            self.h = None


class ConvPlan:
    """One protected layer: packed filters (+ FC checksum-digit rows), the offline
    filter checksum and the per-tile verification workspace."""

    def __init__(self, ls: LayerShape, filters: torch.Tensor, checks: int = 0, block_n: int = 0):
        self.ls = ls
        self.checks = checks
        self.handle = C.c_void_p()
        call("abed_conv_plan_create", C.byref(ls), _p(filters), checks, block_n, C.byref(self.handle))
        self.info = abi.PlanInfo()
        call("abed_conv_plan_info", self.handle, C.byref(self.info))
        self._outcomes = torch.zeros(3 * C.sizeof(VerifyOutcome), dtype=torch.uint8, device="cuda")

    def __del__(self):
        try:
            if self.handle:
                abi.load().abed_conv_plan_destroy(self.handle)
        except Exception:
            pass

    def packed_buffer(self) -> torch.Tensor:
        return torch.zeros(self.info.packed_input_bytes, dtype=torch.int8, device="cuda")

    def pack(self, x_nchw: torch.Tensor, packed: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        packed = self.packed_buffer() if packed is None else packed
        call("abed_pack_input", self.handle, _p(x_nchw), _p(packed), stream or _stream())
        return packed

    def run(self, packed, out=None, out_mode=abi.OUT_I8_NCHW, scale=1.0, bias=None, relu=True, next_plan=None,
            fault_key=-1, fault_bit=0, stream=None, ep=None):
        if ep is None:
            ep = self.epilog_params(scale, bias, relu)
            _keep_alive(self._bias, stream)
        call("abed_conv_plan_run", self.handle, _p(packed), C.byref(ep) if ep is not None else None, out_mode,
             C.c_void_p(out.data_ptr()) if out is not None else None, next_plan.handle if next_plan else None,
             fault_key, fault_bit, stream or _stream())
        return out

    def epilog_params(self, scale=1.0, bias=None, relu=True):
        if bias is None:
            self._bias = None
            return abi.EpilogParams(scale, None, 0, abi.RELU if relu else abi.IDENTITY, I8)
        self._bias = torch.as_tensor(bias, dtype=torch.float32).reshape(-1).cuda()
        return abi.EpilogParams(scale, self._bias.data_ptr(), self._bias.numel(), abi.RELU if relu else abi.IDENTITY, I8)

    def finalize(self, stream=None):
        call("abed_conv_plan_finalize", self.handle, _p(self._outcomes), stream or _stream())

    def set_input_checksum_source(self, source: int = abi.RHS_STAGED):
        """FIC rhs from the staged activation tiles (default) or a re-read of the input (FR)."""
        call("abed_conv_plan_set_input_checksum_source", self.handle, source)

    def set_paired_finalize(self, on: bool = True):
        """IC plans: captured graphs finalize every run they contain (no clearing memsets)."""
        call("abed_conv_plan_set_paired_finalize", self.handle, 1 if on else 0)

    def set_af_input(self, on: bool = True):
        """FIC-AF: this layer's FIC rhs comes from the previous layer's epilogue."""
        call("abed_conv_plan_set_af_input", self.handle, 1 if on else 0)

    def outcomes(self):
        """(FC, FIC, IC) VerifyOutcomes of the last finalize (synchronises)."""
        host = self._outcomes.cpu().numpy()
        res = (VerifyOutcome * 3)()
        C.memmove(res, host.ctypes.data, C.sizeof(res))
        return tuple(res)


class ConvPlanDW(ConvPlan):
    """Depthwise layer (one filter per channel, K == C, filters C x 1 x R x S int8)
    on the strip-plane layout; checks 0 or abi.CHECK_FIC."""

    def __init__(self, ls: LayerShape, filters: torch.Tensor, checks: int = 0):
        self.ls = ls
        self.checks = checks
        self.handle = C.c_void_p()
        call("abed_conv_plan_create_dw", C.byref(ls), _p(filters), checks, C.byref(self.handle))
        self.info = abi.PlanInfo()
        call("abed_conv_plan_info", self.handle, C.byref(self.info))
        self._outcomes = torch.zeros(3 * C.sizeof(VerifyOutcome), dtype=torch.uint8, device="cuda")


class PlanSet:
    """Verdicts of a whole pass: one finalize launch for many plans
    (abed_conv_plan_finalize_many); outcomes()[i] = plan i's (FC, FIC, IC)."""

    def __init__(self, plans):
        self.plans = list(plans)
        self._arr = (C.c_void_p * len(self.plans))(*[pl.handle.value for pl in self.plans])
        self._out = torch.zeros(3 * len(self.plans) * C.sizeof(VerifyOutcome), dtype=torch.uint8, device="cuda")

    def finalize(self, stream=None):
        call("abed_conv_plan_finalize_many", C.cast(self._arr, C.c_void_p), len(self.plans), _p(self._out),
             stream or _stream())

    def outcomes(self):
        host = self._out.cpu().numpy()
        res = (VerifyOutcome * (3 * len(self.plans)))()
        C.memmove(res, host.ctypes.data, C.sizeof(res))
        return [tuple(res[3 * i:3 * i + 3]) for i in range(len(self.plans))]


# ------------------------------------------------------------------ float mode on tensor cores
class ConvPlanH(ConvPlan):
    """Float-mode protected layer (checksum.hpp:471-595 semantics on tcgen05
    kind::f16): f32 filters rounded to fp16 / bf16 (elem_kind abi.F16 / abi.BF16),
    f32 accumulation, FC / FIC with absolute thresholds tau_fc / tau_fic."""

    def __init__(self, ls: LayerShape, filters_f32: torch.Tensor, elem_kind: int = abi.F16, checks: int = 0,
                 tau_fc: float = 0.0, tau_fic: float = 0.0, block_n: int = 0):
        self.ls = ls
        self.checks = checks
        self.elem_kind = elem_kind
        self.handle = C.c_void_p()
        f = filters_f32.contiguous().to(torch.float32)
        call("abed_conv_plan_create_h", C.byref(ls), _p(f), elem_kind, checks, float(tau_fc), float(tau_fic), block_n,
             C.byref(self.handle))
        self.info = abi.PlanInfo()
        call("abed_conv_plan_info", self.handle, C.byref(self.info))
        self._outcomes = torch.zeros(3 * C.sizeof(VerifyOutcome), dtype=torch.uint8, device="cuda")

    def set_tau(self, tau_fc: float, tau_fic: float):
        call("abed_conv_plan_set_tau", self.handle, float(tau_fc), float(tau_fic))

    def pack(self, x_nchw_f32: torch.Tensor, packed: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        packed = self.packed_buffer() if packed is None else packed
        x = x_nchw_f32.contiguous().to(torch.float32)
        call("abed_pack_input_h", self.handle, _p(x), _p(packed), stream or _stream())
        if x is not x_nchw_f32:
            _keep_alive(x, stream)
        return packed

    def run(self, packed, out=None, out_mode=abi.OUT_F32_NCHW, scale=1.0, bias=None, relu=False, next_plan=None,
            fault_key=-1, fault_bit=0, stream=None, ep=None):
        return super().run(packed, out, out_mode, scale, bias, relu, next_plan, fault_key, fault_bit, stream, ep)
