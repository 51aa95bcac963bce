#!/usr/bin/env python3
"""Benchmark of the ABED-protected INT8 convolution hot path on B200.

Workload (BASELINE.json configs[1]): the 16 ResNet-50 3x3 conv layers
(network_config.hpp:233-282, conv2 of every bottleneck) in INT8 at batch 32 per
GPU with fused bias + ReLU + requantise, protected by FIC (headline), FC, and
compared with the same kernel unprotected and with full duplication.  One step =
one pass of all 16 layers over one synthetic batch (SplitMix64 int8 data).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Timing: CUDA events on the launching stream
around a CUDA-graph replay of the whole step, L2 flushed (512 MiB memset + read-back, bench.l2_flush)
before every timed step, max over ranks.  The reference arm times the
reference's own CPU implementation (oracle/_ref, built from the reference
headers) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ResNet-50 3x3 convs (name, n, c, h, w, k, r, s, stride, pad), batch per GPU = 32
RESNET50_3X3 = (
    [(f"layer1.{i}.conv2", 64, 56, 56, 64, 1) for i in range(3)]
    + [("layer2.0.conv2", 128, 56, 56, 128, 2)] + [(f"layer2.{i}.conv2", 128, 28, 28, 128, 1) for i in range(1, 4)]
    + [("layer3.0.conv2", 256, 28, 28, 256, 2)] + [(f"layer3.{i}.conv2", 256, 14, 14, 256, 1) for i in range(1, 6)]
    + [("layer4.0.conv2", 512, 14, 14, 512, 2)] + [(f"layer4.{i}.conv2", 512, 7, 7, 512, 1) for i in range(1, 3)]
)
# BASELINE configs[2]: VGG-16 conv stack (network_config.hpp:163-184), 3x3 s1 p1,
# FP16 at batch 64; conv1_1 (C=3) excluded as in SURVEY.md 8(d)
VGG16_3X3 = [("conv1_2", 64, 224, 64), ("conv2_1", 64, 112, 128), ("conv2_2", 128, 112, 128),
             ("conv3_1", 128, 56, 256), ("conv3_2", 256, 56, 256), ("conv3_3", 256, 56, 256),
             ("conv4_1", 256, 28, 512), ("conv4_2", 512, 28, 512), ("conv4_3", 512, 28, 512),
             ("conv5_1", 512, 14, 512), ("conv5_2", 512, 14, 512), ("conv5_3", 512, 14, 512)]
VGG_BATCH = 64
# BASELINE configs[3]: MobileNetV2 inverted-residual blocks, INT8, batch 32 --
# a builder-defined table: (C_in, H=W, expansion, C_out, dw stride);
# each block = pw expand 1x1 (tensor cores) -> dw 3x3 (CUDA cores) -> pw project 1x1,
# chained through the packed layout
MBV2_BLOCKS = [(16, 112, 6, 24, 2), (24, 56, 6, 24, 1), (32, 28, 6, 32, 1), (64, 14, 6, 64, 1), (160, 7, 6, 160, 1)]
BATCH = 32
METRIC = "ABED conv TOPS & overhead % vs unprotected/duplication; detection coverage"
WORKLOAD = "resnet50-3x3-convs-int8-b32 (16 layers, fused bias+ReLU+requant, FIC-protected)"
PEAK_INT8_NOMINAL = 4500.0


def l2_flush(buf):
    """Evict L2 between timed steps: write the 512 MiB buffer (larger than the
    126 MB L2), then read it back so the lines left in L2 are clean -- otherwise the
    write-back of the flush buffer's dirty lines lands inside the next timed step
    and is charged to the kernel.  ABED_BENCH_FLUSH=write keeps the write-only
    flush (for comparison)."""
    import torch

    buf.zero_()
    if os.environ.get("ABED_BENCH_FLUSH", "clean") != "write":
        buf.view(torch.int64).amax()


def pinned_wc_host(nbytes):
    """Pinned, write-combined host memory as an int8 tensor (cudaHostAlloc with
    cudaHostAllocWriteCombined): the H2D staging side of the e2e leg.  The host only
    writes it, the GPU reads it over PCIe without snooping the CPU caches --
    measured 55 GB/s steady where ordinary pinned memory read 11-55 GB/s on the
    same box (tools/pcie_probe.py).  Falls back to ordinary pinned memory."""
    import ctypes

    import numpy as np
    import torch
    try:
        from cuda.bindings import runtime as rt
        err, ptr = rt.cudaHostAlloc(max(1, nbytes), rt.cudaHostAllocWriteCombined)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(str(err))
        arr = np.ctypeslib.as_array((ctypes.c_int8 * max(1, nbytes)).from_address(int(ptr)))
        t = torch.from_numpy(arr)[:nbytes]
        _WC_KEEP.append(ptr)  # freed at exit with the process
        return t
    except Exception:  # noqa: BLE001
        return torch.empty(nbytes, dtype=torch.int8).pin_memory()


_WC_KEEP = []


def workload_config(per_gpu_batch, world, global_batch=0):
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": WORKLOAD if not global_batch else WORKLOAD.replace("-b32", f"-b{per_gpu_batch * world}"),
            "global_batch": per_gpu_batch * world, "per_gpu_batch": per_gpu_batch, "layers": 16,
            "shapes": "ResNet-50 conv2 3x3 of every bottleneck (network_config.hpp:233-282), stride 2 at the first of "
                      "layer2-4, pad 1", "epilog": "bias linspace(-2,2), scale 0.05, ReLU, int8 requantise",
            "check": "FIC", "parallelism": f"dp{world}",
            "l2": "GPU arm: flushed (512 MiB memset + read-back: clean lines) before every timed step"}


def layer_ops(c, h, w, k, stride, n=BATCH):
    p = (h + 2 - 3) // stride + 1
    q = (w + 2 - 3) // stride + 1
    return 2 * n * k * p * q * c * 9


def total_ops(n=BATCH):
    return sum(layer_ops(c, h, w, k, st, n) for _, c, h, w, k, st in RESNET50_3X3)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ---------------------------------------------------------------- distributed
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- CPU reference
def _cpu_reference_lib():
    from oracle.pyoracle import Oracle, build_oracle, ref_available, ref_kind
    if not ref_available() and os.path.isdir("/root/reference/proj/include/abed"):
        build_oracle()
    if ref_available():
        return Oracle("ref"), "reference", ref_kind()
    return Oracle("ora"), "port", "C oracle"


def cpu_reference_pass(ref, kind, threads, batch, seed):
    """One step of the workload through the reference's own CPU path (oracle/_ref:
    detail::conv_fast_i8 + gen_input_checksum + fic_dot + fic_verify + epilog, the
    batch split over `threads` std::threads).  Returns (ops, seconds)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    ops, secs = 0, 0.0
    for _, c, h, w, k, st in RESNET50_3X3:
        ls = ref.layer_shape(batch, c, h, w, k, 3, 3, st, st, 1, 1)
        x = rng.integers(-128, 128, ls.input_dims(), dtype=np.int8)
        f = rng.integers(-128, 128, ls.filter_dims(), dtype=np.int8)
        if kind == "reference":
            secs += ref.time_layer(ls, 3, threads, x, f)  # scheme 3 = FIC
        else:  # single-threaded C restatement
            t0 = time.perf_counter()
            conv = ref.conv_i8(x, f, ls)
            ref.fic_verify(conv, ref.fic_dot(ref.gen_filter_checksum(f), ref.gen_input_checksum(x, ls)))
            ref.epilog(conv, 0.05, np.zeros(ls.k, np.float32))
            secs += time.perf_counter() - t0
        ops += layer_ops(c, h, w, k, st, n=batch)
    return ops, secs


def cpu_reference_sample(target_s=10.0, batch=BATCH):
    """Bounded sample for cpu_baseline: whole steps (16 layers, batch 32) until
    ~target_s of CPU time.  Returns (TOPS, description, cores, kind)."""
    ref, kind, flavour = _cpu_reference_lib()
    threads = (os.cpu_count() or 1) if kind == "reference" else 1
    ops, secs, reps = 0, 0.0, 0
    while reps == 0 or secs < target_s:
        o, s = cpu_reference_pass(ref, kind, threads, batch, seed=reps)
        ops += o
        secs += s
        reps += 1
    desc = (f"{reps} step(s) of the workload (16 ResNet-50 3x3 layers, batch {batch}) through the reference CPU path "
            f"({flavour}): conv_fast_i8 + FIC check + epilog, batch split over {threads} thread(s); {secs:.2f}s")
    return ops / secs / 1e12, desc, min(threads, batch), kind


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU implementation on this host's cores."""
    if rank != 0:
        return 0
    t_start = time.time()
    ref, kind, flavour = _cpu_reference_lib()
    threads = (os.cpu_count() or 1) if kind == "reference" else 1
    for i in range(args.warmup):
        cpu_reference_pass(ref, kind, threads, BATCH, seed=100 + i)
    ops, secs, per = 0, 0.0, []
    for i in range(args.steps):
        o, s = cpu_reference_pass(ref, kind, threads, BATCH, seed=i)
        ops += o
        secs += s
        per.append(s)
    value = ops / secs / 1e12
    desc = (f"{args.steps} step(s) of the workload through the reference CPU path ({flavour}): conv_fast_i8 + FIC "
            f"check + epilog, batch {BATCH} split over {threads} thread(s)")
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(per), 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic (random int8, numpy)",
        "impl": "reference",
        "config": workload_config(BATCH, world),
        "method": {"where": "host CPU threads (rank 0 only)", "threads": threads},
        "cpu_baseline": {"value": round(value, 5), "unit": "TOPS", "cores": min(threads, BATCH), "kind": kind,
                         "sample": desc},
        "e2e": {"value": round(value, 5), "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t_start, 1),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{device_index}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def keep_busy(self, fn, seconds):
        import torch
        t_end = time.time() + seconds
        while time.time() < t_end:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measure_vgg16_fp16(args, dev, stream, flush, world, dist):
    """BASELINE configs[2]: the 12 VGG-16 3x3 convs (C >= 64) in FP16 on tensor
    cores (f32 accumulate), batch 64 per GPU, epilog ReLU -> fp16 packed output,
    unprotected / FC / FIC (absolute thresholds, float_verify semantics) /
    full duplication.  Thresholds from the f32-accumulation error bound:
    tau = (CRS + 32) * 2^-22 * max|x| * sum|f| (FC per pixel; FIC times N*P*Q)."""
    import torch

    from paper_2006_04984_b200 import abi, api
    gen = torch.Generator(device=dev)
    gen.manual_seed(2006_04984)
    layers = []
    flops = 0
    for name, c, hw, k in VGG16_3X3:
        ls = api.layer_shape(VGG_BATCH, c, hw, hw, k, 3, 3, 1, 1, 1, 1)
        x = torch.empty(ls.input_dims(), dtype=torch.float32, device=dev).uniform_(-1, 1, generator=gen)
        f = torch.empty(ls.filter_dims(), dtype=torch.float32, device=dev).uniform_(-1, 1, generator=gen) * 0.05
        sum_f = float(f.abs().sum())
        crs = c * 9
        tau_fc = (crs + k + 32) * 2.0 ** -22 * sum_f
        tau_fic = (crs + 32) * 2.0 ** -22 * sum_f * ls.p * ls.q * VGG_BATCH
        L = {"name": name, "ls": ls}
        L["plans"] = {"unprotected": api.ConvPlanH(ls, f, abi.F16, 0),
                      "fc": api.ConvPlanH(ls, f, abi.F16, abi.CHECK_FC, tau_fc, tau_fic),
                      "fic": api.ConvPlanH(ls, f, abi.F16, abi.CHECK_FIC, tau_fc, tau_fic)}
        L["packed"] = L["plans"]["unprotected"].pack(x)
        del x
        L["out"] = L["plans"]["unprotected"].packed_buffer() if False else None
        # identity consumer of the fp16 output: 8 channels per 16-byte pixel
        out_elems = VGG_BATCH * ((k + 15) // 16 * 16) * (ls.p + 1) * (ls.q + 1) + (1 << 16)
        L["out"] = torch.zeros(out_elems * 2, dtype=torch.int8, device=dev)
        L["ep"] = {kk: pl.epilog_params(1.0, None, True) for kk, pl in L["plans"].items()}
        flops += 2 * VGG_BATCH * k * ls.p * ls.q * crs
        layers.append(L)
    torch.cuda.synchronize()

    sets = {v: api.PlanSet([L["plans"][v] for L in layers]) for v in ("fc", "fic")}

    def step(variant):
        for L in layers:
            if variant == "dup":
                pl = L["plans"]["unprotected"]
                pl.run(L["packed"], L["out"], abi.OUT_H_PACKED, ep=L["ep"]["unprotected"])
                pl.run(L["packed"], L["out"], abi.OUT_H_COMPARE, ep=L["ep"]["unprotected"])
            else:
                pl = L["plans"][variant]
                pl.run(L["packed"], L["out"], abi.OUT_H_PACKED, ep=L["ep"][variant])
        if variant in sets:
            sets[variant].finalize()

    with torch.cuda.stream(stream):
        for v in ("unprotected", "fc", "fic", "dup"):
            step(v)
    torch.cuda.synchronize()
    graphs = {}
    for v in ("unprotected", "fc", "fic", "dup"):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(v)
        graphs[v] = g
    res = {}
    steps = max(3, min(args.steps, 10))
    for v in ("unprotected", "fc", "dup", "fic"):
        for _ in range(max(3, args.warmup)):
            l2_flush(flush)
            graphs[v].replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ts = []
        cur = torch.cuda.current_stream()
        for _ in range(steps):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            graphs[v].replay()
            e1.record(cur)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.mean(ts)
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        res[v] = {"tflops": round(flops * world / (ms * 1e-3) / 1e12, 2), "ms_per_step": round(ms, 4)}
    fails = sum(o.status for v in ("fc", "fic") for oc in sets[v].outcomes() for o in oc[:2])
    u = res["unprotected"]["ms_per_step"]
    vgg_peak = measured_peaks().get("bf16_tflops") or 1590.0
    return {"workload": "vgg16-3x3-convs-fp16-b64 (12 layers, C>=64; f32 accumulate, ReLU, fp16 packed out)",
            "dtype": "fp16 operands, f32 accumulation (tcgen05 kind::f16)", "global_batch": VGG_BATCH * world,
            "gflop_per_step": round(flops * world / 1e9, 1), "variants": res,
            "overhead_pct": {"fic_vs_unprotected": round(100 * (res["fic"]["ms_per_step"] / u - 1), 2),
                             "fc_vs_unprotected": round(100 * (res["fc"]["ms_per_step"] / u - 1), 2),
                             "duplication_vs_unprotected": round(100 * (res["dup"]["ms_per_step"] / u - 1), 2)},
            "tau": "absolute, (CRS+32)*2^-22*max|x|*sum|f| (FC per pixel; FIC x N*P*Q)",
            "fault_free_verdicts_failed": fails,
            "roofline": {"bound": "tensor", "peak_tflops": vgg_peak,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops" if measured_peaks().get("bf16_tflops")
                         else "fallback 1590 (B200_PROFILING.md)",
                         "frac_unprotected": round(res["unprotected"]["tflops"] / vgg_peak, 3),
                         "frac_fic": round(res["fic"]["tflops"] / vgg_peak, 3),
                         "frac_fic_of_sustained": (round(res["fic"]["tflops"] / measured_peaks()["bf16_tflops_sustained"], 3)
                                                   if measured_peaks().get("bf16_tflops_sustained") else None)},
            "peak_note": "fp16 dense peak = MEASURED_PEAKS bf16_tflops (or the 1590 fallback)"}


def measure_mobilenetv2_int8(args, dev, stream, flush, world, dist):
    """BASELINE configs[3]: 5 MobileNetV2 blocks (15 layers: pointwise on tcgen05,
    depthwise on CUDA cores), INT8 at batch 32 per GPU, bias + ReLU6-free ReLU +
    requant, unprotected / FIC (every layer) / duplication, chained through the
    packed layout (low arithmetic intensity: the checksum-overhead stress case)."""
    import torch

    from paper_2006_04984_b200 import abi, api
    layers, ops, seed = [], 0, 900
    hbm_bytes = 0  # algorithmic: every layer reads its input + filters once and writes its output once
    for ci, hw, t, co, st in MBV2_BLOCKS:
        e = ci * t
        ho = (hw + 2 - 3) // st + 1
        shapes = [("pw", api.layer_shape(BATCH, ci, hw, hw, e, 1, 1, 1, 1, 0, 0)),
                  ("dw", api.layer_shape(BATCH, e, hw, hw, e, 3, 3, st, st, 1, 1)),
                  ("pw", api.layer_shape(BATCH, e, ho, ho, co, 1, 1, 1, 1, 0, 0))]
        block = []
        for kind, ls in shapes:
            seed += 1
            hbm_bytes += ls.n * ls.c * ls.h * ls.w + ls.n * ls.k * ls.p * ls.q
            if kind == "pw":
                f = api.fill_random_i8(ls.k * ls.c, api.derive_seed(seed, 2)).view(ls.filter_dims())
                mk = lambda ch, ls=ls, f=f: api.ConvPlan(ls, f, ch)  # noqa: E731
                ops += 2 * ls.n * ls.k * ls.p * ls.q * ls.c
                hbm_bytes += ls.k * ls.c
            else:
                f = api.fill_random_i8(ls.c * 9, api.derive_seed(seed, 2)).view(ls.c, 1, 3, 3)
                mk = lambda ch, ls=ls, f=f: api.ConvPlanDW(ls, f, ch)  # noqa: E731
                ops += 2 * ls.n * ls.k * ls.p * ls.q * 9
                hbm_bytes += ls.c * 9
            L = {"kind": kind, "ls": ls, "plans": {"unprotected": mk(0), "fic": mk(abi.CHECK_FIC),
                                                    "fic_af": mk(abi.CHECK_FIC)}}
            if block:  # FIC-AF: rhs accumulated by the producing layer's epilogue
                L["plans"]["fic_af"].set_af_input(True)
            L["ep"] = {v: pl.epilog_params(0.02, None, True) for v, pl in L["plans"].items()}
            block.append(L)
        # activation buffers: block input (fresh data), then each layer writes the next one's input
        x = api.fill_random_i8(shapes[0][1].n * ci * hw * hw, api.derive_seed(seed, 1)).view(shapes[0][1].input_dims())
        block[0]["in"] = block[0]["plans"]["unprotected"].pack(x)
        for a, b in zip(block, block[1:]):
            a["out"] = b["plans"]["unprotected"].packed_buffer()
            a["next"] = b
            b["in"] = a["out"]
        last = block[-1]["ls"]
        block[-1]["out"] = torch.zeros(last.n * ((last.k + 15) // 16 * 16) * (last.p + 1) * (last.q + 1) + (1 << 16),
                                       dtype=torch.int8, device=dev)
        block[-1]["next"] = None
        layers += block
    VARIANTS = ("unprotected", "fic", "fic_af", "dup")
    sets = {v: api.PlanSet([L["plans"][v] for L in layers]) for v in ("fic", "fic_af")}

    def step(variant):
        for L in layers:
            nxt = L["next"]["plans"]["fic_af" if variant == "fic_af" else "unprotected"] if L["next"] else None
            if variant == "dup":
                pl = L["plans"]["unprotected"]
                pl.run(L["in"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"]["unprotected"], next_plan=nxt)
                pl.run(L["in"], L["out"], abi.OUT_I8_COMPARE, ep=L["ep"]["unprotected"], next_plan=nxt)
            else:
                pl = L["plans"][variant]
                pl.run(L["in"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"][variant], next_plan=nxt)
        if variant in sets:
            sets[variant].finalize()

    with torch.cuda.stream(stream):
        for v in VARIANTS:
            step(v)
    torch.cuda.synchronize()
    graphs = {}
    for v in VARIANTS:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(v)
        graphs[v] = g
    res = {}
    for v in VARIANTS:
        for _ in range(max(3, args.warmup)):
            l2_flush(flush)
            graphs[v].replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ts = []
        cur = torch.cuda.current_stream()
        for _ in range(max(3, args.steps)):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            graphs[v].replay()
            e1.record(cur)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.mean(ts)
        if dist:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        res[v] = {"tops": round(ops * world / (ms * 1e-3) / 1e12, 2), "ms_per_step": round(ms, 4)}
    fails = sum(oc[1].status for v in ("fic", "fic_af") for oc in sets[v].outcomes())
    u = res["unprotected"]["ms_per_step"]
    return {"workload": "mobilenetv2-5-blocks-int8-b32 (15 layers: pw 1x1 tcgen05 + dw 3x3 CUDA cores, chained)",
            "fic_af": "FIC with each in-block layer's input checksum accumulated by the producing epilogue",
            "blocks": [list(b) for b in MBV2_BLOCKS], "global_batch": BATCH * world,
            "gop_per_step": round(ops * world / 1e9, 2), "variants": res,
            # HBM-bound stress config: algorithmic bytes (each layer's int8 input, output and
            # filters once) per step over the step time, against the measured copy bandwidth
            "roofline": {"bound": "hbm", "algorithmic_bytes_per_step": int(hbm_bytes * world),
                         "achieved_gbs_fic": round(hbm_bytes * world / (res["fic"]["ms_per_step"] * 1e-3) / 1e9, 1),
                         "achieved_gbs_unprotected": round(hbm_bytes * world / (u * 1e-3) / 1e9, 1),
                         "peak_gbs": measured_peaks().get("hbm_gbs") or 7700.0,
                         "frac_fic": round(hbm_bytes * world / (res["fic"]["ms_per_step"] * 1e-3) / 1e9 /
                                           (measured_peaks().get("hbm_gbs") or 7700.0), 3),
                         "note": "15 chained launches of small layers: per-launch latency, not bandwidth, sets "
                                 "the step time"},
            "overhead_pct": {"fic_vs_unprotected": round(100 * (res["fic"]["ms_per_step"] / u - 1), 2),
                             "fic_af_vs_unprotected": round(100 * (res["fic_af"]["ms_per_step"] / u - 1), 2),
                             "duplication_vs_unprotected": round(100 * (res["dup"]["ms_per_step"] / u - 1), 2)},
            "fault_free_verdicts_failed": fails}


def resnet50_chains(batch):
    """Every ResNet-50 conv after the stem (network_config.hpp:245-282 builtin at
    224x224; conv1 is excluded like the reference's exclude_first_layer): per
    bottleneck the chain conv1 1x1 -> conv2 3x3 -> conv3 1x1, plus the 1x1
    projection of each stage's first block as a chain of its own.  The residual
    adds and pooling are not convolutions and are not part of this library, so
    each chain starts from fresh packed data."""
    from paper_2006_04984_b200 import api
    chains, h, c = [], 56, 64
    for st, (blocks, width) in enumerate(((3, 64), (4, 128), (6, 256), (3, 512))):
        out = 4 * width
        for b in range(blocks):
            s = 2 if (b == 0 and st > 0) else 1
            ho = (h + 2 - 3) // s + 1
            chains.append([api.layer_shape(batch, c, h, h, width, 1, 1, 1, 1, 0, 0),
                           api.layer_shape(batch, width, h, h, width, 3, 3, s, s, 1, 1),
                           api.layer_shape(batch, width, ho, ho, out, 1, 1, 1, 1, 0, 0)])
            if b == 0:
                chains.append([api.layer_shape(batch, c, h, h, out, 1, 1, s, s, 0, 0)])
            h, c = ho, out
    return chains


def measure_resnet50_network(args, dev, stream, flush, world, dist):
    """whole-network protected INT8 inference -- all 52
    ResNet-50 convs after the stem at batch 32 per GPU, bias + ReLU + requant,
    chained through the packed layout.  Variants: unprotected, FIC with every
    layer's input checksum from a second read of its input (FR), FIC-AF (inside a
    chain the producing epilogue accumulates the consumer's input checksum from the
    values it stores, cost-model option AF; chain heads stay FR), and full
    duplication.  Overheads here are the inference-level numbers the paper quotes."""
    import torch

    from paper_2006_04984_b200 import abi, api
    layers, ops, seed = [], 0, 5000
    for chain in resnet50_chains(BATCH):
        block = []
        for ls in chain:
            seed += 1
            f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(seed, 2)).view(ls.filter_dims())
            ops += 2 * ls.n * ls.k * ls.p * ls.q * ls.c * ls.r * ls.s
            L = {"ls": ls, "plans": {"unprotected": api.ConvPlan(ls, f, 0), "fic": api.ConvPlan(ls, f, abi.CHECK_FIC),
                                     "fic_sm": api.ConvPlan(ls, f, abi.CHECK_FIC),
                                     "fic_af": api.ConvPlan(ls, f, abi.CHECK_FIC)}}
            L["plans"]["fic_sm"].set_input_checksum_source(abi.RHS_STAGED)
            if block:
                L["plans"]["fic_af"].set_af_input(True)
            bias = torch.linspace(-1.0, 1.0, ls.k).tolist()
            L["ep"] = {v: pl.epilog_params(0.02, bias, True) for v, pl in L["plans"].items()}
            block.append(L)
        ls0 = chain[0]
        x = api.fill_random_i8(ls0.n * ls0.c * ls0.h * ls0.w, api.derive_seed(seed, 1)).view(ls0.input_dims())
        block[0]["in"] = block[0]["plans"]["unprotected"].pack(x)
        for a, b in zip(block, block[1:]):
            a["out"] = b["plans"]["unprotected"].packed_buffer()
            a["next"] = b
            b["in"] = a["out"]
        last = block[-1]["ls"]
        block[-1]["out"] = torch.zeros(last.n * ((last.k + 15) // 16 * 16) * (last.p + 1) * (last.q + 1) + (1 << 16),
                                       dtype=torch.int8, device=dev)
        block[-1]["next"] = None
        layers += block
    VARIANTS = ("unprotected", "fic", "fic_sm", "fic_af", "dup")
    sets = {v: api.PlanSet([L["plans"][v] for L in layers]) for v in ("fic", "fic_sm", "fic_af")}

    def step(variant):
        for L in layers:
            nxt = L["next"]["plans"]["fic_af" if variant == "fic_af" else "unprotected"] if L["next"] else None
            if variant == "dup":
                pl = L["plans"]["unprotected"]
                pl.run(L["in"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"]["unprotected"], next_plan=nxt)
                pl.run(L["in"], L["out"], abi.OUT_I8_COMPARE, ep=L["ep"]["unprotected"], next_plan=nxt)
            else:
                pl = L["plans"][variant]
                pl.run(L["in"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"][variant], next_plan=nxt)
        if variant in sets:
            sets[variant].finalize()

    with torch.cuda.stream(stream):
        for v in VARIANTS:
            step(v)
    torch.cuda.synchronize()
    graphs = {}
    for v in VARIANTS:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(v)
        graphs[v] = g
    res = {}
    cur = torch.cuda.current_stream()
    for v in VARIANTS:
        for _ in range(max(3, args.warmup)):
            l2_flush(flush)
            graphs[v].replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ts = []
        for _ in range(max(3, args.steps)):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            graphs[v].replay()
            e1.record(cur)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.mean(ts)
        if dist:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        res[v] = {"tops": round(ops * world / (ms * 1e-3) / 1e12, 2), "ms_per_step": round(ms, 4)}
    fails = sum(oc[1].status for v in ("fic", "fic_sm", "fic_af") for oc in sets[v].outcomes())
    u = res["unprotected"]["ms_per_step"]
    return {"workload": f"resnet50-all-convs-int8-b{BATCH} ({len(layers)} convs after the stem: 1x1 + 3x3 + "
                        "projections, chained per bottleneck; residual adds / pooling not modelled)",
            "fic_af": "FIC; inside each bottleneck chain the producing epilogue accumulates the consumer's "
                      "input checksum (chain heads re-read their input)",
            "global_batch": BATCH * world, "layers": len(layers), "gop_per_step": round(ops * world / 1e9, 2),
            "variants": res,
            "overhead_pct": {"fic_vs_unprotected": round(100 * (res["fic"]["ms_per_step"] / u - 1), 2),
                             "fic_sm_vs_unprotected": round(100 * (res["fic_sm"]["ms_per_step"] / u - 1), 2),
                             "fic_af_vs_unprotected": round(100 * (res["fic_af"]["ms_per_step"] / u - 1), 2),
                             "duplication_vs_unprotected": round(100 * (res["dup"]["ms_per_step"] / u - 1), 2)},
            "fault_free_verdicts_failed": fails}


# ---------------------------------------------------------------- GPU arm
def measure_hbm_kernels(dev, stream, flush, peaks):
    """The HBM-bound checksum kernels and the layout boundary
    on ResNet-50 layer1 tensors at batch 256 (a batch-32 tensor, 6.4 MB, is launch-latency
    bound, not HBM-bound): a CUDA graph of 8 launches, each on its own copy of the
    tensors (8 x 106 MB > L2, so no launch finds its inputs in L2), timed after an
    L2 flush, per-launch = total / 8 (the event clock ticks in ~2 us steps, too
    coarse for one launch), median of 20.  The
    standalone epilog (K9) validates its bias on the host (synchronously, as the
    reference throws on non-finite values) and is read from the ncu launch list.  Achieved =
    algorithmic bytes (every input byte read once, every output byte written once) /
    time, against the measured HBM copy bandwidth."""
    import ctypes as C

    import torch

    from paper_2006_04984_b200 import abi, api

    n, c, h, w, k = 256, 64, 56, 56, 64
    R = 8  # launches per graph, each on its own buffers (8 x 106 MB: no L2 reuse between them)
    xs = [api.fill_random_i8(n * c * h * w, api.derive_seed(77, 1 + 10 * i)).view(n, c, h, w) for i in range(R)]
    f4s = [api.fill_random_i8(512 * 512 * 9, api.derive_seed(77, 2 + 10 * i)).view(512, 512, 3, 3) for i in range(R)]
    ls = api.layer_shape(n, c, h, w, k, 3, 3, 1, 1, 1, 1)
    f1 = api.fill_random_i8(k * c * 9, api.derive_seed(77, 3)).view(k, c, 3, 3)
    plan = api.ConvPlan(ls, f1, 0)
    packs = [plan.packed_buffer() for _ in range(R)]
    sums_f = [torch.empty((1, 512, 3, 3), dtype=torch.int32, device=dev) for _ in range(R)]
    sums_x = [torch.empty((1, c, h, w), dtype=torch.int32, device=dev) for _ in range(R)]
    st = C.c_void_p(stream.cuda_stream)
    cases = {
        "gen_filter_checksum (K6, 512x512x3x3 filters)": (
            lambda i: abi.call("abed_gen_filter_checksum", f4s[i].data_ptr(), api._dims(f4s[i]), sums_f[i].data_ptr(),
                               st),
            f4s[0].numel() + sums_f[0].numel() * 4),
        "ic_batch_checksum (K7, 256x64x56x56 input)": (
            lambda i: abi.call("abed_ic_batch_checksum", xs[i].data_ptr(), api._dims(xs[i]), sums_x[i].data_ptr(), st),
            xs[0].numel() + sums_x[0].numel() * 4),
        "pack_input (NCHW -> strip planes, 256x64x56x56)": (
            lambda i: abi.call("abed_pack_input", plan.handle, xs[i].data_ptr(), packs[i].data_ptr(), st),
            xs[0].numel() + plan.info.packed_input_bytes),
    }
    peak = peaks.get("hbm_gbs") or 7700.0
    res = {}
    with torch.cuda.stream(stream):
        for name, (fn, nbytes) in cases.items():
            for i in range(R):
                fn(i)
            g = torch.cuda.CUDAGraph()  # R launches per replay on distinct buffers: no host gaps
            with torch.cuda.graph(g, stream=stream):
                for i in range(R):
                    fn(i)
            ts = []
            for _ in range(20):
                l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / R)
            us = statistics.median(ts)
            gbs = nbytes / (us * 1e-6) / 1e9
            res[name] = {"us": round(us, 2), "bytes": int(nbytes), "achieved_gbs": round(gbs, 1),
                         "frac_of_hbm": round(gbs / peak, 3)}
    torch.cuda.synchronize()
    return {"peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks.get("hbm_gbs") else "fallback 7700",
            "timing": "CUDA graph of 8 launches on 8 distinct buffer sets (no L2 reuse) after an L2 flush, CUDA events / 8, median of 20", "kernels": res}


def measure_abft_gemm(dev, stream, flush):
    """the classical row/column-checksum ABFT (reference
    abft_gemm.hpp) on the B200 against the same GEMM unprotected and with the ABED
    style check fused into the GEMM epilogue (the filter-checksum column = ABFT's
    row check).  GEMMs = the im2col products of ResNet-50 3x3 layers at batch 32
    (m = N.P.Q, k = C.R.S, n = K).  All three modes run the same pipeline on the
    tcgen05 kernel with both operands supplied at run time (pack A, pack B, GEMM,
    copy-out; "weights_offline" keeps B packed from the warm-up, as ABED's offline
    filter checksum assumes); ABFT adds its online tasks (checksum row / column as digit rows,
    the larger GEMM, the dual output-checksum passes over the i64 c_aug).  Each
    mode: one captured CUDA graph, L2 flushed before every replay, median of 20."""
    import torch

    from paper_2006_04984_b200 import api

    shapes = {"layer2 (25088x1152x128)": (25088, 1152, 128), "layer3 (6272x2304x256)": (6272, 2304, 256)}
    out = {}
    with torch.cuda.stream(stream):
        for name, (m, k, n) in shapes.items():
            a = api.fill_random_i8(m * k, api.derive_seed(91, 1)).view(m, k)
            b = api.fill_random_i8(k * n, api.derive_seed(91, 2)).view(k, n)
            c = torch.empty((m, n), dtype=torch.int32, device=dev)
            ca = torch.empty((m + 1, n + 1), dtype=torch.int64, device=dev)
            plan = api.AbftPlan(m, n, k)
            res = {}
            for label, mode in (("plain", api.ABFT_PLAIN), ("abed_fused_row", api.ABFT_FUSED_ROW),
                                ("abft", api.ABFT_CHECKED)):
                for _ in range(3):
                    plan.run(a, b, c, ca, mode)
                torch.cuda.synchronize()
                row, col = plan.verdicts()
                assert row.status == 0 and col.status == 0, (name, label)
                for setting, bb in (("online", b), ("weights_offline", None)):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        plan.run(a, bb, c, ca, mode)
                    ts = []
                    for _ in range(20):
                        l2_flush(flush)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        g.replay()
                        e1.record(stream)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    us = statistics.median(ts)
                    res.setdefault(setting, {})[label] = {"us": round(us, 2),
                                                          "tops": round(2.0 * m * n * k / (us * 1e-6) / 1e12, 1)}
            row, col = plan.verdicts()
            out[name] = res
            for setting, r in res.items():
                r["abft_overhead_pct"] = round(100 * (r["abft"]["us"] / r["plain"]["us"] - 1), 1)
                r["abed_fused_row_overhead_pct"] = round(100 * (r["abed_fused_row"]["us"] / r["plain"]["us"] - 1), 1)
            out[name]["abft_verdicts"] = [row.status, col.status]
            del plan
    torch.cuda.synchronize()
    return {"what": "int8 GEMM (im2col shapes of ResNet-50 3x3 layers, batch 32): plain / ABED-style fused row check / "
                    "classical row+column ABFT (abft_gemm.hpp tasks 2-6), all on the tcgen05 GEMM",
            "timing": "one CUDA graph per mode, L2 flushed before each replay, CUDA events, median of 20",
            "gemms": out}


def measure_dropin_calls(dev):
    """The reference-facing one-shot call a drop-in caller makes per layer
    (conv_fast_i8 / conv_direct -> abed_conv_i8, convolution.hpp:224,237): device
    tensors in / out, synchronous like the reference.  First call (plan built and
    cached), then the mean of 20 cached calls, against the plan API's one kernel
    launch for the same layer (ResNet-50 layer1.0.conv2, batch 32).  Host wall
    clock around each synchronous call (the call itself synchronizes)."""
    import time

    import torch

    from paper_2006_04984_b200 import abi, api

    ls = api.layer_shape(32, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(91, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(91, 2)).view(ls.filter_dims())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = api.conv_direct(x, f, ls)
    first = (time.perf_counter() - t0) * 1e3
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        api.conv_direct(x, f, ls)
        ts.append((time.perf_counter() - t0) * 1e3)
    plan = api.ConvPlan(ls, f, 0)
    packed = plan.pack(x)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device=dev)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    e1.record()
    torch.cuda.synchronize()
    assert torch.equal(out, y)
    ops = 2.0 * ls.n * ls.k * ls.p * ls.q * ls.c * 9
    cached = statistics.mean(ts)
    return {"call": "abed_conv_i8 (conv_fast_i8 / conv_direct drop-in), layer1.0.conv2 b32, int32 NCHW out",
            "first_call_ms": round(first, 3), "cached_call_ms": round(cached, 3),
            "cached_call_tops": round(ops / (cached * 1e-3) / 1e12, 2),
            "plan_api_kernel_ms": round(e0.elapsed_time(e1) / 20, 4),
            "note": "one-shot calls pack the filters and the input, run the tensor-core conv and synchronize; "
                    "the plan and its buffers are cached per (device, shape)"}


def measure_campaign_cfg5(args, dev, world, rank, dist):
    """BASELINE configs[4]'s fault-injection campaign: ResNet-50 layer1.0.conv2
    (64 -> 64, 3x3, 56x56) at batch 1024, the batch sharded over the ranks
    (1024 / N images each, generated from the same SplitMix64 stream as the whole
    batch).  Every rank evaluates every trial on its shard with the trial-parallel
    kernel (one CTA per trial: the flip's perturbed ConvOut elements against the
    golden ConvOut), writing per-trial records {check failed, output differs, sum
    delta}; ONE NCCL all-reduce (sum) of the records over NVLink, then a classify
    launch gives the campaign report -- identical for every N.  Timed on the device
    (CUDA events, max over ranks), golden ConvOut excluded (created once).  Rank 0
    also re-runs a few trials through the exhaustive path (one fused protected conv
    of the whole batch per trial) as a cross-check."""
    import torch

    from paper_2006_04984_b200 import abi, api

    n_glob = 1024
    ls = api.layer_shape(n_glob, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)
    n0, n1 = n_glob * rank // world, n_glob * (rank + 1) // world
    trials = args.campaign_trials
    out = {"layer": "resnet50 layer1.0.conv2 64x56x56 -> 64, 3x3 p1, batch 1024 (random int8 data)",
           "images_per_rank": n1 - n0, "trials": trials, "reduction": "NCCL all_reduce(sum) of int64 [trials, 3] records"
           if world > 1 else "none (1 GPU)", "schemes": {}}
    for name, scheme, target, seed in [("fic_input", abi.FIC, abi.TARGET_INPUT, 0xD1),
                                       ("fic_filter", abi.FIC, abi.TARGET_FILTER, 0xD2),
                                       ("fic_convout", abi.FIC, abi.TARGET_CONVOUT, 0xD3),
                                       ("fc_filter", abi.FC, abi.TARGET_FILTER, 0xD4)]:
        camp = api.Campaign(ls, scheme, target, trials, seed, mode=abi.DATA_RANDOM_I8, images=(n0, n1))
        rec = torch.zeros(trials, 3, dtype=torch.int64, device=dev)
        cnt = torch.zeros(4, dtype=torch.int64, device=dev)
        camp.run_records(rec)  # warm-up
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec.zero_()
        cnt.zero_()
        camp.run_records(rec)
        if dist:
            dist.all_reduce(rec)
        camp.classify(rec, cnt)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        c = cnt.tolist()
        out["schemes"][name] = {"detected": c[abi.DETECTED], "detected_benign": c[abi.DETECTED_BENIGN],
                                "sdc": c[abi.SDC], "masked": c[abi.MASKED],
                                "coverage": round((c[abi.DETECTED] + c[abi.DETECTED_BENIGN]) / trials, 4),
                                "ms": round(ms, 3), "trials_per_s": round(trials / (ms * 1e-3), 1)}
        del camp
    if rank == 0:
        # exhaustive cross-check: the first few trials through the fused protected
        # conv of the whole batch per trial, against the trial-parallel kernel
        xc = {}
        for name, scheme, target, seed in [("fic_input", abi.FIC, abi.TARGET_INPUT, 0xD1),
                                           ("fic_filter", abi.FIC, abi.TARGET_FILTER, 0xD2)]:
            k = 8
            a = api.run_campaign(ls, scheme, target, trials, seed, mode=abi.DATA_RANDOM_I8, begin=0, end=k)
            b = api.run_campaign(ls, scheme, target, trials, seed, mode=abi.DATA_RANDOM_I8, begin=0, end=k,
                                 batched=True)
            xc[name] = {"trials": k, "exhaustive": list(a.astuple()), "batched": list(b.astuple()),
                        "equal": a.astuple() == b.astuple()}
        out["exhaustive_crosscheck"] = xc
    torch.cuda.synchronize()
    return out


def run_ours(args, world, rank, local):
    import ctypes as C

    import torch

    from paper_2006_04984_b200 import abi, api

    # ABED_BENCH_SHARED_GPU=1: code-path check of the multi-rank bench on a box with
    # fewer GPUs than ranks (ranks share devices, gloo instead of NCCL); its
    # timings are not measurements
    shared = os.environ.get("ABED_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    # per-GPU batch: BASELINE configs[1] (32 per GPU, weak scaling) by default;
    # --global-batch B shards a fixed batch over the ranks (configs[4]: 1024, strong)
    rb = args.global_batch // world if args.global_batch else BATCH
    if args.global_batch and args.global_batch % world:
        raise SystemExit("--global-batch must be divisible by the number of GPUs")
    abi.check(abi.load().abed_device_check())
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream()
    peaks = measured_peaks()

    # ------------------------------------------------ layers, data, plans
    layers = []
    for li, (name, c, h, w, k, st) in enumerate(RESNET50_3X3):
        ls = api.layer_shape(rb, c, h, w, k, 3, 3, st, st, 1, 1)
        seed = 1000 * (rank + 1) + li  # each rank owns its own batch shard
        x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(seed, 1)).view(ls.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(seed, 2)).view(ls.filter_dims())
        bias = torch.linspace(-2.0, 2.0, k).tolist()
        L = {"name": name, "ls": ls, "x": x, "f": f, "ops": layer_ops(c, h, w, k, st)}
        L["plans"] = {"unprotected": api.ConvPlan(ls, f, 0), "fc": api.ConvPlan(ls, f, abi.CHECK_FC),
                      "fic": api.ConvPlan(ls, f, abi.CHECK_FIC), "fic_sm": api.ConvPlan(ls, f, abi.CHECK_FIC),
                      "ic": api.ConvPlan(ls, f, abi.CHECK_IC), "icbatch": api.ConvPlan(ls, f, abi.CHECK_ICBATCH)}
        # FIC with the input checksum dotted from the staged shared-memory tiles
        # instead of the default second read of the stored input (FR)
        L["plans"]["fic_sm"].set_input_checksum_source(abi.RHS_STAGED)
        # the captured pass finalizes every IC run it contains
        L["plans"]["ic"].set_paired_finalize(True)
        L["plans"]["icbatch"].set_paired_finalize(True)
        L["packed"] = L["plans"]["unprotected"].pack(x)
        # ICBatch: the packed input also holds the batch-sum digit images (written in-kernel)
        L["packed_icb"] = L["plans"]["icbatch"].pack(x)
        for v, pl in L["plans"].items():
            if v != "icbatch":
                assert pl.info.packed_input_bytes == L["plans"]["unprotected"].info.packed_input_bytes
        L["ep"] = {kk: pl.epilog_params(0.05, bias, True) for kk, pl in L["plans"].items()}
        out_bytes = ls.n * k * (ls.p + 1) * (ls.q + 1) + (1 << 16)
        L["out"] = torch.zeros(out_bytes, dtype=torch.int8, device=dev)
        L["out2"] = torch.zeros(out_bytes, dtype=torch.int8, device=dev)
        layers.append(L)
    torch.cuda.synchronize()
    # one verdict launch per pass: every layer's FC / FIC / IC / ICBatch VerifyOutcome
    CHECKED = ("fc", "fic", "fic_sm", "ic", "icbatch")
    VARIANTS = ("unprotected",) + CHECKED + ("dup",)
    sets = {v: api.PlanSet([L["plans"][v] for L in layers]) for v in CHECKED}
    # multi-GPU verdicts: each rank packs its shard's VerifyOutcomes into
    # records, ONE all-gather per step moves them (NCCL over NVLink), and a one-block
    # kernel folds them into the global outcomes (FC counts / first locus, FIC sums)
    from paper_2006_04984_b200.dist import ShardedVerdicts
    shards = {v: ShardedVerdicts(sets[v]._out, [abi.FC, abi.FIC, abi.IC if v == "ic" else abi.ICBATCH] * len(layers),
                                 n_offset=rank * rb) for v in CHECKED}

    def step(variant):
        for L in layers:
            if variant == "dup":
                pl = L["plans"]["unprotected"]
                pl.run(L["packed"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"]["unprotected"])
                pl.run(L["packed"], L["out"], abi.OUT_I8_COMPARE, ep=L["ep"]["unprotected"])
            else:
                # one launch per layer: conv + checks (+ the in-kernel input checksum);
                # each CTA leaves its partial verdict record
                pl = L["plans"][variant]
                pl.run(L["packed_icb"] if variant == "icbatch" else L["packed"], L["out"], abi.OUT_I8_PACKED,
                       ep=L["ep"][variant])
        if variant in sets:
            sets[variant].finalize()
            shards[variant].record()

    # kernels of this library per step: conv per layer, + ICBatch scan per layer,
    # + one verdict launch (IC: the two batched IC-verdict launches instead)
    # (+ with several ranks the verdict-record kernel in the graph and the fold
    # kernel after the all-gather)
    xr = 2 if world > 1 else 0
    launches_per_step = {"unprotected": 16, "dup": 32, "fc": 17 + xr, "fic": 17 + xr, "fic_sm": 17 + xr,
                         "ic": 18 + xr, "icbatch": 33 + xr}

    # warm up eagerly (sets kernel attributes), then capture each variant as one graph
    with torch.cuda.stream(stream):
        for v in VARIANTS:
            step(v)
    torch.cuda.synchronize()
    graphs = {}
    for v in VARIANTS:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(v)
        graphs[v] = g
    torch.cuda.synchronize()

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def timed(v, steps, warmup, sampler=None):
        for _ in range(warmup):
            l2_flush(flush)
            graphs[v].replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if sampler:
            # nvidia-smi needs a few hundred ms for its first sample: keep the same
            # step running under load until samples flow, time the K steps, then keep
            # the load on briefly so the samples bracket the timed region
            sampler.start()
            sampler.keep_busy(lambda: (l2_flush(flush), graphs[v].replay()), 1.0)
        cur = torch.cuda.current_stream()
        for i in range(steps):
            l2_flush(flush)
            evs[i][0].record(cur)
            graphs[v].replay()
            if v in shards:  # the only collective: the per-shard verdict records, then the fold
                shards[v].reduce()
            evs[i][1].record(cur)
        torch.cuda.synchronize()
        if sampler:
            sampler.keep_busy(lambda: (l2_flush(flush), graphs[v].replay()), 0.4)
        clocks = sampler.stop() if sampler else None
        ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms, clocks

    ops_step = total_ops(rb) * world
    res = {}
    sampler = ClockSampler(local)
    for v in ("unprotected", "fc", "dup", "fic_sm", "ic", "icbatch", "fic"):
        ms, clk = timed(v, args.steps, args.warmup, sampler if v == "fic" else None)
        res[v] = {"ms": ms, "tops": ops_step / (ms * 1e-3) / 1e12}
        if v == "fic":
            clocks = clk

    vgg = None
    if not args.skip_vgg:
        vgg = measure_vgg16_fp16(args, dev, stream, flush, world, dist)
    hbm = measure_hbm_kernels(dev, stream, flush, peaks) if rank == 0 else None
    abft = measure_abft_gemm(dev, stream, flush) if (rank == 0 and not args.skip_abft) else None
    r50 = None
    if not args.skip_r50net:
        r50 = measure_resnet50_network(args, dev, stream, flush, world, dist)
    mbv2 = None
    if not args.skip_mbv2:
        mbv2 = measure_mobilenetv2_int8(args, dev, stream, flush, world, dist)

    # global verdicts of the last pass of every checked variant, folded over the ranks
    # (fault-free => all pass); slots are {FC, FIC, IC/ICBatch} per layer
    fails = 0
    for v in CHECKED:
        glob = shards[v].outcomes_global()
        want = {"fc": (0,), "fic": (1,), "fic_sm": (1,), "ic": (2,), "icbatch": (2,)}[v]
        fails += sum(glob[3 * i + j].status for i in range(len(layers)) for j in want)

    # ------------------------------------------------ roofline of the dominant kernel
    # the FIC conv kernel of each layer (the whole per-layer FIC work: conv, checks,
    # input checksum, verdict) timed as a captured graph of R back-to-back launches
    # after an L2 flush, CUDA events on the launching stream; per-launch = total / R
    R = 10

    def per_layer_ms(variant):
        out = []
        for L in layers:
            pl = L["plans"][variant]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(R):
                    pl.run(L["packed"], L["out"], abi.OUT_I8_PACKED, ep=L["ep"][variant])
            ts = []
            for i in range(4):
                l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                cur = torch.cuda.current_stream()
                e0.record(cur)
                g.replay()
                e1.record(cur)
                torch.cuda.synchronize()
                if i:
                    ts.append(e0.elapsed_time(e1) / R)
            out.append(statistics.mean(ts))
        return out

    conv_ms = per_layer_ms("fic")
    unprot_ms = per_layer_ms("unprotected")
    staged_ms = per_layer_ms("fic_sm")
    conv_tops = total_ops(rb) / (sum(conv_ms) * 1e-3) / 1e12
    # denominator: the tcgen05 kind::i8 dense peak MEASURED in this run on this device
    # (all SMs issuing back-to-back M128 N256 K32 MMAs, CUDA events; abed_probe_mma_i8_peak)
    pk_tops, pk_ms = C.c_double(), C.c_double()
    abi.call("abed_probe_mma_i8_peak", 4000, C.byref(pk_tops), C.byref(pk_ms))
    peak = pk_tops.value
    bf16 = peaks.get("bf16_tflops")
    ncu = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            ncu = json.load(fh)
    except (OSError, ValueError):
        pass
    roofline = {"bound": "tensor", "achieved": round(conv_tops, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
                "frac": round(conv_tops / peak, 4), "traffic": ncu.get("traffic_bytes_per_launch"),
                "traffic_source": "profiles/ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum of one "
                                  "launch of " + str(ncu.get("traffic_layer")) + " (ncu --set full)",
                "kernel": "conv_i8_tc_kernel<int8, packed out, FIC> (conv + input-checksum warps + output sums + verdict)",
                "peak_source": ("measured in this run: tcgen05.mma kind::i8 M128xN256xK32 back to back on all "
                                f"{torch.cuda.get_device_properties(dev).multi_processor_count} SMs, operands in "
                                f"shared memory, CUDA events ({pk_ms.value:.2f} ms; abed_probe_mma_i8_peak)"),
                "frac_of_nominal_4500": round(conv_tops / PEAK_INT8_NOMINAL, 4),
                "frac_of_2x_bf16_measured": round(conv_tops / (2.0 * bf16), 4) if bf16 else None,
                "conv_share_of_step": round(sum(conv_ms) / res["fic"]["ms"], 3),
                "per_layer_conv_us": [round(t * 1e3, 2) for t in conv_ms],
                "per_layer_unprotected_us": [round(t * 1e3, 2) for t in unprot_ms],
                "per_layer_fic_staged_us": [round(t * 1e3, 2) for t in staged_ms],
                "timing": f"per layer: graph of {R} back-to-back launches after an L2 flush, CUDA events / {R}"}

    # ------------------------------------------------ e2e through the C ABI with host buffers
    e2e = None
    if True:
        in_n = [L["x"].numel() for L in layers]
        out_n = [L["ls"].n * L["ls"].k * L["ls"].p * L["ls"].q for L in layers]
        # issue order: the smallest input first and the smallest output last, so the
        # pipeline's lone first H2D and lone last D2H are short
        first = min(range(len(layers)), key=lambda i: in_n[i])
        last = min((i for i in range(len(layers)) if i != first), key=lambda i: out_n[i])
        order = [first] + [i for i in range(len(layers)) if i not in (first, last)] + [last]
        # host and device buffers: one block per direction, laid out in issue order,
        # so consecutive layers' copies coalesce -- pairs of layers share one H2D and
        # one D2H (measured: 8 copies per direction 1.465 ms, 16 per-layer copies
        # 1.55-1.58 ms, tools/e2e_timeline.py); the first and last layers travel
        # alone so the pipeline's fill and drain are one small layer each (~2%)
        pair = 2
        mid = order[1:-1]
        groups = [order[:1]] + [mid[g:g + pair] for g in range(0, len(mid), pair)] + [order[-1:]]
        if os.environ.get("ABED_E2E_PAIRS_ONLY"):  # comparison: pairs from the first layer on
            groups = [order[g:g + pair] for g in range(0, len(order), pair)]
        in_off, out_off, oi, oo = {}, {}, 0, 0
        for i in order:
            in_off[i], out_off[i] = oi, oo
            oi += in_n[i]
            oo += out_n[i]
        host_in_blk = pinned_wc_host(oi)
        host_out_blk = torch.empty(oo, dtype=torch.int8).pin_memory()
        dev_in_blk = torch.empty(oi, dtype=torch.int8, device=dev)
        dev_out_blk = torch.empty(oo, dtype=torch.int8, device=dev)
        dev_in = {i: dev_in_blk[in_off[i]:in_off[i] + in_n[i]].view(layers[i]["x"].shape) for i in order}
        dev_out = {i: dev_out_blk[out_off[i]:out_off[i] + out_n[i]].view(layers[i]["ls"].output_dims())
                   for i in order}
        for i in order:
            host_in_blk[in_off[i]:in_off[i] + in_n[i]].copy_(layers[i]["x"].reshape(-1).cpu())
        oc_host = torch.empty(3 * 72 * len(layers), dtype=torch.uint8).pin_memory()
        oc_dev = torch.empty(3 * 72 * len(layers), dtype=torch.uint8, device=dev)  # every plan's verdicts
        h2d = host_in_blk.numel()
        d2h = host_out_blk.numel() + oc_host.numel()

        # three streams pipelined across the layer pairs: the copy engines move the
        # next pair's inputs in and the previous pair's outputs out while a pair
        # computes (every layer owns its slice of the device blocks: no hazards)
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        sp = C.c_void_p(s_cmp.cuda_stream)

        def e2e_step():
            cur = torch.cuda.current_stream()
            for st_ in (s_in, s_cmp, s_out):
                st_.wait_stream(cur)
            for grp in groups:
                i0, i1 = in_off[grp[0]], in_off[grp[-1]] + in_n[grp[-1]]
                o0, o1 = out_off[grp[0]], out_off[grp[-1]] + out_n[grp[-1]]
                with torch.cuda.stream(s_in):
                    dev_in_blk[i0:i1].copy_(host_in_blk[i0:i1], non_blocking=True)
                s_cmp.wait_stream(s_in)
                for i in grp:
                    L = layers[i]
                    pl = L["plans"]["fic"]
                    pl.pack(dev_in[i], L["packed"], stream=sp)
                    pl.run(L["packed"], dev_out[i], abi.OUT_I8_NCHW, ep=L["ep"]["fic"], stream=sp)
                    abi.call("abed_conv_plan_finalize", pl.handle, oc_dev[i * 216:].data_ptr(), sp)
                s_out.wait_stream(s_cmp)
                with torch.cuda.stream(s_out):
                    host_out_blk[o0:o1].copy_(dev_out_blk[o0:o1], non_blocking=True)
            with torch.cuda.stream(s_out):  # the 16 layers' VerifyOutcomes in one read-back
                s_out.wait_stream(s_cmp)
                oc_host.copy_(oc_dev, non_blocking=True)
            for st_ in (s_in, s_cmp, s_out):
                cur.wait_stream(st_)

        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()

        def time_e2e(run):
            ts = []
            for _ in range(args.steps):
                l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return statistics.mean(ts)

        # eager: ~100 host calls per step (ctypes + torch copies) -- host-launch
        # bound on a slow host; graph: the same C-ABI calls and the same pinned
        # H2D / D2H copies captured once and replayed (every byte still crosses
        # PCIe inside the timed region)
        eager_ms = time_e2e(e2e_step)
        g_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_e2e):
            e2e_step()
        g_e2e.replay()
        torch.cuda.synchronize()
        e_ms = time_e2e(g_e2e.replay)
        if dist:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        # the read-back verdicts of the last replay: every layer's FIC must pass
        torch.cuda.synchronize()
        st_words = oc_host.view(torch.int32).view(len(layers), 3, 18)[:, 1, 0]
        e2e_failed = int((st_words != 0).sum())
        # the PCIe floor of the same bytes: one H2D of the step's inputs and one D2H of
        # its outputs + verdicts, concurrently on two streams, nothing else
        fl_in = pinned_wc_host(int(h2d))  # the same host memory type as the step's inputs
        fl_out = torch.empty(int(d2h), dtype=torch.int8).pin_memory()
        fl_din = torch.empty(int(h2d), dtype=torch.int8, device=dev)
        fl_dout = torch.empty(int(d2h), dtype=torch.int8, device=dev)

        def copies_only():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            s_out.wait_stream(cur)
            with torch.cuda.stream(s_in):
                fl_din.copy_(fl_in, non_blocking=True)
            with torch.cuda.stream(s_out):
                fl_out.copy_(fl_dout, non_blocking=True)
            cur.wait_stream(s_in)
            cur.wait_stream(s_out)

        copies_only()
        floor_ms = time_e2e(copies_only)
        e2e = {"value": round(ops_step / (e_ms * 1e-3) / 1e12, 3), "unit": "TOPS", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3), "eager_ms_per_step": round(eager_ms, 3),
               "pcie_floor_ms": round(floor_ms, 3), "frac_of_pcie_floor": round(floor_ms / e_ms, 3),
               "fic_verdicts_failed": e2e_failed,
               "path": "per layer: pinned (write-combined) H2D NCHW -> abed_pack_input -> abed_conv_plan_run(FIC, OUT_I8_NCHW) -> "
                       "abed_conv_plan_finalize -> D2H output, copies coalesced per pair of layers (8 H2D + 8 D2H); the 16 "
                       "layers' verdicts in one D2H at the end; H2D / compute / D2H on three streams, "
                       "pipelined across the pairs; the step's calls captured once as a CUDA graph and replayed "
                       "(eager_ms_per_step: the same calls issued from Python every step)"}

    # ------------------------------------------------ detection coverage (GPU fault campaigns)
    cfg1 = api.layer_shape(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)
    trials = args.campaign_trials
    b0, b1 = trials * rank // world, trials * (rank + 1) // world  # trials sharded by index across GPUs
    det = {}
    for name, scheme, target in [("fic_convout", abi.FIC, abi.TARGET_CONVOUT), ("fic_input", abi.FIC, abi.TARGET_INPUT),
                                 ("fic_filter", abi.FIC, abi.TARGET_FILTER), ("fc_convout", abi.FC, abi.TARGET_CONVOUT),
                                 ("fc_filter", abi.FC, abi.TARGET_FILTER), ("fc_input", abi.FC, abi.TARGET_INPUT)]:
        seed = {"fc_filter": 0xC2, "fc_convout": 0xC3, "fc_input": 0xC4, "fic_input": 0xC5, "fic_filter": 0xC6,
                "fic_convout": 0xC7}[name]
        rep = api.run_campaign(cfg1, scheme, target, trials, seed, begin=b0, end=b1)
        cnt = torch.tensor(list(rep.astuple()), dtype=torch.int64, device=dev)
        if dist:
            dist.all_reduce(cnt)
        c = cnt.tolist()
        det[name] = {"detected": c[0], "detected_benign": c[1], "sdc": c[2], "masked": c[3],
                     "coverage": round((c[0] + c[1]) / trials, 4)}

    camp5 = None if args.skip_campaign5 else measure_campaign_cfg5(args, dev, world, rank, dist)
    dropin = measure_dropin_calls(dev) if rank == 0 else None

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    # ------------------------------------------------ CPU baseline (reference, host cores, rank 0, N=1)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            tops, desc, cores, kind = cpu_reference_sample(target_s=args.cpu_seconds)
            cpu = {"value": round(tops, 4), "unit": "TOPS", "cores": cores, "kind": kind, "sample": desc}
        except Exception as exc:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "TOPS", "cores": 0, "kind": "unavailable", "sample": f"failed: {exc}"}

    fic = res["fic"]
    line = {
        "metric": METRIC,
        "value": round(fic["tops"], 2),
        "unit": "TOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(fic["ms"], 4),
        "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak",
        "vs_baseline": None,
        "dtype": "int8",
        "data": "synthetic: SplitMix64 int8 activations/filters generated on device; bias linspace(-2,2), scale 0.05",
        "config": workload_config(rb, world, args.global_batch),
        "method": {"scheme": "FIC-FR in one kernel per layer (input checksum x.G with dp4a from a second read of the stored input, by input-checksum warps or, where the conv grid leaves SMs free, input-checksum CTAs; epilogue output sums; per-CTA verdict records) + one verdict launch per pass for all 16 VerifyOutcomes",
                   "parallelism": f"dp{world} (batch shards; one NCCL all-gather of the per-shard verdict records "
                                  "per step, folded on the device)",
                   "timing": "CUDA graph replay, CUDA events"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step["fic"] * args.steps,
        "clocks": clocks,
        "variants": {v: {"tops": round(r["tops"], 2), "ms_per_step": round(r["ms"], 4)} for v, r in res.items()},
        "overhead_pct": {"fic_vs_unprotected": round(100 * (res["fic"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "fic_sm_vs_unprotected": round(100 * (res["fic_sm"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "fc_vs_unprotected": round(100 * (res["fc"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "ic_vs_unprotected": round(100 * (res["ic"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "icbatch_vs_unprotected": round(100 * (res["icbatch"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "duplication_vs_unprotected": round(100 * (res["dup"]["ms"] / res["unprotected"]["ms"] - 1), 2),
                         "fic_throughput_vs_duplication": round(res["dup"]["ms"] / res["fic"]["ms"], 3)},
        "detection": {"layer": "cfg1 1x64x56x56 K=64 3x3 p1, ones data, scale 0.05, trials %d" % trials, **det},
        "fault_free_verdicts_failed": fails,
        "int8_peak_nominal_tops": PEAK_INT8_NOMINAL,
        "cfg3_vgg16_fp16": vgg,
        "cfg4_mobilenetv2_int8": mbv2,
        "hbm_kernels": hbm,
        "resnet50_network_int8": r50,
        "abft_gemm_int8": abft,
        "cfg5_campaign_b1024": camp5,
        "dropin_one_shot": dropin,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--campaign-trials", type=int, default=1000)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-vgg", action="store_true", help="skip the VGG-16 FP16 block (BASELINE configs[2])")
    ap.add_argument("--skip-mbv2", action="store_true", help="skip the MobileNetV2 INT8 block (BASELINE configs[3])")
    ap.add_argument("--skip-r50net", action="store_true", help="skip the whole-network ResNet-50 INT8 block")
    ap.add_argument("--skip-abft", action="store_true", help="skip the ABFT-GEMM comparison block")
    ap.add_argument("--skip-campaign5", action="store_true",
                    help="skip the batch-1024 batch-sharded fault campaign (BASELINE configs[4])")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="shard this fixed ResNet-50 batch over the GPUs (BASELINE configs[4]: 1024); default 32 per GPU")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
