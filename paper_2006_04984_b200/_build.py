"""Builds libabed_b200.so (all CUDA sources under csrc/) in-tree for sm_100a.

Plain nvcc, no torch extension machinery: the library is a C-ABI shared object
(include/abed_b200.h) that ctypes, the C++ drop-in headers and bench.py load.
Incremental: an object is rebuilt when its .cu or any csrc header is newer.
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libabed_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-diag-suppress", "177", "-I", os.path.join(ROOT, "include")]
# diagnostics builds only (e.g. ABED_NVCC_EXTRA=-DABED_CONV_DEBUG=1 for the conv
# kernel's timing-experiment flags used by tools/epi_probe.py); a change of flags
# rebuilds every object
FLAGS += os.environ.get("ABED_NVCC_EXTRA", "").split()


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    return r


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_mtime = max((os.path.getmtime(h) for h in headers), default=0)
    # objects built with other flags (ABED_NVCC_EXTRA, a different nvcc) are stale
    stamp = os.path.join(BUILD, "flags.txt")
    flags_now = " ".join([NVCC, *ARCH, *FLAGS])
    if not os.path.exists(stamp) or open(stamp).read() != flags_now:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
        with open(stamp, "w") as fh:
            fh.write(flags_now)
    objs, cmds = [], []
    for src in sources:
        obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        cmds.append(cmd)
    # translation units are independent: compile them concurrently
    with concurrent.futures.ThreadPoolExecutor(max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(_run, cmds))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs])
    build_cli()
    return LIB


# nlohmann/json for the CLI's --config files and JSON reports (the reference's own
# dependency; this image ships a copy inside the cudnn frontend headers)
JSON_DIRS = [os.environ.get("ABED_JSON_INCLUDE", ""),
             os.path.join(sys.prefix, "lib", "python3.12", "site-packages", "include", "cudnn_frontend",
                          "thirdparty", "nlohmann"),
             "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"]
# The CLI is the reference's own driver, UNMODIFIED, compiled where it lies
# (tools/abed_main.cpp of the reference) against this repository's drop-in headers
# include/abed/*.hpp and linked to libabed_b200.so: every `abed verify / inject /
# cost / abft` call runs on the B200 library.  CLI11 (vendored by the reference,
# absent from its tree) is replaced by the minimal compatible parser in
# tools/dropin_cli/CLI11.hpp.  The binary is built here (where the reference
# exists) and travels with the repository snapshot.
REF_CLI_SRC = os.environ.get("ABED_REF_CLI", "/root/reference/proj/tools/abed_main.cpp")
CLI_DIR = os.path.join(ROOT, "tools", "dropin_cli")
CLI_BIN = os.path.join(CLI_DIR, "abed")


def build_cli() -> str | None:
    """g++ the reference CLI against the drop-in headers and libabed_b200.so (tools/dropin_cli/abed)."""
    if not os.path.exists(REF_CLI_SRC):
        return CLI_BIN if os.path.exists(CLI_BIN) else None
    jdir = next((d for d in JSON_DIRS if d and os.path.exists(os.path.join(d, "json.hpp"))), None)
    if jdir is None:
        sys.stderr.write("abed CLI not built: no nlohmann json.hpp found (set ABED_JSON_INCLUDE)\n")
        return None
    deps = [REF_CLI_SRC, LIB, os.path.join(CLI_DIR, "CLI11.hpp")] + \
        glob.glob(os.path.join(ROOT, "include", "abed", "*.hpp"))
    if os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) >= max(os.path.getmtime(d) for d in deps):
        return CLI_BIN
    _run(["g++", "-std=c++20", "-O2", "-I", CLI_DIR, "-I", os.path.join(ROOT, "include"), "-I", jdir,
          "-I", "/usr/local/cuda/include", REF_CLI_SRC, "-o", CLI_BIN, "-L", PKG, "-labed_b200",
          "-Wl,-rpath,$ORIGIN/../../paper_2006_04984_b200", "-L/usr/local/cuda/lib64", "-lcudart"])
    return CLI_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
