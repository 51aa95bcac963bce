"""The C-ABI library loads and exports every symbol include/abed_b200.h declares;
without a device every compute entry point fails loudly (no host fallback); the
C++ drop-in headers compile and their host-only parts pass; on a GPU the whole
C++ suite (the reference's test assertions through include/abed/*.hpp) passes."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "abed_b200.h")
LIB = os.path.join(ROOT, "paper_2006_04984_b200", "libabed_b200.so")
BIN = os.path.join(ROOT, "build", "abed_api_test")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(abed_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2006_04984_b200 import abi
    syms = declared_symbols()
    assert len(syms) >= 50
    lib = C.CDLL(LIB)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(abi.SIGNATURES) == syms, set(syms) ^ set(abi.SIGNATURES)


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2006_04984_b200 import abi
    lib = abi.load()
    assert lib.abed_device_check() == abi.ERR_NO_DEVICE
    assert b"no host fallback" in lib.abed_last_error()
    ls = abi.layer_shape(1, 1, 3, 3, 1, 3, 3)  # pure host validation works
    assert (ls.p, ls.q) == (1, 1)
    with pytest.raises(abi.AbedError):
        abi.call("abed_conv_i8", None, None, C.byref(ls), None, None)
    with pytest.raises(abi.InvalidArgument):
        abi.layer_shape(1, 1, 3, 3, 1, 5, 5)


def build_cpp():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "tests", "cpp"),
           os.path.join(ROOT, "tests", "cpp", "abed_api_test.cpp"), "-L", os.path.dirname(LIB), "-labed_b200",
           "-Wl,-rpath," + os.path.dirname(LIB), "-o", BIN]
    subprocess.run(cmd, check=True)


def test_cpp_dropin_headers_compile_and_host_suites_pass():
    build_cpp()
    r = subprocess.run([BIN, "Host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_full_suite_on_gpu():
    build_cpp()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
