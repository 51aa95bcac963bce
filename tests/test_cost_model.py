"""The analytic op / byte model drop-in (include/abed/cost_model.hpp) against the
reference's cost_model.hpp: tests/cpp/cost_dump.cpp compiled against include/abed
must print exactly what the same source printed against the reference headers
(tests/golden/cost.json: 96 layer rows x 4 schemes x 3 options x plane / padding
variants, 72 whole-network reports).  Plus the numbers SURVEY 8(d) quotes and the
reference's acceptance criterion 3 bounds.  Host only (no GPU)."""
import json
import os
import subprocess

import pytest

from paper_2006_04984_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "cost.json")))


@pytest.fixture(scope="module")
def ours():
    jdir = next((d for d in _build.JSON_DIRS if d and os.path.exists(os.path.join(d, "json.hpp"))), None)
    if jdir is None:
        pytest.skip("nlohmann json.hpp not available")
    exe = os.path.join(ROOT, "build", "cost_dump")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    lib = os.path.dirname(_build.LIB)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", jdir,
                    "-I", "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "cost_dump.cpp"), "-o", exe,
                    "-L", lib, "-labed_b200", "-Wl,-rpath," + lib], check=True)
    return json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)


def test_layer_rows_equal_reference(ours):
    assert len(ours["layers"]) == len(GOLDEN["layers"]) == 96
    for a, b in zip(ours["layers"], GOLDEN["layers"]):
        assert a == b, (a["dims"], a["scheme"], a["planes"])


def test_network_reports_equal_reference(ours):
    assert len(ours["networks"]) == len(GOLDEN["networks"]) == 72
    for a, b in zip(ours["networks"], GOLDEN["networks"]):
        assert a == b, (a["net"], a["scheme"], a["option"])


def test_survey_byte_counts(ours):  # ResNet-50 layer1 at batch 32
    row = {r["scheme"]: r for r in ours["layers"] if r["dims"] == [32, 64, 56, 64, 3] and r["planes"] == 4}
    assert sum(row["fc"]["base"][0]) == 12_881_920
    assert sum(row["fc"]["bytes"]["fr"]) == 12_884_232
    assert sum(row["fic"]["bytes"]["fr"]) == 19_311_376
    assert sum(row["fic"]["bytes"]["af"]) == 12_888_848


def test_acceptance_criterion3_bounds(ours):  # acceptance_main.cpp:184-200
    for net in ("vgg16-1080p", "resnet18-1080p", "resnet50-1080p"):
        rep = {(r["scheme"], r["option"]): r for r in ours["networks"] if r["net"] == net}
        fic, fc = rep[("fic", "fr")]["op_pct"], rep[("fc", "fr")]["op_pct"]
        assert 0.0 < fic < 1.0 and 0.0 < fc < 7.0, (net, fic, fc)
