"""The reference's own CLI (tools/abed_main.cpp, UNMODIFIED) compiled against the
drop-in headers include/abed/*.hpp and libabed_b200.so (tools/dropin_cli/abed,
built by paper_2006_04984_b200/_build.py), and the drop-in network_config.hpp,
mirroring the reference's cli_test.cpp: usage errors
exit 1 (no GPU needed), fault-free verification exits 0 with the plan table, the
forced-32 negative control exits 2, float mode with tau 0 passes on integer data,
.abed dump / reload round-trips, and an injection campaign reproduces the
reference's counts for the cfg1 layer (tests/golden/golden.json)."""
import json
import os
import subprocess

import pytest

from paper_2006_04984_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def cli():
    path = _build.build_cli()
    if path is None:
        pytest.skip("drop-in CLI not built (reference driver source or nlohmann json.hpp not available)")
    return path


def run(cli, args):
    r = subprocess.run([cli] + args.split(), capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("args", [
    "verify --scheme fic --layer 0",                                    # no network source
    "verify --network resnet18 --layer nope --scheme fic",              # unknown layer
    "frobnicate",                                                       # unknown subcommand
    "inject --network resnet18 --layer 1 --scheme fic --target convout --trials 0",
    "inject --network resnet18 --layer 1 --scheme icbatch --target convout",
    "verify --network resnet18 --layer 1 --scheme nope",
    "verify --network resnet18 --image 4k --layer 1 --scheme fic",
    "verify --network resnet18 --layer 1",                              # --scheme required
    "verify --network resnet18 --layer 1 --scheme fic --bogus 1",
    "verify --network resnet18 --layer 1 --scheme fic --seed -1",       # uint64 seed: negative rejected
    "verify --network resnet18 --layer 1 --scheme fic --seed 18446744073709551616",  # > 2^64 - 1
    "verify --config x.json --network resnet18 --layer 1 --scheme fic",  # --config excludes --network
    "verify --image 224 --layer 1 --scheme fic",                        # --image needs --network
])
def test_usage_errors_exit_1(cli, args):
    code, out = run(cli, args)
    assert code == 1, out
    assert "error" in out


def test_builtin_networks_match_reference():
    """network_config.hpp builtins: every layer id, shape and activation equal the
    reference's (golden generated from the reference header itself)."""
    import tempfile
    want = json.load(open(os.path.join(GOLDEN, "networks.json")))["networks"]
    src = r'''
#include <iostream>
#include "abed/network_config.hpp"
int main() {
  for (const char* net : {"vgg16", "resnet18", "resnet50"})
    for (const char* img : {"224", "1080p"}) {
      const auto cfg = abed::builtin_network(net, img);
      std::cout << cfg.name << " " << cfg.exclude_first_layer << " " << cfg.layers.size() << "\n";
      for (const auto& l : cfg.layers) {
        const auto& s = l.shape;
        std::cout << l.id << " " << s.n << " " << s.c << " " << s.h << " " << s.w << " " << s.k << " " << s.r << " "
                  << s.s << " " << s.stride_h << " " << s.stride_w << " " << s.pad_h << " " << s.pad_w << " "
                  << l.activation << "\n";
      }
    }
}
'''
    with tempfile.TemporaryDirectory() as d:
        cpp, exe = os.path.join(d, "n.cpp"), os.path.join(d, "n")
        open(cpp, "w").write(src)
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), cpp, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    i = 0
    for net in want:
        name, excl, count = lines[i].split()
        i += 1
        assert name == net["name"] and int(excl) == int(net["exclude_first_layer"]) and int(count) == len(net["layers"])
        for layer in net["layers"]:
            f = lines[i].split()
            i += 1
            keys = ["n", "c", "h", "w", "k", "r", "s", "stride_h", "stride_w", "pad_h", "pad_w"]
            assert f[0] == layer["id"]
            assert [int(v) for v in f[1:12]] == [layer[k] for k in keys], layer["id"]
            assert int(f[12]) == int(layer["activation"]), layer["id"]


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["fc", "ic", "icbatch", "fic"])
def test_verify_every_scheme_passes(cli, scheme):
    code, out = run(cli, f"verify --network resnet18 --image 224 --layer layer1.0.conv1 --scheme {scheme} --seed 7")
    assert code == 0, out
    assert "layer,scheme,mode,status,lhs,rhs,locus,seed" in out
    assert f"{scheme},int,pass" in out and "plan,b," in out


@pytest.mark.gpu
def test_verify_full_uint64_seed(cli):  # CLI11 reads --seed as std::uint64_t (abed_main.cpp:499)
    code, out = run(cli, "verify --network resnet18 --layer 1 --cap-hw 8 --scheme fc --seed 18446744073709551615")
    assert code == 0, out
    assert out.strip().split("\n")[1].endswith(",18446744073709551615")


@pytest.mark.gpu
def test_verify_json_and_plan_widths(cli):
    code, out = run(cli, "verify --network resnet18 --layer 1 --scheme fic --seed 7 --json")
    assert code == 0, out
    doc = json.loads(out)
    assert doc["status"] == "pass" and doc["lhs"] == doc["rhs"] and doc["layer"] == "layer1.0.conv1"
    # checksum.hpp plan_precision on cfg1's shape (PlanPrecision.TableRows)
    p = doc["plan"]
    assert (p["bits_output_fmap"], p["bits_reduced_fc"], p["bits_reduced_fic"], p["bits_filter_checksum"],
            p["bits_input_checksum"]) == (26, 32, 43, 14, 20)


@pytest.mark.gpu
def test_negative_control_exits_2(cli):
    code, out = run(cli, "verify --network vgg16 --image 224 --layer conv3_1 --scheme fic --data max --cap-hw 16 "
                         "--force-reduce32")
    assert code == 2, out
    assert "mismatch" in out


@pytest.mark.gpu
def test_float_mode_tau0_on_integer_data(cli):
    code, out = run(cli, "verify --network resnet18 --layer 1 --cap-hw 16 --scheme fic --float --tau 0")
    assert code == 0, out
    assert "float,pass" in out


@pytest.mark.gpu
def test_dump_and_reload(cli, tmp_path):
    base = "verify --network resnet18 --layer 1 --cap-hw 12 --scheme fc --seed 3"
    code, first = run(cli, base + f" --dump-dir {tmp_path}")
    assert code == 0, first
    for f in ("input.abed", "filters.abed", "convout.abed"):
        assert (tmp_path / f).stat().st_size > 21
    code, again = run(cli, base.replace("--seed 3", "--seed 99") +
                      f" --load-input {tmp_path}/input.abed --load-filters {tmp_path}/filters.abed")
    assert code == 0, again
    # same tensors, same checksums (only the echoed seed differs)
    assert first.split("\n")[1].rsplit(",", 1)[0] == again.split("\n")[1].rsplit(",", 1)[0]
    code, wrong = run(cli, "verify --network resnet18 --layer 1 --cap-hw 8 --scheme fc "
                           f"--load-input {tmp_path}/input.abed")
    assert code == 1, wrong


@pytest.mark.gpu
def test_inject_reproduces_reference_campaign(cli):
    gold = json.load(open(os.path.join(GOLDEN, "golden.json")))["campaigns"]
    names = {0: "fc", 1: "ic", 3: "fic"}
    targets = {0: "input", 1: "filter", 2: "convout"}
    done = 0
    for c in gold:
        if c["dims"] != [1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1] or c["mode"] != 0:
            continue
        code, out = run(cli, f"inject --network resnet18 --layer 1 --scheme {names[c['scheme']]} "
                             f"--target {targets[c['target']]} --trials {c['trials']} --seed {c['root_seed']} --mode ones")
        assert code == 0, out
        row = out.split("\n")[1].split(",")
        assert [int(v) for v in row[3:7]] == c["counts"], (c, row)
        done += 1
    assert done == 6


@pytest.mark.parametrize("args", ["abft --m 0", "abft --k x", "abft --trials 5 --bogus"])
def test_abft_usage_errors_exit_1(cli, args):
    code, out = run(cli, args)
    assert code == 1 and "error" in out, out


@pytest.mark.gpu
def test_abft_report_and_copy_accounting(cli):  # cli_test.cpp:138-147
    code, out = run(cli, "abft --m 16 --n 12 --k 20 --trials 25 --seed 9")
    assert code == 0, out
    assert "m,n,k,trials,faultfree_pass,detected,detection_rate,copy_elements,seed" in out
    assert "16,12,20,25,25,25,1,944,9" in out
    assert "copy_in," in out and "gemm," in out
    code, out = run(cli, "abft --m 16 --n 12 --k 20 --trials 3 --seed 9 --single-pass --json")
    doc = json.loads(out)
    assert code == 0 and doc["copy_elements"] == 944 and doc["detected"] == 3 and len(doc["tasks"]) == 5


def test_cost_report_columns_and_pruned_override(cli):  # cli_test.cpp:86, 107-129
    code, out = run(cli, "cost --network vgg16 --image 224 --scheme fc --option uf")
    assert code == 0, out
    assert "network,layer,scheme,option,fma,add,mul,act,cast,read_bytes,write_bytes,op_overhead_pct,byte_overhead_pct" in out
    assert "TOTAL" in out and "conv1_1 (excluded)" in out
    code, pruned = run(cli, "cost --network vgg16 --image 224 --scheme fc --option uf --pruned "
                       + os.path.join(GOLDEN, "vgg16_pruned.json"))
    assert code == 0, pruned

    def total_op_pct(text):
        line = next(ln for ln in text.splitlines() if ",TOTAL," in ln)
        return float(line.split(",")[-2])
    assert total_op_pct(pruned) < total_op_pct(out)
    assert run(cli, "cost --network resnet18 --image 1080p --scheme fic --option xx")[0] == 1


def test_cost_json_matches_reference_model(cli):  # cli_test.cpp:130-136 + tests/golden/cost.json
    code, out = run(cli, "cost --network resnet50 --image 1080p --scheme fic --option fr --json")
    assert code == 0, out
    doc = json.loads(out)
    assert doc["network"] == "resnet50-1080p" and "op_overhead_pct" in doc["total"]
    gold = next(r for r in json.load(open(os.path.join(GOLDEN, "cost.json")))["networks"]
                if r["net"] == "resnet50-1080p" and r["scheme"] == "fic" and r["option"] == "fr")
    t = doc["total"]
    assert [t["fma"], t["add"], t["mul"], t["act"], t["cast"]] == gold["ops"]
    assert [t["read_bytes"], t["write_bytes"]] == gold["bytes"]


def test_cost_fc_plane_options(cli):  # cost --fc-pad8 / --fc-planes (abed_main.cpp:531-532)
    def total_bytes(args):
        code, out = run(cli, "cost --network resnet18 --image 224 --scheme fc --option fr --json " + args)
        assert code == 0, out
        t = json.loads(out)["total"]
        return t["read_bytes"] + t["write_bytes"], t["fma"]
    base, fma4 = total_bytes("")
    pad, _ = total_bytes("--fc-pad8")
    _, fma2 = total_bytes("--fc-planes 2")
    assert pad > base and fma2 < fma4
    assert run(cli, "cost --network resnet18 --image 224 --scheme fc --fc-planes 5")[0] == 1
