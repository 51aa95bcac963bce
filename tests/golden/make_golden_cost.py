"""Golden analytic cost model: compiles tests/cpp/cost_dump.cpp against the
REFERENCE's own cost_model.hpp / network_config.hpp (json via the nlohmann copy in
this image) and stores its output as tests/golden/cost.json.  Needs
/root/reference (this container only); tests/test_cost_model.py compiles the same
source against include/abed and compares."""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def main():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "cost_ref")
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", "/root/reference/proj/include", "-I", JSON_DIR,
                        os.path.join(ROOT, "tests", "cpp", "cost_dump.cpp"), "-o", exe], check=True)
        out = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    out["generator"] = "tests/golden/make_golden_cost.py (reference cost_model.hpp)"
    with open(os.path.join(HERE, "cost.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote cost.json", len(out["layers"]), "layer rows", len(out["networks"]), "network rows")


if __name__ == "__main__":
    main()
