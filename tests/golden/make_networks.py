"""Golden builtin network tables: compiles a 20-line program against the
reference's own network_config.hpp (network_config.hpp:163-299, json via the
nlohmann copy in this image) and records network_to_json for vgg16 / resnet18 /
resnet50 at 224 and 1080p into tests/golden/networks.json.  Needs
/root/reference (this container only); the test that reads the file does not."""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
SRC = r'''
#include <iostream>
#include "abed/network_config.hpp"
int main() {
  nlohmann::json all = nlohmann::json::array();
  for (const char* net : {"vgg16", "resnet18", "resnet50"})
    for (const char* img : {"224", "1080p"}) all.push_back(abed::network_to_json(abed::builtin_network(net, img)));
  std::cout << all.dump() << "\n";
}
'''


def main():
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "nets.cpp"), os.path.join(d, "nets")
        open(src, "w").write(SRC)
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", "/root/reference/proj/include", "-I", JSON_DIR, src, "-o", exe],
                       check=True)
        nets = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    with open(os.path.join(HERE, "networks.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_networks.py (reference network_config.hpp)", "networks": nets}, f)
    print(len(nets), "networks,", sum(len(n["layers"]) for n in nets), "layers")


if __name__ == "__main__":
    main()
