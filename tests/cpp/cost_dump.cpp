// Prints the analytic op / byte model (cost_model.hpp) for a fixed set of layer
// shapes and the builtin networks as JSON.  The SAME source is compiled against
// the reference headers (tests/golden/make_golden_cost.py -> tests/golden/cost.json)
// and against the drop-in (tests/test_cost_model.py), and the outputs compared.
#include <cstdio>
#include <string>

#include "abed/cost_model.hpp"
#include "abed/network_config.hpp"

using namespace abed;

static void ops_json(const OpCounts& o) {
  std::printf("[%lld,%lld,%lld,%lld,%lld]", (long long)o.fma, (long long)o.add, (long long)o.mul,
              (long long)o.activation_eval, (long long)o.cast);
}
static void bytes_json(const ByteCounts& b) { std::printf("[%lld,%lld]", (long long)b.read_bytes, (long long)b.write_bytes); }

int main() {
  const LayerShape shapes[] = {
      LayerShape::make(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),   LayerShape::make(32, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),
      LayerShape::make(32, 128, 56, 56, 128, 3, 3, 2, 2, 1, 1), LayerShape::make(2, 3, 224, 224, 64, 3, 3, 1, 1, 1, 1),
      LayerShape::make(4, 256, 14, 14, 1024, 1, 1, 1, 1, 0, 0), LayerShape::make(3, 5, 9, 7, 6, 5, 3, 2, 1, 2, 1)};
  const Scheme schemes[] = {Scheme::FC, Scheme::IC, Scheme::ICBatch, Scheme::FIC};
  const ImplOption options[] = {ImplOption::UF, ImplOption::FR, ImplOption::AF};
  std::printf("{\"layers\":[");
  bool first = true;
  for (const auto& ls : shapes)
    for (Scheme sc : schemes) {
      for (int planes = 1; planes <= 4; ++planes) {
        std::printf("%s{\"dims\":[%lld,%lld,%lld,%lld,%lld],\"scheme\":\"%s\",\"planes\":%d,\"ops\":", first ? "" : ",",
                    (long long)ls.n, (long long)ls.c, (long long)ls.h, (long long)ls.k, (long long)ls.r, to_string(sc),
                    planes);
        first = false;
        ops_json(count_ops(ls, sc, planes != 2, planes));
        std::printf(",\"bytes\":{");
        for (ImplOption op : options)
          for (int pad = 0; pad < 2; ++pad) {
            CostOptions o;
            o.fc_planes = planes;
            o.fc_pad_to_8 = pad != 0;
            std::printf("%s\"%s%s\":", (op == ImplOption::UF && pad == 0) ? "" : ",", to_string(op), pad ? "8" : "");
            bytes_json(count_bytes(ls, sc, op, o));
          }
        std::printf("},\"base\":[");
        bytes_json(baseline_bytes(ls, true));
        std::printf(",");
        bytes_json(baseline_bytes(ls, false));
        std::printf("]}");
      }
    }
  std::printf("],\"networks\":[");
  first = true;
  for (const char* net : {"vgg16", "resnet18", "resnet50"})
    for (const char* img : {"224", "1080p"}) {
      const NetworkConfig cfg = builtin_network(net, img);
      for (Scheme sc : schemes)
        for (ImplOption op : options) {
          const CostReport r = aggregate_network(cfg, sc, op);
          std::printf("%s{\"net\":\"%s\",\"scheme\":\"%s\",\"option\":\"%s\",\"ops\":", first ? "" : ",", r.network.c_str(),
                      to_string(sc), to_string(op));
          first = false;
          ops_json(r.total_ops);
          std::printf(",\"ops_base\":");
          ops_json(r.total_ops_baseline);
          std::printf(",\"bytes\":");
          bytes_json(r.total_bytes);
          std::printf(",\"bytes_base\":");
          bytes_json(r.total_bytes_baseline);
          std::printf(",\"op_pct\":%.9g,\"byte_pct\":%.9g,\"rows\":%zu,\"excluded0\":%d}", r.op_overhead_pct(),
                      r.byte_overhead_pct(), r.rows.size(), r.rows[0].excluded ? 1 : 0);
        }
    }
  std::printf("]}\n");
  return 0;
}
