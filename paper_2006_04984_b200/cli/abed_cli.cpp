// abed_b200: the reference CLI's `verify` and `inject` front ends
// (tools/abed_main.cpp:167-344) over the B200 drop-in headers, so every
// convolution, checksum, verdict and fault-injection trial runs through
// libabed_b200.so.  Same flags, the same CSV / JSON report schemas and the same
// exit codes (0 success, 1 usage / config / IO error, 2 verification mismatch,
// abed_main.cpp:29-31), plus `abft` (abed_main.cpp:425-487), the row/column
// checksum ABFT-GEMM comparison, whose GEMMs and checks run on the B200 too,
// and `cost` (abed_main.cpp:350-417), the analytic op / byte model (host only).
//
// Flags are parsed by hand (the reference uses CLI11, which this image lacks);
// the JSON reports use nlohmann/json like the reference.
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "abed/abed.hpp"
#include "abed/network_config.hpp"

#ifndef ABED_HAVE_JSON
#error "abed_cli needs nlohmann/json (<json.hpp>) on the include path"
#endif

namespace {

using namespace abed;

constexpr int kExitOk = 0;
constexpr int kExitUsage = 1;
constexpr int kExitMismatch = 2;

struct UsageError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// --opt value / --flag parsing against a per-subcommand option table
struct Args {
  std::map<std::string, std::string> values;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return values.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt) const {
    auto it = values.find(k);
    return it == values.end() ? dflt : it->second;
  }
};

Args parse(int argc, char** argv, const std::set<std::string>& options, const std::set<std::string>& flags) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    const std::string tok = argv[i];
    if (flags.count(tok)) {
      a.flags.insert(tok);
    } else if (options.count(tok)) {
      if (i + 1 >= argc) throw UsageError(tok + " needs a value");
      a.values[tok] = argv[++i];
    } else {
      throw UsageError("unknown argument '" + tok + "'");
    }
  }
  return a;
}

std::int64_t to_i64(const std::string& s, const char* what) {
  try {
    std::size_t pos = 0;
    const long long v = std::stoll(s, &pos, 0);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw UsageError(std::string(what) + ": not an integer: '" + s + "'");
  }
}
double to_f64(const std::string& s, const char* what) {
  try {
    std::size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw UsageError(std::string(what) + ": not a number: '" + s + "'");
  }
}

void emit(const Args& a, const std::string& csv, const nlohmann::json& doc) {
  const std::string text = a.flags.count("--json") ? doc.dump(2) + "\n" : csv;
  const std::string out = a.get("--out", "");
  if (out.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream f(out);
  if (!f) throw std::runtime_error("cannot open output file " + out);
  f << text;
}

// abed_main.cpp:68-92 resolve_network / resolve_layer
NetworkConfig resolve_network(const Args& a) {
  if (a.has("--config") && a.has("--network")) throw UsageError("--config excludes --network");
  if (a.has("--image") && !a.has("--network")) throw UsageError("--image needs --network");
  if (a.has("--config")) return load_network(a.get("--config", ""));
  if (a.has("--network")) return builtin_network(a.get("--network", ""), a.get("--image", "224"));
  throw std::invalid_argument("one of --config or --network is required");
}

LayerConfig resolve_layer(const Args& a) {
  const NetworkConfig cfg = resolve_network(a);
  const std::string id = a.get("--layer", "");
  LayerConfig layer;
  if (cfg.has_layer(id)) {
    layer = cfg.layer(id);
  } else {
    try {
      const std::size_t index = std::stoul(id);
      if (index >= cfg.layers.size()) throw std::out_of_range("index");
      layer = cfg.layers[index];
    } catch (const std::exception&) {
      throw std::invalid_argument("no layer '" + id + "' in " + cfg.name);
    }
  }
  const std::int64_t cap = a.has("--cap-hw") ? to_i64(a.get("--cap-hw", "0"), "--cap-hw") : 0;
  if (cap > 0) layer.shape = capped_spatial(layer.shape, cap);
  return layer;
}

Scheme parse_scheme(const std::string& s) {
  if (s == "fc") return Scheme::FC;
  if (s == "ic") return Scheme::IC;
  if (s == "icbatch") return Scheme::ICBatch;
  if (s == "fic") return Scheme::FIC;
  throw std::invalid_argument("unknown scheme '" + s + "'");
}
InjectionTarget parse_target(const std::string& s) {
  if (s == "input") return InjectionTarget::InputFmap;
  if (s == "filter") return InjectionTarget::Filter;
  if (s == "convout") return InjectionTarget::ConvOut;
  throw std::invalid_argument("unknown target '" + s + "'");
}

std::string locus_string(const VerifyOutcome& o) {
  if (!o.locus) return "";
  std::ostringstream os;
  const auto& l = *o.locus;
  os << l[0];
  if (l[1] >= 0) os << ":" << l[1] << ":" << l[2];
  return os.str();
}

// abed_main.cpp:143-165 make_data_tensor (seeds derive_seed(seed, 1 | 2))
Tensor4D make_data_tensor(const LayerShape& ls, const std::string& data, bool use_float, std::uint64_t seed,
                          bool filters) {
  const Dims4 dims = filters ? ls.filter_dims() : ls.input_dims();
  SplitMix64 rng(derive_seed(seed, filters ? 2 : 1));
  if (data != "random" && data != "ones" && data != "extreme" && data != "max")
    throw std::invalid_argument("unknown data mode '" + data + "' (random|ones|extreme|max)");
  if (use_float) {
    if (data == "ones") return Tensor4D::filled(dims, ElemKind::F32, 1.0);
    if (data == "max") return Tensor4D::filled(dims, ElemKind::F32, 127.0);
    Tensor4D t(dims, ElemKind::F32);
    if (data == "extreme")
      fill_random_f32(t, rng, -128.0f, 127.0f);
    else
      fill_random_f32_integers(t, rng);
    return t;
  }
  if (data == "ones") return Tensor4D::filled(dims, ElemKind::I8, 1);
  if (data == "max") return Tensor4D::filled(dims, ElemKind::I8, 127);
  Tensor4D t(dims, ElemKind::I8);
  if (data == "extreme")
    fill_random_extreme(t, rng);
  else
    fill_random_i8(t, rng);
  return t;
}

// abed_main.cpp:167-289 run_verify
int run_verify(const Args& a) {
  if (!a.has("--layer")) throw UsageError("--layer is required");
  if (!a.has("--scheme")) throw UsageError("--scheme is required");
  const LayerConfig layer = resolve_layer(a);
  const LayerShape& ls = layer.shape;
  const std::string scheme_name = a.get("--scheme", "fic");
  const Scheme scheme = parse_scheme(scheme_name);
  const bool use_float = a.flags.count("--float") != 0;
  const bool force32 = a.flags.count("--force-reduce32") != 0;
  const std::uint64_t seed = static_cast<std::uint64_t>(to_i64(a.get("--seed", "1"), "--seed"));
  const double tau = to_f64(a.get("--tau", "0"), "--tau");
  const int operand_bits = static_cast<int>(to_i64(a.get("--operand-bits", "8"), "--operand-bits"));
  const std::string data = a.get("--data", "random");
  if (use_float && (scheme == Scheme::ICBatch || force32))
    throw std::invalid_argument("--float supports fc|ic|fic without --force-reduce32");
  if (force32 && scheme != Scheme::FIC) throw std::invalid_argument("--force-reduce32 applies to the fic scheme");

  Tensor4D input = a.has("--load-input") ? load_tensor(a.get("--load-input", ""))
                                          : make_data_tensor(ls, data, use_float, seed, false);
  Tensor4D filters = a.has("--load-filters") ? load_tensor(a.get("--load-filters", ""))
                                              : make_data_tensor(ls, data, use_float, seed, true);
  if (input.dims() != ls.input_dims() || filters.dims() != ls.filter_dims())
    throw std::invalid_argument("loaded tensor dims do not match the selected layer");

  VerifyOutcome outcome;
  std::optional<PrecisionPlan> plan;
  Tensor4D convout;
  if (use_float) {
    convout = conv_direct_f32(input, filters, ls);
    if (scheme == Scheme::FC) {
      const auto sums = filter_checksum_f64(filters);
      Tensor4D cs({1, ls.c, ls.r, ls.s}, ElemKind::F32);
      for (std::size_t i = 0; i < sums.size(); ++i) cs.view<float>()[i] = static_cast<float>(sums[i]);
      LayerShape cs_shape = ls;
      cs_shape.k = 1;
      outcome = fc_verify_f32(convout, conv_direct_f32(input, cs, cs_shape), tau);
    } else if (scheme == Scheme::IC) {
      outcome = ic_verify_k_f32(convout, filters, input_checksum_f64(input, ls), tau);
    } else {
      outcome = fic_verify_f32(convout, fic_dot_f64(filter_checksum_f64(filters), input_checksum_f64(input, ls)),
                               tau);
    }
  } else {
    plan = plan_precision(ls, operand_bits);
    convout = detail::conv_fast_i8(input, filters, ls);
    switch (scheme) {
      case Scheme::FC: {
        const FilterChecksum fc = gen_filter_checksum_decomposed(filters);
        outcome = fc_verify(convout, recombine_extra_fmaps(conv_checksum_planes(input, ls, *fc.decomposed)));
        break;
      }
      case Scheme::IC:
        outcome = ic_verify_k(convout, filters, gen_input_checksum(input, ls));
        break;
      case Scheme::ICBatch:
        outcome = ic_batch_verify(convout, conv_batch_checksum(ic_batch_checksum(input), filters, ls));
        break;
      case Scheme::FIC: {
        const std::int64_t expected = fic_dot(gen_filter_checksum(filters), gen_input_checksum(input, ls));
        outcome = force32 ? fic_verify_forced32(convout, expected) : fic_verify(convout, expected);
        break;
      }
    }
  }

  if (a.has("--dump-dir")) {
    const std::filesystem::path dir(a.get("--dump-dir", ""));
    std::filesystem::create_directories(dir);
    save_tensor(dir / "input.abed", input);
    save_tensor(dir / "filters.abed", filters);
    save_tensor(dir / "convout.abed", convout);
  }

  const bool pass = outcome.pass();
  std::ostringstream csv;
  csv << "layer,scheme,mode,status,lhs,rhs,locus,seed\n";
  csv << layer.id << "," << scheme_name << "," << (use_float ? "float" : "int") << ","
      << (pass ? "pass" : "mismatch") << ",";
  if (use_float)
    csv << outcome.lhs_f << "," << outcome.rhs_f;
  else
    csv << outcome.lhs << "," << outcome.rhs;
  csv << "," << locus_string(outcome) << "," << seed << "\n";
  if (plan) {
    csv << "plan,b,output_fmap,reduced_fc,reduced_fic,filter_checksum,input_checksum\n";
    csv << "bits," << plan->operand_bits << "," << plan->bits_output_fmap << "," << plan->bits_reduced_fc << ","
        << plan->bits_reduced_fic << "," << plan->bits_filter_checksum << "," << plan->bits_input_checksum << "\n";
    csv << "kinds,," << to_string(plan->output_fmap_kind) << "," << to_string(plan->reduced_fc_kind) << ","
        << to_string(plan->reduced_fic_kind) << "," << to_string(plan->filter_checksum_kind) << ","
        << to_string(plan->input_checksum_kind) << "\n";
  }
  nlohmann::json doc{{"layer", layer.id},
                     {"scheme", scheme_name},
                     {"mode", use_float ? "float" : "int"},
                     {"status", pass ? "pass" : "mismatch"},
                     {"seed", seed}};
  if (use_float) {
    doc["lhs"] = outcome.lhs_f;
    doc["rhs"] = outcome.rhs_f;
    doc["tau"] = tau;
  } else {
    doc["lhs"] = outcome.lhs;
    doc["rhs"] = outcome.rhs;
  }
  if (outcome.locus) doc["locus"] = locus_string(outcome);
  if (plan) {
    doc["plan"] = {{"b", plan->operand_bits},
                   {"bits_output_fmap", plan->bits_output_fmap},
                   {"bits_reduced_fc", plan->bits_reduced_fc},
                   {"bits_reduced_fic", plan->bits_reduced_fic},
                   {"bits_filter_checksum", plan->bits_filter_checksum},
                   {"bits_input_checksum", plan->bits_input_checksum},
                   {"output_fmap_kind", to_string(plan->output_fmap_kind)},
                   {"reduced_fic_kind", to_string(plan->reduced_fic_kind)}};
  }
  emit(a, csv.str(), doc);
  return pass ? kExitOk : kExitMismatch;
}

// abed_main.cpp:307-344 run_inject (the campaign runs on the B200; reports are
// independent of --jobs, faults.hpp:293-317)
int run_inject(const Args& a) {
  for (const char* req : {"--layer", "--scheme", "--target"})
    if (!a.has(req)) throw UsageError(std::string(req) + " is required");
  const LayerConfig layer = resolve_layer(a);
  CampaignConfig config;
  config.shape = layer.shape;
  config.scheme = parse_scheme(a.get("--scheme", "fic"));
  if (config.scheme == Scheme::ICBatch) throw std::invalid_argument("inject supports fc|ic|fic");
  config.target = parse_target(a.get("--target", "convout"));
  config.trials = to_i64(a.get("--trials", "1000"), "--trials");
  if (config.trials < 1) throw UsageError("--trials must be positive");
  config.root_seed = static_cast<std::uint64_t>(to_i64(a.get("--seed", "1"), "--seed"));
  const std::string mode = a.get("--mode", "ones");
  config.mode = mode == "random" ? DataMode::RandomI8 : DataMode::Ones;
  config.jobs = static_cast<int>(to_i64(a.get("--jobs", "0"), "--jobs"));
  config.epilog.scale = static_cast<float>(to_f64(a.get("--scale", "0.05"), "--scale"));
  config.epilog.activation = layer.activation ? Activation::ReLU : Activation::Identity;

  const CampaignReport report = run_campaign(config);

  std::ostringstream csv;
  csv << "scheme,target,trials,detected,detected_benign,sdc,masked,detection_rate,sdc_rate,seed\n";
  csv << to_string(report.scheme) << "," << to_string(report.target) << "," << report.trials << ","
      << report.detected << "," << report.detected_benign << "," << report.sdc << "," << report.masked << ","
      << report.detection_rate() << "," << report.sdc_rate() << "," << report.seed << "\n";
  const nlohmann::json doc{{"scheme", to_string(report.scheme)},
                           {"target", to_string(report.target)},
                           {"layer", layer.id},
                           {"trials", report.trials},
                           {"detected", report.detected},
                           {"detected_benign", report.detected_benign},
                           {"sdc", report.sdc},
                           {"masked", report.masked},
                           {"detection_rate", report.detection_rate()},
                           {"sdc_rate", report.sdc_rate()},
                           {"seed", report.seed}};
  emit(a, csv.str(), doc);
  return kExitOk;
}

// abed_main.cpp:436-487 run_abft: per trial a fresh SplitMix64(derive_seed(seed, t))
// draws A, B, then (i, j, bit) of a single c_aug corruption; same CSV / JSON schema
int run_abft(const Args& a) {
  const std::int64_t m = to_i64(a.get("--m", "64"), "--m"), n = to_i64(a.get("--n", "64"), "--n");
  const std::int64_t k = to_i64(a.get("--k", "64"), "--k"), trials = to_i64(a.get("--trials", "1000"), "--trials");
  if (m < 1 || n < 1 || k < 1 || trials < 1) throw UsageError("--m/--n/--k/--trials must be positive");
  const std::uint64_t seed = static_cast<std::uint64_t>(to_i64(a.get("--seed", "1"), "--seed"));
  const bool single_pass = a.flags.count("--single-pass") != 0;
  std::int64_t faultfree_pass = 0, detected = 0;
  for (std::int64_t t = 0; t < trials; ++t) {
    SplitMix64 rng(derive_seed(seed, static_cast<std::uint64_t>(t)));
    Matrix am(m, k, ElemKind::I8), bm(k, n, ElemKind::I8);
    for (auto& v : am.view<std::int8_t>()) v = rng.next_i8();
    for (auto& v : bm.view<std::int8_t>()) v = rng.next_i8();
    AbftResult result = abft_gemm(am, bm, single_pass);
    if (result.pass()) ++faultfree_pass;
    const auto i = static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(m)));
    const auto j = static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(n)));
    const int bit = static_cast<int>(rng.below(63));
    result.c_aug.at<std::int64_t>(i, j) ^= std::int64_t{1} << bit;
    const auto [row_check, col_check] = abft_check(result.c_aug);
    if (!row_check.pass() || !col_check.pass()) ++detected;
  }
  const AbftCosts costs = abft_costs(m, n, k, single_pass);
  const double rate = static_cast<double>(detected) / static_cast<double>(trials);
  std::ostringstream csv;
  csv << "m,n,k,trials,faultfree_pass,detected,detection_rate,copy_elements,seed\n";
  csv << m << "," << n << "," << k << "," << trials << "," << faultfree_pass << "," << detected << "," << rate << ","
      << costs.copy_elements() << "," << seed << "\n";
  csv << "task,ops,read_bytes,write_bytes,elements_moved\n";
  nlohmann::json tasks = nlohmann::json::array();
  for (const auto& task : costs.tasks) {
    csv << task.name << "," << task.ops << "," << task.read_bytes << "," << task.write_bytes << ","
        << task.elements_moved << "\n";
    tasks.push_back({{"task", std::string(task.name)},
                     {"ops", task.ops},
                     {"read_bytes", task.read_bytes},
                     {"write_bytes", task.write_bytes},
                     {"elements_moved", task.elements_moved}});
  }
  const nlohmann::json doc{{"m", m}, {"n", n}, {"k", k}, {"trials", trials}, {"faultfree_pass", faultfree_pass},
                           {"detected", detected}, {"detection_rate", rate}, {"copy_elements", costs.copy_elements()},
                           {"tasks", tasks}, {"seed", seed}};
  emit(a, csv.str(), doc);
  return kExitOk;
}

// abed_main.cpp:360-417 run_cost: per-layer and total op / byte counts of a
// scheme and implementation option over a network, same CSV / JSON schema
int run_cost(const Args& a) {
  if (!a.has("--scheme")) throw UsageError("--scheme is required");
  NetworkConfig cfg = resolve_network(a);
  const Scheme scheme = parse_scheme(a.get("--scheme", "fic"));
  const std::string opt = a.get("--option", "fr");
  if (opt != "uf" && opt != "fr" && opt != "af") throw std::invalid_argument("unknown option '" + opt + "' (uf|fr|af)");
  const ImplOption option = opt == "uf" ? ImplOption::UF : opt == "fr" ? ImplOption::FR : ImplOption::AF;
  CostOptions opts;
  opts.fc_planes = static_cast<int>(to_i64(a.get("--fc-planes", "4"), "--fc-planes"));
  opts.fc_pad_to_8 = a.flags.count("--fc-pad8") != 0;
  const NetworkConfig unpruned = cfg;
  const bool pruned = a.has("--pruned");
  if (pruned) cfg = load_pruned(cfg, a.get("--pruned", ""));
  const CostReport rep = aggregate_network(cfg, scheme, option, opts, pruned ? &unpruned : nullptr);

  std::ostringstream csv;
  csv << "network,layer,scheme,option,fma,add,mul,act,cast,read_bytes,write_bytes,op_overhead_pct,byte_overhead_pct\n";
  auto line = [&](const std::string& id, const OpCounts& o, const ByteCounts& b, double op_pct, double byte_pct) {
    csv << rep.network << "," << id << "," << to_string(scheme) << "," << to_string(option) << "," << o.fma << ","
        << o.add << "," << o.mul << "," << o.activation_eval << "," << o.cast << "," << b.read_bytes << ","
        << b.write_bytes << "," << op_pct << "," << byte_pct << "\n";
  };
  auto fields = [](const OpCounts& o, const ByteCounts& b, double op_pct, double byte_pct) {
    return nlohmann::json{{"fma", o.fma}, {"add", o.add}, {"mul", o.mul}, {"act", o.activation_eval},
                          {"cast", o.cast}, {"read_bytes", b.read_bytes}, {"write_bytes", b.write_bytes},
                          {"op_overhead_pct", op_pct}, {"byte_overhead_pct", byte_pct}};
  };
  nlohmann::json rows = nlohmann::json::array();
  for (const auto& r : rep.rows) {
    line(r.layer + (r.excluded ? " (excluded)" : ""), r.ops, r.bytes, r.op_overhead_pct(), r.byte_overhead_pct());
    nlohmann::json j = {{"layer", r.layer}, {"excluded", r.excluded}};
    j.update(fields(r.ops, r.bytes, r.op_overhead_pct(), r.byte_overhead_pct()));
    rows.push_back(j);
  }
  line("TOTAL", rep.total_ops, rep.total_bytes, rep.op_overhead_pct(), rep.byte_overhead_pct());
  const nlohmann::json doc{{"network", rep.network}, {"scheme", to_string(scheme)}, {"option", to_string(option)},
                           {"layers", rows},
                           {"total", fields(rep.total_ops, rep.total_bytes, rep.op_overhead_pct(), rep.byte_overhead_pct())}};
  emit(a, csv.str(), doc);
  return kExitOk;
}

const std::set<std::string> kLayerOpts = {"--config", "--network", "--image", "--layer", "--cap-hw", "--out"};

std::set<std::string> with(std::set<std::string> base, std::initializer_list<const char*> more) {
  for (const char* m : more) base.insert(m);
  return base;
}

void usage(std::ostream& os) {
  os << "abed_b200 -- checksum-verified int8 convolutions on B200 (ABED)\n"
        "usage:\n"
        "  abed_b200 verify (--network NAME [--image 224|1080p] | --config FILE) --layer ID --scheme fc|ic|icbatch|fic\n"
        "            [--seed S] [--data random|ones|extreme|max] [--float] [--tau T] [--force-reduce32]\n"
        "            [--operand-bits 4|8] [--cap-hw N] [--dump-dir DIR] [--load-input F] [--load-filters F]\n"
        "            [--json] [--out FILE]\n"
        "  abed_b200 inject (--network NAME [--image ..] | --config FILE) --layer ID --scheme fc|ic|fic\n"
        "            --target input|filter|convout [--trials N] [--seed S] [--mode ones|random] [--jobs J]\n"
        "            [--scale X] [--cap-hw N] [--json] [--out FILE]\n"
        "  abed_b200 cost (--network NAME [--image ..] | --config FILE) --scheme fc|ic|icbatch|fic [--option uf|fr|af]\n"
        "            [--pruned FILE] [--fc-pad8] [--fc-planes 1..4] [--json] [--out FILE]\n"
        "  abed_b200 abft [--m M] [--n N] [--k K] [--trials T] [--seed S] [--single-pass] [--json] [--out FILE]\n"
        "exit codes: 0 success, 1 usage/config/IO error, 2 verification mismatch\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") {
    usage(std::cout);
    return kExitOk;
  }
  try {
    if (cmd == "verify") {
      const Args a = parse(argc, argv,
                           with(kLayerOpts, {"--scheme", "--seed", "--data", "--tau", "--operand-bits", "--dump-dir",
                                             "--load-input", "--load-filters"}),
                           {"--float", "--force-reduce32", "--json"});
      return run_verify(a);
    }
    if (cmd == "inject") {
      const Args a = parse(argc, argv,
                           with(kLayerOpts, {"--scheme", "--target", "--trials", "--seed", "--mode", "--jobs",
                                             "--scale"}),
                           {"--json"});
      return run_inject(a);
    }
    if (cmd == "cost") {
      const Args a = parse(argc, argv, {"--config", "--network", "--image", "--scheme", "--option", "--pruned",
                                        "--fc-planes", "--out"},
                           {"--fc-pad8", "--json"});
      return run_cost(a);
    }
    if (cmd == "abft") {
      const Args a = parse(argc, argv, {"--m", "--n", "--k", "--trials", "--seed", "--out"}, {"--single-pass", "--json"});
      return run_abft(a);
    }
    std::cerr << "error: unknown subcommand '" << cmd << "'\n";
    usage(std::cerr);
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}
