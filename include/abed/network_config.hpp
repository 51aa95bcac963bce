// abed/network_config.hpp -- drop-in for the reference's network_config.hpp
// (per-layer conv geometry of a network, network_config.hpp:14-282).
//
// Same types and entry points: LayerConfig / NetworkConfig (:14-37), the builtin
// VGG16 / ResNet18 / ResNet50 tables at 224x224 and 1080x1920 (:163-282: same
// layer ids, shapes, activations and exclude_first_layer), builtin_network, and
// the JSON schema of network_from_json / load_network (:58-101).  JSON goes
// through nlohmann/json (the reference's own dependency); it is only compiled in
// when <json.hpp> is on the include path (the CLI build adds the copy this image
// ships), so the rest of the drop-in stays dependency-free.
#pragma once

#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tensor.hpp"

#if __has_include(<json.hpp>)
#include <json.hpp>
#define ABED_HAVE_JSON 1
#endif

namespace abed {

struct LayerConfig {
  std::string id;
  LayerShape shape;
  bool activation = true;
};

struct NetworkConfig {
  std::string name;
  bool exclude_first_layer = false;
  std::vector<LayerConfig> layers;

  const LayerConfig& layer(const std::string& id) const {
    for (const auto& l : layers)
      if (l.id == id) return l;
    throw std::invalid_argument("NetworkConfig: no layer with id '" + id + "'");
  }
  bool has_layer(const std::string& id) const {
    for (const auto& l : layers)
      if (l.id == id) return true;
    return false;
  }
};

namespace detail {

// the builtins chain their stages through these pooling steps
inline std::int64_t halve(std::int64_t v) { return v / 2; }                 // 2x2 max pool, stride 2
inline std::int64_t pool3s2(std::int64_t v) { return (v - 1) / 2 + 1; }     // 3x3 max pool, stride 2, pad 1

inline LayerConfig conv_layer(std::string id, std::int64_t c, std::int64_t h, std::int64_t w, std::int64_t k,
                              std::int64_t rs, std::int64_t st, std::int64_t pad, bool act) {
  return LayerConfig{std::move(id), LayerShape::make(1, c, h, w, k, rs, rs, st, st, pad, pad), act};
}

inline NetworkConfig vgg16(std::int64_t h, std::int64_t w, const std::string& tag) {
  NetworkConfig cfg{"vgg16-" + tag, true, {}};
  const std::vector<std::vector<std::int64_t>> stages = {
      {64, 64}, {128, 128}, {256, 256, 256}, {512, 512, 512}, {512, 512, 512}};
  std::int64_t c = 3;
  for (std::size_t s = 0; s < stages.size(); ++s) {
    for (std::size_t i = 0; i < stages[s].size(); ++i) {
      const std::string id = "conv" + std::to_string(s + 1) + "_" + std::to_string(i + 1);
      cfg.layers.push_back(conv_layer(id, c, h, w, stages[s][i], 3, 1, 1, true));
      c = stages[s][i];
    }
    h = halve(h);
    w = halve(w);
  }
  return cfg;
}

// ResNet18: both 3x3 convs of every basic block, identity shortcuts; ReLU after
// conv1 of a block, after the residual add for conv2 (activation false here)
inline NetworkConfig resnet18(std::int64_t h, std::int64_t w, const std::string& tag) {
  NetworkConfig cfg{"resnet18-" + tag, true, {}};
  cfg.layers.push_back(conv_layer("conv1", 3, h, w, 64, 7, 2, 3, true));
  h = pool3s2(cfg.layers.back().shape.p);
  w = pool3s2(cfg.layers.back().shape.q);
  const std::int64_t widths[4] = {64, 128, 256, 512};
  std::int64_t c = 64;
  for (int s = 0; s < 4; ++s) {
    for (int b = 0; b < 2; ++b) {
      const std::int64_t st = (b == 0 && s > 0) ? 2 : 1;
      const std::string pre = "layer" + std::to_string(s + 1) + "." + std::to_string(b);
      const LayerConfig c1 = conv_layer(pre + ".conv1", c, h, w, widths[s], 3, st, 1, true);
      cfg.layers.push_back(c1);
      cfg.layers.push_back(conv_layer(pre + ".conv2", widths[s], c1.shape.p, c1.shape.q, widths[s], 3, 1, 1, false));
      h = c1.shape.p;
      w = c1.shape.q;
      c = widths[s];
    }
  }
  return cfg;
}

// ResNet50 (v1.5: the stride sits on the 3x3): conv1 1x1, conv2 3x3, conv3 1x1
// per bottleneck, plus the 1x1 projection ("downsample") on each stage's first block
inline NetworkConfig resnet50(std::int64_t h, std::int64_t w, const std::string& tag) {
  NetworkConfig cfg{"resnet50-" + tag, true, {}};
  cfg.layers.push_back(conv_layer("conv1", 3, h, w, 64, 7, 2, 3, true));
  h = pool3s2(cfg.layers.back().shape.p);
  w = pool3s2(cfg.layers.back().shape.q);
  const int blocks[4] = {3, 4, 6, 3};
  const std::int64_t width[4] = {64, 128, 256, 512};
  std::int64_t c = 64;
  for (int s = 0; s < 4; ++s) {
    const std::int64_t out = 4 * width[s];
    for (int b = 0; b < blocks[s]; ++b) {
      const std::int64_t st = (b == 0 && s > 0) ? 2 : 1;
      const std::string pre = "layer" + std::to_string(s + 1) + "." + std::to_string(b);
      cfg.layers.push_back(conv_layer(pre + ".conv1", c, h, w, width[s], 1, 1, 0, true));
      const LayerConfig c2 = conv_layer(pre + ".conv2", width[s], h, w, width[s], 3, st, 1, true);
      cfg.layers.push_back(c2);
      cfg.layers.push_back(conv_layer(pre + ".conv3", width[s], c2.shape.p, c2.shape.q, out, 1, 1, 0, false));
      if (b == 0) cfg.layers.push_back(conv_layer(pre + ".downsample", c, h, w, out, 1, st, 0, false));
      h = c2.shape.p;
      w = c2.shape.q;
      c = out;
    }
  }
  return cfg;
}

}  // namespace detail

/// network_config.hpp:284 builtin_network: name vgg16|resnet18|resnet50, image 224|1080p
inline NetworkConfig builtin_network(const std::string& name, const std::string& image) {
  std::int64_t h = 0, w = 0;
  if (image == "224") {
    h = w = 224;
  } else if (image == "1080p") {
    h = 1080;
    w = 1920;
  } else {
    throw std::invalid_argument("builtin_network: unknown image size '" + image + "' (224|1080p)");
  }
  if (name == "vgg16") return detail::vgg16(h, w, image);
  if (name == "resnet18") return detail::resnet18(h, w, image);
  if (name == "resnet50") return detail::resnet50(h, w, image);
  throw std::invalid_argument("builtin_network: unknown network '" + name + "' (vgg16|resnet18|resnet50)");
}

#ifdef ABED_HAVE_JSON
/// network_config.hpp:58-88 network_from_json (same keys, defaults and errors)
inline NetworkConfig network_from_json(const nlohmann::json& j) {
  NetworkConfig cfg;
  cfg.name = j.at("name").get<std::string>();
  cfg.exclude_first_layer = j.value("exclude_first_layer", false);
  if (!j.contains("layers") || !j.at("layers").is_array() || j.at("layers").empty())
    throw std::invalid_argument("network config: missing or empty layers array");
  for (const auto& l : j.at("layers")) {
    LayerConfig layer;
    layer.id = l.at("id").get<std::string>();
    auto g = [&](const char* key) { return l.at(key).get<std::int64_t>(); };
    layer.shape = LayerShape::make(g("n"), g("c"), g("h"), g("w"), g("k"), g("r"), g("s"),
                                   l.value("stride_h", std::int64_t{1}), l.value("stride_w", std::int64_t{1}),
                                   l.value("pad_h", std::int64_t{0}), l.value("pad_w", std::int64_t{0}));
    layer.activation = l.value("activation", true);
    if (cfg.has_layer(layer.id))
      throw std::invalid_argument("network config: duplicate layer id '" + layer.id + "'");
    cfg.layers.push_back(std::move(layer));
  }
  return cfg;
}

/// network_config.hpp:90-96 load_network
inline NetworkConfig load_network(const std::filesystem::path& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("load_network: cannot open " + path.string());
  nlohmann::json j;
  f >> j;
  return network_from_json(j);
}

/// network_config.hpp apply_pruned_k / load_pruned: per-layer output-channel
/// overrides {"layers": [{"id", "k"}], "name"?}; 1 <= k <= the layer's K
inline NetworkConfig apply_pruned_k(const NetworkConfig& cfg, const nlohmann::json& pruned) {
  NetworkConfig out = cfg;
  for (const auto& e : pruned.at("layers")) {
    const std::string id = e.at("id").get<std::string>();
    const std::int64_t k = e.at("k").get<std::int64_t>();
    auto it = std::find_if(out.layers.begin(), out.layers.end(), [&](const LayerConfig& l) { return l.id == id; });
    if (it == out.layers.end()) throw std::invalid_argument("pruned config: unknown layer id '" + id + "'");
    if (k < 1 || k > it->shape.k) throw std::invalid_argument("pruned config: bad k for layer '" + id + "'");
    it->shape.k = k;
  }
  if (pruned.contains("name")) out.name = pruned.at("name").get<std::string>();
  return out;
}
inline NetworkConfig load_pruned(const NetworkConfig& cfg, const std::filesystem::path& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("load_pruned: cannot open " + path.string());
  nlohmann::json j;
  f >> j;
  return apply_pruned_k(cfg, j);
}
#endif

}  // namespace abed
