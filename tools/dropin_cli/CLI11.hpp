// Minimal CLI11-compatible command-line parser (drop-in build support only).
//
// The reference's CLI (/root/reference/proj/tools/abed_main.cpp) includes
// <CLI11.hpp>, a vendored third-party header that is absent from the reference
// tree.  This file provides the subset of the CLI11 interface that abed_main.cpp
// uses -- App / add_subcommand / add_option / add_flag / require_subcommand /
// parse / exit / parsed, Option::required / needs / excludes / check,
// CLI::PositiveNumber, CLI::ParseError / CLI::CallForHelp -- so that the
// UNMODIFIED reference driver compiles against this repository's drop-in
// headers (include/abed/*.hpp) and runs on the B200 library
// (tools/dropin_cli/build.sh).  Behaviour follows CLI11's documented defaults
// for that subset: unknown arguments, missing values, failed conversions,
// failed validators, missing required options and needs / excludes violations
// throw ParseError; --help / -h throws CallForHelp.
#pragma once

#include <cerrno>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& msg, int code = 106) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

class CallForHelp : public ParseError {
 public:
  CallForHelp() : ParseError("help requested", 0) {}
};

// a validator maps the raw string to an error message ("" = accepted)
struct Validator {
  std::function<std::string(const std::string&)> fn;
};

inline const Validator PositiveNumber{[](const std::string& s) -> std::string {
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s.c_str(), &end);
  if (s.empty() || end != s.c_str() + s.size() || errno != 0) return "Value " + s + " could not be converted";
  if (!(v > 0.0)) return "Value " + s + " not in range (0 - inf)";
  return "";
}};

namespace detail {

template <typename T>
bool convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
    return true;
  } else if constexpr (std::is_same_v<T, bool>) {
    if (s == "true" || s == "1" || s == "on" || s == "yes") return out = true, true;
    if (s == "false" || s == "0" || s == "off" || s == "no") return out = false, true;
    return false;
  } else if constexpr (std::is_integral_v<T>) {
    if (s.empty()) return false;
    if (std::is_unsigned_v<T> && s[0] == '-') return false;
    const char* b = s.c_str() + (s[0] == '+' ? 1 : 0);
    const char* e = s.c_str() + s.size();
    T v{};
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc() || r.ptr != e) return false;
    out = v;
    return true;
  } else if constexpr (std::is_floating_point_v<T>) {
    if (s.empty()) return false;
    char* end = nullptr;
    errno = 0;
    const long double v = std::strtold(s.c_str(), &end);
    if (end != s.c_str() + s.size() || errno == ERANGE) return false;
    out = static_cast<T>(v);
    return true;
  } else {
    static_assert(sizeof(T) == 0, "CLI shim: unsupported option type");
  }
}

}  // namespace detail

class Option {
 public:
  Option(std::string name, std::string desc, bool flag, std::function<bool(const std::string&)> set)
      : name_(std::move(name)), desc_(std::move(desc)), flag_(flag), set_(std::move(set)) {}

  Option* required(bool on = true) {
    required_ = on;
    return this;
  }
  Option* needs(Option* other) {
    needs_.push_back(other);
    return this;
  }
  Option* excludes(Option* other) {
    excludes_.push_back(other);
    other->excludes_.push_back(this);
    return this;
  }
  Option* check(const Validator& v) {
    checks_.push_back(v);
    return this;
  }
  std::size_t count() const { return count_; }
  const std::string& get_name() const { return name_; }

 private:
  friend class App;
  void take(const std::string& value) {
    for (const Validator& v : checks_) {
      const std::string err = v.fn(value);
      if (!err.empty()) throw ParseError(name_ + ": " + err);
    }
    if (!set_(value)) throw ParseError("Could not convert: " + name_ + " = " + value);
    ++count_;
  }

  std::string name_, desc_;
  bool flag_;
  std::function<bool(const std::string&)> set_;
  bool required_ = false;
  std::vector<Option*> needs_, excludes_;
  std::vector<Validator> checks_;
  std::size_t count_ = 0;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  App* require_subcommand(int n = 1) {
    require_sub_ = n;
    return this;
  }
  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    subs_.back()->parent_ = this;
    return subs_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& name, T& var, const std::string& desc = "") {
    opts_.push_back(std::make_unique<Option>(name, desc, false,
                                             [&var](const std::string& s) { return detail::convert(s, var); }));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& var, const std::string& desc = "") {
    opts_.push_back(std::make_unique<Option>(name, desc, true, [&var](const std::string& s) {
      if (s.empty()) return var = true, true;
      return detail::convert(s, var);
    }));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parsed_ = true;
    App* cur = this;
    for (std::size_t i = 0; i < args.size(); ++i) {
      const std::string& tok = args[i];
      if (tok == "--help" || tok == "-h") throw CallForHelp();
      if (tok.rfind("--", 0) == 0) {
        const std::size_t eq = tok.find('=');
        const std::string key = tok.substr(0, eq);
        Option* o = cur->find(key);
        if (!o) throw ParseError("The following argument was not expected: " + tok);
        if (o->flag_) {
          o->take(eq == std::string::npos ? "" : tok.substr(eq + 1));
        } else if (eq != std::string::npos) {
          o->take(tok.substr(eq + 1));
        } else {
          if (i + 1 >= args.size()) throw ParseError(key + ": 1 required argument(s) missing");
          o->take(args[++i]);
        }
        continue;
      }
      // positional tokens: only a subcommand name of this (top-level) app
      App* sub = nullptr;
      if (cur == this)
        for (auto& s : subs_)
          if (s->name_ == tok) sub = s.get();
      if (!sub) throw ParseError("The following argument was not expected: " + tok);
      sub->parsed_ = true;
      cur = sub;
    }
    int nsub = 0;
    for (auto& s : subs_) nsub += s->parsed_ ? 1 : 0;
    if (require_sub_ > 0 && nsub < require_sub_) throw ParseError("A subcommand is required");
    validate();
    for (auto& s : subs_)
      if (s->parsed_) s->validate();
  }
  void parse(int argc, char** argv) { parse(argc, const_cast<const char* const*>(argv)); }

  int exit(const ParseError& e) const {
    if (dynamic_cast<const CallForHelp*>(&e)) {
      std::cout << help();
      return 0;
    }
    std::cerr << "error: " << e.what() << "\nRun with --help for more information.\n";
    return e.get_exit_code();
  }

  std::string help() const {
    std::string h = desc_ + "\n";
    if (!subs_.empty()) {
      h += "Subcommands:\n";
      for (auto& s : subs_) h += "  " + s->name_ + "  " + s->desc_ + "\n";
    }
    if (!opts_.empty()) {
      h += "Options:\n";
      for (auto& o : opts_) h += "  " + o->name_ + "  " + o->desc_ + (o->required_ ? " (required)" : "") + "\n";
    }
    return h;
  }

 private:
  Option* find(const std::string& key) {
    for (auto& o : opts_)
      if (o->name_ == key) return o.get();
    return nullptr;
  }
  void validate() const {
    for (auto& o : opts_) {
      if (o->required_ && o->count_ == 0) throw ParseError(o->name_ + " is required");
      if (o->count_ == 0) continue;
      for (Option* n : o->needs_)
        if (n->count_ == 0) throw ParseError(o->name_ + " requires " + n->name_);
      for (Option* x : o->excludes_)
        if (x->count_ > 0) throw ParseError(o->name_ + " excludes " + x->name_);
    }
  }

  std::string desc_, name_;
  App* parent_ = nullptr;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
