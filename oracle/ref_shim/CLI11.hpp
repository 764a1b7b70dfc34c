// CLI11-lite — TEST INFRASTRUCTURE ONLY.  The subset of CLI11's API that the
// reference's command line (sim.cpp:736-872) uses: subcommands, positional and
// --named options with a value, required(), parse(), got_subcommand(), exit().
#pragma once

#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>
#include <functional>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

class Option {
 public:
  template <class T>
  Option(std::string name, T& target) : name_(std::move(name)) {
    set_ = [&target](const std::string& v) {
      std::istringstream is(v);
      if constexpr (std::is_same<T, std::string>::value) target = v;
      else if (!(is >> target)) throw ParseError("invalid value '" + v + "'", 2);
    };
  }
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  bool positional() const { return name_.rfind("--", 0) != 0; }
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool required_ = false, seen_ = false;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
  void require_subcommand(int n) { need_sub_ = n; }
  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <class T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, target));
    return opts_.back().get();
  }
  void parse(int argc, char** argv) {
    std::vector<std::string> a(argv + 1, argv + argc);
    parse_args(a, 0);
  }
  bool got_subcommand(const App* s) const { return s == chosen_; }
  int exit(const ParseError& e) const {
    std::cerr << e.what() << "\n";
    return e.code;
  }

 private:
  void parse_args(const std::vector<std::string>& a, size_t i) {
    if (!subs_.empty()) {
      if (i >= a.size()) throw ParseError("a subcommand is required", 2);
      for (auto& s : subs_)
        if (s->name_ == a[i]) {
          chosen_ = s.get();
          s->parse_own(a, i + 1);
          return;
        }
      throw ParseError("unknown subcommand '" + a[i] + "'", 2);
    }
    parse_own(a, i);
  }
  void parse_own(const std::vector<std::string>& a, size_t i) {
    size_t pos = 0;
    for (; i < a.size(); ++i) {
      if (a[i].rfind("--", 0) == 0) {
        std::string key = a[i], val;
        const size_t eq = key.find('=');
        if (eq != std::string::npos) {
          val = key.substr(eq + 1);
          key = key.substr(0, eq);
        } else {
          if (i + 1 >= a.size()) throw ParseError("option " + key + " needs a value", 2);
          val = a[++i];
        }
        Option* o = find(key);
        if (!o) throw ParseError("unknown option " + key, 2);
        o->set_(val);
        o->seen_ = true;
      } else {
        Option* o = nth_positional(pos++);
        if (!o) throw ParseError("unexpected argument '" + a[i] + "'", 2);
        o->set_(a[i]);
        o->seen_ = true;
      }
    }
    for (auto& o : opts_)
      if (o->required_ && !o->seen_) throw ParseError(o->name_ + " is required", 2);
  }
  Option* find(const std::string& k) {
    for (auto& o : opts_)
      if (o->name_ == k) return o.get();
    return nullptr;
  }
  Option* nth_positional(size_t n) {
    for (auto& o : opts_)
      if (o->positional() && n-- == 0) return o.get();
    return nullptr;
  }
  std::string desc_, name_;
  int need_sub_ = 0;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  App* chosen_ = nullptr;
};

}  // namespace CLI
