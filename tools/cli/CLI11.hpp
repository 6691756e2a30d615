// Minimal stand-in for the CLI11 command-line parser (the reference's vendor/
// directory is not shipped, proj/.gitignore:2), covering exactly the API the
// reference's tools/veil_cli.cpp uses: App::add_option for scalars and
// vectors with ->expected(n) / ->check(Range), App::add_flag, --help, and
// the CLI11_PARSE macro. With it the reference CLI compiles unmodified
// against libveil.so (tools/cli/Makefile), showing that its C-ABI-only
// driver runs on the device renderer.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help", 0) {}
};

struct Range {
  double lo, hi;
  Range(double a, double b) : lo(a), hi(b) {}
};

namespace detail {
template <typename T>
bool convert(const std::string& s, T* out) {
  std::istringstream in(s);
  if constexpr (std::is_same_v<T, std::string>) {
    *out = s;
    return true;
  } else if constexpr (std::is_unsigned_v<T>) {
    if (!s.empty() && s[0] == '-') return false;
    unsigned long long v = 0;
    in >> v;
    *out = T(v);
  } else {
    in >> *out;
  }
  return bool(in) && (in >> std::ws).eof();
}
template <typename T>
struct is_vector : std::false_type {};
template <typename T>
struct is_vector<std::vector<T>> : std::true_type {};
}  // namespace detail

class Option {
 public:
  Option(std::string name, std::string desc, bool flag) : name_(std::move(name)), desc_(std::move(desc)), flag_(flag) {}
  Option* expected(int n) {
    expected_ = n;
    return this;
  }
  Option* check(const Range& r) {
    range_ = std::make_unique<Range>(r);
    return this;
  }
  const std::string& name() const { return name_; }
  const std::string& description() const { return desc_; }
  bool is_flag() const { return flag_; }
  int expected_count() const { return expected_; }
  std::function<bool(const std::vector<std::string>&)> assign;
  const Range* range() const { return range_.get(); }

 private:
  std::string name_, desc_;
  bool flag_;
  int expected_ = 1;
  std::unique_ptr<Range> range_;
};

class App {
 public:
  explicit App(std::string description) : description_(std::move(description)) {}

  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& desc = "") {
    auto opt = std::make_unique<Option>(name, desc, false);
    Option* o = opt.get();
    if constexpr (detail::is_vector<T>::value) {
      o->expected(-1);
      o->assign = [&target](const std::vector<std::string>& v) {
        target.clear();
        for (const auto& s : v) {
          typename T::value_type x{};
          if (!detail::convert(s, &x)) return false;
          target.push_back(x);
        }
        return true;
      };
    } else {
      o->assign = [&target, o](const std::vector<std::string>& v) {
        T x{};
        if (v.size() != 1 || !detail::convert(v[0], &x)) return false;
        if constexpr (std::is_arithmetic_v<T>) {
          if (o->range() && (double(x) < o->range()->lo || double(x) > o->range()->hi)) return false;
        }
        target = x;
        return true;
      };
    }
    options_.push_back(std::move(opt));
    return o;
  }

  Option* add_flag(const std::string& name, bool& target, const std::string& desc = "") {
    auto opt = std::make_unique<Option>(name, desc, true);
    opt->assign = [&target](const std::vector<std::string>&) {
      target = true;
      return true;
    };
    Option* o = opt.get();
    options_.push_back(std::move(opt));
    return o;
  }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    for (size_t i = 0; i < args.size();) {
      std::string a = args[i++];
      if (a == "--help" || a == "-h") throw CallForHelp();
      std::string inline_value;
      bool has_inline = false;
      if (auto eq = a.find('='); eq != std::string::npos && a.rfind("--", 0) == 0) {
        inline_value = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_inline = true;
      }
      Option* o = find(a);
      if (!o) throw ParseError("The following argument was not expected: " + a, 109);
      std::vector<std::string> values;
      if (!o->is_flag()) {
        if (has_inline) values.push_back(inline_value);
        const int want = o->expected_count();
        while (i < args.size() && (want < 0 || int(values.size()) < want)) {
          if (args[i].rfind("--", 0) == 0 && find(args[i].substr(0, args[i].find('='))) ) break;
          values.push_back(args[i++]);
        }
        if (values.empty() || (want > 0 && int(values.size()) != want))
          throw ParseError(a + ": expected " + std::to_string(want < 0 ? 1 : want) + " value(s)", 107);
      }
      if (!o->assign(values)) throw ParseError(a + ": invalid value", 105);
    }
  }

  int exit(const ParseError& e) const {
    if (dynamic_cast<const CallForHelp*>(&e)) {
      std::cout << description_ << "\n\nOptions:\n  -h,--help  Print this help message and exit\n";
      for (const auto& o : options_) std::cout << "  " << o->name() << "  " << o->description() << "\n";
      return 0;
    }
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return e.code;
  }

 private:
  Option* find(const std::string& name) {
    for (auto& o : options_)
      if (o->name() == name) return o.get();
    return nullptr;
  }
  std::string description_;
  std::vector<std::unique_ptr<Option>> options_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)      \
  try {                                   \
    (app).parse((argc), (argv));          \
  } catch (const CLI::ParseError& e) {    \
    return (app).exit(e);                 \
  }
