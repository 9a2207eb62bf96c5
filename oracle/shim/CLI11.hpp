// Minimal CLI11 subset for the reference CLI (proj/tools/main.cpp), built
// only as a parity oracle. TEST INFRASTRUCTURE ONLY. Supports subcommands,
// positional and `--name value` options, flags, required(), parsed() and
// CLI11_PARSE (usage errors exit with code 106 like CLI11's ArgumentMismatch
// family; the reference maps nothing else to that path).
#ifndef VEQ_ORACLE_CLI11_SHIM_H
#define VEQ_ORACLE_CLI11_SHIM_H
#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

namespace CLI {
struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string &m, int c) : std::runtime_error(m), code(c) {}
};
struct Option {
  std::string name;
  bool positional = false, flag = false, is_required = false, seen = false;
  std::function<void(const std::string &)> set;
  Option *required() { is_required = true; return this; }
};
class App {
public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
  void require_subcommand(int) { need_sub_ = true; }
  App *add_subcommand(const std::string &name, const std::string &desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <class T> Option *add_option(const std::string &name, T &target, const std::string & = "") {
    auto o = std::make_unique<Option>();
    o->name = name;
    o->positional = name.empty() || name[0] != '-';
    o->set = [&target](const std::string &v) {
      if constexpr (std::is_same_v<T, std::string>) target = v;
      else {
        std::istringstream is(v);
        T x{};
        if (!(is >> x) || !is.eof()) throw ParseError("invalid value '" + v + "'", 106);
        target = x;
      }
    };
    opts_.push_back(std::move(o));
    return opts_.back().get();
  }
  Option *add_flag(const std::string &name, bool &target, const std::string & = "") {
    auto o = std::make_unique<Option>();
    o->name = name;
    o->flag = true;
    o->set = [&target](const std::string &) { target = true; };
    opts_.push_back(std::move(o));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }
  void parse(int argc, char **argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_vec(args, 0);
  }

private:
  void parse_vec(const std::vector<std::string> &args, size_t i) {
    parsed_ = true;
    size_t pos_idx = 0;
    for (; i < args.size(); i++) {
      const std::string &a = args[i];
      if (a.size() > 1 && a[0] == '-') {
        std::string key = a, val;
        bool has_eq = false;
        if (auto eq = a.find('='); eq != std::string::npos) {
          key = a.substr(0, eq);
          val = a.substr(eq + 1);
          has_eq = true;
        }
        Option *o = find(key);
        if (!o) throw ParseError("unknown option " + key, 109);
        o->seen = true;
        if (o->flag) { o->set(""); continue; }
        if (!has_eq) {
          if (i + 1 >= args.size()) throw ParseError(key + " needs a value", 106);
          val = args[++i];
        }
        o->set(val);
        continue;
      }
      bool matched_sub = false;
      if (pos_idx == 0 || subs_.size()) {
        for (auto &s : subs_)
          if (s->name_ == a) { s->parse_vec(args, i + 1); matched_sub = true; break; }
      }
      if (matched_sub) { i = args.size(); break; }
      Option *p = nth_positional(pos_idx++);
      if (!p) throw ParseError("unexpected argument " + a, 109);
      p->seen = true;
      p->set(a);
    }
    for (auto &o : opts_)
      if (o->is_required && !o->seen) throw ParseError(o->name + " is required", 106);
    if (need_sub_) {
      bool any = false;
      for (auto &s : subs_) any = any || s->parsed_;
      if (!any) throw ParseError("a subcommand is required", 106);
    }
  }
  Option *find(const std::string &k) {
    for (auto &o : opts_) if (!o->positional && o->name == k) return o.get();
    return nullptr;
  }
  Option *nth_positional(size_t n) {
    for (auto &o : opts_) if (o->positional && n-- == 0) return o.get();
    return nullptr;
  }
  std::string desc_, name_;
  bool need_sub_ = false, parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};
} // namespace CLI

#define CLI11_PARSE(app, argc, argv)                                           \
  try {                                                                        \
    (app).parse((argc), (argv));                                               \
  } catch (const CLI::ParseError &e) {                                         \
    std::cerr << e.what() << "\n";                                             \
    return e.code;                                                             \
  }
#endif
