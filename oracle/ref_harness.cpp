// ref_harness — TEST INFRASTRUCTURE ONLY (parity oracle + CPU baseline).
//
// Links the reference checker compiled from /root/reference/proj (see
// oracle/Makefile) and:
//   pair  OUTDIR A.mk B.mk CFG      elaborate both kernels with the REFERENCE
//                                   frontend, write them as packed IR
//                                   (a.veqir, b.veqir) plus golden.json: the
//                                   reference's run() results for each side and
//                                   its full check_equivalence report.
//   gen   OUTDIR SEED               same for the reference's property-test
//                                   program generator (tests/prog_gen.hpp).
//   bench A.mk B.mk CFGLIST THREADS SECONDS   (CFGLIST line: cfg [TAB b.mk])
//                                   CPU baseline: times the reference's own
//                                   run(A) + run(B) + eq() per CTA pair (the
//                                   t_exec_a + t_exec_b + t_decide span of
//                                   pipeline.cpp:182-243) over the configs
//                                   listed in CFGLIST, on THREADS host threads,
//                                   until SECONDS elapse; prints JSON.
// Nothing in the product links or calls this.
#include <atomic>
#include <chrono>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

#include <json.hpp>

#include "ctaeq/decide.hpp"
#include "ctaeq/expr.hpp"
#include "ctaeq/frontend.hpp"
#include "ctaeq/ir.hpp"
#include "ctaeq/pipeline.hpp"
#include "ctaeq/symexec.hpp"
#include "/root/reference/proj/tests/prog_gen.hpp"
#include "veq_ir.hpp"
#include "ref_pack.hpp"

using namespace ctaeq;
using ojson = nlohmann::ordered_json;

namespace {

std::string read_file(const std::string &p) {
  std::ifstream in(p, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + p);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

using refpack::to_ir;

ojson loc_j(const SrcLoc &l) { return ojson{{"line", l.line}, {"col", l.col}}; }

ojson access_j(const AccessRef &a) {
  return ojson{{"tid", a.tid}, {"access", access_kind_str(a.kind)}, {"loc", loc_j(a.loc)}, {"step", a.step}};
}

ojson safety_j(const SafetyReport &s) {
  ojson j;
  j["kind"] = safety_kind_str(s.kind);
  j["tid"] = s.tid;
  j["loc"] = loc_j(s.loc);
  if (s.addr) {
    j["array"] = s.addr->array;
    j["offset"] = s.addr->offset;
  }
  j["reg"] = s.reg;
  j["is_store"] = s.is_store;
  j["detail"] = s.detail;
  j["step"] = s.step;
  return j;
}

ojson deadlock_j(const DeadlockReport &d) {
  ojson j;
  j["threads"] = ojson::array();
  for (const auto &t : d.threads) {
    ojson tj;
    tj["tid"] = t.tid;
    tj["state"] = thread_state_str(t.state);
    if (t.waiting) tj["waiting"] = t.waiting->to_vector();
    if (t.state == ThreadState::Blocked) tj["loc"] = loc_j(t.loc);
    j["threads"].push_back(tj);
  }
  if (d.conflict_tids) {
    j["conflict_tids"] = {d.conflict_tids->first, d.conflict_tids->second};
    j["conflict_sets"] = {d.conflict_sets->first.to_vector(), d.conflict_sets->second.to_vector()};
  }
  j["str"] = d.str();
  return j;
}

ojson run_j(const RunResult &rr) {
  ojson j;
  j["steps"] = rr.steps;
  j["releases"] = rr.releases;
  const char *ok[] = {"final", "race", "deadlock", "safety"};
  j["outcome"] = ok[(int)rr.outcome.kind];
  j["races"] = ojson::array();
  for (const auto &r : rr.races) {
    ojson x;
    x["array"] = r.addr.array;
    x["offset"] = r.addr.offset;
    x["first"] = access_j(r.first);
    x["second"] = access_j(r.second);
    x["str"] = r.str();
    j["races"].push_back(x);
  }
  j["safeties"] = ojson::array();
  for (const auto &s : rr.safeties) {
    ojson x = safety_j(s);
    x["str"] = s.str();
    j["safeties"].push_back(x);
  }
  j["deadlock"] = rr.deadlock ? deadlock_j(*rr.deadlock) : ojson(nullptr);
  j["shared"] = ojson::object();
  if (rr.outcome.kind == Outcome::Kind::Final)
    for (const auto &[addr, v] : rr.outcome.shared) j["shared"][addr.str()] = to_string(v);
  // Final register files (Outcome::regs): per thread, register -> to_string
  // (programs of at most 256 threads: the fixtures stay small)
  j["regs"] = ojson::array();
  if (rr.outcome.kind == Outcome::Kind::Final && rr.outcome.regs.size() <= 256)
    for (const RegFile &rf : rr.outcome.regs) {
      ojson t = ojson::object();
      for (const auto &[name, v] : rf) t[name] = to_string(v);
      j["regs"].push_back(t);
    }
  return j;
}

void write_json(const std::string &path, const ojson &j) {
  std::ofstream out(path);
  out << j.dump(1) << "\n";
}

ojson inputs_j(const std::vector<std::string> &order, const std::map<std::string, uint64_t> &sizes) {
  ojson j = ojson::array();
  for (auto &n : order) j.push_back({{"name", n}, {"size", sizes.at(n)}});
  return j;
}

int cmd_pair(const std::string &dir, const std::string &pa_path, const std::string &pb_path,
             const std::string &cfg_path) {
  LaunchConfig cfg = parse_config(read_file(cfg_path));
  CheckRequest req;
  req.kernel_a_src = read_file(pa_path);
  req.kernel_b_src = read_file(pb_path);
  req.cfg = cfg;
  ojson g;
  // the reference's full pipeline report (minus timings)
  Report rep = check_equivalence(req, 1);
  ojson rj = report_to_json(rep);
  rj.erase("timings");
  g["report"] = rj;
  Program pa, pb;
  try {
    pa = elaborate(parse_kernel(req.kernel_a_src), cfg, cfg.for_a());
    validate_structured(pa);
    pb = elaborate(parse_kernel(req.kernel_b_src), cfg, cfg.for_b());
    validate_structured(pb);
  } catch (const std::exception &e) {
    g["elab_error"] = e.what();
    write_json(dir + "/golden.json", g);
    return 0;
  }
  SharedMem init = make_symbolic_inputs(cfg, pa.arrays);
  std::vector<std::string> order;
  std::map<std::string, uint64_t> sizes;
  for (const auto &name : cfg.inputs)
    for (const auto &a : pa.arrays)
      if (a.name == name && !sizes.count(name)) {
        order.push_back(name);
        sizes[name] = a.size;
      }
  g["inputs"] = inputs_j(order, sizes);
  to_ir(pa, sizes, order).save(dir + "/a.veqir");
  to_ir(pb, sizes, order).save(dir + "/b.veqir");
  RunResult ra = run(pa, init, SchedulePolicy::round_robin());
  RunResult rb = run(pb, init, SchedulePolicy::round_robin());
  g["run_a"] = run_j(ra);
  g["run_b"] = run_j(rb);
  // fast-path bit per VC: canonical structures identical (decide.cpp:765)
  ojson fp = ojson::array();
  if (ra.outcome.kind == Outcome::Kind::Final && rb.outcome.kind == Outcome::Kind::Final) {
    std::vector<const ArrayDecl *> outs;
    for (const auto &a : pa.arrays)
      if (a.role == Role::Out) outs.push_back(&a);
    std::sort(outs.begin(), outs.end(), [](auto *x, auto *y) { return x->name < y->name; });
    for (auto *a : outs)
      for (uint64_t i = 0; i < a->size; i++) {
        Addr ad{a->name, (int64_t)i};
        auto ia = ra.outcome.shared.find(ad), ib = rb.outcome.shared.find(ad);
        ojson v;
        v["array"] = a->name;
        v["index"] = i;
        if (ia == ra.outcome.shared.end() || ib == rb.outcome.shared.end()) {
          v["missing"] = true;
        } else {
          Expr cf = canonicalize(ia->second), cg = canonicalize(ib->second);
          v["fast_equal"] = (cf == cg);
          std::vector<SideCondition> sc;
          std::set<Expr> seen;
          collect_side_conditions(cf, sc, seen);
          collect_side_conditions(cg, sc, seen);
          ojson scj = ojson::array();
          for (auto &c : sc) scj.push_back({{"denominator", to_string(c.denominator)}, {"discharged", c.discharged}});
          v["side_conditions"] = scj;
        }
        fp.push_back(v);
      }
  }
  g["fast_path"] = fp;
  write_json(dir + "/golden.json", g);
  return 0;
}

// CRC-32 (IEEE, as zlib.crc32) of a byte string: digests of strings too large
// to commit (canonical forms of full-size outputs, packed IR images).
uint32_t crc32_of(const std::string &s) {
  static uint32_t tab[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; i++) {
      uint32_t c = i;
      for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      tab[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (unsigned char ch : s) c = tab[(c ^ ch) & 0xff] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}
ojson digest_j(const std::string &s) {
  char h[16];
  snprintf(h, sizeof h, "%08x", crc32_of(s));
  return ojson{{"crc32", h}, {"len", s.size()}};
}
std::string ir_image(const veq::HostBatch &b) {
  char *buf = nullptr;
  size_t n = 0;
  FILE *f = open_memstream(&buf, &n);
  b.write(f);
  fclose(f);
  std::string s(buf, n);
  free(buf);
  return s;
}

// Digest golden for full-size workloads: the reference's report (one
// check_equivalence, VCs decided on all host threads) with long strings
// replaced by CRC-32 digests, per-output digests of to_string of both
// kernels' canonical outputs (env_a / env_b), full strings of a few sample
// outputs, and digests of the reference's packed-IR elaboration.
int cmd_digest(const std::string &dir, const std::string &pa_path, const std::string &pb_path,
               const std::string &cfg_path) {
  LaunchConfig cfg = parse_config(read_file(cfg_path));
  CheckRequest req;
  req.kernel_a_src = read_file(pa_path);
  req.kernel_b_src = read_file(pb_path);
  req.cfg = cfg;
  ojson g;
  {
    Program pa = elaborate(parse_kernel(req.kernel_a_src), cfg, cfg.for_a());
    Program pb = elaborate(parse_kernel(req.kernel_b_src), cfg, cfg.for_b());
    std::vector<std::string> order;
    std::map<std::string, uint64_t> sizes;
    for (const auto &name : cfg.inputs)
      for (const auto &a : pa.arrays)
        if (a.name == name && !sizes.count(name)) {
          order.push_back(name);
          sizes[name] = a.size;
        }
    g["inputs"] = inputs_j(order, sizes);
    g["ir_a"] = digest_j(ir_image(to_ir(pa, sizes, order)));
    g["ir_b"] = digest_j(ir_image(to_ir(pb, sizes, order)));
  }
  const unsigned jobs = std::max(1u, std::thread::hardware_concurrency());
  auto t0 = std::chrono::steady_clock::now();
  Report rep = check_equivalence(req, jobs);
  g["ref_seconds"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  g["ref_jobs"] = jobs;
  ojson rj = report_to_json(rep);
  rj.erase("timings");
  for (auto &sc : rj["side_conditions"]) {
    const std::string d = sc["denominator"].get<std::string>();
    sc["denominator_digest"] = digest_j(d);
    if (d.size() > 2048) sc.erase("denominator");
  }
  g["report"] = rj;
  for (auto side : {std::make_pair("env_a", &rep.env_a), std::make_pair("env_b", &rep.env_b)}) {
    ojson e = ojson::array();
    for (const EnvEntry &x : *side.second) {
      const std::string str = to_string(x.value);
      ojson v{{"array", x.array}, {"index", x.index}};
      v["digest"] = digest_j(str);
      if (&x == &side.second->front() || &x == &side.second->back())
        if (str.size() <= 65536) v["text"] = str;
      e.push_back(v);
    }
    g[side.first] = e;
  }
  write_json(dir + "/golden.json", g);
  return 0;
}

int cmd_gen(const std::string &dir, uint64_t seed) {
  auto gp = testutil::gen_program(seed);
  std::vector<std::string> order;
  std::map<std::string, uint64_t> sizes;
  for (const auto &a : gp.prog.arrays) {
    order.push_back(a.name);
    sizes[a.name] = a.size;
  }
  ojson g;
  g["inputs"] = inputs_j(order, sizes);
  to_ir(gp.prog, sizes, order).save(dir + "/a.veqir");
  RunResult r = run(gp.prog, gp.inputs, SchedulePolicy::round_robin());
  g["run_a"] = run_j(r);
  write_json(dir + "/golden.json", g);
  return 0;
}

// CPU baseline: per CTA pair, time run(A)+run(B)+eq over all Out cells.
int cmd_bench(const std::string &pa_path, const std::string &pb_path, const std::string &list_path,
              unsigned threads, double seconds) {
  std::string sa = read_file(pa_path), sb = read_file(pb_path);
  KernelAst ka = parse_kernel(sa), kb = parse_kernel(sb);
  // CFGLIST lines: "cfg_path" or "cfg_path<TAB>b_kernel_path" (a batch of
  // candidate kernels against one reference kernel A, config C5)
  std::vector<std::string> cfgs;
  std::vector<std::shared_ptr<KernelAst>> kbs;
  {
    std::ifstream in(list_path);
    std::string line;
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      const size_t tab = line.find('\t');
      cfgs.push_back(read_file(line.substr(0, tab)));
      kbs.push_back(tab == std::string::npos ? nullptr
                                             : std::make_shared<KernelAst>(parse_kernel(read_file(line.substr(tab + 1)))));
    }
  }
  struct Job {
    Program pa, pb;
    SharedMem init;
    uint64_t n_out = 0;
  };
  // Parse, elaboration and make_symbolic_inputs are the reference's t_parse
  // and setup (pipeline.cpp:147-180) and are excluded from the metric; they
  // run per job inside the worker, outside the timed span, so memory stays
  // bounded by the thread count.
  std::atomic<size_t> cursor{0};
  std::atomic<uint64_t> done_elems{0}, done_pairs{0}, equal{0};
  std::mutex mu;
  double busy = 0, t_parse = 0;
  auto t0 = std::chrono::steady_clock::now();
  auto worker = [&]() {
    double my = 0, my_parse = 0;
    for (;;) {
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > seconds) break;
      size_t i = cursor++;
      if (i >= cfgs.size()) break;
      auto p0 = std::chrono::steady_clock::now();
      Job j;
      {
        LaunchConfig c = parse_config(cfgs[i]);
        j.pa = elaborate(ka, c, c.for_a());
        j.pb = elaborate(kbs[i] ? *kbs[i] : kb, c, c.for_b());
        j.init = make_symbolic_inputs(c, j.pa.arrays);
        for (auto &a : j.pa.arrays)
          if (a.role == Role::Out) j.n_out += a.size;
      }
      auto s0 = std::chrono::steady_clock::now();
      my_parse += std::chrono::duration<double>(s0 - p0).count();
      RunResult ra = run(j.pa, j.init, SchedulePolicy::round_robin());
      RunResult rb = run(j.pb, j.init, SchedulePolicy::round_robin());
      uint64_t eqn = 0;
      if (ra.outcome.kind == Outcome::Kind::Final && rb.outcome.kind == Outcome::Kind::Final)
        for (auto &a : j.pa.arrays)
          if (a.role == Role::Out)
            for (uint64_t k = 0; k < a.size; k++) {
              Addr ad{a.name, (int64_t)k};
              auto ia = ra.outcome.shared.find(ad), ib = rb.outcome.shared.find(ad);
              if (ia == ra.outcome.shared.end() || ib == rb.outcome.shared.end()) continue;
              Verdict v = eq(ia->second, ib->second, DecideBudget{}, 0, 64);
              if (v.kind == VerdictKind::Equal) eqn++;
            }
      clear_canon_cache();
      my += std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
      done_elems += j.n_out;
      done_pairs++;
      equal += eqn;
    }
    std::lock_guard<std::mutex> g(mu);
    busy += my;
    t_parse += my_parse;
  };
  std::vector<std::thread> th;
  for (unsigned t = 0; t < threads; t++) th.emplace_back(worker);
  for (auto &x : th) x.join();
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ojson o;
  o["pairs"] = done_pairs.load();
  o["pairs_total"] = cfgs.size();
  o["elements"] = done_elems.load();
  o["equal"] = equal.load();
  o["wall_s"] = wall;
  o["busy_s"] = busy;  // summed over threads: exec + decide only
  o["threads"] = threads;
  o["t_parse_s"] = t_parse;
  // throughput of the timed span with all threads busy on it
  o["elements_per_s"] = busy > 0 ? done_elems.load() / (busy / threads) : 0.0;
  std::cout << o.dump() << std::endl;
  return 0;
}

} // namespace

// parse_config of one config file, printed in veqh_parse_config's format
// (or the exception text): pins the product config reader.
int cmd_config(const char *path) {
  std::ifstream f(path);
  std::stringstream ss;
  ss << f.rdbuf();
  try {
    LaunchConfig c = parse_config(ss.str());
    std::cout << "threads=" << c.threads << "\nthreads_a=" << c.threads_a << "\nthreads_b=" << c.threads_b
              << "\nwarp_size=" << c.warp_size;
    for (auto &[k, v] : c.params) std::cout << "\nparams." << k << "=" << v;
    auto join = [](const std::vector<std::string> &v) {
      std::string r;
      for (size_t i = 0; i < v.size(); i++) r += (i ? "," : "") + v[i];
      return r;
    };
    std::cout << "\ninputs=" << join(c.inputs) << "\noutputs=" << join(c.outputs) << "\n";
    return 0;
  } catch (const std::exception &e) {
    std::cout << e.what();
    return 3;
  }
}

int main(int argc, char **argv) {
  try {
    std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "config" && argc == 3) return cmd_config(argv[2]);
    if (cmd == "pair" && argc == 6) return cmd_pair(argv[2], argv[3], argv[4], argv[5]);
    if (cmd == "digest" && argc == 6) return cmd_digest(argv[2], argv[3], argv[4], argv[5]);
    if (cmd == "gen" && argc == 4) return cmd_gen(argv[2], std::stoull(argv[3]));
    if (cmd == "bench" && argc == 7)
      return cmd_bench(argv[2], argv[3], argv[4], (unsigned)std::stoul(argv[5]), std::stod(argv[6]));
    std::cerr << "usage: ref_harness pair OUTDIR A.mk B.mk CFG | gen OUTDIR SEED | "
                 "bench A.mk B.mk CFGLIST THREADS SECONDS\n";
    return 4;
  } catch (const std::exception &e) {
    std::cerr << "ref_harness: " << e.what() << "\n";
    return 4;
  }
}
