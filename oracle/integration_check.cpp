// integration_check.cpp — TEST INFRASTRUCTURE (oracle/): the C++ binding a
// maintainer adds to the reference checker, compiled and
// run. It links the reference's own objects (oracle/_ref/obj, built from
// /root/reference/proj/src) and the product's C-ABI library (libveq.so) and
// re-states check_equivalence (proj/src/pipeline.cpp:141-267) with the two
// hot calls swapped in:
//   run()  (pipeline.cpp:183, 199)  -> veq_load_batch + veq_run +
//          veq_run_report + veq_fetch_cells / veq_export_dag (gpu_run below)
//   eq()   (pipeline.cpp:227)       -> veq_compare's canonical fast path;
//          a VC whose canonical forms differ goes to the reference's own
//          eq() on the imported forms (the host verdict API stays host code)
// For every manifest pair (proj/kernels/manifest.txt) it prints the product
// report and the reference report (report_to_json minus timings) and exits
// non-zero on any difference.
//   usage: integration_check KERNELS_DIR [pair-index ...]
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "ctaeq/decide.hpp"
#include "ctaeq/expr.hpp"
#include "ctaeq/frontend.hpp"
#include "ctaeq/ir.hpp"
#include "ctaeq/pipeline.hpp"
#include "ctaeq/symexec.hpp"
#include "ref_pack.hpp"
#include "veq.h"

using namespace ctaeq;

namespace {

std::string read_file(const std::string &p) {
  std::ifstream in(p, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + p);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void check(veq_ctx *ctx, int st, const char *what) {
  if (st != VEQ_OK)
    throw std::runtime_error(std::string(what) + ": " + veq_strerror(st) + ": " + veq_last_error(ctx));
}

// ---- import: device DAG -> reference Expr (smart constructors applied to
// already-canonical kids reproduce the exact canonical structure)
std::vector<Expr> import_exprs(veq_ctx *ctx, const std::vector<uint32_t> &roots,
                               const std::vector<std::string> &input_names) {
  if (roots.empty()) return {};
  veq_dag_buf buf{};
  check(ctx, veq_export_dag(ctx, roots.data(), roots.size(), &buf), "veq_export_dag");
  std::vector<veq_dag_node> nodes(buf.n_nodes);
  std::vector<uint32_t> kids(buf.n_kids), ridx(roots.size());
  buf.cap_nodes = buf.n_nodes;
  buf.cap_kids = buf.n_kids;
  buf.nodes = nodes.data();
  buf.kids = kids.data();
  buf.root_index = ridx.data();
  check(ctx, veq_export_dag(ctx, roots.data(), roots.size(), &buf), "veq_export_dag");
  std::vector<Expr> ex(nodes.size());
  for (size_t i = 0; i < nodes.size(); i++) {  // post-order: kids first
    const veq_dag_node &n = nodes[i];
    std::vector<Expr> k;
    for (uint32_t j = 0; j < n.nkids; j++) k.push_back(ex[kids[n.kid_off + j]]);
    switch (n.kind) {
    case VEQ_K_CONST:
      if (n.den == 0) {
        std::cerr << "import: Const with zero denominator at dag node " << i << " of " << nodes.size() << " (roots";
        for (uint32_t r : roots) std::cerr << " " << r;
        std::cerr << ")\n";
        throw std::runtime_error("bad Const");
      }
      ex[i] = cst(Rat(mpz_class((long)n.num), mpz_class((long)n.den)));
      break;
    case VEQ_K_NEGINF: ex[i] = neg_inf(); break;
    case VEQ_K_VAR:
      ex[i] = var(n.var_input >= 0 ? input_names[n.var_input] + "_" + std::to_string(n.var_index)
                                    : "!undef<" + std::to_string(n.var_index) + ">");
      break;
    case VEQ_K_EXP: ex[i] = exp_e(k[0]); break;
    case VEQ_K_MAX: ex[i] = max_of(k); break;
    case VEQ_K_DIV: ex[i] = div(k[0], k[1]); break;
    case VEQ_K_NEG: ex[i] = neg(k[0]); break;
    case VEQ_K_MUL: ex[i] = mul(k); break;
    case VEQ_K_ADD: ex[i] = add(k); break;
    default: throw std::runtime_error("bad node kind");
    }
  }
  std::vector<Expr> out;
  for (uint32_t r : ridx) out.push_back(ex[r]);
  return out;
}

// ---- gpu_run: one program on the device, rebuilt as the reference RunResult
struct Loaded {
  uint32_t batch;
  veq::HostBatch hb;
};

RunResult import_run(veq_ctx *ctx, const Loaded &L, const Program &p, const std::vector<std::string> &inputs) {
  RunResult rr;
  veq_report rep{};
  std::vector<uint64_t> locs;
  for (auto &l : L.hb.locs) locs.push_back(((uint64_t)l.line << 32) | l.col);
  check(ctx, veq_batch_locs(ctx, L.batch, locs.data()), "veq_batch_locs");
  check(ctx, veq_run_report(ctx, L.batch, 0, &rep), "veq_run_report");
  rr.steps = rep.steps;
  rr.releases = rep.releases;
  auto loc = [&](uint32_t s) { return SrcLoc{L.hb.locs[s].line, L.hb.locs[s].col}; };
  auto arr = [&](uint32_t a) { return L.hb.array_names[a]; };
  auto reg = [&](uint32_t tid, uint32_t r) {
    return L.hb.reg_names[L.hb.thread_reg_off[tid] + r];
  };
  const char *details[] = {"", "-inf is not a valid operand of Add", "-inf is not a valid operand of Mul",
                           "-inf is not a valid operand of Neg", "-inf is not a valid operand of Div",
                           "-inf is not a valid operand of Exp", "zero denominator"};
  for (uint64_t k = 0; k < rep.n_races; k++) {
    const veq_race_report &r = rep.races[k];
    RaceReport x;
    x.addr = Addr{arr(r.arr), r.offset};
    x.first = AccessRef{r.first.tid, r.first.is_write ? AccessKind::Write : AccessKind::Read, loc(r.first.stmt),
                        r.first.step};
    x.second = AccessRef{r.second.tid, r.second.is_write ? AccessKind::Write : AccessKind::Read, loc(r.second.stmt),
                         r.second.step};
    rr.races.push_back(x);
  }
  for (uint64_t k = 0; k < rep.n_safeties; k++) {
    const veq_safety_report &s = rep.safeties[k];
    SafetyReport x;
    x.kind = (SafetyKind)s.kind;
    x.tid = s.tid;
    x.loc = loc(s.stmt);
    x.step = s.step;
    if (s.has_addr) x.addr = Addr{arr(s.arr), s.offset};
    else x.reg = reg(s.tid, s.reg);
    x.is_store = s.is_store != 0;
    x.detail = details[s.detail];
    rr.safeties.push_back(x);
  }
  auto members = [&](uint32_t set) {
    uint32_t n = 0;
    check(ctx, veq_set_members(ctx, L.batch, 0, set, nullptr, 0, &n), "veq_set_members");
    std::vector<uint32_t> t(n);
    check(ctx, veq_set_members(ctx, L.batch, 0, set, t.data(), n, &n), "veq_set_members");
    TidSet ts;
    for (uint32_t x : t) ts.insert(x);
    return ts;
  };
  if (rep.deadlocked) {
    DeadlockReport d;
    for (uint32_t t = 0; t < rep.n_threads; t++) {
      ThreadStatusReport ts;
      ts.tid = t;
      ts.state = rep.threads[t].state == VEQ_TS_BLOCKED ? ThreadState::Blocked
                 : rep.threads[t].state == VEQ_TS_RETURNED ? ThreadState::Returned : ThreadState::Runnable;
      if (ts.state == ThreadState::Blocked) {
        ts.waiting = members(rep.threads[t].set);
        ts.loc = loc(rep.threads[t].stmt);
      }
      d.threads.push_back(ts);
    }
    if (rep.conflict_a >= 0) {
      d.conflict_tids = std::make_pair((Tid)rep.conflict_a, (Tid)rep.conflict_b);
      d.conflict_sets = std::make_pair(members(rep.conflict_set_a), members(rep.conflict_set_b));
    }
    rr.deadlock = d;
  }
  rr.outcome.kind = rep.outcome == VEQ_OUT_RACE ? Outcome::Kind::Race
                    : rep.outcome == VEQ_OUT_SAFETY ? Outcome::Kind::Safety
                    : rep.outcome == VEQ_OUT_DEADLOCK ? Outcome::Kind::Deadlock : Outcome::Kind::Final;
  if (rr.outcome.kind == Outcome::Kind::Final) {
    // final shared memory: every written cell (inputs keep their symbols)
    std::vector<uint32_t> roots;
    std::vector<Addr> addrs;
    for (size_t a = 0; a < p.arrays.size(); a++) {
      std::vector<uint32_t> cells(p.arrays[a].size);
      check(ctx, veq_fetch_cells(ctx, L.batch, 0, (uint32_t)a, cells.data(), cells.size()), "veq_fetch_cells");
      for (size_t i = 0; i < cells.size(); i++)
        if (cells[i] != 0xFFFFFFFFu) {
          roots.push_back(cells[i]);
          addrs.push_back(Addr{p.arrays[a].name, (int64_t)i});
        }
    }
    std::vector<Expr> ex = import_exprs(ctx, roots, inputs);
    for (size_t i = 0; i < ex.size(); i++) rr.outcome.shared[addrs[i]] = ex[i];
  }
  return rr;
}

std::vector<const ArrayDecl *> with_role(const Program &p, Role r) {
  std::vector<const ArrayDecl *> v;
  for (const auto &a : p.arrays)
    if (a.role == r) v.push_back(&a);
  std::sort(v.begin(), v.end(), [](auto *x, auto *y) { return x->name < y->name; });
  return v;
}

Report check_programs_gpu(veq_ctx *ctx, const Program &pa, const Program &pb, const std::vector<std::string> &order,
                          const std::map<std::string, uint64_t> &sizes, Report r);

// check_equivalence (proj/src/pipeline.cpp:141-267) with gpu_run and the
// device fast path of eq().
Report check_equivalence_gpu(veq_ctx *ctx, const CheckRequest &req) {
  Report r;
  r.kernel_a = req.kernel_a_name;
  r.kernel_b = req.kernel_b_name;
  Program pa, pb;
  try {
    pa = elaborate(parse_kernel(req.kernel_a_src), req.cfg, req.cfg.for_a());
    validate_structured(pa);
  } catch (const std::runtime_error &e) {
    r.verdict = ReportVerdict::KernelAError;
    r.error_kernel = "a";
    r.error_detail = e.what();
    return r;
  }
  try {
    pb = elaborate(parse_kernel(req.kernel_b_src), req.cfg, req.cfg.for_b());
    validate_structured(pb);
  } catch (const std::runtime_error &e) {
    r.verdict = ReportVerdict::KernelBError;
    r.error_kernel = "b";
    r.error_detail = e.what();
    return r;
  }
  for (Role role : {Role::In, Role::Out}) {  // signature_mismatch (pipeline.cpp:39-60)
    auto as = with_role(pa, role), bs = with_role(pb, role);
    std::string rs = role == Role::In ? "in" : "out", m;
    if (as.size() != bs.size()) m = "kernels declare a different number of " + rs + " arrays";
    for (size_t i = 0; m.empty() && i < as.size(); i++) {
      if (as[i]->name != bs[i]->name) m = rs + " array name mismatch: " + as[i]->name + " vs " + bs[i]->name;
      else if (as[i]->size != bs[i]->size)
        m = rs + " array " + as[i]->name + " size mismatch: " + std::to_string(as[i]->size) + " vs " +
            std::to_string(bs[i]->size);
    }
    if (!m.empty()) {
      r.verdict = ReportVerdict::KernelBError;
      r.error_kernel = "b";
      r.error_detail = m;
      return r;
    }
  }
  // the session's symbolic inputs (make_symbolic_inputs, pipeline.cpp:107-119)
  std::vector<std::string> order;
  std::map<std::string, uint64_t> sizes;
  for (const auto &name : req.cfg.inputs)
    for (const auto &a : pa.arrays)
      if (a.name == name && !sizes.count(name)) {
        order.push_back(name);
        sizes[name] = a.size;
      }
  return check_programs_gpu(ctx, pa, pb, order, sizes, r);
}

// Everything after elaboration and the signature check: both runs on the
// device, the VC compare on the device, the slow path and aggregation here.
Report check_programs_gpu(veq_ctx *ctx, const Program &pa, const Program &pb, const std::vector<std::string> &order,
                          const std::map<std::string, uint64_t> &sizes, Report r) {
  std::vector<veq_input_desc> in;
  for (auto &n : order) in.push_back(veq_input_desc{n.c_str(), sizes.at(n)});
  check(ctx, veq_declare_inputs(ctx, in.data(), (uint32_t)in.size()), "veq_declare_inputs");
  Loaded La{0, refpack::to_ir(pa, sizes, order)}, Lb{0, refpack::to_ir(pb, sizes, order)};
  for (Loaded *L : {&La, &Lb}) {
    veq_batch_desc d = L->hb.desc();
    check(ctx, veq_load_batch(ctx, &d, &L->batch), "veq_load_batch");
    veq_run_out o{};
    check(ctx, veq_run(ctx, L->batch, &o), "veq_run");
  }
  auto harvest = [&](const RunResult &rr) {  // harvest_errors (pipeline.cpp:63-71)
    if (rr.outcome.kind == Outcome::Kind::Final && rr.races.empty() && rr.safeties.empty()) return false;
    r.races = rr.races;
    r.safeties = rr.safeties;
    r.deadlock = rr.deadlock;
    return true;
  };
  auto missing = [&](const Program &p, const RunResult &rr) -> bool {  // missing_output (pipeline.cpp:73-87)
    for (const ArrayDecl *a : with_role(p, Role::Out))
      for (uint64_t i = 0; i < a->size; i++) {
        Addr ad{a->name, (int64_t)i};
        if (!rr.outcome.shared.count(ad)) {
          SafetyReport s;
          s.kind = SafetyKind::UninitMemoryRead;
          s.addr = ad;
          s.detail = "output element never written";
          r.safeties.push_back(s);
          return true;
        }
      }
    return false;
  };
  RunResult ra = import_run(ctx, La, pa, order);
  if (harvest(ra) || missing(pa, ra)) {
    r.verdict = ReportVerdict::KernelAError;
    r.error_kernel = "a";
    return r;
  }
  r.env_a = output_env(ra.outcome.shared, pa.arrays);
  RunResult rb = import_run(ctx, Lb, pb, order);
  if (harvest(rb) || missing(pb, rb)) {
    r.verdict = ReportVerdict::KernelBError;
    r.error_kernel = "b";
    return r;
  }
  r.env_b = output_env(rb.outcome.shared, pb.arrays);
  // VCs: the device compare (canonical fast path + side conditions)
  std::vector<uint32_t> oa, ob;
  for (const ArrayDecl *a : with_role(pa, Role::Out)) {
    for (size_t k = 0; k < pa.arrays.size(); k++)
      if (&pa.arrays[k] == a) oa.push_back((uint32_t)k);
    for (size_t k = 0; k < pb.arrays.size(); k++)
      if (pb.arrays[k].name == a->name) ob.push_back((uint32_t)k);
  }
  veq_vc_out vc{};
  check(ctx, veq_compare(ctx, La.batch, Lb.batch, oa.data(), ob.data(), (uint32_t)oa.size(), &vc), "veq_compare");
  std::vector<uint32_t> sc_nodes(vc.sc_node, vc.sc_node + vc.n_sc);
  std::vector<uint8_t> sc_dis(vc.sc_discharged, vc.sc_discharged + vc.n_sc);
  std::vector<veq_vc> vcs(vc.vcs, vc.vcs + vc.n_vcs);
  std::vector<Expr> sc_ex = import_exprs(ctx, sc_nodes, order);
  size_t v = 0;
  for (const ArrayDecl *a : with_role(pa, Role::Out))
    for (uint64_t i = 0; i < a->size; i++, v++) {
      Addr ad{a->name, (int64_t)i};
      VcResult res{a->name, i, Verdict{}};
      if (vcs[v].equal) {
        res.verdict.kind = VerdictKind::Equal;
        for (uint32_t q = vcs[v].sc_off; q < vcs[v].sc_off + vcs[v].sc_n; q++)
          res.verdict.side_conditions.push_back(SideCondition{sc_ex[q], sc_dis[q] != 0});
      } else {
        // canonically different: the host verdict API (slow path) decides
        const std::string key = a->name + "[" + std::to_string(i) + "]";
        uint64_t seed = 1469598103934665603ull;  // fnv1a as pipeline.cpp:18-25 seeds it
        for (unsigned char c : key) {
          seed ^= c;
          seed *= 1099511628211ull;
        }
        res.verdict = eq(ra.outcome.shared.at(ad), rb.outcome.shared.at(ad), DecideBudget{}, seed, 64);
      }
      r.vcs.push_back(res);
    }
  // aggregation (pipeline.cpp:245-266)
  std::set<std::string> seen;
  bool any_ne = false, any_unknown = false, residual = false;
  for (const VcResult &vr : r.vcs) {
    for (const SideCondition &sc : vr.verdict.side_conditions)
      if (seen.insert(to_string(sc.denominator)).second) {
        r.side_conditions.push_back(sc);
        if (!sc.discharged) residual = true;
      }
    any_ne |= vr.verdict.kind == VerdictKind::NotEqual;
    any_unknown |= vr.verdict.kind == VerdictKind::Unknown;
  }
  r.verdict = any_ne ? ReportVerdict::NotEquivalent
                     : (any_unknown || residual) ? ReportVerdict::Unknown : ReportVerdict::Equivalent;
  return r;
}

// Golden mode (GPU box, no /root/reference there): each fixture directory
// holds the reference's own elaboration (a.veqir, b.veqir, with register
// names and locations) and its report (golden.json, made by
// oracle/_ref/ref_harness pair); the programs are rebuilt from the packed IR
// and checked through the C-ABI; the report must equal the reference's.
int golden_main(int n, char **dirs) {
  veq_ctx *ctx = nullptr;
  veq_limits lim{1u << 22, 1u << 24, 1ull << 30};
  int st = veq_open(0, &lim, &ctx);
  if (st != VEQ_OK) {
    std::cerr << "veq_open: " << veq_strerror(st) << "\n";
    return 3;
  }
  int diffs = 0, done = 0;
  for (int i = 0; i < n; i++) {
    const std::string d = dirs[i];
    auto g = nlohmann::ordered_json::parse(read_file(d + "/golden.json"));
    if (g.contains("elab_error")) continue;  // rejected before the hot path
    auto want = g["report"];
    if (want.contains("error") && !want.contains("race") && !want.contains("safety") && !want.contains("deadlock"))
      continue;  // parse / structural / signature errors: host frontend only
    veq::HostBatch ha = veq::HostBatch::load(d + "/a.veqir"), hb = veq::HostBatch::load(d + "/b.veqir");
    Program pa = refpack::from_ir(ha), pb = refpack::from_ir(hb);
    std::vector<std::string> order;
    std::map<std::string, uint64_t> sizes;
    for (auto &x : g["inputs"]) {
      order.push_back(x["name"].get<std::string>());
      sizes[order.back()] = x["size"].get<uint64_t>();
    }
    Report r;
    r.kernel_a = want["kernels"]["a"].get<std::string>();
    r.kernel_b = want["kernels"]["b"].get<std::string>();
    Report got = check_programs_gpu(ctx, pa, pb, order, sizes, r);
    auto j = report_to_json(got);
    j.erase("timings");
    const bool same = j.dump() == want.dump();
    std::cout << (same ? "MATCH " : "DIFF  ") << d << " -> " << report_verdict_str(got.verdict) << "\n";
    if (!same) {
      diffs++;
      std::cout << "  ref: " << want.dump().substr(0, 1500) << "\n  gpu: " << j.dump().substr(0, 1500) << "\n";
    }
    done++;
    clear_canon_cache();
  }
  veq_close(ctx);
  std::cout << (diffs ? "FAILED " : "OK ") << done << " checked, " << diffs << " difference(s)\n";
  return diffs ? 1 : 0;
}

}  // namespace

void on_fault(int sig) {
  void *bt[64];
  const int n = backtrace(bt, 64);
  fprintf(stderr, "integration_check: signal %d\n", sig);
  backtrace_symbols_fd(bt, n, 2);
  _exit(128 + sig);
}

int main(int argc, char **argv) {
  signal(SIGFPE, on_fault);
  signal(SIGSEGV, on_fault);
  if (argc < 2) {
    std::cerr << "usage: integration_check KERNELS_DIR [pair-index ...]\n";
    return 2;
  }
  if (std::string(argv[1]) == "--golden") return golden_main(argc - 2, argv + 2);
  const std::string kd = argv[1];
  std::vector<std::vector<std::string>> rows;
  {
    std::istringstream ms(read_file(kd + "/manifest.txt"));
    std::string line;
    while (std::getline(ms, line)) {
      if (line.empty() || line[0] == '#') continue;
      std::istringstream ls(line);
      std::vector<std::string> f;
      std::string x;
      while (ls >> x) f.push_back(x);
      if (f.size() >= 4) rows.push_back(f);
    }
  }
  std::set<int> only;
  for (int i = 2; i < argc; i++) only.insert(std::stoi(argv[i]));
  veq_ctx *ctx = nullptr;
  veq_limits lim{1u << 22, 1u << 24, 1ull << 30};
  int st = veq_open(0, &lim, &ctx);
  if (st != VEQ_OK) {
    std::cerr << "veq_open: " << veq_strerror(st) << "\n";
    return 3;
  }
  int diffs = 0;
  for (size_t k = 0; k < rows.size(); k++) {
    if (!only.empty() && !only.count((int)k)) continue;
    CheckRequest req;
    req.kernel_a_src = read_file(kd + "/" + rows[k][0]);
    req.kernel_b_src = read_file(kd + "/" + rows[k][1]);
    req.cfg = parse_config(read_file(kd + "/" + rows[k][2]));
    Report ref = check_equivalence(req, 1);
    Report gpu = check_equivalence_gpu(ctx, req);
    auto strip = [](nlohmann::ordered_json j) {
      j.erase("timings");
      return j.dump();
    };
    const std::string a = strip(report_to_json(ref)), b = strip(report_to_json(gpu));
    const bool same = a == b && report_verdict_str(ref.verdict) == rows[k][3];
    std::cout << (same ? "MATCH " : "DIFF  ") << k << " " << rows[k][0] << " " << rows[k][1] << " " << rows[k][2]
              << " -> " << report_verdict_str(gpu.verdict) << " (manifest " << rows[k][3] << ")\n";
    if (!same) {
      diffs++;
      std::cout << "  ref: " << a.substr(0, 2000) << "\n  gpu: " << b.substr(0, 2000) << "\n";
    }
    clear_canon_cache();
  }
  veq_close(ctx);
  std::cout << (diffs ? "FAILED " : "OK ") << diffs << " difference(s)\n";
  return diffs ? 1 : 0;
}
