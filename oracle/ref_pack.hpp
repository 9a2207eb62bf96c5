// ref_pack.hpp — TEST INFRASTRUCTURE (oracle/): packs a reference Program
// (proj/include/ctaeq/ir.hpp:148-156) into the product's packed IR
// (include/veq_ir.hpp). Used by the golden-dump harness and by the C++
// integration test of the C-ABI (integration_check.cpp). Only tests/ and
// the CPU-baseline leg of bench.py execute binaries built from oracle/.
#pragma once
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "ctaeq/ir.hpp"
#include "veq_ir.hpp"

namespace refpack {
using namespace ctaeq;

// ref Program -> packed IR (one program). `seeded` maps array name -> number
// of cells that carry input symbols (from the init SharedMem).
inline veq::HostBatch to_ir(const Program &p, const std::map<std::string, uint64_t> &seeded,
                     const std::vector<std::string> &input_order) {
  veq::HostBatch b;
  veq_program_meta m{};
  m.n_threads = p.n_threads;
  m.warp_size = p.warp_size;
  m.thread_off = 0;
  m.array_off = 0;
  m.n_arrays = (uint32_t)p.arrays.size();
  b.progs.push_back(m);
  b.prog_names.push_back(p.name);
  std::map<std::string, uint16_t> arr_idx;
  std::vector<bool> stored(p.arrays.size(), false);
  for (size_t i = 0; i < p.arrays.size(); i++) arr_idx[p.arrays[i].name] = (uint16_t)i;
  std::map<std::string, uint32_t> const_idx;
  std::map<std::string, uint32_t> set_idx;
  TidSet all = TidSet::full(p.n_threads);
  for (Tid t = 0; t < p.n_threads; t++) {
    std::map<std::string, uint32_t> regs;
    std::vector<std::string> names;
    auto reg = [&](const std::string &n) {
      auto it = regs.find(n);
      if (it != regs.end()) return it->second;
      uint32_t id = (uint32_t)names.size();
      regs[n] = id;
      names.push_back(n);
      return id;
    };
    for (const Stmt &s : p.threads[t].stmts) {
      veq_stmt o{};
      o.kind = (uint8_t)s.kind;
      switch (s.kind) {
      case StmtKind::SetConst: {
        o.dst = reg(s.set_const.dst);
        if (s.set_const.neg_infinity) {
          o.op = 1;
        } else {
          std::string key = s.set_const.value.get_str();
          auto it = const_idx.find(key);
          if (it == const_idx.end()) {
            Rat q = s.set_const.value;
            if (!mpz_fits_slong(q.get_num()) || !mpz_fits_slong(q.get_den()))
              throw std::runtime_error("constant out of int64 range");
            b.consts.push_back({q.get_num().get_si(), q.get_den().get_si()});
            it = const_idx.emplace(key, (uint32_t)b.consts.size() - 1).first;
          }
          o.a = it->second;
        }
        break;
      }
      case StmtKind::BinOp:
        o.op = (uint8_t)s.bin_op.op;
        o.a = reg(s.bin_op.a);
        o.b = reg(s.bin_op.b);
        o.dst = reg(s.bin_op.dst);
        break;
      case StmtKind::UnOp:
        o.op = (uint8_t)s.un_op.op;
        o.a = reg(s.un_op.a);
        o.dst = reg(s.un_op.dst);
        break;
      case StmtKind::Copy:
        o.a = reg(s.copy.src);
        o.dst = reg(s.copy.dst);
        break;
      case StmtKind::Load:
        o.arr = arr_idx.at(s.load.addr.array);
        if (s.load.addr.offset < INT32_MIN || s.load.addr.offset > INT32_MAX)
          throw std::runtime_error("offset out of int32 range");
        o.a = (uint32_t)(int32_t)s.load.addr.offset;
        o.dst = reg(s.load.dst);
        break;
      case StmtKind::Store:
        o.arr = arr_idx.at(s.store.addr.array);
        if (s.store.addr.offset < INT32_MIN || s.store.addr.offset > INT32_MAX)
          throw std::runtime_error("offset out of int32 range");
        o.a = (uint32_t)(int32_t)s.store.addr.offset;
        o.dst = reg(s.store.src);
        stored[o.arr] = true;
        break;
      case StmtKind::Sync: {
        std::string key = s.sync.set.str();
        auto it = set_idx.find(key);
        if (it == set_idx.end()) {
          veq_syncset q{};
          if (s.sync.set == all) {
            q.full = 1;
            q.lo = 0;
            q.n_bits = p.n_threads;
          } else {
            q.full = 0;
            q.lo = s.sync.set.min_tid();
            q.n_bits = s.sync.set.max_tid() - q.lo + 1;
            q.word_off = (uint32_t)b.set_words.size();
            std::vector<uint64_t> w((q.n_bits + 63) / 64, 0);
            for (Tid x : s.sync.set.to_vector()) w[(x - q.lo) / 64] |= 1ull << ((x - q.lo) % 64);
            b.set_words.insert(b.set_words.end(), w.begin(), w.end());
          }
          b.syncsets.push_back(q);
          it = set_idx.emplace(key, (uint32_t)b.syncsets.size() - 1).first;
        }
        o.a = it->second;
        break;
      }
      }
      b.stmts.push_back(o);
      b.locs.push_back({s.loc.line, s.loc.col});
    }
    b.thread_stmt.push_back(b.stmts.size());
    b.thread_nregs.push_back((uint32_t)names.size());
    b.reg_names.insert(b.reg_names.end(), names.begin(), names.end());
    b.thread_reg_off.push_back(b.reg_names.size());
  }
  for (size_t i = 0; i < p.arrays.size(); i++) {
    const ArrayDecl &a = p.arrays[i];
    veq_array o{};
    o.size = a.size;
    o.role = (uint32_t)a.role;
    o.flags = stored[i] ? VEQ_ARR_STORED : 0;
    o.input = -1;
    o.seeded = 0;
    for (size_t k = 0; k < input_order.size(); k++)
      if (input_order[k] == a.name) {
        o.input = (int32_t)k;
        o.seeded = (uint32_t)seeded.at(a.name);
      }
    b.arrays.push_back(o);
    b.array_names.push_back(a.name);
  }
  return b;
}


// Packed IR (one program of a batch) -> reference Program: the inverse of
// to_ir for batches elaborated with register names (the golden fixtures).
inline Program from_ir(const veq::HostBatch &b, uint32_t prog = 0) {
  const veq_program_meta &m = b.progs.at(prog);
  Program p;
  p.name = b.prog_names.at(prog);
  p.n_threads = m.n_threads;
  p.warp_size = m.warp_size;
  for (uint32_t a = 0; a < m.n_arrays; a++) {
    const veq_array &x = b.arrays[m.array_off + a];
    p.arrays.push_back(ArrayDecl{b.array_names[m.array_off + a], x.size, (Role)x.role});
  }
  auto set_of = [&](uint32_t s) {
    const veq_syncset &q = b.syncsets.at(s);
    if (q.full) return TidSet::full(m.n_threads);
    TidSet t;
    for (uint32_t k = 0; k < q.n_bits; k++)
      if ((b.set_words[q.word_off + k / 64] >> (k % 64)) & 1ull) t.insert(q.lo + k);
    return t;
  };
  for (uint32_t t = 0; t < m.n_threads; t++) {
    const uint32_t g = m.thread_off + t;
    const uint64_t r0 = b.thread_reg_off.at(g), r1 = b.thread_reg_off.at(g + 1);
    auto reg = [&](uint32_t r) {
      if (r0 + r >= r1) throw std::runtime_error("from_ir: batch has no register names");
      return b.reg_names[r0 + r];
    };
    ThreadProg tp;
    for (uint64_t i = b.thread_stmt[g]; i < b.thread_stmt[g + 1]; i++) {
      const veq_stmt &s = b.stmts[i];
      const SrcLoc loc{b.locs[i].line, b.locs[i].col};
      const std::string an = s.kind == VEQ_ST_LOAD || s.kind == VEQ_ST_STORE ? p.arrays.at(s.arr).name : "";
      switch (s.kind) {
      case VEQ_ST_SETCONST:
        if (s.op == 1) tp.stmts.push_back(Stmt::mk_neg_inf(reg(s.dst), loc));
        else tp.stmts.push_back(Stmt::mk_const(reg(s.dst), Rat(mpz_class((long)b.consts[s.a].num),
                                                                mpz_class((long)b.consts[s.a].den)), loc));
        break;
      case VEQ_ST_BINOP: tp.stmts.push_back(Stmt::mk_bin(reg(s.dst), (Bin)s.op, reg(s.a), reg(s.b), loc)); break;
      case VEQ_ST_UNOP: tp.stmts.push_back(Stmt::mk_un(reg(s.dst), (Un)s.op, reg(s.a), loc)); break;
      case VEQ_ST_COPY: tp.stmts.push_back(Stmt::mk_copy(reg(s.dst), reg(s.a), loc)); break;
      case VEQ_ST_LOAD: tp.stmts.push_back(Stmt::mk_load(reg(s.dst), Addr{an, (int32_t)s.a}, loc)); break;
      case VEQ_ST_STORE: tp.stmts.push_back(Stmt::mk_store(Addr{an, (int32_t)s.a}, reg(s.dst), loc)); break;
      case VEQ_ST_SYNC: tp.stmts.push_back(Stmt::mk_sync(set_of(s.a), loc)); break;
      default: throw std::runtime_error("from_ir: bad statement kind");
      }
    }
    p.threads.push_back(std::move(tp));
  }
  return p;
}

}  // namespace refpack
