// veq_ir.hpp — host-side owner of a packed IR batch (header-only C++17).
//
// A HostBatch holds everything veq_batch_desc points at plus the host-only
// report metadata the device never needs: program/array names, per-thread
// register names, and per-statement source locations (ctaeq::SrcLoc,
// proj/include/ctaeq/ir.hpp:21-25). It serialises to a flat binary file
// ("VEQIR02") so batches can be produced by one tool and consumed by another.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "veq.h"

namespace veq {

struct Loc {
  uint32_t line = 0, col = 0;
};

struct HostBatch {
  // device-visible
  std::vector<veq_program_meta> progs;
  std::vector<uint64_t> thread_stmt{0};
  std::vector<uint32_t> thread_nregs;
  std::vector<veq_stmt> stmts;
  std::vector<veq_array> arrays;
  std::vector<veq_rat> consts;
  std::vector<veq_syncset> syncsets;
  std::vector<uint64_t> set_words;
  // host-only
  std::vector<std::string> prog_names;
  std::vector<std::string> array_names;        // parallel to arrays
  std::vector<uint64_t> thread_reg_off{0};     // [T+1] into reg_names
  std::vector<std::string> reg_names;          // per-thread register names
  std::vector<Loc> locs;                       // parallel to stmts

  uint32_t n_threads_total() const { return (uint32_t)thread_nregs.size(); }

  veq_batch_desc desc() const {
    veq_batch_desc d{};
    d.n_progs = (uint32_t)progs.size();
    d.n_threads_total = n_threads_total();
    d.n_stmts = stmts.size();
    d.n_arrays_total = (uint32_t)arrays.size();
    d.n_consts = (uint32_t)consts.size();
    d.n_syncsets = (uint32_t)syncsets.size();
    d.n_set_words = (uint32_t)set_words.size();
    d.progs = progs.data();
    d.thread_stmt = thread_stmt.data();
    d.thread_nregs = thread_nregs.data();
    d.stmts = stmts.data();
    d.arrays = arrays.data();
    d.consts = consts.data();
    d.syncsets = syncsets.data();
    d.set_words = set_words.data();
    return d;
  }

  // thread index of a batch-global statement (binary search)
  uint32_t thread_of_stmt(uint64_t s) const {
    size_t lo = 0, hi = thread_nregs.size();
    while (hi - lo > 1) {
      size_t mid = (lo + hi) / 2;
      if (thread_stmt[mid] <= s) lo = mid; else hi = mid;
    }
    return (uint32_t)lo;
  }
  const std::string &reg_name(uint32_t thread, uint32_t reg) const {
    return reg_names.at(thread_reg_off.at(thread) + reg);
  }

  // ---- serialisation ---------------------------------------------------
  template <class T> static void wvec(FILE *f, const std::vector<T> &v) {
    uint64_t n = v.size();
    fwrite(&n, 8, 1, f);
    if (n) fwrite(v.data(), sizeof(T), n, f);
  }
  static void wstrs(FILE *f, const std::vector<std::string> &v) {
    uint64_t n = v.size();
    fwrite(&n, 8, 1, f);
    for (auto &s : v) {
      uint32_t l = (uint32_t)s.size();
      fwrite(&l, 4, 1, f);
      fwrite(s.data(), 1, l, f);
    }
  }
  template <class T> static void rvec(FILE *f, std::vector<T> &v) {
    uint64_t n = 0;
    if (fread(&n, 8, 1, f) != 1) throw std::runtime_error("veq ir: truncated");
    v.resize(n);
    if (n && fread(v.data(), sizeof(T), n, f) != n) throw std::runtime_error("veq ir: truncated");
  }
  static void rstrs(FILE *f, std::vector<std::string> &v) {
    uint64_t n = 0;
    if (fread(&n, 8, 1, f) != 1) throw std::runtime_error("veq ir: truncated");
    v.resize(n);
    for (auto &s : v) {
      uint32_t l = 0;
      if (fread(&l, 4, 1, f) != 1) throw std::runtime_error("veq ir: truncated");
      s.resize(l);
      if (l && fread(&s[0], 1, l, f) != l) throw std::runtime_error("veq ir: truncated");
    }
  }
  void save(const std::string &path) const {
    FILE *f = fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("veq ir: cannot write " + path);
    write(f);
    fclose(f);
  }
  void write(FILE *f) const {
    fwrite("VEQIR02", 1, 8, f);
    wvec(f, progs); wvec(f, thread_stmt); wvec(f, thread_nregs); wvec(f, stmts);
    wvec(f, arrays); wvec(f, consts); wvec(f, syncsets); wvec(f, set_words);
    wstrs(f, prog_names); wstrs(f, array_names); wvec(f, thread_reg_off);
    wstrs(f, reg_names); wvec(f, locs);
  }
  static HostBatch load(const std::string &path) {
    FILE *f = fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("veq ir: cannot read " + path);
    char magic[8];
    if (fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "VEQIR02", 8) != 0) {
      fclose(f);
      throw std::runtime_error("veq ir: bad magic in " + path);
    }
    HostBatch b;
    rvec(f, b.progs); rvec(f, b.thread_stmt); rvec(f, b.thread_nregs); rvec(f, b.stmts);
    rvec(f, b.arrays); rvec(f, b.consts); rvec(f, b.syncsets); rvec(f, b.set_words);
    rstrs(f, b.prog_names); rstrs(f, b.array_names); rvec(f, b.thread_reg_off);
    rstrs(f, b.reg_names); rvec(f, b.locs);
    fclose(f);
    return b;
  }

  // Appends all programs of `o` (pools re-based).
  void append(const HostBatch &o) {
    uint32_t t0 = n_threads_total(), a0 = (uint32_t)arrays.size();
    uint32_t c0 = (uint32_t)consts.size(), q0 = (uint32_t)syncsets.size();
    uint32_t w0 = (uint32_t)set_words.size();
    uint64_t s0 = stmts.size(), r0 = reg_names.size();
    for (auto p : o.progs) {
      p.thread_off += t0;
      p.array_off += a0;
      progs.push_back(p);
    }
    for (size_t t = 0; t < o.thread_nregs.size(); t++) {
      thread_stmt.push_back(o.thread_stmt[t + 1] + s0);
      thread_nregs.push_back(o.thread_nregs[t]);
      thread_reg_off.push_back(o.thread_reg_off[t + 1] + r0);
    }
    for (auto s : o.stmts) {
      if (s.kind == VEQ_ST_SETCONST && s.op == 0) s.a += c0;
      if (s.kind == VEQ_ST_SYNC) s.a += q0;
      stmts.push_back(s);
    }
    arrays.insert(arrays.end(), o.arrays.begin(), o.arrays.end());
    consts.insert(consts.end(), o.consts.begin(), o.consts.end());
    for (auto q : o.syncsets) {
      q.word_off += w0;
      syncsets.push_back(q);
    }
    set_words.insert(set_words.end(), o.set_words.begin(), o.set_words.end());
    prog_names.insert(prog_names.end(), o.prog_names.begin(), o.prog_names.end());
    array_names.insert(array_names.end(), o.array_names.begin(), o.array_names.end());
    reg_names.insert(reg_names.end(), o.reg_names.begin(), o.reg_names.end());
    locs.insert(locs.end(), o.locs.begin(), o.locs.end());
  }
};

} // namespace veq
