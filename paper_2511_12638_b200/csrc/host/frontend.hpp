// frontend.hpp — kernel-language frontend and packed-IR elaborator (host).
//
// Drop-in for the reference frontend (proj/include/ctaeq/frontend.hpp,
// proj/src/frontend.cpp): same lexer, grammar, launch-config format, error
// messages and per-thread full unrolling, but it emits packed IR
// (veq::HostBatch) directly instead of per-thread vectors of string-keyed
// Stmt objects, and it elaborates the blocks of a grid in parallel.
#pragma once
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/veq_ir.hpp"

namespace veqh {

struct SrcLoc {
  uint32_t line = 0, col = 0;
  std::string str() const { return line == 0 ? "<synthetic>" : std::to_string(line) + ":" + std::to_string(col); }
};

// ParseError / StructuredCtaError of the reference (frontend.hpp:19-23,
// ir.hpp:27-29): what() carries the same text.
struct ParseError : std::runtime_error {
  SrcLoc loc;
  ParseError(SrcLoc l, const std::string &m) : std::runtime_error(l.str() + ": " + m), loc(l) {}
};
struct StructuredCtaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Template elaboration only: the kernel's control or data does not depend on
// the block parameter through array offsets alone (see elaborate_template).
struct TemplateUnsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct LaunchConfig {
  uint32_t threads = 0, threads_a = 0, threads_b = 0, warp_size = 32;
  std::map<std::string, int64_t> params;
  std::vector<std::string> inputs, outputs;
  uint32_t for_a() const { return threads_a ? threads_a : threads; }
  uint32_t for_b() const { return threads_b ? threads_b : threads; }
};

LaunchConfig parse_config(const std::string &text);

struct Kernel;  // parsed AST (opaque)
struct KernelDeleter {
  void operator()(Kernel *) const;
};

// Parsed kernel, reusable across elaborations.
struct ParsedKernel {
  Kernel *k = nullptr;
  explicit ParsedKernel(const std::string &src);
  ~ParsedKernel();
  ParsedKernel(const ParsedKernel &) = delete;
  ParsedKernel &operator=(const ParsedKernel &) = delete;
  const std::string &name() const;
};

// Input symbols of a pair (make_symbolic_inputs, pipeline.cpp:107-119):
// for each config input that names one of kernel A's arrays, that array's
// name and A's size.
struct InputDecl {
  std::string name;
  uint64_t size;
};

// Elaborates one CTA program into a one-program batch. `inputs` marks which
// arrays are seeded (and how many cells). want_names=false skips per-thread
// register name strings (reports then name registers r<id>).
veq::HostBatch elaborate(const ParsedKernel &k, const LaunchConfig &cfg, uint32_t n_threads,
                         const std::vector<InputDecl> &inputs, bool want_names = true);

// Elaborates ONE program for a whole grid: params.<block_param> is symbolic
// over blocks [block_lo, block_lo + n_blocks). The result is block-
// independent except for array offsets; CTA b is the template with every
// Load/Store offset on array a shifted by deltas[(b - block_lo) * n_arrays + a].
// Throws TemplateUnsupported when that does not hold (branches, bounds,
// constants or sync sets depending on the block, non-uniform shifts); the
// caller then elaborates per CTA. Errors the concrete elaboration raises for
// every CTA are raised as they would be there.
veq::HostBatch elaborate_template(const ParsedKernel &k, const LaunchConfig &cfg, uint32_t n_threads,
                                  const std::vector<InputDecl> &inputs, bool want_names,
                                  const std::string &block_param, int64_t block_lo, uint32_t n_blocks,
                                  std::vector<int32_t> &deltas);

// Inputs of a pair given kernel A's elaboration (array names/sizes).
std::vector<InputDecl> pair_inputs(const ParsedKernel &ka, const LaunchConfig &cfg);

}  // namespace veqh
