// decide.hpp — the slow path of the verdict API on a DAG exported from the
// device term table: the exp-polynomial zero test of a canonical difference
// (opaque-max pass) and the rigorous random witness search. Restates
// proj/src/decide.cpp:338-477 (rationalize, to_exp_poly), 686-718
// (refute_random), 728-859 (eq) and proj/src/interval.cpp (MPFR intervals,
// loaded at run time from libmpfr.so.6).
#pragma once
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace veqdec {

// A canonical DAG in post-order (kids before parents), the format of
// veq_export_dag.
struct DNode {
  uint8_t kind;  // veq.h VEQ_K_* (ctaeq::Kind order)
  std::vector<uint32_t> kids;
  int64_t num = 0, den = 1;  // Const
  std::string name;          // Var
};
struct Dag {
  std::vector<DNode> nodes;
};

enum class Kind { Equal, NotEqual, Unknown };
struct Result {
  Kind kind = Kind::Unknown;
  std::string reason;
  std::vector<std::pair<std::string, std::string>> assignment;  // witness, name order
  std::string f_enclosure, g_enclosure;
  unsigned precision = 0;
};

// Exp-polynomial zero test of node `d` of `dag` with every Max node an
// opaque atom (decide.cpp:740-745, 789-813). Returns true when the
// rationalized numerator vanishes identically; throws DecideError carrying
// the reference's reason text otherwise-undecidable shapes.
struct DecideError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
bool zero_by_exp_poly(const Dag &dag, uint32_t d, uint64_t max_monomials = 1000000);
bool contains_max(const Dag &dag, uint32_t d);

// refute_random (decide.cpp:686-718) on f and g; false when MPFR is
// unavailable or no separating point was found.
// want_witness false: only the outcome (and w.precision) is filled.
bool refute_random(const Dag &dag, uint32_t f, uint32_t g, uint64_t trials, uint64_t seed, Result &w,
                   bool want_witness = true);
bool mpfr_available();

}  // namespace veqdec
