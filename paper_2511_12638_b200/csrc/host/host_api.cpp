// host_api.cpp — C-ABI of libveq_host.so (include/veq_host.h).
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>

#include "../../../include/veq_host.h"
#include "frontend.hpp"

namespace {

void put_err(char *err, size_t n, const std::string &m) {
  if (!err || !n) return;
  size_t k = std::min(n - 1, m.size());
  std::memcpy(err, m.data(), k);
  err[k] = 0;
}

uint8_t *to_image(const veq::HostBatch &b, size_t *len) {
  char *buf = nullptr;
  size_t sz = 0;
  FILE *f = open_memstream(&buf, &sz);
  if (!f) throw std::runtime_error("open_memstream failed");
  b.write(f);
  fclose(f);
  *len = sz;
  return reinterpret_cast<uint8_t *>(buf);
}

}  // namespace

extern "C" int veqh_parse_config(const char *cfg_src, char *out, size_t outlen) {
  if (!cfg_src) return VEQH_E_ARG;
  try {
    const veqh::LaunchConfig c = veqh::parse_config(cfg_src);
    std::string s = "threads=" + std::to_string(c.threads) + "\nthreads_a=" + std::to_string(c.threads_a) +
                    "\nthreads_b=" + std::to_string(c.threads_b) + "\nwarp_size=" + std::to_string(c.warp_size);
    for (const auto &[k, v] : c.params) s += "\nparams." + k + "=" + std::to_string(v);
    auto join = [](const std::vector<std::string> &v) {
      std::string r;
      for (size_t i = 0; i < v.size(); i++) r += (i ? "," : "") + v[i];
      return r;
    };
    s += "\ninputs=" + join(c.inputs) + "\noutputs=" + join(c.outputs) + "\n";
    put_err(out, outlen, s);
    return VEQH_OK;
  } catch (const std::exception &e) {
    put_err(out, outlen, e.what());
    return VEQH_E_CONFIG;
  }
}

extern "C" int veqh_elaborate_grid(const char *kernel_a, const char *kernel_b, const char *cfg_src,
                                   const char *block_param, uint32_t block_base, uint32_t n_blocks,
                                   uint32_t n_workers, int want_names, veqh_pair *out, char *err, size_t errlen) {
  if (!kernel_a || !kernel_b || !cfg_src || !out || n_blocks == 0) return VEQH_E_ARG;
  std::memset(out, 0, sizeof(*out));
  veqh::LaunchConfig cfg;
  try {
    cfg = veqh::parse_config(cfg_src);
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_CONFIG;
  }
  std::unique_ptr<veqh::ParsedKernel> ka, kb;
  try {
    ka.reset(new veqh::ParsedKernel(kernel_a));
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_A;
  }
  try {
    kb.reset(new veqh::ParsedKernel(kernel_b));
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_B;
  }
  const bool grid = block_param && *block_param;
  auto cfg_for = [&](uint32_t blk) {
    veqh::LaunchConfig c = cfg;
    if (grid) c.params[block_param] = (int64_t)block_base + blk;
    return c;
  };
  std::vector<veqh::InputDecl> inputs;
  try {
    inputs = veqh::pair_inputs(*ka, cfg_for(0));
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_A;
  }
  std::vector<veq::HostBatch> A(n_blocks), B(n_blocks);
  std::vector<std::string> errs(n_blocks);
  std::vector<int> codes(n_blocks, 0);
  std::atomic<uint32_t> next{0};
  auto work = [&]() {
    for (uint32_t b; (b = next++) < n_blocks;) {
      veqh::LaunchConfig c = cfg_for(b);
      try {
        A[b] = veqh::elaborate(*ka, c, c.for_a(), inputs, want_names != 0);
      } catch (const std::exception &e) {
        errs[b] = e.what();
        codes[b] = VEQH_E_KERNEL_A;
        continue;
      }
      try {
        B[b] = veqh::elaborate(*kb, c, c.for_b(), inputs, want_names != 0);
      } catch (const std::exception &e) {
        errs[b] = e.what();
        codes[b] = VEQH_E_KERNEL_B;
      }
    }
  };
  uint32_t nw = std::max<uint32_t>(1, std::min<uint32_t>(n_workers ? n_workers : 1, n_blocks));
  std::vector<std::thread> th;
  for (uint32_t i = 1; i < nw; i++) th.emplace_back(work);
  work();
  for (auto &t : th) t.join();
  for (uint32_t b = 0; b < n_blocks; b++)
    if (codes[b]) {
      put_err(err, errlen, errs[b]);
      return codes[b];
    }
  veq::HostBatch ga, gb;
  for (uint32_t b = 0; b < n_blocks; b++) {
    ga.append(A[b]);
    gb.append(B[b]);
    A[b] = veq::HostBatch();
    B[b] = veq::HostBatch();
  }
  try {
    out->ir_a = to_image(ga, &out->ir_a_len);
    out->ir_b = to_image(gb, &out->ir_b_len);
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_ARG;
  }
  std::string in;
  for (auto &i : inputs) in += i.name + "\t" + std::to_string(i.size) + "\n";
  out->inputs = strdup(in.c_str());
  return VEQH_OK;
}

extern "C" void veqh_free(veqh_pair *p) {
  if (!p) return;
  free(p->ir_a);
  free(p->ir_b);
  free(p->inputs);
  std::memset(p, 0, sizeof(*p));
}

extern "C" int veqh_elaborate_template(const char *kernel_a, const char *kernel_b, const char *cfg_src,
                                       const char *block_param, int64_t block_base, uint32_t n_blocks,
                                       int want_names, veqh_template *out, char *err, size_t errlen) {
  if (!kernel_a || !kernel_b || !cfg_src || !out || !block_param || !*block_param || n_blocks == 0) return VEQH_E_ARG;
  std::memset(out, 0, sizeof(*out));
  veqh::LaunchConfig cfg;
  try {
    cfg = veqh::parse_config(cfg_src);
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_CONFIG;
  }
  std::unique_ptr<veqh::ParsedKernel> ka, kb;
  try {
    ka.reset(new veqh::ParsedKernel(kernel_a));
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_A;
  }
  try {
    kb.reset(new veqh::ParsedKernel(kernel_b));
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_B;
  }
  // the config as the first block sees it: inputs and sizes are block-free
  veqh::LaunchConfig c0 = cfg;
  c0.params[block_param] = block_base;
  std::vector<veqh::InputDecl> inputs;
  try {
    inputs = veqh::pair_inputs(*ka, c0);
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_KERNEL_A;
  }
  veq::HostBatch ta, tb;
  std::vector<int32_t> da, db;
  int side = VEQH_E_KERNEL_A;
  try {
    ta = veqh::elaborate_template(*ka, c0, c0.for_a(), inputs, want_names != 0, block_param, block_base, n_blocks, da);
    side = VEQH_E_KERNEL_B;
    tb = veqh::elaborate_template(*kb, c0, c0.for_b(), inputs, want_names != 0, block_param, block_base, n_blocks, db);
  } catch (const veqh::TemplateUnsupported &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_TEMPLATE;
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return side;
  }
  try {
    out->ir_a = to_image(ta, &out->ir_a_len);
    out->ir_b = to_image(tb, &out->ir_b_len);
  } catch (const std::exception &e) {
    put_err(err, errlen, e.what());
    return VEQH_E_ARG;
  }
  std::string in;
  for (auto &i : inputs) in += i.name + "\t" + std::to_string(i.size) + "\n";
  out->inputs = strdup(in.c_str());
  out->n_blocks = n_blocks;
  out->n_arrays_a = (uint32_t)ta.arrays.size();
  out->n_arrays_b = (uint32_t)tb.arrays.size();
  out->deltas_a = (int32_t *)malloc(std::max<size_t>(1, da.size()) * 4);
  out->deltas_b = (int32_t *)malloc(std::max<size_t>(1, db.size()) * 4);
  std::memcpy(out->deltas_a, da.data(), da.size() * 4);
  std::memcpy(out->deltas_b, db.data(), db.size() * 4);
  return VEQH_OK;
}

extern "C" void veqh_free_template(veqh_template *p) {
  if (!p) return;
  free(p->ir_a);
  free(p->ir_b);
  free(p->inputs);
  free(p->deltas_a);
  free(p->deltas_b);
  std::memset(p, 0, sizeof(*p));
}
