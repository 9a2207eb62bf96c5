// veq_api.cu — C-ABI implementation (include/veq.h): device memory,
// batch preparation and the launch sequence of one check.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <functional>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <string>
#include <vector>
#include <atomic>
#include <thread>

#include "veq_pipeline.cuh"
#include "host/decide.hpp"

// Open-addressing set of W-word keys (report identities in veq_run_report):
// sized once for the number of inserts, no per-key allocation.
template <int W> struct FlatSet {
  std::vector<std::array<uint64_t, W>> keys;
  std::vector<uint8_t> used;
  uint64_t mask = 0;
  void init(uint64_t n) {
    uint64_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    keys.assign(cap, {});
    used.assign(cap, 0);
    mask = cap - 1;
  }
  bool insert(const std::array<uint64_t, W> &k) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int i = 0; i < W; i++) {
      h = (h ^ k[i]) * 0xff51afd7ed558ccdull;
      h ^= h >> 32;
    }
    for (uint64_t j = h & mask;; j = (j + 1) & mask) {
      if (!used[j]) {
        used[j] = 1;
        keys[j] = k;
        return true;
      }
      if (keys[j] == k) return false;
    }
  }
};

using namespace veqd;

namespace {

const char *kErr[] = {"ok",
                      "term table or arena capacity exhausted",
                      "rational coefficient overflow (outside exact int64 range)",
                      "device out of memory",
                      "invalid IR",
                      "CUDA error",
                      "bad argument",
                      "unsupported input",
                      "no CUDA device",
                      "canonicalisation scratch exhausted"};

struct DevBuf {
  void *p = nullptr;
  size_t n = 0;
};

struct BatchDev {
  // host copies needed for reports / compare
  std::vector<veq_program_meta> progs;
  std::vector<veq_array> arrays;
  std::vector<uint64_t> arr_cell_base;
  std::vector<uint64_t> thread_stmt;
  uint64_t n_stmts = 0, n_cells = 0, n_segs = 0, n_rel_cap = 0, n_regs = 0, n_access_max = 0;
  uint64_t n_arith = 0;  // BinOp/UnOp statements: bound of the work list and chain logs
  unsigned long long *d_stats = nullptr;  // [0..7] table counters at run start, [8] work items
  bool started = false;                   // veq_run_start enqueued, veq_run_finish pending
  bool timing_run = false;                // phase events recorded by this run
  bool no_defer = false;                  // deferral off for this batch (set after an E_DEFER fallback)
  bool keep_regs = false;                 // this batch's runs keep final register files
  uint32_t run_launches = 0;
  unsigned long long n_work_last = 0;  // work items of the last run (read back with its results)
  uint32_t n_threads = 0;
  unsigned int sched_flags = 0;  // written by k_prep_syncs (valid after the load's final sync)
  // device arrays (owned)
  std::vector<void *> owned;
  veq_rat *dconsts = nullptr;
  uint32_t n_consts = 0;
  Batch B{};
  // host-visible run results
  std::vector<veq_prog_result> res;
  std::vector<veq_fault> faults;
  std::vector<uint64_t> prog_fault_off;   // faults sorted by (prog, step, sub): program p's are [off[p], off[p+1])
  std::vector<uint64_t> locs;             // optional per-statement location keys (veq_batch_locs)
  std::vector<veq_syncset> syncsets;      // host copies for reports (set membership)
  std::vector<uint64_t> set_words;
  // veq_run_report output of the last call
  // veq_run_report / veq_run_reports output (ctx-owned, per call)
  struct RepStore {
    std::vector<veq_race_report> races;
    std::vector<veq_safety_report> safeties;
    std::vector<veq_thread_report> threads;
  };
  RepStore rep;
  std::vector<RepStore> rep_many;
  std::vector<uint8_t> th_state;
  std::vector<uint32_t> th_bset;
  std::vector<uint64_t> th_bstmt;
  bool ran = false;
};

// A template batch (veq_load_template): small tables on the host, statements
// resident on the device; veq_instantiate expands it into regular batches.
struct TemplateDev {
  std::vector<veq_program_meta> progs;
  std::vector<uint64_t> thread_stmt;
  std::vector<uint32_t> thread_nregs;
  std::vector<veq_array> arrays;
  std::vector<veq_rat> consts;
  std::vector<veq_syncset> syncsets;
  std::vector<uint64_t> set_words;
  uint64_t n_stmts = 0;
  veq_stmt *stmts = nullptr;
};

}  // namespace

struct veq_ctx {
  int device = 0;
  // grow-only run workspace: one slot per veq_run/veq_compare temporary, so
  // steady-state runs make no allocation at all (cudaMalloc only when a
  // slot grows; runs on the ctx's single stream never overlap)
  std::vector<std::pair<void *, size_t>> ws;
  // all-returned thread states handed out by runs without a deadlock
  std::vector<uint8_t> ret_state;
  std::vector<uint32_t> unset_set;
  std::vector<uint64_t> unset_stmt;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // side stream: long-thread executor alongside the short-thread one
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string last_error;
  Table T{};
  veq_limits lim{};
  // term table storage
  Node *nodes = nullptr;
  uint32_t *kids = nullptr, *slots = nullptr;
  unsigned long long *counters = nullptr;
  int *error = nullptr;
  unsigned long long *dbg = nullptr;
  uint32_t *session_ids = nullptr;
  uint64_t *in_base = nullptr, *in_size = nullptr;
  uint32_t *in_cache = nullptr;
  uint64_t in_cache_n = 0, in_cells = 0;
  uint64_t n_slots = 0;
  // scratch pool
  char *pool = nullptr;
  unsigned long long *pool_used = nullptr;
  uint64_t pool_cap = 0;
  // session
  std::vector<std::string> input_names;
  std::vector<uint64_t> input_sizes;
  std::vector<BatchDev *> batches;    // dropped batches leave a null slot
  std::vector<TemplateDev *> templates;
  // compare outputs
  std::vector<veq_vc> vcs;
  std::vector<uint32_t> sc_node;
  std::vector<uint8_t> sc_dis;
  // deferred-scaling merge memo (EvalCtx::mkeys/mvals), grown per run
  unsigned long long *mkeys = nullptr;
  uint32_t *mvals = nullptr;
  uint64_t mslots = 0;
  bool keep_regs = false;  // VEQ_OPT_KEEP_REGS for runs started from now on
  // multi-GPU: NCCL communicator (veq_comm_init) and veq_comm_combine output
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  std::vector<uint8_t> all_verdict;
  std::vector<uint64_t> all_sc_hash;
  std::vector<uint8_t> all_sc_dis;
  std::vector<uint64_t> rank_vc_off, rank_sc_off;
  // host snapshot of the term table (append-only between clears): later
  // exports copy only what was created since the previous one
  std::vector<Node> hnodes;
  std::vector<uint32_t> hkids;
  // veq_decide output
  std::string dec_reason, dec_f, dec_g;
  std::vector<std::string> dec_names, dec_values;
  std::vector<const char *> dec_name_p, dec_value_p;
  // veq_render output
  std::string render_text;
  std::vector<uint64_t> render_offs;
  uint64_t last_equal = 0, last_missing = 0, last_vcs = 0, last_faults = 0;
  // instrumentation
  bool timing = false;
  cudaEvent_t ev0[VEQ_MAX_PHASES] = {}, ev1[VEQ_MAX_PHASES] = {};
  uint32_t launches = 0;
};

namespace {

int fail(veq_ctx *c, int code, const std::string &msg) {
  if (c) c->last_error = msg;
  return code;
}

bool live_batch(const veq_ctx *ctx, uint32_t b) { return b < ctx->batches.size() && ctx->batches[b] != nullptr; }

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) return fail(ctx, VEQ_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

int ws_get(veq_ctx *ctx, int slot, void **out, size_t bytes) {
  if ((int)ctx->ws.size() <= slot) ctx->ws.resize(slot + 1, {nullptr, 0});
  auto &w = ctx->ws[slot];
  bytes = std::max<size_t>(bytes, 256);
  if (w.second < bytes) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(w.first);
    w = {nullptr, 0};
    size_t cap = bytes + bytes / 8;
    if (cudaMalloc(&w.first, cap) != cudaSuccess) return fail(ctx, VEQ_E_OOM, "run workspace");
    w.second = cap;
  }
  *out = w.first;
  return VEQ_OK;
}

template <class X> int dalloc(veq_ctx *ctx, BatchDev *bd, X **out, size_t n) {
  void *p = nullptr;
  size_t bytes = std::max<size_t>(n, 1) * sizeof(X);
  cudaError_t e = cudaMallocAsync(&p, bytes, ctx->stream);
  if (e != cudaSuccess) return fail(ctx, VEQ_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (bd) bd->owned.push_back(p);
  *out = reinterpret_cast<X *>(p);
  return VEQ_OK;
}
template <class X> int dupload(veq_ctx *ctx, BatchDev *bd, X **out, const X *src, size_t n) {
  int r = dalloc(ctx, bd, out, n);
  if (r) return r;
  if (n) {
    cudaError_t e = cudaMemcpyAsync(*out, src, n * sizeof(X), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return fail(ctx, VEQ_E_CUDA, cudaGetErrorString(e));
  }
  return VEQ_OK;
}

uint32_t blocks(uint64_t n, uint32_t b) { return (uint32_t)((n + b - 1) / b); }

int check_error_flag(veq_ctx *ctx) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, ctx->error, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (h) {
    if (h == E_BUDGET) return fail(ctx, VEQ_E_BUDGET, "term table / arena capacity exhausted");
    if (h == E_OVERFLOW) return fail(ctx, VEQ_E_RATIONAL_OVERFLOW, "rational coefficient overflow");
    if (h == E_SCRATCH) {
      unsigned long long d[3] = {0, 0, 0};
      cudaMemcpy(d, ctx->dbg, sizeof(d), cudaMemcpyDeviceToHost);
      return fail(ctx, VEQ_E_SCRATCH, "canonicalisation scratch exhausted (request " + std::to_string(d[0]) +
                                          " B at pool offset " + std::to_string(d[1]) + ", item " +
                                          std::to_string(d[2]) + ", pool " + std::to_string(ctx->pool_cap) + " B)");
    }
    return fail(ctx, VEQ_E_INVALID_IR, "internal invariant violated on device (code " + std::to_string(h) + ")");
  }
  return VEQ_OK;
}

// NCCL is resolved at run time (dlopen of libnccl.so.2): a process that
// already loaded one (e.g. PyTorch's) shares it, and the library still loads
// on hosts without NCCL (veq_comm_* then report VEQ_E_UNSUPPORTED).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi &nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.GetErrorString;
    return a;
  }();
  return api;
}

}  // namespace

static void veq_comm_destroy_(veq_ctx *ctx) {
  if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
  ctx->comm = nullptr;
  ctx->nranks = 1;
  ctx->rank = 0;
}

#define NK(call)                                                                                      \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) return fail(ctx, VEQ_E_CUDA, std::string(#call ": ") + nccl().GetErrorString(r_)); \
  } while (0)

extern "C" {

const char *veq_strerror(int s) {
  if (s >= 0 && s < (int)(sizeof(kErr) / sizeof(kErr[0]))) return kErr[s];
  return "unknown status";
}

const char *veq_last_error(veq_ctx *ctx) { return ctx ? ctx->last_error.c_str() : "null ctx"; }

int veq_open(int device, const veq_limits *lim, veq_ctx **out) {
  if (!out) return VEQ_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return VEQ_E_NO_DEVICE;
  if (device < 0 || device >= ndev) return VEQ_E_ARG;
  veq_ctx *ctx = new veq_ctx();
  ctx->device = device;
  if (lim) ctx->lim = *lim;
  if (!ctx->lim.max_nodes) ctx->lim.max_nodes = 64ull << 20;
  if (!ctx->lim.max_kid_words) ctx->lim.max_kid_words = 256ull << 20;
  if (!ctx->lim.scratch_bytes) ctx->lim.scratch_bytes = 4ull << 30;
  if (ctx->lim.max_nodes >= (1ull << 31)) ctx->lim.max_nodes = (1ull << 31) - 1;
  // kid-arena offsets travel as u32 in the eval kernel's shared working sets
  if (ctx->lim.max_kid_words >= (1ull << 32)) ctx->lim.max_kid_words = (1ull << 32) - 1;
  auto bail = [&](int code, const char *what) {
    fprintf(stderr, "veq_open: %s\n", what);
    delete ctx;
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(VEQ_E_CUDA, "cudaSetDevice");
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(VEQ_E_CUDA, "stream");

  if (cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess)
    return bail(VEQ_E_CUDA, "side stream");
  {
    // keep freed stream-ordered allocations in the pool across syncs: the
    // per-run work buffers are re-allocated every run
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  uint64_t slots = 1;
  while (slots < ctx->lim.max_nodes * 2) slots <<= 1;
  ctx->n_slots = slots;
  if (cudaMalloc(&ctx->nodes, ctx->lim.max_nodes * sizeof(Node)) != cudaSuccess) return bail(VEQ_E_OOM, "nodes");
  if (cudaMalloc(&ctx->kids, ctx->lim.max_kid_words * sizeof(uint32_t)) != cudaSuccess) return bail(VEQ_E_OOM, "kids");
  if (cudaMalloc(&ctx->slots, slots * sizeof(uint32_t)) != cudaSuccess) return bail(VEQ_E_OOM, "slots");
  if (cudaMalloc(&ctx->counters, 8 * sizeof(unsigned long long)) != cudaSuccess) return bail(VEQ_E_OOM, "counters");
  if (cudaMalloc(&ctx->error, sizeof(int)) != cudaSuccess) return bail(VEQ_E_OOM, "error");
  if (cudaMalloc(&ctx->dbg, 4 * sizeof(unsigned long long)) != cudaSuccess) return bail(VEQ_E_OOM, "dbg");
  if (cudaMalloc(&ctx->session_ids, 4 * sizeof(uint32_t)) != cudaSuccess) return bail(VEQ_E_OOM, "ids");
  ctx->pool_cap = ctx->lim.scratch_bytes;
  if (cudaMalloc(&ctx->pool, ctx->pool_cap) != cudaSuccess) return bail(VEQ_E_OOM, "scratch pool");
  if (cudaMalloc(&ctx->pool_used, sizeof(unsigned long long)) != cudaSuccess) return bail(VEQ_E_OOM, "pool ctr");
  Table &T = ctx->T;
  T.nodes = ctx->nodes;
  T.kids = ctx->kids;
  T.slots = ctx->slots;
  T.counters = ctx->counters;
  T.max_nodes = ctx->lim.max_nodes;
  T.max_kids = ctx->lim.max_kid_words;
  T.slot_mask = slots - 1;
  T.error = ctx->error;
  T.dbg = ctx->dbg;
  *out = ctx;
  // an empty session so the ctx is usable without declared inputs
  return veq_declare_inputs(ctx, nullptr, 0);
}

void veq_close(veq_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (BatchDev *b : ctx->batches) {
    if (!b) continue;
    for (void *p : b->owned) cudaFreeAsync(p, ctx->stream);
    delete b;
  }
  for (TemplateDev *t : ctx->templates)
    if (t) {
      cudaFreeAsync(t->stmts, ctx->stream);
      delete t;
    }
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->nodes);
  cudaFree(ctx->kids);
  cudaFree(ctx->slots);
  cudaFree(ctx->counters);
  cudaFree(ctx->error);
  cudaFree(ctx->dbg);
  cudaFree(ctx->session_ids);
  cudaFree(ctx->pool);
  cudaFree(ctx->pool_used);
  cudaFree(ctx->mkeys);
  cudaFree(ctx->mvals);
  if (ctx->comm) veq_comm_destroy_(ctx);
  cudaFree(ctx->in_base);
  cudaFree(ctx->in_size);
  cudaFree(ctx->in_cache);
  for (auto &w : ctx->ws) cudaFree(w.first);
  cudaStreamDestroy(ctx->stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

int veq_declare_inputs(veq_ctx *ctx, const veq_input_desc *inputs, uint32_t n) {
  if (!ctx) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  // drop batches and templates of the previous session
  for (BatchDev *b : ctx->batches) {
    if (!b) continue;
    for (void *p : b->owned) cudaFreeAsync(p, ctx->stream);
    delete b;
  }
  ctx->batches.clear();
  for (TemplateDev *t : ctx->templates)
    if (t) {
      cudaFreeAsync(t->stmts, ctx->stream);
      delete t;
    }
  ctx->templates.clear();
  ctx->input_names.clear();
  ctx->input_sizes.clear();
  // Byte order of "<name>_<i>" symbols: groups "<name>_" in byte order, then
  // the decimal-string order inside a group (lexrank on the device). Exact
  // unless one group string is a proper prefix of another ("x_" / "x_1_").
  std::vector<std::string> g(n);
  for (uint32_t i = 0; i < n; i++) {
    if (!inputs[i].name) return fail(ctx, VEQ_E_ARG, "null input name");
    ctx->input_names.push_back(inputs[i].name);
    ctx->input_sizes.push_back(inputs[i].size);
    g[i] = std::string(inputs[i].name) + "_";
  }
  for (uint32_t i = 0; i < n; i++)
    for (uint32_t j = 0; j < n; j++)
      if (i != j && g[j].size() > g[i].size() && g[j].compare(0, g[i].size(), g[i]) == 0)
        return fail(ctx, VEQ_E_UNSUPPORTED, "input array names " + g[i] + " / " + g[j] + " interleave in byte order");
  std::vector<uint32_t> ord(n);
  for (uint32_t i = 0; i < n; i++) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return g[a] < g[b]; });
  std::vector<uint64_t> base(n ? n : 1, 0), size(n ? n : 1, 0);
  uint64_t acc = 0;
  for (uint32_t k = 0; k < n; k++) {
    base[ord[k]] = acc;
    acc += inputs[ord[k]].size;
  }
  for (uint32_t i = 0; i < n; i++) size[i] = inputs[i].size;
  if (acc >= (1ull << 43)) return fail(ctx, VEQ_E_UNSUPPORTED, "too many input symbols");
  cudaFree(ctx->in_base);
  cudaFree(ctx->in_size);
  // input-symbol cache (dense rank -> node id), kept across sessions when
  // large enough; inputs beyond 2^28 symbols go uncached
  ctx->in_cells = acc;
  if (acc <= (1ull << 28) && acc > ctx->in_cache_n) {
    cudaFree(ctx->in_cache);
    ctx->in_cache = nullptr;
    ctx->in_cache_n = 0;
    if (cudaMalloc(&ctx->in_cache, std::max<uint64_t>(acc, 1) * 4) == cudaSuccess) ctx->in_cache_n = acc;
  }
  CK(cudaMalloc(&ctx->in_base, base.size() * 8));
  CK(cudaMalloc(&ctx->in_size, size.size() * 8));
  CK(cudaMemcpyAsync(ctx->in_base, base.data(), base.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->in_size, size.data(), size.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  Table &T = ctx->T;
  T.in_base = ctx->in_base;
  T.in_size = ctx->in_size;
  T.n_inputs = n;
  T.in_cache = (acc <= ctx->in_cache_n && acc) ? ctx->in_cache : nullptr;
  int r = veq_clear_terms(ctx);
  if (r) return r;
  CK(cudaStreamSynchronize(ctx->stream));
  return VEQ_OK;
}

// Fills n 32-bit words with a value, 16 bytes per thread per iteration
// (grid-stride over all SMs): the per-step table clear.
__global__ void k_fill_u32(uint32_t *p, uint64_t n, uint32_t v) {
  const uint64_t n4 = n / 4;
  uint4 *q = reinterpret_cast<uint4 *>(p);
  const uint4 w = make_uint4(v, v, v, v);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    q[i] = w;
  if (blockIdx.x == 0 && threadIdx.x < n - 4 * n4) p[4 * n4 + threadIdx.x] = v;
}

int veq_clear_terms(veq_ctx *ctx) {
  if (!ctx) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  ctx->hnodes.clear();
  ctx->hkids.clear();
  Table &T = ctx->T;
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    k_fill_u32<<<nsm * 8, 256, 0, ctx->stream>>>(ctx->slots, ctx->n_slots, 0xFFFFFFFFu);
    ctx->launches++;
  }
  CK(cudaMemsetAsync(ctx->counters, 0, 8 * sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->error, 0, sizeof(int), ctx->stream));
  CK(cudaMemsetAsync(ctx->dbg, 0, 4 * sizeof(unsigned long long), ctx->stream));
  if (T.in_cache) k_fill_u32<<<148, 256, 0, ctx->stream>>>(T.in_cache, ctx->in_cells, 0xFFFFFFFFu);
  // a single thread interns -inf, 0, 1, -1 first into an empty table, so
  // their ids are 0..3 without a host round trip
  k_session_init<<<1, 32, 0, ctx->stream>>>(T, ctx->session_ids);
  ctx->launches++;
  CK(cudaGetLastError());
  T.id_neginf = 0;
  T.id_zero = 1;
  T.id_one = 2;
  T.id_mone = 3;
  return VEQ_OK;
}

void *veq_stream(veq_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int veq_set_timing(veq_ctx *ctx, int on) {
  if (!ctx) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  if (on && !ctx->ev0[0])
    for (int i = 0; i < VEQ_MAX_PHASES; i++) {
      CK(cudaEventCreate(&ctx->ev0[i]));
      CK(cudaEventCreate(&ctx->ev1[i]));
    }
  ctx->timing = on != 0;
  return VEQ_OK;
}

// Frees a batch's device buffers (stream-ordered) and the batch itself.
void drop_batch(veq_ctx *ctx, BatchDev *bd) {
  for (void *p : bd->owned) cudaFreeAsync(p, ctx->stream);
  delete bd;
}

static int load_impl(veq_ctx *ctx, const veq_batch_desc *d, veq_stmt *dev_stmts, uint32_t *out);

int veq_load_batch(veq_ctx *ctx, const veq_batch_desc *d, uint32_t *out) {
  if (!ctx || !d || !out) return VEQ_E_ARG;
  return load_impl(ctx, d, nullptr, out);
}

// d->stmts is ignored when dev_stmts is given: the statements are already on
// the device (an instantiated template) and the batch takes ownership.
static int load_impl(veq_ctx *ctx, const veq_batch_desc *d, veq_stmt *dev_stmts, uint32_t *out) {
  static const bool lprof = getenv("VEQ_PROF") && getenv("VEQ_PROF")[0] == '1';
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto lt0 = now();
  CK(cudaSetDevice(ctx->device));
  const uint32_t P = d->n_progs, Tn = d->n_threads_total;
  const uint64_t S = d->n_stmts;
  if (S >= (1ull << 31) || P >= (1u << 20)) {
    if (dev_stmts) cudaFreeAsync(dev_stmts, ctx->stream);
    return fail(ctx, VEQ_E_UNSUPPORTED, S >= (1ull << 31) ? "batch has more than 2^31 statements"
                                                          : "batch has more than 2^20 programs");
  }
  BatchDev *bd = new BatchDev();
  bd->progs.assign(d->progs, d->progs + P);
  bd->arrays.assign(d->arrays, d->arrays + d->n_arrays_total);
  bd->n_stmts = S;
  bd->n_threads = Tn;
  Batch &B = bd->B;
  B.n_progs = P;
  B.n_threads = Tn;
  B.n_stmts = S;
  int r = 0;
  cudaStream_t s = ctx->stream;
#define UP(field, src, n, T_)                                                            \
  do {                                                                                   \
    T_ *p_ = nullptr;                                                                    \
    if ((r = dupload(ctx, bd, &p_, (const T_ *)(src), (n)))) { drop_batch(ctx, bd); return r; }   \
    B.field = p_;                                                                        \
  } while (0)
#define AL(field, n, T_)                                                  \
  do {                                                                    \
    T_ *p_ = nullptr;                                                     \
    if ((r = dalloc(ctx, bd, &p_, (n)))) { drop_batch(ctx, bd); return r; }        \
    B.field = p_;                                                         \
  } while (0)
  // the caller's big buffers go first: their DMA overlaps the host
  // preparation below (async when the caller's memory is pinned)
  if (dev_stmts) {
    bd->owned.push_back(dev_stmts);
    B.stmts = dev_stmts;
  } else {
    UP(stmts, d->stmts, S, veq_stmt);
  }
  UP(thread_stmt, d->thread_stmt, Tn + 1, uint64_t);
  UP(progs, d->progs, P, veq_program_meta);
  UP(arrays, d->arrays, d->n_arrays_total, veq_array);
  UP(set_words, d->set_words, d->n_set_words, uint64_t);
  // ---- host preparation (per program / array / pool entry only): program
  // ranges, register offsets, sync-set pool canonicalisation, cell bases.
  // Everything per statement runs on the device (k_prep_*).
  std::vector<uint64_t> reg_off(Tn + 1, 0);
  for (uint32_t p = 0; p < P; p++) {
    const veq_program_meta &m = d->progs[p];
    if ((uint64_t)m.thread_off + m.n_threads > Tn || (uint64_t)m.array_off + m.n_arrays > d->n_arrays_total) {
      drop_batch(ctx, bd);
      return fail(ctx, VEQ_E_INVALID_IR, "program " + std::to_string(p) + " out of range");
    }
  }
  for (uint32_t t = 0; t < Tn; t++) {
    if (d->thread_stmt[t + 1] < d->thread_stmt[t] || d->thread_stmt[t + 1] > S) {
      drop_batch(ctx, bd);
      return fail(ctx, VEQ_E_INVALID_IR, "thread statement ranges are not monotone");
    }
    reg_off[t + 1] = reg_off[t] + d->thread_nregs[t];
  }
  // content-equal sync sets share the id of their first pool entry; the
  // full set of every program is the extra entry n_syncsets
  const uint32_t NS = d->n_syncsets;
  std::vector<uint32_t> set_canon(NS), set_pop(NS);
  std::vector<veq_syncset> sets(d->syncsets, d->syncsets + NS);
  sets.push_back(veq_syncset{1, 0, 0, 0});
  {
    std::unordered_map<std::string, uint32_t> seen;
    std::string key;
    for (uint32_t i = 0; i < NS; i++) {
      const veq_syncset &q = d->syncsets[i];
      uint32_t pop = 0;
      key.assign(reinterpret_cast<const char *>(&q.full), 4);
      if (!q.full) {
        if ((uint64_t)q.word_off + (q.n_bits + 63) / 64 > d->n_set_words) {
          drop_batch(ctx, bd);
          return fail(ctx, VEQ_E_INVALID_IR, "sync set words out of range");
        }
        key.append(reinterpret_cast<const char *>(&q.lo), 8);
        for (uint32_t w = 0; w < (q.n_bits + 63) / 64; w++) {
          uint64_t x = d->set_words[q.word_off + w];
          if (w == (q.n_bits - 1) / 64 && q.n_bits % 64) x &= (1ull << (q.n_bits % 64)) - 1;
          pop += __builtin_popcountll(x);
          key.append(reinterpret_cast<const char *>(&x), 8);
        }
      }
      set_canon[i] = seen.emplace(key, i).first->second;
      set_pop[i] = q.full ? ~0u : pop;
    }
  }
  std::vector<uint64_t> cell_base(d->n_arrays_total, UNSET64);
  uint64_t cells = 0;
  for (uint32_t a = 0; a < d->n_arrays_total; a++) {
    const veq_array &ar = d->arrays[a];
    bool direct = !(ar.flags & VEQ_ARR_STORED) && ar.input >= 0 && ar.seeded >= ar.size;
    if (ar.input >= (int32_t)ctx->input_names.size()) {
      drop_batch(ctx, bd);
      return fail(ctx, VEQ_E_INVALID_IR, "array refers to an undeclared input");
    }
    if (!direct) {
      cell_base[a] = cells;
      cells += ar.size;
    }
  }
  if (cells >= (1ull << 32)) {
    drop_batch(ctx, bd);
    return fail(ctx, VEQ_E_UNSUPPORTED, "more than 2^32 checked memory cells in one batch");
  }
  bd->arr_cell_base = cell_base;
  bd->syncsets.assign(d->syncsets, d->syncsets + NS);
  bd->set_words.assign(d->set_words, d->set_words + d->n_set_words);
  bd->n_cells = cells;
  bd->n_regs = reg_off[Tn];
  // programs laid out in order (thread and statement ranges contiguous)
  // allow a statement -> program search over P+1 boundaries
  std::vector<uint64_t> prog_stmt(P + 1, 0);
  bool in_order = true;
  for (uint32_t p = 0; p < P; p++) {
    const veq_program_meta &m = d->progs[p];
    if (p + 1 < P && d->progs[p + 1].thread_off != m.thread_off + m.n_threads) in_order = false;
    prog_stmt[p] = d->thread_stmt[m.thread_off];
  }
  if (P) prog_stmt[P] = d->thread_stmt[d->progs[P - 1].thread_off + d->progs[P - 1].n_threads];
  // sort-key field widths: steps of a program are at most its statements
  // plus its releases (<= statements), programs < P
  {
    uint64_t maxps = 0;
    for (uint32_t p = 0; p < P; p++) {
      const veq_program_meta &m = d->progs[p];
      maxps = std::max<uint64_t>(maxps, d->thread_stmt[m.thread_off + m.n_threads] - d->thread_stmt[m.thread_off]);
    }
    uint32_t sb = 1, pb = 1;
    while ((1ull << sb) < 2 * maxps + 2 && sb < 32) sb++;
    while ((1ull << pb) < (uint64_t)P + 1 && pb < 20) pb++;
    bd->B.step_bits = sb;
    bd->B.prog_bits = pb;
  }
  const auto lt1 = now();
  // ---- upload
  UP(arr_cell_base, cell_base.data(), cell_base.size(), uint64_t);
  B.n_cells = cells;
  UP(sets, sets.data(), sets.size(), veq_syncset);
  UP(reg_off, reg_off.data(), Tn + 1, uint64_t);
  if (in_order && P) UP(prog_stmt, prog_stmt.data(), P + 1, uint64_t);
  else B.prog_stmt = nullptr;
  AL(thread_prog, Tn, uint32_t);
  AL(prog_full_set, P, uint32_t);
  const auto lt2 = now();
  // ---- device preparation
  uint32_t *d_canon = nullptr, *d_pop = nullptr, *d_long = nullptr;
  unsigned long long *d_cnt = nullptr, *d_nlong = nullptr;
  uint64_t *d_psync = nullptr;
  if ((r = dupload(ctx, nullptr, &d_canon, set_canon.data(), NS)) || (r = dupload(ctx, nullptr, &d_pop, set_pop.data(), NS)) ||
      (r = dalloc(ctx, nullptr, &d_cnt, S + 1)) || (r = dalloc(ctx, nullptr, &d_nlong, 1)) ||
      (r = dalloc(ctx, nullptr, &d_psync, P + 1)) || (r = dalloc(ctx, bd, &d_long, Tn))) {
    drop_batch(ctx, bd);
    return r;
  }
  B.long_threads = d_long;
  unsigned int *d_flags = nullptr;
  unsigned long long *d_narith = nullptr;
  if ((r = dalloc(ctx, nullptr, &d_flags, 1)) || (r = dalloc(ctx, nullptr, &d_narith, 1))) {
    drop_batch(ctx, bd);
    return r;
  }
  CK(cudaMemsetAsync(d_flags, 0, 4, s));
  CK(cudaMemsetAsync(d_narith, 0, 8, s));
  PrepArgs PA{P, Tn, NS, d->n_arrays_total, S, B.progs, B.thread_stmt, B.thread_prog, B.stmts, B.sets, d_canon, d_pop,
              d_cnt, ctx->error, B.set_words, d_flags, B.arrays, d_narith};
  CK(cudaMemsetAsync(ctx->error, 0, sizeof(int), s));
  CK(cudaMemsetAsync(d_cnt + S, 0, 8, s));
  CK(cudaMemsetAsync(d_nlong, 0, 8, s));
  if (P) k_prep_thread_prog<<<P, 256, 0, s>>>(PA, (uint32_t *)B.thread_prog);
  if (S) k_prep_stmts<<<blocks(S, 256), 256, 0, s>>>(PA);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_cnt, (int64_t)(S + 1), s);
    void *tmp = nullptr;
    CK(cudaMallocAsync(&tmp, tb, s));
    cub::DeviceScan::ExclusiveSum(tmp, tb, d_cnt, d_cnt, (int64_t)(S + 1), s);
    CK(cudaFreeAsync(tmp, s));
  }
  if (Tn) k_prep_long<<<blocks(Tn, 256), 256, 0, s>>>(PA, d_long, d_nlong, EXEC_WARP_MIN);
  unsigned long long tot = 0, nlong = 0, narith = 0;
  int perr = 0;
  CK(cudaMemcpyAsync(&narith, d_narith, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&tot, d_cnt + S, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&nlong, d_nlong, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&perr, ctx->error, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (perr) {
    cudaFreeAsync(d_canon, s);
    cudaFreeAsync(d_pop, s);
    cudaFreeAsync(d_cnt, s);
    cudaFreeAsync(d_nlong, s);
    cudaFreeAsync(d_psync, s);
    cudaMemsetAsync(ctx->error, 0, sizeof(int), s);
    drop_batch(ctx, bd);
    return fail(ctx, VEQ_E_INVALID_IR, perr == 1 ? "bad statement kind"
                                       : perr == 2 ? "array index out of range"
                                                   : "sync set index out of range");
  }
  const auto lt3 = now();
  const uint64_t n_syncs = tot & 0xffffffffull, n_access = tot >> 32;
  bd->n_arith = narith;
  B.n_long = (uint32_t)nlong;
  bd->n_segs = (uint64_t)Tn + n_syncs;
  bd->n_rel_cap = n_syncs;
  bd->n_access_max = n_access;
  AL(seg_off, Tn + 1, uint64_t);
  AL(seg_start, bd->n_segs, uint64_t);
  AL(seg_set, bd->n_segs, uint32_t);
  AL(rel_off, P + 1, uint64_t);
  k_prep_threads<<<blocks((uint64_t)Tn + 1, 256), 256, 0, s>>>(PA, (uint64_t *)B.seg_off, (uint64_t *)B.seg_start,
                                                               (uint32_t *)B.seg_set);
  if (S) k_prep_syncs<<<blocks(S, 256), 256, 0, s>>>(PA, (uint64_t *)B.seg_start, (uint32_t *)B.seg_set);
  AL(set_chunk, (uint64_t)NS + 1, unsigned long long);
  k_prep_set_chunks<<<blocks((uint64_t)NS + 1, 256), 256, 0, s>>>(B.sets, B.set_words, NS,
                                                                   (unsigned long long *)B.set_chunk);
  if (P) {
    k_prep_progs<<<blocks(P, 256), 256, 0, s>>>(PA, d_psync, (uint32_t *)B.prog_full_set);
    CK(cudaMemsetAsync(d_psync + P, 0, 8, s));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, d_psync, (uint64_t *)B.rel_off, (int64_t)(P + 1), s);
    void *tmp = nullptr;
    CK(cudaMallocAsync(&tmp, tb, s));
    cub::DeviceScan::ExclusiveSum(tmp, tb, d_psync, (uint64_t *)B.rel_off, (int64_t)(P + 1), s);
    CK(cudaFreeAsync(tmp, s));
  } else {
    CK(cudaMemsetAsync((void *)B.rel_off, 0, 8, s));
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&bd->sched_flags, d_flags, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d_flags, s));
  CK(cudaFreeAsync(d_narith, s));
  CK(cudaFreeAsync(d_canon, s));
  CK(cudaFreeAsync(d_pop, s));
  CK(cudaFreeAsync(d_cnt, s));
  CK(cudaFreeAsync(d_nlong, s));
  CK(cudaFreeAsync(d_psync, s));
  uint32_t *cn = nullptr;
  veq_rat *dconsts = nullptr;
  if ((r = dalloc(ctx, bd, &cn, d->n_consts)) || (r = dupload(ctx, bd, &dconsts, d->consts, d->n_consts))) {
    drop_batch(ctx, bd);
    return r;
  }
  B.const_node = cn;
  bd->dconsts = dconsts;
  bd->n_consts = d->n_consts;
  // run-state buffers
  AL(seg_base, bd->n_segs, uint32_t);
  AL(rel_step, bd->n_rel_cap, uint32_t);
  AL(rel_set, bd->n_rel_cap, uint32_t);
  AL(prog_nrel, P, uint32_t);
  AL(prog_dead, P, uint32_t);
  AL(prog_steps, P, unsigned long long);
  AL(th_state, Tn, uint8_t);
  AL(th_seg, Tn, uint32_t);
  AL(th_bset, Tn, uint32_t);
  AL(regfile, bd->n_regs, uint32_t);
  AL(ref_a, S, uint32_t);
  AL(ref_b, S, uint32_t);
  AL(st_step, S, uint32_t);
  AL(canon, S, uint32_t);
  AL(chain_head, S, uint32_t);
  AL(chain_pos, S, uint32_t);
  AL(chain_len, S, uint32_t);
  AL(uses, S, uint32_t);
  AL(continued, S, uint8_t);
  AL(user, S, uint32_t);
  AL(defer, (S + 4) & ~3ull, uint8_t);
  AL(tup_key, n_access, unsigned long long);
  AL(tup_val, n_access, unsigned long long);
  AL(n_tup, 1, unsigned long long);
  AL(final_val, cells, uint32_t);
  AL(final_node, cells, uint32_t);
  uint64_t fcap = std::min<uint64_t>(std::max<uint64_t>(3 * S, 1024), 16ull << 20);
  AL(faults, fcap, veq_fault);
  AL(n_faults, 1, unsigned long long);
  B.fault_cap = fcap;
#undef AL
#undef UP
  if ((r = dalloc(ctx, bd, &bd->d_stats, 16))) {
    drop_batch(ctx, bd);
    return r;
  }
  ctx->batches.push_back(bd);
  *out = (uint32_t)(ctx->batches.size() - 1);
  const int rc = check_error_flag(ctx);
  if (lprof)
    fprintf(stderr, "[veq load] S=%llu host prep %.2f upload-issue %.2f device prep+sync %.2f rest %.2f ms\n",
            (unsigned long long)S, ms(lt0, lt1), ms(lt1, lt2), ms(lt2, lt3), ms(lt3, now()));
  return rc;
}

int veq_run(veq_ctx *ctx, uint32_t batch, veq_run_out *out) {
  int r = veq_run_start(ctx, batch);
  if (r) return r;
  return veq_run_finish(ctx, batch, out);
}

int veq_run_start(veq_ctx *ctx, uint32_t batch) {
  if (!ctx || !live_batch(ctx, batch)) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (bd->started) return fail(ctx, VEQ_E_ARG, "veq_run_start: previous run of this batch not finished");
  Batch &B = bd->B;
  cudaStream_t s = ctx->stream;
  const uint64_t S = bd->n_stmts;
  // reset run state; the table counters are snapshot on the device (stats)
  CK(cudaMemcpyAsync(bd->d_stats, ctx->counters, 64, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(B.seg_base, 0xff, bd->n_segs * 4, s));
  CK(cudaMemsetAsync(B.regfile, 0xff, std::max<uint64_t>(bd->n_regs, 1) * 4, s));
  CK(cudaMemsetAsync(B.st_step, 0xff, S * 4, s));
  CK(cudaMemsetAsync(B.canon, 0xff, S * 4, s));
  CK(cudaMemsetAsync(B.uses, 0, S * 4, s));
  CK(cudaMemsetAsync(B.continued, 0, S, s));
  CK(cudaMemsetAsync(B.defer, 0, (S + 4) & ~3ull, s));
  {
    static const bool env_off = getenv("VEQ_NO_DEFER") && getenv("VEQ_NO_DEFER")[0] == '1';
    B.no_defer = (env_off || bd->no_defer) ? 1u : 0u;
    B.keep_regs = ctx->keep_regs ? 1u : 0u;
    bd->keep_regs = ctx->keep_regs;
  }
  // the tuple buffer holds every checked access; slots of accesses that
  // never execute (deadlock) keep key ~0 and sort last, so the sort needs no
  // host read-back of the tuple count
  if (bd->n_access_max) CK(cudaMemsetAsync(B.tup_key, 0xff, bd->n_access_max * 8, s));
  CK(cudaMemsetAsync(B.n_tup, 0, 8, s));
  CK(cudaMemsetAsync(B.n_faults, 0, 8, s));
  CK(cudaMemsetAsync(B.final_val, 0xff, std::max<uint64_t>(bd->n_cells, 1) * 4, s));
  CK(cudaMemsetAsync(ctx->pool_used, 0, 8, s));
  const uint32_t launches0 = ctx->launches;
#define PH0(p) do { if (ctx->timing) CK(cudaEventRecord(ctx->ev0[p], s)); } while (0)
#define PH1(p) do { if (ctx->timing) CK(cudaEventRecord(ctx->ev1[p], s)); } while (0)
#define LAUNCH(...) do { __VA_ARGS__; ctx->launches++; } while (0)
  // constants are interned per run so a cleared term table stays consistent
  if (bd->n_consts)
    LAUNCH(k_intern_consts<<<blocks(bd->n_consts, 256), 256, 0, s>>>(ctx->T, bd->dconsts, bd->n_consts,
                                                                       (uint32_t *)B.const_node));
  // K0
  PH0(VEQ_PH_SCHEDULE);
  if (B.n_progs) {
    uint32_t maxT = 0;
    for (const veq_program_meta &m : bd->progs) maxT = std::max(maxT, m.n_threads);
    if (maxT <= 1024 && !(bd->sched_flags & 1u)) {
      // one warp per CTA, chunked round-robin emulation
      const size_t smem = SW_WARPS * sizeof(SchedWarpSmem);
      CK(cudaFuncSetAttribute(k_schedule_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LAUNCH(k_schedule_warp<<<blocks(B.n_progs, SW_WARPS), SW_WARPS * 32, smem, s>>>(B));
    } else if (maxT <= 1024) {
      // one CUDA thread per symbolic thread, control state in registers
      const uint32_t bt = std::max<uint32_t>(32, (maxT + 31) / 32 * 32);
      LAUNCH(k_schedule_lanes<<<B.n_progs, bt, 0, s>>>(B));
    } else {
      // on-chip control state sized to the largest CTA of the batch, so small
      // CTAs keep many scheduler blocks resident per SM
      size_t smem = maxT <= SCHED_SMEM_T ? ((size_t)maxT * 9 + 15) / 16 * 16 : 0;
      B.sched_on_chip = smem > 0 ? maxT : 0;
      if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(k_schedule_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LAUNCH(k_schedule_smem<<<B.n_progs, SCHED_BLOCK, smem, s>>>(B));
    }
  }
  PH1(VEQ_PH_SCHEDULE);
  CK(cudaGetLastError());
  // K3 (direct input loads are interned first, in parallel)
  PH0(VEQ_PH_EXEC);
  if (S && ctx->T.in_cache) {
    LAUNCH(k_mark_inputs<<<blocks(S, 256), 256, 0, s>>>(B, ctx->T));
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    LAUNCH(k_intern_marked<<<nsm * 8, 256, 0, s>>>(ctx->T, ctx->in_cells));
  }
  if (S) LAUNCH(k_pre_inputs<<<blocks(S, 256), 256, 0, s>>>(B, ctx->T));
  // short threads: one CUDA thread each; long threads: one warp each
  // long threads (warp executor) run on the side stream alongside the short
  // ones: a batch mixing both kinds of CTA (e.g. kernel A's 1-thread CTAs
  // and kernel B's 1024-thread CTAs) keeps the GPU busy with both
  if (B.n_long && B.n_threads > B.n_long) {
    CK(cudaEventRecord(ctx->ev_fork, s));
    CK(cudaStreamWaitEvent(ctx->stream2, ctx->ev_fork, 0));
    LAUNCH(k_exec_warp<<<blocks((uint64_t)B.n_long * 32, 128), 128, 0, ctx->stream2>>>(B, ctx->T));
    CK(cudaEventRecord(ctx->ev_join, ctx->stream2));
    LAUNCH(k_exec<<<blocks(B.n_threads, 128), 128, 0, s>>>(B, ctx->T));
    CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
  } else {
    if (B.n_threads) LAUNCH(k_exec<<<blocks(B.n_threads, 128), 128, 0, s>>>(B, ctx->T));
    if (B.n_long) LAUNCH(k_exec_warp<<<blocks((uint64_t)B.n_long * 32, 128), 128, 0, s>>>(B, ctx->T));
  }
  PH1(VEQ_PH_EXEC);
  CK(cudaGetLastError());
  const unsigned long long n_tup = bd->n_access_max;
  // K4: sort access tuples by (cell, step) and scan per cell
  PH0(VEQ_PH_SORT);
  if (n_tup) {
    unsigned long long *k2 = nullptr, *v2 = nullptr;
    uint32_t *starts = nullptr;
    unsigned long long *n_starts = nullptr;
    Reader *rs = nullptr;
    { int r_ = ws_get(ctx, 1, (void **)&k2, n_tup * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 2, (void **)&v2, n_tup * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 3, (void **)&starts, n_tup * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 4, (void **)&n_starts, 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 5, (void **)&rs, n_tup * sizeof(Reader)); if (r_) return r_; }
    int cb = 1;
    while ((1ull << cb) < bd->n_cells + 1) cb++;
    int end_bit = (int)B.step_bits + cb;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, B.tup_key, k2, B.tup_val, v2, (int64_t)n_tup, 0, end_bit, s);
    void *tmp = nullptr;
    { int r_ = ws_get(ctx, 6, (void **)&tmp, tmp_bytes); if (r_) return r_; }
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, B.tup_key, k2, B.tup_val, v2, (int64_t)n_tup, 0, end_bit, s);
    ctx->launches += (end_bit + 7) / 8 + 1;
    CK(cudaMemsetAsync(n_starts, 0, 8, s));
    LAUNCH(k_seg_heads<<<blocks(n_tup, APP_NT * APP_ITEMS), APP_NT, 0, s>>>(k2, n_tup, starts, n_starts, B.step_bits));
    PH1(VEQ_PH_SORT);
    PH0(VEQ_PH_MEMSCAN);
    // one thread per segment head; the head count stays on the device
    LAUNCH(k_mem_scan<<<blocks(n_tup, 128), 128, 0, s>>>(B, ctx->T, k2, v2, starts, n_starts, n_tup, rs));
    PH1(VEQ_PH_MEMSCAN);
    CK(cudaGetLastError());
  } else {
    PH1(VEQ_PH_SORT);
    PH0(VEQ_PH_MEMSCAN);
    PH1(VEQ_PH_MEMSCAN);
  }
  // resolve operands through loads, count uses (incl. final cells), size
  // the chain logs — one pass over the statements
  uint32_t *sz = nullptr, *base = nullptr, *log = nullptr, *log_stmt = nullptr;
  unsigned long long n_work = 0;
  PH0(VEQ_PH_RESOLVE);
  if (S) {
    { int r_ = ws_get(ctx, 7, (void **)&sz, S * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 8, (void **)&base, S * 4); if (r_) return r_; }
    LAUNCH(k_resolve_all<<<blocks(S, 256), 256, 0, s>>>(B, sz));
  }
  if (bd->n_cells) LAUNCH(k_resolve_finals<<<blocks(bd->n_cells, 256), 256, 0, s>>>(B));
  if (B.keep_regs && bd->n_regs) LAUNCH(k_resolve_regs<<<blocks(bd->n_regs, 256), 256, 0, s>>>(B, bd->n_regs));
  // deferred scaling: products of a used-once sum feeding a chain (k_mark_defer)
  B.prog_split = nullptr;
  if (S && !B.no_defer) {
    { int r_ = ws_get(ctx, 40, (void **)&B.n_defer_chains, 4); if (r_) return r_; }
    CK(cudaMemsetAsync(B.n_defer_chains, 0, 4, s));
    LAUNCH(k_mark_defer<<<blocks(S, 256), 256, 0, s>>>(B));
    { int r_ = ws_get(ctx, 28, (void **)&B.prog_split, (uint64_t)B.n_progs * 4); if (r_) return r_; }
    CK(cudaMemsetAsync(B.prog_split, 0xff, (uint64_t)B.n_progs * 4, s));
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    LAUNCH(k_defer_split<<<nsm * 16, 256, 0, s>>>(B));
  }
  PH1(VEQ_PH_RESOLVE);
  CK(cudaGetLastError());
  // chain logs
  if (S) {
    PH0(VEQ_PH_CHAINS);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, sz, base, (int64_t)S, s);
    void *tmp = nullptr;
    { int r_ = ws_get(ctx, 9, (void **)&tmp, tb); if (r_) return r_; }
    cub::DeviceScan::ExclusiveSum(tmp, tb, sz, base, (int64_t)S, s);
    ctx->launches += 2;
    // log capacity bound: a chain of L links has L + 1 entries <= 2L
    const uint64_t nlog = 2 * bd->n_arith + 2;
    { int r_ = ws_get(ctx, 10, (void **)&log, std::max<uint64_t>(nlog, 1) * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 11, (void **)&log_stmt, std::max<uint64_t>(nlog, 1) * 4); if (r_) return r_; }
    PH1(VEQ_PH_CHAINS);
    // chain-log entries and the work list, one pass; work sorted by
    // (step, program)
    PH0(VEQ_PH_WORKLIST);
    unsigned long long *wk = nullptr, *wk2 = nullptr, *nw = nullptr;
    uint32_t *wv = nullptr, *wv2 = nullptr;
    // capacity U = BinOp/UnOp statements (static bound); unused slots keep
    // key ~0 and sort last; the true length stays on the device
    const uint64_t U = std::max<uint64_t>(bd->n_arith, 1);
    { int r_ = ws_get(ctx, 12, (void **)&wk, U * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 13, (void **)&wk2, U * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 14, (void **)&wv, U * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 15, (void **)&wv2, U * 4); if (r_) return r_; }
    // nw = {items, pass-2 items}
    { int r_ = ws_get(ctx, 16, (void **)&nw, 16); if (r_) return r_; }
    CK(cudaMemsetAsync(nw, 0, 16, s));
    // large lists: read the exact item count back (one short wait) and sort
    // only the items; small ones sort the whole capacity with no host wait
    // (unused slots keep key ~0 and sort last)
    const bool exact = U >= (1ull << 22);
    if (!exact) CK(cudaMemsetAsync(wk, 0xff, U * 8, s));
    LAUNCH(k_scatter_work<<<blocks(S, APP_NT * APP_ITEMS), APP_NT, 0, s>>>(B, base, log, log_stmt, wk, wv, nw));
    void *tmp2 = nullptr;
    n_work = bd->n_arith;
    uint64_t n_sort = U;
    if (exact) {
      unsigned long long h_nw = 0;
      CK(cudaMemcpyAsync(&h_nw, nw, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      n_sort = h_nw;
      n_work = h_nw;
    }
    if (n_work) {
      // key = pass << (step_bits + prog_bits) | step << prog_bits | program:
      // sort only the bits in use
      const int end_bit = (int)(B.prog_bits + B.step_bits) + (B.prog_split ? 1 : 0);
      size_t tb2 = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb2, wk, wk2, wv, wv2, (int64_t)n_sort, 0, end_bit, s);
      { int r_ = ws_get(ctx, 17, (void **)&tmp2, tb2); if (r_) return r_; }
      cub::DeviceRadixSort::SortPairs(tmp2, tb2, wk, wk2, wv, wv2, (int64_t)n_sort, 0, end_bit, s);
      ctx->launches += (end_bit + 7) / 8 + 1;
    }
    PH1(VEQ_PH_WORKLIST);
    PH0(VEQ_PH_EVAL);
    if (n_work) {
      unsigned long long *cursor = nullptr;
      { int r_ = ws_get(ctx, 18, (void **)&cursor, 16); if (r_) return r_; }
      CK(cudaMemsetAsync(cursor, 0, 16, s));
      static const bool prof_on = getenv("VEQ_PROF") && getenv("VEQ_PROF")[0] == '1';
      unsigned long long *prof = nullptr;
      if (prof_on) {
        { int r_ = ws_get(ctx, 19, (void **)&prof, 256 * 8); if (r_) return r_; }
        CK(cudaMemsetAsync(prof, 0, 256 * 8, s));
      }
      static const uint32_t eval_off = getenv("VEQ_EVAL_OFF") ? (uint32_t)atoi(getenv("VEQ_EVAL_OFF")) : 0u;
      // merge memo: sized from the arithmetic statements, cleared per run
      uint64_t want = 1ull << 16;
      while (want < (bd->n_arith / 8) && want < (1ull << 24)) want <<= 1;
      if (want > ctx->mslots) {
        CK(cudaStreamSynchronize(s));
        cudaFree(ctx->mkeys);
        cudaFree(ctx->mvals);
        ctx->mkeys = nullptr;
        ctx->mvals = nullptr;
        ctx->mslots = 0;
        if (cudaMalloc(&ctx->mkeys, want * 8) != cudaSuccess || cudaMalloc(&ctx->mvals, want * 4) != cudaSuccess)
          return fail(ctx, VEQ_E_OOM, "merge memo");
        ctx->mslots = want;
      }
      CK(cudaMemsetAsync(ctx->mkeys, 0xff, ctx->mslots * 8, s));
      CK(cudaMemsetAsync(ctx->mvals, 0xff, ctx->mslots * 4, s));
      static const uint32_t bucket_us = getenv("VEQ_PROF_BUCKET_US") ? (uint32_t)atoi(getenv("VEQ_PROF_BUCKET_US")) : 400u;
      static const bool no_memo = getenv("VEQ_NO_MEMO") && getenv("VEQ_NO_MEMO")[0] == '1';
      EvalCtx E{log, log_stmt, base, prof, eval_off, no_memo ? nullptr : ctx->mkeys, ctx->mvals, ctx->mslots - 1,
                bucket_us ? bucket_us : 400u};
      uint4 *desc = nullptr;
      { int r_ = ws_get(ctx, 20, (void **)&desc, n_work * sizeof(uint4)); if (r_) return r_; }
      LAUNCH(k_make_desc<<<blocks(n_work, 256), 256, 0, s>>>(B, E, wv2, nw, desc));
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
      // one warp per work item, persistent over the sorted work list;
      // persistent grid: exactly the resident capacity (no second wave)
      const int smem = (int)(EVAL_PAGES * SPAGE);
      int per_sm = 1;
      eval_warp_config(smem, &per_sm);
      if (per_sm < 1) per_sm = 1;
      // every resident slot is launched (warps spread over all SMs); the
      // kernel reads the work-list length and picks its claim size
      uint64_t threads = (uint64_t)nsm * per_sm * EVAL_BLOCK;
      // per-warp allocation chunks: at most 1/16 of the table's capacity is
      // held in chunk tails when every warp holds one
      {
        const uint64_t warps = threads / 32;
        ctx->T.wa_ids = (uint32_t)std::min<uint64_t>(WA_IDS, std::max<uint64_t>(1, ctx->lim.max_nodes / (16 * warps)));
        ctx->T.wa_kids = (uint32_t)std::min<uint64_t>(WA_KIDS, std::max<uint64_t>(32, ctx->lim.max_kid_words / (16 * warps)));
      }
      uint64_t chunk = std::min<uint64_t>(1ull << 20, std::max<uint64_t>(16ull << 10, ctx->pool_cap / (4 * threads)));
      LAUNCH(launch_eval_warp(blocks(threads, EVAL_BLOCK), EVAL_BLOCK, smem, s, B, ctx->T, E, desc, nw, cursor,
                              ctx->pool, ctx->pool_used, ctx->pool_cap, chunk, false));
      // pass 2: items from each program's first deferred expansion on
      if (B.prog_split)
        LAUNCH(launch_eval_warp(blocks(threads, EVAL_BLOCK), EVAL_BLOCK, smem, s, B, ctx->T, E, desc, nw, cursor + 1,
                                ctx->pool, ctx->pool_used, ctx->pool_cap, chunk, true));
      CK(cudaGetLastError());
      if (prof) {
        unsigned long long hp[256], nwh = 0;
        CK(cudaMemcpyAsync(hp, prof, 256 * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&nwh, nw, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fprintf(stderr, "[veq prof] items %llu warps %llu | wait %.1f us/item |", nwh, (unsigned long long)(threads / 32),
                hp[0] / 1965.0 / std::max<double>(1, nwh));
        const char *nm[5] = {"other", "lean", "smem", "small", "global"};
        for (int k = 0; k < 5; k++)
          if (hp[6 + k]) fprintf(stderr, " %s n=%llu %.2f us", nm[k], hp[6 + k], hp[1 + k] / 1965.0 / hp[6 + k]);
        if (hp[7])
          fprintf(stderr, " | lean phases: loads %.2f sort %.2f intern %.2f us", hp[11] / 1965.0 / hp[7],
                  hp[12] / 1965.0 / hp[7], hp[13] / 1965.0 / hp[7]);
        if (hp[8])
          fprintf(stderr, " | smem: pool wait %.2f us/item, %.1f pages/item; runs %.2f gather %.2f merge %.2f intern %.2f us",
                  hp[14] / 1965.0 / hp[8], (double)hp[15] / hp[8], hp[16] / 1965.0 / hp[8], hp[17] / 1965.0 / hp[8],
                  hp[18] / 1965.0 / hp[8], hp[19] / 1965.0 / hp[8]);
        if (hp[27])
          fprintf(stderr, " | deferred: n=%llu expand %.1f terms %.1f sum %.1f us", hp[27], hp[24] / 1965.0 / hp[27],
                  hp[25] / 1965.0 / hp[27], hp[26] / 1965.0 / hp[27]);
        {
          const char *on[8] = {"mul", "div", "max", "neg", "exp", "?", "?", "?"};
          fprintf(stderr, "\n[veq prof] lane items (n, us/item incl. waits):");
          for (int k = 0; k < 5; k++)
            if (hp[128 + k]) fprintf(stderr, " %s n=%llu %.1f", on[k], hp[128 + k], hp[136 + k] / 1965.0 / hp[128 + k]);
        }
        fprintf(stderr, "\n[veq prof] timeline (per %u us: items, smem items, warps done):", bucket_us ? bucket_us : 400u);
        for (int k = 0; k < 32; k++)
          if (hp[32 + k] || hp[96 + k]) fprintf(stderr, " %d:%llu/%llu/%llu", k, hp[32 + k], hp[64 + k], hp[96 + k]);
        fprintf(stderr, "\n");
      }
    }
    PH1(VEQ_PH_EVAL);
    CK(cudaMemcpyAsync(bd->d_stats + 8, nw, 8, cudaMemcpyDeviceToDevice, s));
  }
  PH0(VEQ_PH_FINALS);
  if (bd->n_cells) LAUNCH(k_final_nodes<<<blocks(bd->n_cells, 256), 256, 0, s>>>(B));
  PH1(VEQ_PH_FINALS);
  CK(cudaGetLastError());
  bd->started = true;
  bd->timing_run = ctx->timing;
  bd->run_launches = ctx->launches - launches0;
  return VEQ_OK;
}

int veq_run_finish(veq_ctx *ctx, uint32_t batch, veq_run_out *out) {
  if (!ctx || !live_batch(ctx, batch)) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (!bd->started) return fail(ctx, VEQ_E_ARG, "veq_run_finish: no run started on this batch");
  bd->started = false;
  Batch &B = bd->B;
  cudaStream_t s = ctx->stream;
  // ---- results to host (the first read-back waits for the run)
  unsigned long long st16[16] = {0};
  CK(cudaMemcpyAsync(st16, bd->d_stats, 128, cudaMemcpyDeviceToHost, s));
  const unsigned long long *cnt0 = st16;
  bd->n_work_last = st16[8];
  const uint32_t P = B.n_progs;
  std::vector<uint32_t> nrel(P);
  std::vector<unsigned long long> steps(P);
  unsigned long long nf = 0;
  CK(cudaMemcpyAsync(nrel.data(), B.prog_nrel, P * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(steps.data(), B.prog_steps, P * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&nf, B.n_faults, 8, cudaMemcpyDeviceToHost, s));
  std::vector<uint32_t> dead(P);
  CK(cudaMemcpyAsync(dead.data(), B.prog_dead, P * 4, cudaMemcpyDeviceToHost, s));
  unsigned long long nn[8] = {0};
  CK(cudaMemcpyAsync(nn, ctx->counters, 64, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  {
    // -inf met inside a deferred expansion: repeat the run without deferral
    // so faults are reported exactly where the reference raises them
    int h = 0;
    CK(cudaMemcpy(&h, ctx->error, sizeof(int), cudaMemcpyDeviceToHost));
    if (h == E_DEFER && !bd->no_defer) {
      CK(cudaMemsetAsync(ctx->error, 0, sizeof(int), s));
      bd->no_defer = true;
      int r = veq_run_start(ctx, batch);
      if (r) return r;
      return veq_run_finish(ctx, batch, out);
    }
  }
  int er = check_error_flag(ctx);
  if (er) return er;
  if (nf > B.fault_cap) return fail(ctx, VEQ_E_BUDGET, "fault buffer overflow");
  bd->faults.resize(nf);
  // many faults (racy kernels): ordered on the device before the copy
  const bool dev_order = nf >= (1u << 14) && B.n_progs < (1u << 23);
  if (dev_order) {
    unsigned long long *k1 = nullptr, *k2 = nullptr;
    uint32_t *i1 = nullptr, *i2 = nullptr;
    veq_fault *sorted = nullptr;
    { int r_ = ws_get(ctx, 32, (void **)&k1, nf * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 33, (void **)&k2, nf * 8); if (r_) return r_; }
    { int r_ = ws_get(ctx, 34, (void **)&i1, nf * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 35, (void **)&i2, nf * 4); if (r_) return r_; }
    { int r_ = ws_get(ctx, 36, (void **)&sorted, nf * sizeof(veq_fault)); if (r_) return r_; }
    k_fault_keys<<<blocks(nf, 256), 256, 0, s>>>(B.faults, nf, k1, i1);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, i1, i2, (int64_t)nf, 0, 63, s);
    void *tmp = nullptr;
    { int r_ = ws_get(ctx, 37, &tmp, tb); if (r_) return r_; }
    cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k2, i1, i2, (int64_t)nf, 0, 63, s);
    k_fault_gather<<<blocks(nf, 256), 256, 0, s>>>(B.faults, i2, nf, sorted);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(bd->faults.data(), sorted, nf * sizeof(veq_fault), cudaMemcpyDeviceToHost, s));
  } else if (nf) {
    CK(cudaMemcpyAsync(bd->faults.data(), B.faults, nf * sizeof(veq_fault), cudaMemcpyDeviceToHost, s));
  }
  bool any_dead = false;
  for (uint32_t p = 0; p < P; p++) any_dead |= dead[p] != 0;
  // final thread states are per-thread only after a deadlock; otherwise every
  // thread returned and the ctx's shared all-returned arrays are handed out
  bd->th_state.clear();
  bd->th_bset.clear();
  bd->th_bstmt.clear();
  if (ctx->ret_state.size() < B.n_threads) {
    ctx->ret_state.assign(B.n_threads, TS_RET);
    ctx->unset_set.assign(B.n_threads, UNSET);
    ctx->unset_stmt.assign(B.n_threads, ~0ull);
  }
  if (any_dead) {
    // final thread states only matter for deadlock reports (symexec.cpp:335-365)
    bd->th_state.assign(B.n_threads, TS_RET);
    bd->th_bset.assign(B.n_threads, UNSET);
    bd->th_bstmt.assign(B.n_threads, ~0ull);
    std::vector<uint32_t> th_seg(B.n_threads);
    CK(cudaMemcpyAsync(bd->th_state.data(), B.th_state, B.n_threads, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(bd->th_bset.data(), B.th_bset, B.n_threads * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(th_seg.data(), B.th_seg, B.n_threads * 4, cudaMemcpyDeviceToHost, s));
    std::vector<uint64_t> seg_off_h(B.n_threads + 1), seg_start_h(bd->n_segs);
    CK(cudaMemcpyAsync(seg_off_h.data(), B.seg_off, (B.n_threads + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(seg_start_h.data(), B.seg_start, bd->n_segs * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint32_t t = 0; t < B.n_threads; t++)
      if (bd->th_state[t] == TS_BLOCK) bd->th_bstmt[t] = seg_start_h[seg_off_h[t] + th_seg[t] + 1] - 1;
  }
  CK(cudaStreamSynchronize(s));
  bd->res.assign(P, veq_prog_result{});
  for (uint32_t p = 0; p < P; p++) {
    bd->res[p].steps = steps[p];
    bd->res[p].releases = nrel[p];
    bd->res[p].deadlocked = dead[p];
  }
  for (const veq_fault &f : bd->faults) bd->res[f.prog].n_faults++;
  // reference order within a program: execution order (step, then the
  // order of checks inside one statement); programs grouped. A stable
  // counting pass by program, then each program's range stable-sorted on
  // its own (threads when there are many faults): the order of one global
  // stable sort by (prog, step, sub)
  const auto tf0 = std::chrono::steady_clock::now();
  bd->prog_fault_off.assign(P + 1, 0);
  for (const veq_fault &f : bd->faults) bd->prog_fault_off[f.prog + 1]++;
  for (uint32_t p = 0; p < P; p++) bd->prog_fault_off[p + 1] += bd->prog_fault_off[p];
  if (nf && !dev_order) {
    std::vector<veq_fault> by_prog(nf);
    std::vector<uint64_t> at(bd->prog_fault_off.begin(), bd->prog_fault_off.end() - 1);
    for (const veq_fault &f : bd->faults) by_prog[at[f.prog]++] = f;
    bd->faults.swap(by_prog);
    auto sort_prog = [&](uint32_t p) {
      std::stable_sort(bd->faults.begin() + bd->prog_fault_off[p], bd->faults.begin() + bd->prog_fault_off[p + 1],
                       [](const veq_fault &a, const veq_fault &b) {
                         if (a.step != b.step) return a.step < b.step;
                         return a.sub < b.sub;
                       });
    };
    const unsigned nt = nf < (1u << 16) ? 1u : std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
      for (uint32_t p; (p = next.fetch_add(1)) < P;) sort_prog(p);
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; t++) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
  }
  static const bool prof_f = getenv("VEQ_PROF") && getenv("VEQ_PROF")[0] == '1';
  if (prof_f)
    fprintf(stderr, "[veq run_finish] faults %llu, order %.1f ms\n", nf,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tf0).count());
  bd->ran = true;
  ctx->last_faults = nf;
  if (out) {
    out->n_progs = P;
    out->progs = bd->res.data();
    out->n_faults = nf;
    out->faults = bd->faults.data();
    out->n_threads_total = B.n_threads;
    const bool own = !bd->th_state.empty();
    out->thread_state = own ? bd->th_state.data() : ctx->ret_state.data();
    out->thread_block_set = own ? bd->th_bset.data() : ctx->unset_set.data();
    out->thread_block_stmt = own ? bd->th_bstmt.data() : ctx->unset_stmt.data();
    out->n_nodes = nn[0] - nn[4];
    out->n_kid_words = nn[1] - nn[5];
    out->n_work = bd->n_work_last;
    out->n_access = bd->n_access_max;
    uint64_t executed = 0;
    for (uint32_t p = 0; p < P; p++) executed += bd->res[p].steps - bd->res[p].releases;
    out->n_stmts_executed = executed;
    // allocation chunks leave holes (counters[4], [5]); stats count real nodes
    out->n_new_nodes = (nn[0] - nn[4]) - (cnt0[0] - cnt0[4]);
    out->n_new_kid_words = (nn[1] - nn[5]) - (cnt0[1] - cnt0[5]);
    out->n_launches = bd->run_launches;
    out->n_phases = VEQ_MAX_PHASES;
    for (int i = 0; i < VEQ_MAX_PHASES; i++) {
      float ms = 0;
      if (bd->timing_run) cudaEventElapsedTime(&ms, ctx->ev0[i], ctx->ev1[i]);
      out->phase_ms[i] = ms;
    }
  }
  return VEQ_OK;
}

int veq_compare(veq_ctx *ctx, uint32_t ba, uint32_t bb, const uint32_t *out_a, const uint32_t *out_b,
                uint32_t n_out, veq_vc_out *out) {
  if (!ctx || !live_batch(ctx, ba) || !live_batch(ctx, bb)) return VEQ_E_ARG;
  BatchDev *A = ctx->batches[ba], *Bd = ctx->batches[bb];
  if (A->progs.size() != Bd->progs.size()) return fail(ctx, VEQ_E_ARG, "batches differ in program count");
  return veq_compare_progs(ctx, ba, 0, bb, 0, (uint32_t)A->progs.size(), out_a, out_b, n_out, out);
}

// Pair q compares program pa0 + q * a_stride of batch a with pb0 + q of b.
static int compare_impl(veq_ctx *ctx, uint32_t ba, uint32_t pa0, uint32_t a_stride, uint32_t bb, uint32_t pb0,
                        uint32_t n_pairs, const uint32_t *out_a, const uint32_t *out_b, uint32_t n_out,
                        veq_vc_out *out) {
  if (!ctx || !live_batch(ctx, ba) || !live_batch(ctx, bb)) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *A = ctx->batches[ba], *Bd = ctx->batches[bb];
  if (!A->ran || !Bd->ran) return fail(ctx, VEQ_E_ARG, "compare before run");
  if ((uint64_t)pa0 + (uint64_t)(n_pairs ? n_pairs - 1 : 0) * a_stride + (n_pairs ? 1 : 0) > A->progs.size() ||
      (uint64_t)pb0 + n_pairs > Bd->progs.size())
    return fail(ctx, VEQ_E_ARG, "program range out of the batch");
  std::vector<uint32_t> ca, cb;
  for (size_t q = 0; q < n_pairs; q++)
    for (uint32_t k = 0; k < n_out; k++) {
      const size_t p = pa0 + q * a_stride, pb = pb0 + q;
      uint32_t ga = A->progs[p].array_off + out_a[k], gb = Bd->progs[pb].array_off + out_b[k];
      if (out_a[k] >= A->progs[p].n_arrays || out_b[k] >= Bd->progs[pb].n_arrays)
        return fail(ctx, VEQ_E_ARG, "out array index out of range");
      uint64_t n = A->arrays[ga].size;
      uint64_t cba = A->arr_cell_base[ga], cbb = Bd->arr_cell_base[gb];
      for (uint64_t i = 0; i < n; i++) {
        ca.push_back(cba == UNSET64 ? UNSET : (uint32_t)(cba + i));
        cb.push_back(cbb == UNSET64 || i >= Bd->arrays[gb].size ? UNSET : (uint32_t)(cbb + i));
      }
    }
  uint64_t nv = ca.size();
  cudaStream_t s = ctx->stream;
  uint32_t *dca = nullptr, *dcb = nullptr, *scn = nullptr;
  uint8_t *scd = nullptr;
  veq_vc *dv = nullptr;
  unsigned long long *cnt = nullptr;
  uint64_t sc_cap = std::max<uint64_t>(nv * 2, 1024);
  { int r_ = ws_get(ctx, 21, (void **)&dca, std::max<uint64_t>(nv, 1) * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 22, (void **)&dcb, std::max<uint64_t>(nv, 1) * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 23, (void **)&dv, std::max<uint64_t>(nv, 1) * sizeof(veq_vc)); if (r_) return r_; }
  { int r_ = ws_get(ctx, 24, (void **)&scn, sc_cap * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 25, (void **)&scd, sc_cap); if (r_) return r_; }
  { int r_ = ws_get(ctx, 26, (void **)&cnt, 3 * 8); if (r_) return r_; }
  CK(cudaMemsetAsync(cnt, 0, 24, s));
  CK(cudaMemsetAsync(ctx->pool_used, 0, 8, s));
  if (nv) {
    CK(cudaMemcpyAsync(dca, ca.data(), nv * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dcb, cb.data(), nv * 4, cudaMemcpyHostToDevice, s));
    CmpArgs C{dca, dcb, nv, dv, scn, scd, cnt, sc_cap, cnt + 1, cnt + 2};
    uint64_t chunk = std::min<uint64_t>(1ull << 20, std::max<uint64_t>(16ull << 10, ctx->pool_cap / (4 * nv)));
    k_compare<<<blocks(nv, 128), 128, 0, s>>>(ctx->T, A->B.final_node, Bd->B.final_node, C, ctx->pool, ctx->pool_used,
                                              ctx->pool_cap, chunk);
    CK(cudaGetLastError());
  }
  unsigned long long h[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(h, cnt, 24, cudaMemcpyDeviceToHost, s));
  ctx->vcs.resize(nv);
  if (nv) CK(cudaMemcpyAsync(ctx->vcs.data(), dv, nv * sizeof(veq_vc), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  uint64_t nsc = std::min<uint64_t>(h[0], sc_cap);
  ctx->sc_node.resize(nsc);
  ctx->sc_dis.resize(nsc);
  if (nsc) {
    CK(cudaMemcpyAsync(ctx->sc_node.data(), scn, nsc * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->sc_dis.data(), scd, nsc, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  int er = check_error_flag(ctx);
  if (er) return er;
  if (h[0] > sc_cap) return fail(ctx, VEQ_E_BUDGET, "side-condition buffer overflow");
  ctx->last_equal = h[1];
  ctx->last_missing = h[2];
  ctx->last_vcs = nv;
  if (out) {
    out->n_vcs = nv;
    out->vcs = ctx->vcs.data();
    out->n_sc = nsc;
    out->sc_node = ctx->sc_node.data();
    out->sc_discharged = ctx->sc_dis.data();
    out->n_equal = h[1];
    out->n_missing = h[2];
  }
  return VEQ_OK;
}

int veq_compare_progs(veq_ctx *ctx, uint32_t ba, uint32_t pa0, uint32_t bb, uint32_t pb0, uint32_t n_pairs,
                      const uint32_t *out_a, const uint32_t *out_b, uint32_t n_out, veq_vc_out *out) {
  return compare_impl(ctx, ba, pa0, 1, bb, pb0, n_pairs, out_a, out_b, n_out, out);
}

int veq_compare_fan(veq_ctx *ctx, uint32_t ba, uint32_t pa, uint32_t bb, uint32_t pb0, uint32_t n_pairs,
                    const uint32_t *out_a, const uint32_t *out_b, uint32_t n_out, veq_vc_out *out) {
  return compare_impl(ctx, ba, pa, 0, bb, pb0, n_pairs, out_a, out_b, n_out, out);
}

// Host snapshot of the term table: nodes and kid words are append-only
// between veq_clear_terms calls and complete whenever no run is in flight,
// so each sync copies only the ranges created since the previous one.
static int sync_table(veq_ctx *ctx) {
  cudaStream_t s = ctx->stream;
  unsigned long long nn[2];
  CK(cudaMemcpyAsync(nn, ctx->counters, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t NN = std::min<uint64_t>(nn[0], ctx->lim.max_nodes), NK = std::min<uint64_t>(nn[1], ctx->lim.max_kid_words);
  const uint64_t n0 = std::min<uint64_t>(ctx->hnodes.size(), NN), k0 = std::min<uint64_t>(ctx->hkids.size(), NK);
  ctx->hnodes.resize(NN);
  ctx->hkids.resize(NK);
  if (NN > n0)
    CK(cudaMemcpyAsync(ctx->hnodes.data() + n0, ctx->nodes + n0, (NN - n0) * sizeof(Node), cudaMemcpyDeviceToHost, s));
  if (NK > k0) CK(cudaMemcpyAsync(ctx->hkids.data() + k0, ctx->kids + k0, (NK - k0) * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return VEQ_OK;
}

int veq_export_dag(veq_ctx *ctx, const uint32_t *roots, size_t n_roots, veq_dag_buf *buf) {
  if (!ctx || !buf || (n_roots && !roots)) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  if (int r = sync_table(ctx)) return r;
  const std::vector<Node> &nodes = ctx->hnodes;
  const std::vector<uint32_t> &kids = ctx->hkids;
  const uint64_t NN = nodes.size();
  // iterative post-order DFS over the reachable nodes, dense renumbering
  struct Idx {
    std::unordered_map<uint32_t, uint32_t> m;
    uint32_t &operator[](uint32_t x) { return m.try_emplace(x, UNSET).first->second; }
  } idx;
  std::vector<uint32_t> order;
  for (size_t r = 0; r < n_roots; r++) {
    if (roots[r] >= NN) return fail(ctx, VEQ_E_ARG, "root id out of range");
    std::vector<std::pair<uint32_t, uint32_t>> st{{roots[r], 0}};
    while (!st.empty()) {
      auto &[x, k] = st.back();
      if (idx[x] != UNSET) {
        st.pop_back();
        continue;
      }
      const Node &n = nodes[x];
      bool comp = n.kind != K_CONST && n.kind != K_VAR && n.kind != K_NEGINF;
      if (comp && k < n.nkids) {
        uint32_t kid = kids[n.p0 + k];
        k++;
        if (kid >= NN) return fail(ctx, VEQ_E_INVALID_IR, "kid id out of range");
        if (idx[kid] == UNSET) st.push_back({kid, 0});
        continue;
      }
      idx[x] = (uint32_t)order.size();
      order.push_back(x);
      st.pop_back();
    }
  }
  uint64_t total_kids = 0;
  for (uint32_t x : order) {
    const Node &n = nodes[x];
    if (n.kind != K_CONST && n.kind != K_VAR && n.kind != K_NEGINF) total_kids += n.nkids;
  }
  uint64_t cap_n = buf->cap_nodes, cap_k = buf->cap_kids;
  buf->n_nodes = order.size();
  buf->n_kids = total_kids;
  // sizing call: capacities too small or no node buffer (the kid buffer may
  // be null when there are no kids)
  if (cap_n < order.size() || cap_k < total_kids || !buf->nodes || !buf->root_index || (total_kids && !buf->kids))
    return VEQ_OK;
  uint64_t ko = 0;
  for (size_t i = 0; i < order.size(); i++) {
    const Node &n = nodes[order[i]];
    veq_dag_node &o = buf->nodes[i];
    o.kind = n.kind;
    o.nkids = 0;
    o.kid_off = ko;
    o.num = 0;
    o.den = 1;
    o.var_input = -1;
    o.var_index = 0;
    if (n.kind == K_CONST) {
      o.num = (int64_t)n.p0;
      o.den = (int64_t)n.p1;
    } else if (n.kind == K_VAR) {
      if (n.p0 >= INPUT_KEY) {
        o.var_input = (int64_t)(n.p1 >> 40);
        o.var_index = n.p1 & ((1ull << 40) - 1);
      } else {
        o.var_input = -1;
        o.var_index = n.p1;
      }
    } else if (n.kind != K_NEGINF) {
      o.nkids = n.nkids;
      for (uint32_t k = 0; k < n.nkids; k++) buf->kids[ko++] = idx[kids[n.p0 + k]];
    }
  }
  for (size_t r = 0; r < n_roots; r++) buf->root_index[r] = idx[roots[r]];
  return VEQ_OK;
}

}  // extern "C"

// ---- to_string of device terms (proj/src/expr.cpp:735-822) ----------------
namespace {

// Byte sinks: a string, or CRC-32 (IEEE, zlib.crc32) + length.
struct StrSink {
  std::string *out;
  void put(const char *p, size_t n) { out->append(p, n); }
};
struct CrcSink {
  uint32_t c = 0xFFFFFFFFu;
  uint64_t n = 0;
  static const uint32_t *table() {
    static uint32_t t[256];
    static bool init = false;
    if (!init) {
      for (uint32_t i = 0; i < 256; i++) {
        uint32_t x = i;
        for (int k = 0; k < 8; k++) x = (x & 1) ? 0xEDB88320u ^ (x >> 1) : x >> 1;
        t[i] = x;
      }
      init = true;
    }
    return t;
  }
  void put(const char *p, size_t len) {
    const uint32_t *t = table();
    for (size_t i = 0; i < len; i++) c = t[(c ^ (unsigned char)p[i]) & 0xff] ^ (c >> 8);
    n += len;
  }
};

// CRC-32 of a concatenation from the parts' CRCs and lengths (GF(2)
// polynomial arithmetic modulo the reflected IEEE polynomial, the method of
// zlib's crc32_combine): memoised per node, a DAG's text digest costs one
// combine per edge instead of one table step per byte of its (possibly
// exponentially larger) text.
struct CrcCat {
  static uint32_t mulmod(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
      if (a & m) {
        p ^= b;
        if ((a & (m - 1)) == 0) break;
      }
      m >>= 1;
      b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
  }
  uint32_t x2n[64];
  CrcCat() {
    uint32_t p = 1u << 30;  // x^1
    x2n[0] = p;
    for (int k = 1; k < 64; k++) x2n[k] = p = mulmod(p, p);
  }
  uint32_t xpow8(uint64_t n) const {  // x^(8n) mod P
    uint32_t p = 1u << 31;
    for (int k = 3; n; n >>= 1, k++)
      if (n & 1) p = mulmod(x2n[k & 63], p);
    return p;
  }
  struct D {
    uint32_t crc;
    uint64_t len;
  };
  D cat(D a, D b) const { return b.len == 0 ? a : D{mulmod(xpow8(b.len), a.crc) ^ b.crc, a.len + b.len}; }
  static D of(const char *s, size_t n) {
    CrcSink k;
    k.put(s, n);
    return D{k.c ^ 0xFFFFFFFFu, k.n};
  }
};

struct Printer {
  const std::vector<Node> &N;
  const std::vector<uint32_t> &K;
  const std::vector<std::string> &inputs;
  static int prec(uint8_t k) { return k == K_ADD ? 1 : (k == K_MUL || k == K_DIV) ? 2 : k == K_NEG ? 3 : 4; }
  template <class S> void lit(S &o, const char *s) { o.put(s, strlen(s)); }
  template <class S> void print(uint32_t id, int ctx, S &o) {
    const Node &n = N[id];
    const bool paren = prec(n.kind) < ctx;
    if (paren) o.put("(", 1);
    char buf[64];
    switch (n.kind) {
    case K_CONST: {
      const long long num = (long long)n.p0, den = (long long)n.p1;
      int l = den == 1 ? snprintf(buf, sizeof buf, "%lld", num) : snprintf(buf, sizeof buf, "%lld/%lld", num, den);
      o.put(buf, l);
      break;
    }
    case K_VAR: {
      if (n.p0 >= INPUT_KEY) {
        const std::string &nm = inputs[n.p1 >> 40];
        o.put(nm.data(), nm.size());
        int l = snprintf(buf, sizeof buf, "_%llu", (unsigned long long)(n.p1 & ((1ull << 40) - 1)));
        o.put(buf, l);
      } else {
        int l = snprintf(buf, sizeof buf, "!undef<%llx>", (unsigned long long)n.p1);
        o.put(buf, l);
      }
      break;
    }
    case K_NEGINF: lit(o, "-inf"); break;
    case K_ADD:
    case K_MUL:
    case K_MAX: {
      const char *sep = n.kind == K_ADD ? " + " : (n.kind == K_MUL ? "*" : ", ");
      const int kc = n.kind == K_ADD ? 2 : (n.kind == K_MUL ? 3 : 0);
      if (n.kind == K_MAX) lit(o, "max(");
      for (uint32_t i = 0; i < n.nkids; i++) {
        if (i) lit(o, sep);
        print(K[n.p0 + i], kc, o);
      }
      if (n.kind == K_MAX) lit(o, ")");
      break;
    }
    case K_DIV:
      print(K[n.p0], 3, o);
      lit(o, " / ");
      print(K[n.p0 + 1], 3, o);
      break;
    case K_NEG:
      lit(o, "-");
      print(K[n.p0], 3, o);
      break;
    case K_EXP:
      lit(o, "exp(");
      print(K[n.p0], 0, o);
      lit(o, ")");
      break;
    default: break;
    }
    if (paren) o.put(")", 1);
  }
};

}  // namespace

extern "C" {

int veq_render(veq_ctx *ctx, const uint32_t *roots, size_t n_roots, const char **text, const uint64_t **offs) {
  if (!ctx || (n_roots && !roots) || !text || !offs) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  if (int r = sync_table(ctx)) return r;
  const std::vector<Node> &nodes = ctx->hnodes;
  Printer P{ctx->hnodes, ctx->hkids, ctx->input_names};
  ctx->render_text.clear();
  ctx->render_offs.assign(1, 0);
  StrSink sink{&ctx->render_text};
  for (size_t i = 0; i < n_roots; i++) {
    if (roots[i] >= nodes.size()) return fail(ctx, VEQ_E_ARG, "root id out of range");
    P.print(roots[i], 0, sink);
    ctx->render_offs.push_back(ctx->render_text.size());
  }
  *text = ctx->render_text.data();
  *offs = ctx->render_offs.data();
  return VEQ_OK;
}

int veq_render_digest(veq_ctx *ctx, const uint32_t *roots, size_t n_roots, uint32_t *crc32, uint64_t *len) {
  if (!ctx || (n_roots && (!roots || !crc32 || !len))) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  if (int r = sync_table(ctx)) return r;
  const std::vector<Node> &nodes = ctx->hnodes;
  const std::vector<uint32_t> &kids = ctx->hkids;
  Printer P{ctx->hnodes, ctx->hkids, ctx->input_names};
  static const CrcCat C;
  using D = CrcCat::D;
  // memo of each node's unparenthesised text digest; atoms are printed
  std::vector<D> memo(nodes.size(), D{0, ~0ull});
  const D lp = CrcCat::of("(", 1), rp = CrcCat::of(")", 1);
  std::function<D(uint32_t, int)> dig = [&](uint32_t id, int c) -> D {
    const Node &n = nodes[id];
    D core;
    if (n.kind == K_CONST || n.kind == K_VAR || n.kind == K_NEGINF) {
      std::string t;
      StrSink sk{&t};
      P.print(id, 0, sk);
      core = CrcCat::of(t.data(), t.size());
    } else if (memo[id].len != ~0ull) {
      core = memo[id];
    } else {
      const char *sep = n.kind == K_ADD ? " + " : (n.kind == K_MUL ? "*" : (n.kind == K_MAX ? ", " : " / "));
      const D ds = CrcCat::of(sep, strlen(sep));
      const int kc = n.kind == K_ADD ? 2 : (n.kind == K_MAX || n.kind == K_EXP) ? 0 : 3;
      core = n.kind == K_MAX ? CrcCat::of("max(", 4) : n.kind == K_EXP ? CrcCat::of("exp(", 4)
                                                     : n.kind == K_NEG ? CrcCat::of("-", 1) : D{0, 0};
      for (uint32_t k = 0; k < n.nkids; k++) {
        if (k) core = C.cat(core, ds);
        core = C.cat(core, dig(kids[n.p0 + k], kc));
      }
      if (n.kind == K_MAX || n.kind == K_EXP) core = C.cat(core, rp);
      memo[id] = core;
    }
    return Printer::prec(n.kind) < c ? C.cat(C.cat(lp, core), rp) : core;
  };
  for (size_t i = 0; i < n_roots; i++) {
    if (roots[i] >= nodes.size()) return fail(ctx, VEQ_E_ARG, "root id out of range");
    const D d = dig(roots[i], 0);
    crc32[i] = d.crc;
    len[i] = d.len;
  }
  return VEQ_OK;
}

int veq_fetch_cells(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t array, uint32_t *out_nodes, uint64_t n) {
  if (!ctx || !live_batch(ctx, batch) || (n && !out_nodes)) return VEQ_E_ARG;
  BatchDev *bd = ctx->batches[batch];
  if (!bd->ran || prog >= bd->progs.size() || array >= bd->progs[prog].n_arrays) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  uint32_t ga = bd->progs[prog].array_off + array;
  uint64_t size = bd->arrays[ga].size, cb = bd->arr_cell_base[ga];
  if (n > size) n = size;
  if (cb == UNSET64) {
    std::fill(out_nodes, out_nodes + n, UNSET);
    return VEQ_OK;
  }
  if (n) {
    CK(cudaMemcpyAsync(out_nodes, bd->B.final_node + cb, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return VEQ_OK;
}

int veq_drop_batch(veq_ctx *ctx, uint32_t batch) {
  if (!ctx || !live_batch(ctx, batch)) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (bd->started) return fail(ctx, VEQ_E_ARG, "veq_drop_batch: run not finished");
  drop_batch(ctx, bd);
  ctx->batches[batch] = nullptr;
  return VEQ_OK;
}

int veq_load_template(veq_ctx *ctx, const veq_batch_desc *d, uint32_t *out) {
  if (!ctx || !d || !out || !d->n_progs) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  TemplateDev *t = new TemplateDev();
  t->progs.assign(d->progs, d->progs + d->n_progs);
  t->thread_stmt.assign(d->thread_stmt, d->thread_stmt + d->n_threads_total + 1);
  t->thread_nregs.assign(d->thread_nregs, d->thread_nregs + d->n_threads_total);
  t->arrays.assign(d->arrays, d->arrays + d->n_arrays_total);
  t->consts.assign(d->consts, d->consts + d->n_consts);
  t->syncsets.assign(d->syncsets, d->syncsets + d->n_syncsets);
  t->set_words.assign(d->set_words, d->set_words + d->n_set_words);
  t->n_stmts = d->n_stmts;
  for (uint32_t p = 0; p < d->n_progs; p++) {
    const veq_program_meta &m = t->progs[p];
    // programs must be laid out in order (threads, arrays and statements)
    const bool ok = m.thread_off + m.n_threads <= d->n_threads_total && m.array_off + m.n_arrays <= d->n_arrays_total &&
                    (p == 0 ? m.thread_off == 0 && m.array_off == 0
                            : m.thread_off == t->progs[p - 1].thread_off + t->progs[p - 1].n_threads &&
                                  m.array_off == t->progs[p - 1].array_off + t->progs[p - 1].n_arrays);
    if (!ok) {
      delete t;
      return fail(ctx, VEQ_E_INVALID_IR, "template programs are not laid out in order");
    }
  }
  if (cudaMallocAsync(&t->stmts, std::max<uint64_t>(d->n_stmts, 1) * sizeof(veq_stmt), ctx->stream) != cudaSuccess) {
    delete t;
    return fail(ctx, VEQ_E_OOM, "template statements");
  }
  if (d->n_stmts)
    CK(cudaMemcpyAsync(t->stmts, d->stmts, d->n_stmts * sizeof(veq_stmt), cudaMemcpyHostToDevice, ctx->stream));
  ctx->templates.push_back(t);
  *out = (uint32_t)(ctx->templates.size() - 1);
  return VEQ_OK;
}

int veq_drop_template(veq_ctx *ctx, uint32_t tmpl) {
  if (!ctx || tmpl >= ctx->templates.size() || !ctx->templates[tmpl]) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  cudaFreeAsync(ctx->templates[tmpl]->stmts, ctx->stream);
  delete ctx->templates[tmpl];
  ctx->templates[tmpl] = nullptr;
  return VEQ_OK;
}

int veq_instantiate(veq_ctx *ctx, uint32_t tmpl, uint32_t n_inst, const int32_t *deltas, uint32_t *out) {
  if (!ctx || !out || !n_inst || tmpl >= ctx->templates.size() || !ctx->templates[tmpl]) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  const TemplateDev &t = *ctx->templates[tmpl];
  const uint32_t Q = (uint32_t)t.progs.size(), NA = (uint32_t)t.arrays.size();
  // program-major expansion: program q * n_inst + i is template program q of
  // instance i, so each template program's instances form one range
  // sized up front and filled by block copies: every instance of template
  // program q repeats q's thread table shifted by a constant
  uint64_t n_thr = 0, n_arr = 0;
  for (uint32_t q = 0; q < Q; q++) {
    n_thr += (uint64_t)t.progs[q].n_threads * n_inst;
    n_arr += (uint64_t)t.progs[q].n_arrays * n_inst;
  }
  if (n_thr >= (1ull << 32)) return fail(ctx, VEQ_E_UNSUPPORTED, "instantiated batch has more than 2^32 threads");
  std::vector<veq_program_meta> progs((size_t)Q * n_inst);
  std::vector<uint64_t> thread_stmt(n_thr + 1);
  std::vector<uint32_t> thread_nregs(n_thr);
  std::vector<veq_array> arrays(n_arr);
  std::vector<ExpandSeg> segs;
  uint64_t so = 0, to = 0, ao = 0;
  thread_stmt[0] = 0;
  for (uint32_t q = 0; q < Q; q++) {
    const veq_program_meta &m = t.progs[q];
    const uint64_t s0 = t.thread_stmt[m.thread_off], s1 = t.thread_stmt[m.thread_off + m.n_threads];
    segs.push_back(ExpandSeg{so, s0, s1 - s0, m.array_off});
    const uint64_t *ts = t.thread_stmt.data() + m.thread_off;
    for (uint32_t i = 0; i < n_inst; i++) {
      veq_program_meta pm = m;
      pm.thread_off = (uint32_t)to;
      pm.array_off = (uint32_t)ao;
      progs[(size_t)q * n_inst + i] = pm;
      std::copy(t.thread_nregs.begin() + m.thread_off, t.thread_nregs.begin() + m.thread_off + m.n_threads,
                thread_nregs.begin() + to);
      const uint64_t shift = so + (s1 - s0) * i - s0;  // instance i's first statement, minus the template's
      for (uint32_t k = 1; k <= m.n_threads; k++) thread_stmt[to + k] = ts[k] + shift;
      std::copy(t.arrays.begin() + m.array_off, t.arrays.begin() + m.array_off + m.n_arrays, arrays.begin() + ao);
      to += m.n_threads;
      ao += m.n_arrays;
    }
    so += (s1 - s0) * n_inst;
  }
  const uint64_t S = so;
  if (S >= (1ull << 31)) return fail(ctx, VEQ_E_UNSUPPORTED, "instantiated batch has more than 2^31 statements");
  veq_stmt *ds = nullptr;
  int32_t *dd = nullptr;
  ExpandSeg *dseg = nullptr;
  cudaStream_t s = ctx->stream;
  if (cudaMallocAsync(&ds, std::max<uint64_t>(S, 1) * sizeof(veq_stmt), s) != cudaSuccess)
    return fail(ctx, VEQ_E_OOM, "instantiated statements");
  if (cudaMallocAsync(&dd, std::max<uint64_t>((uint64_t)n_inst * NA, 1) * 4, s) != cudaSuccess ||
      cudaMallocAsync(&dseg, Q * sizeof(ExpandSeg), s) != cudaSuccess) {
    cudaFreeAsync(ds, s);
    return fail(ctx, VEQ_E_OOM, "instance deltas");
  }
  if (NA) CK(cudaMemcpyAsync(dd, deltas, (uint64_t)n_inst * NA * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dseg, segs.data(), Q * sizeof(ExpandSeg), cudaMemcpyHostToDevice, s));
  if (S) {
    ctx->launches++;
    k_expand_stmts<<<blocks(S, 256), 256, 0, s>>>(t.stmts, dseg, Q, n_inst, dd, NA, ds, S);
  }
  CK(cudaGetLastError());
  CK(cudaFreeAsync(dd, s));
  CK(cudaFreeAsync(dseg, s));
  veq_batch_desc bd{};
  bd.n_progs = (uint32_t)progs.size();
  bd.n_threads_total = (uint32_t)thread_nregs.size();
  bd.n_stmts = S;
  bd.n_arrays_total = (uint32_t)arrays.size();
  bd.n_consts = (uint32_t)t.consts.size();
  bd.n_syncsets = (uint32_t)t.syncsets.size();
  bd.n_set_words = (uint32_t)t.set_words.size();
  bd.progs = progs.data();
  bd.thread_stmt = thread_stmt.data();
  bd.thread_nregs = thread_nregs.data();
  bd.stmts = nullptr;
  bd.arrays = arrays.data();
  bd.consts = t.consts.data();
  bd.syncsets = t.syncsets.data();
  bd.set_words = t.set_words.data();
  return load_impl(ctx, &bd, ds, out);
}

int veq_set_option(veq_ctx *ctx, int option, int value) {
  if (!ctx) return VEQ_E_ARG;
  switch (option) {
  case VEQ_OPT_KEEP_REGS: ctx->keep_regs = value != 0; return VEQ_OK;
  default: return fail(ctx, VEQ_E_ARG, "unknown option");
  }
}

int veq_fetch_regs(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t tid, uint32_t *out_nodes, uint32_t n,
                   uint32_t *n_regs) {
  if (!ctx || !live_batch(ctx, batch) || !n_regs) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (!bd->ran || prog >= bd->progs.size() || tid >= bd->progs[prog].n_threads) return VEQ_E_ARG;
  if (!bd->keep_regs) return fail(ctx, VEQ_E_ARG, "veq_fetch_regs: run without VEQ_OPT_KEEP_REGS");
  const uint32_t g = bd->progs[prog].thread_off + tid;
  uint64_t off[2];
  CK(cudaMemcpy(off, bd->B.reg_off + g, 16, cudaMemcpyDeviceToHost));
  const uint32_t nr = (uint32_t)(off[1] - off[0]);
  *n_regs = nr;
  if (!out_nodes) return VEQ_OK;
  std::vector<uint32_t> v(nr);
  if (nr) CK(cudaMemcpy(v.data(), bd->B.regfile + off[0], nr * 4, cudaMemcpyDeviceToHost));
  for (uint32_t k = 0; k < nr && k < n; k++) {
    uint32_t x = v[k];
    if (x == UNSET) {
      out_nodes[k] = UNSET;
    } else if (x & REF_NODE) {
      out_nodes[k] = x & ~REF_NODE;
    } else {
      CK(cudaMemcpy(&out_nodes[k], bd->B.canon + x, 4, cudaMemcpyDeviceToHost));
    }
  }
  return VEQ_OK;
}

int veq_batch_locs(veq_ctx *ctx, uint32_t batch, const uint64_t *loc_keys) {
  if (!ctx || !live_batch(ctx, batch)) return VEQ_E_ARG;
  BatchDev *bd = ctx->batches[batch];
  if (loc_keys) bd->locs.assign(loc_keys, loc_keys + bd->n_stmts);
  else bd->locs.clear();
  return VEQ_OK;
}

static bool set_has(const BatchDev *bd, uint32_t set, uint32_t n_threads, uint32_t tid) {
  if (set >= bd->syncsets.size()) return tid < n_threads;  // the program's full set
  const veq_syncset &q = bd->syncsets[set];
  if (q.full) return tid < n_threads;
  if (tid < q.lo || tid >= q.lo + q.n_bits) return false;
  const uint32_t k = tid - q.lo;
  return (bd->set_words[q.word_off + k / 64] >> (k % 64)) & 1ull;
}

int veq_set_members(veq_ctx *ctx, uint32_t batch, uint32_t prog, uint32_t set, uint32_t *tids, uint32_t cap,
                    uint32_t *n) {
  if (!ctx || !live_batch(ctx, batch) || !n) return VEQ_E_ARG;
  BatchDev *bd = ctx->batches[batch];
  if (prog >= bd->progs.size()) return VEQ_E_ARG;
  const uint32_t T = bd->progs[prog].n_threads;
  uint32_t k = 0;
  for (uint32_t t = 0; t < T; t++)
    if (set_has(bd, set, T, t)) {
      if (tids && k < cap) tids[k] = t;
      k++;
    }
  *n = k;
  return VEQ_OK;
}

// One program's RunResult from the ordered raw faults (Collector,
// symexec.cpp:308-328; make_deadlock_report, 335-365; precedence, 838-845).
// `st`: the statements of the batch's safety faults (register operands).
static void assemble_report(BatchDev *bd, uint32_t prog, const std::unordered_map<uint32_t, veq_stmt> &st,
                            BatchDev::RepStore &R, veq_report *out) {
  const veq_program_meta &pm = bd->progs[prog];
  auto loc = [&](uint32_t stmt) -> uint64_t { return bd->locs.empty() ? stmt : bd->locs[stmt]; };
  const uint64_t f0 = bd->prog_fault_off[prog], f1 = bd->prog_fault_off[prog + 1];
  R.races.clear();
  R.safeties.clear();
  R.threads.clear();
  // Collector (proj/src/symexec.cpp:308-328): distinct reports in order of
  // first occurrence; identity excludes step numbers
  FlatSet<5> rkeys;
  FlatSet<3> skeys;
  rkeys.init(f1 - f0);
  skeys.init(f1 - f0);
  for (uint64_t k = f0; k < f1; k++) {
    const veq_fault &f = bd->faults[k];
    if (f.type == VEQ_FAULT_RACE) {
      veq_race_report r{};
      r.arr = f.arr;
      r.offset = f.offset;
      r.first = veq_access{f.tid2, f.stmt2, f.step2, f.is_write2, 0};
      r.second = veq_access{f.tid, f.stmt, f.step, f.is_write, 0};
      if (rkeys.insert({((uint64_t)r.arr << 32) | (uint32_t)r.offset,
                        ((uint64_t)f.tid2 << 32) | ((uint64_t)f.is_write2 << 1) | f.is_write, loc(f.stmt2),
                        (uint64_t)f.tid, loc(f.stmt)}))
        R.races.push_back(r);
      continue;
    }
    veq_safety_report s{};
    s.kind = f.kind;
    s.tid = f.tid;
    s.stmt = f.stmt;
    s.step = f.step;
    s.detail = f.detail;
    s.reg = UNSET;
    const veq_stmt &x = st.at(f.stmt);
    if (f.kind == VEQ_SAFE_UNINIT_REG) {
      s.reg = f.reg_slot == 1 ? x.b : (x.kind == VEQ_ST_STORE ? x.dst : x.a);
    } else if (f.kind == VEQ_SAFE_UNINIT_MEM || f.kind == VEQ_SAFE_OOB) {
      s.has_addr = 1;
      s.arr = f.arr;
      s.offset = f.offset;
      s.is_store = f.kind == VEQ_SAFE_OOB ? f.is_write : 0;
    } else {
      s.reg = x.dst;  // invalid arithmetic: the destination register
    }
    if (skeys.insert({((uint64_t)s.kind << 56) | ((uint64_t)s.detail << 48) | ((uint64_t)s.is_store << 40) |
                          ((uint64_t)s.has_addr << 32) | s.tid,
                      loc(s.stmt),
                      ((uint64_t)(s.has_addr ? s.arr : s.reg) << 32) | (uint32_t)(s.has_addr ? s.offset : 0)}))
      R.safeties.push_back(s);
  }
  const veq_prog_result &pr = bd->res[prog];
  out->steps = pr.steps;
  out->releases = pr.releases;
  out->deadlocked = pr.deadlocked;
  out->conflict_a = out->conflict_b = -1;
  out->conflict_set_a = out->conflict_set_b = UNSET;
  out->n_threads = 0;
  if (pr.deadlocked && !bd->th_state.empty()) {
    // make_deadlock_report (symexec.cpp:335-365): every thread's state; the
    // first a < b blocked on different sets with a, b in both sets
    const uint32_t T = pm.n_threads, g0 = pm.thread_off;
    for (uint32_t t = 0; t < T; t++) {
      const uint8_t sv = bd->th_state[g0 + t];
      R.threads.push_back(veq_thread_report{sv, sv == TS_BLOCK ? bd->th_bset[g0 + t] : UNSET,
                                                  sv == TS_BLOCK ? (uint32_t)bd->th_bstmt[g0 + t] : UNSET, 0});
    }
    for (uint32_t a = 0; a < T && out->conflict_a < 0; a++) {
      if (R.threads[a].state != TS_BLOCK) continue;
      const uint32_t ia = R.threads[a].set;
      for (uint32_t b = a + 1; b < T; b++) {
        if (R.threads[b].state != TS_BLOCK) continue;
        const uint32_t ib = R.threads[b].set;
        if (ia == ib) continue;  // canonical set ids: equal content <=> equal id
        if (set_has(bd, ia, T, a) && set_has(bd, ia, T, b) && set_has(bd, ib, T, a) && set_has(bd, ib, T, b)) {
          out->conflict_a = (int32_t)a;
          out->conflict_b = (int32_t)b;
          out->conflict_set_a = ia;
          out->conflict_set_b = ib;
          break;
        }
      }
    }
    out->n_threads = T;
  }
  out->n_races = R.races.size();
  out->races = R.races.data();
  out->n_safeties = R.safeties.size();
  out->safeties = R.safeties.data();
  out->threads = R.threads.data();
  // precedence (symexec.cpp:838-845): race, else safety, else deadlock, else final
  out->outcome = !R.races.empty() ? VEQ_OUT_RACE
                 : !R.safeties.empty() ? VEQ_OUT_SAFETY
                 : pr.deadlocked ? VEQ_OUT_DEADLOCK : VEQ_OUT_FINAL;
}

// The statements of the safety faults of some programs, in one gather.
static int fetch_fault_stmts(veq_ctx *ctx, BatchDev *bd, const uint32_t *progs, uint32_t n,
                             std::unordered_map<uint32_t, veq_stmt> &st) {
  std::vector<uint32_t> ids;
  for (uint32_t q = 0; q < n; q++)
    for (uint64_t k = bd->prog_fault_off[progs[q]]; k < bd->prog_fault_off[progs[q] + 1]; k++)
      if (bd->faults[k].type == VEQ_FAULT_SAFETY && st.emplace(bd->faults[k].stmt, veq_stmt{}).second)
        ids.push_back(bd->faults[k].stmt);
  if (ids.empty()) return VEQ_OK;
  cudaStream_t s = ctx->stream;
  uint32_t *di = nullptr;
  veq_stmt *dst = nullptr;
  { int r_ = ws_get(ctx, 38, (void **)&di, ids.size() * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 39, (void **)&dst, ids.size() * sizeof(veq_stmt)); if (r_) return r_; }
  CK(cudaMemcpyAsync(di, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, s));
  k_gather_stmts<<<blocks(ids.size(), 256), 256, 0, s>>>(bd->B.stmts, di, ids.size(), dst);
  CK(cudaGetLastError());
  std::vector<veq_stmt> h(ids.size());
  CK(cudaMemcpyAsync(h.data(), dst, ids.size() * sizeof(veq_stmt), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (size_t k = 0; k < ids.size(); k++) st[ids[k]] = h[k];
  return VEQ_OK;
}

int veq_run_report(veq_ctx *ctx, uint32_t batch, uint32_t prog, veq_report *out) {
  if (!ctx || !live_batch(ctx, batch) || !out) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (!bd->ran || prog >= bd->progs.size()) return fail(ctx, VEQ_E_ARG, "veq_run_report: no finished run / bad program");
  std::unordered_map<uint32_t, veq_stmt> st;
  if (int r = fetch_fault_stmts(ctx, bd, &prog, 1, st)) return r;
  assemble_report(bd, prog, st, bd->rep, out);
  return VEQ_OK;
}

int veq_run_reports(veq_ctx *ctx, uint32_t batch, const uint32_t *progs, uint32_t n, veq_report *outs) {
  if (!ctx || !live_batch(ctx, batch) || (n && (!progs || !outs))) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  BatchDev *bd = ctx->batches[batch];
  if (!bd->ran) return fail(ctx, VEQ_E_ARG, "veq_run_reports: no finished run");
  for (uint32_t q = 0; q < n; q++)
    if (progs[q] >= bd->progs.size()) return fail(ctx, VEQ_E_ARG, "veq_run_reports: bad program");
  std::unordered_map<uint32_t, veq_stmt> st;
  if (int r = fetch_fault_stmts(ctx, bd, progs, n, st)) return r;
  bd->rep_many.resize(n);
  // programs are independent: assembled on a thread pool
  const unsigned nt = (unsigned)std::min<uint64_t>(n, std::max(1u, std::thread::hardware_concurrency()));
  std::atomic<uint32_t> next{0};
  auto work = [&]() {
    for (uint32_t q; (q = next.fetch_add(1)) < n;) assemble_report(bd, progs[q], st, bd->rep_many[q], outs + q);
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; t++) th.emplace_back(work);
  work();
  for (auto &t : th) t.join();
  return VEQ_OK;
}

int veq_comm_unique_id(void *id_out) {
  if (!id_out) return VEQ_E_ARG;
  if (!nccl().ok) return VEQ_E_UNSUPPORTED;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return VEQ_E_CUDA;
  memcpy(id_out, &id, sizeof(id));
  return VEQ_OK;
}

int veq_comm_init(veq_ctx *ctx, const void *nccl_unique_id, int nranks, int rank) {
  if (!ctx || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return VEQ_E_ARG;
  if (!nccl().ok) return fail(ctx, VEQ_E_UNSUPPORTED, "libnccl.so.2 not available");
  CK(cudaSetDevice(ctx->device));
  veq_comm_destroy_(ctx);
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  NK(nccl().CommInitRank(&ctx->comm, nranks, id, rank));
  ctx->nranks = nranks;
  ctx->rank = rank;
  return VEQ_OK;
}

// The one exchange of a sharded check: every rank calls it
// after its veq_compare / veq_compare_progs. Sum all-reduce of the verdict
// counters, min all-reduce of the first failing VC index, and all-gather of
// every rank's per-VC verdict bytes and side-condition (Merkle hash,
// discharged) pairs in rank order, so any rank can aggregate the report as
// check_equivalence does (proj/src/pipeline.cpp:245-266). Without a
// communicator it returns this rank's own results.
int veq_comm_combine(veq_ctx *ctx, uint64_t first_fail_local, veq_combined *out) {
  if (!ctx || !out) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const uint64_t nv = ctx->vcs.size(), ns = ctx->sc_node.size();
  // this rank's verdict bytes and side-condition hashes
  std::vector<uint8_t> verd(nv);
  for (uint64_t i = 0; i < nv; i++) verd[i] = ctx->vcs[i].equal ? 1 : 0;
  std::vector<uint64_t> hs(ns);
  for (uint64_t i = 0; i < ns; i++)
    CK(cudaMemcpy(&hs[i], reinterpret_cast<const char *>(ctx->nodes + ctx->sc_node[i]) + 8, 8, cudaMemcpyDeviceToHost));
  const int R = ctx->comm ? ctx->nranks : 1;
  std::vector<unsigned long long> h(6 * (size_t)R, 0);
  unsigned long long mine[6] = {ctx->last_equal, ctx->last_vcs, ctx->last_faults, ctx->last_missing,
                                (unsigned long long)nv, (unsigned long long)ns};
  ctx->rank_vc_off.assign(R + 1, 0);
  ctx->rank_sc_off.assign(R + 1, 0);
  unsigned long long first = first_fail_local;
  if (!ctx->comm) {
    for (int k = 0; k < 6; k++) h[k] = mine[k];
  } else {
    // sizes and counters of every rank, then the min first-failing index
    unsigned long long *d = nullptr;
    if (cudaMallocAsync(&d, (6 + 6 * (size_t)R + 1) * 8, s) != cudaSuccess) return fail(ctx, VEQ_E_OOM, "comm");
    CK(cudaMemcpyAsync(d, mine, 48, cudaMemcpyHostToDevice, s));
    NK(nccl().AllGather(d, d + 6, 6, ncclUint64, ctx->comm, s));
    CK(cudaMemcpyAsync(d + 6 + 6 * R, &first, 8, cudaMemcpyHostToDevice, s));
    NK(nccl().AllReduce(d + 6 + 6 * R, d + 6 + 6 * R, 1, ncclUint64, ncclMin, ctx->comm, s));
    CK(cudaMemcpyAsync(h.data(), d + 6, 6 * R * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&first, d + 6 + 6 * R, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaFreeAsync(d, s));
  }
  uint64_t maxv = 0, maxs = 0;
  for (int r = 0; r < R; r++) {
    ctx->rank_vc_off[r + 1] = ctx->rank_vc_off[r] + h[6 * r + 4];
    ctx->rank_sc_off[r + 1] = ctx->rank_sc_off[r] + h[6 * r + 5];
    maxv = std::max<uint64_t>(maxv, h[6 * r + 4]);
    maxs = std::max<uint64_t>(maxs, h[6 * r + 5]);
  }
  ctx->all_verdict.assign(ctx->rank_vc_off[R], 0);
  ctx->all_sc_hash.assign(ctx->rank_sc_off[R], 0);
  ctx->all_sc_dis.assign(ctx->rank_sc_off[R], 0);
  if (!ctx->comm) {
    std::copy(verd.begin(), verd.end(), ctx->all_verdict.begin());
    std::copy(hs.begin(), hs.end(), ctx->all_sc_hash.begin());
    std::copy(ctx->sc_dis.begin(), ctx->sc_dis.end(), ctx->all_sc_dis.begin());
  } else if (maxv || maxs) {
    // equal-size all-gathers of padded per-rank buffers (verdict bytes,
    // hashes, discharged bytes), compacted to rank order on the host
    const uint64_t rec = maxv + maxs * 9;
    char *d = nullptr;
    if (cudaMallocAsync(&d, rec * (R + 1) + 8, s) != cudaSuccess) return fail(ctx, VEQ_E_OOM, "comm");
    std::vector<char> me(rec, 0);
    memcpy(me.data(), verd.data(), nv);
    memcpy(me.data() + maxv, hs.data(), ns * 8);
    memcpy(me.data() + maxv + maxs * 8, ctx->sc_dis.data(), ns);
    CK(cudaMemcpyAsync(d, me.data(), rec, cudaMemcpyHostToDevice, s));
    NK(nccl().AllGather(d, d + rec, rec, ncclChar, ctx->comm, s));
    std::vector<char> all(rec * R);
    CK(cudaMemcpyAsync(all.data(), d + rec, rec * R, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaFreeAsync(d, s));
    for (int r = 0; r < R; r++) {
      const char *b = all.data() + rec * r;
      const uint64_t v0 = ctx->rank_vc_off[r], s0 = ctx->rank_sc_off[r];
      memcpy(ctx->all_verdict.data() + v0, b, h[6 * r + 4]);
      memcpy(ctx->all_sc_hash.data() + s0, b + maxv, h[6 * r + 5] * 8);
      memcpy(ctx->all_sc_dis.data() + s0, b + maxv + maxs * 8, h[6 * r + 5]);
    }
  }
  for (int k = 0; k < 4; k++) {
    out->totals[k] = 0;
    for (int r = 0; r < R; r++) out->totals[k] += h[6 * r + k];
  }
  out->first_fail = first;
  out->n_ranks = (uint32_t)R;
  out->rank_vc_off = ctx->rank_vc_off.data();
  out->verdict = ctx->all_verdict.data();
  out->rank_sc_off = ctx->rank_sc_off.data();
  out->sc_hash = ctx->all_sc_hash.data();
  out->sc_discharged = ctx->all_sc_dis.data();
  return VEQ_OK;
}

// The roots' DAG on the host (veq_export_dag, size call then fill) as the
// decision procedure's Dag; ridx[k] = index of roots[k].
static int export_to_dag(veq_ctx *ctx, const std::vector<uint32_t> &roots, veqdec::Dag &dag,
                         std::vector<uint32_t> &ridx) {
  veq_dag_buf buf{};
  if (int r = veq_export_dag(ctx, roots.data(), roots.size(), &buf)) return r;
  std::vector<veq_dag_node> nodes(buf.n_nodes);
  std::vector<uint32_t> kids(buf.n_kids);
  ridx.assign(roots.size(), 0);
  buf.cap_nodes = buf.n_nodes;
  buf.cap_kids = buf.n_kids;
  buf.nodes = nodes.data();
  buf.kids = kids.data();
  buf.root_index = ridx.data();
  if (int r = veq_export_dag(ctx, roots.data(), roots.size(), &buf)) return r;
  dag.nodes.resize(nodes.size());
  for (size_t i = 0; i < nodes.size(); i++) {
    const veq_dag_node &n = nodes[i];
    veqdec::DNode &o = dag.nodes[i];
    o.kind = (uint8_t)n.kind;
    o.num = n.num;
    o.den = n.den;
    o.kids.assign(kids.begin() + n.kid_off, kids.begin() + n.kid_off + n.nkids);
    if (n.kind == VEQ_K_VAR) {
      char hx[32];
      snprintf(hx, sizeof hx, "%llx", (unsigned long long)n.var_index);
      o.name = n.var_input >= 0 ? ctx->input_names[n.var_input] + "_" + std::to_string(n.var_index)
                                : std::string("!undef<") + hx + ">";
    }
  }
  return VEQ_OK;
}

// Host half of one decision (decide.cpp:749-859 after the fast path) on an
// exported DAG: f, g, and d = canon(f - g) as DAG indices (have_d false when
// the difference could not be formed; res.reason then says why). Returns
// VEQ_EQUAL .. VEQ_UNDECIDED, or -1 when MPFR is missing for a witness.
static int decide_on_dag(const veqdec::Dag &dag, uint32_t f, uint32_t g, uint32_t d, bool have_d, uint64_t trials,
                         uint64_t seed, veqdec::Result &res, bool want_witness = true) {
  using veqdec::DecideError;
  if (have_d) {
    const veqdec::DNode &dn = dag.nodes[d];
    if (dn.kind == VEQ_K_CONST && dn.num == 0) return VEQ_EQUAL;
    // opaque-max pass: Max subtrees are atoms (decide.cpp:789-813)
    const bool has_max = veqdec::contains_max(dag, d);
    bool opaque_done = false;
    try {
      if (veqdec::zero_by_exp_poly(dag, d)) return VEQ_EQUAL;
      opaque_done = true;
      if (!has_max) res.reason = "difference is a nonzero exp-polynomial";
    } catch (const DecideError &e) {
      res.reason = e.what();
    }
    if (has_max && (opaque_done || res.reason.empty())) {
      // The reference now runs the max case split (split_max,
      // decide.cpp:677-681), which is not restated. A rigorous witness
      // settles NotEqual regardless of its outcome (it could not have
      // proved equality); without one the VC stays undecided, not guessed.
      if (!veqdec::mpfr_available()) return -1;
      try {
        if (veqdec::refute_random(dag, f, g, trials, seed, res, want_witness)) return VEQ_NOT_EQUAL;
      } catch (const DecideError &) {
      }
      res.reason = "max case analysis not available";
      res.assignment.clear();
      return VEQ_UNDECIDED;
    }
  }
  // no proof of equality: a rigorous separating point (refute_random)
  if (!veqdec::mpfr_available()) return -1;
  try {
    if (veqdec::refute_random(dag, f, g, trials, seed, res, want_witness)) return VEQ_NOT_EQUAL;
  } catch (const DecideError &e) {
    res.reason = e.what();
  }
  if (res.reason.empty()) res.reason = "no decision within budget";
  res.reason += "; no separating point found in " + std::to_string(trials) + " trials";
  return VEQ_UNKNOWN;
}

static const char *no_diff_reason(uint32_t d) {
  return d == ~0u ? "cannot form the difference: -inf is not a valid operand of Neg"
                  : "cannot form the difference: -inf is not a valid operand of Add";
}

int veq_decide(veq_ctx *ctx, uint32_t f, uint32_t g, uint64_t seed, uint64_t trials, veq_decision *out) {
  if (!ctx || !out) return VEQ_E_ARG;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  veqdec::Result res;
  ctx->dec_reason.clear();
  auto finish = [&](int kind) {
    out->kind = (uint32_t)kind;
    ctx->dec_reason = res.reason;
    ctx->dec_f = res.f_enclosure;
    ctx->dec_g = res.g_enclosure;
    ctx->dec_names.clear();
    ctx->dec_values.clear();
    for (auto &[n, v] : res.assignment) {
      ctx->dec_names.push_back(n);
      ctx->dec_values.push_back(v);
    }
    ctx->dec_name_p.clear();
    ctx->dec_value_p.clear();
    for (size_t i = 0; i < ctx->dec_names.size(); i++) {
      ctx->dec_name_p.push_back(ctx->dec_names[i].c_str());
      ctx->dec_value_p.push_back(ctx->dec_values[i].c_str());
    }
    out->reason = ctx->dec_reason.c_str();
    out->n_assign = (uint32_t)ctx->dec_names.size();
    out->names = ctx->dec_name_p.data();
    out->values = ctx->dec_value_p.data();
    out->f_enclosure = ctx->dec_f.c_str();
    out->g_enclosure = ctx->dec_g.c_str();
    out->precision = res.precision;
    return VEQ_OK;
  };
  if (f == g) return finish(VEQ_EQUAL);
  // d = canon(f - g) on the device (decide.cpp:779-787)
  uint32_t *dd = nullptr;
  { int r_ = ws_get(ctx, 27, (void **)&dd, 16); if (r_) return r_; }
  CK(cudaMemsetAsync(ctx->pool_used, 0, 8, s));
  k_canon_sub<<<1, 32, 0, s>>>(ctx->T, f, g, dd, ctx->pool, ctx->pool_used, ctx->pool_cap);
  CK(cudaGetLastError());
  uint32_t d = 0;
  CK(cudaMemcpyAsync(&d, dd, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (int er = check_error_flag(ctx)) return er;
  // the three DAGs on the host
  veqdec::Dag dag;
  std::vector<uint32_t> roots{f, g}, ridx;
  const bool have_d = d != ~0u && d != ~1u;
  if (have_d) roots.push_back(d);
  else res.reason = no_diff_reason(d);
  if (int r = export_to_dag(ctx, roots, dag, ridx)) return r;
  const int k = decide_on_dag(dag, ridx[0], ridx[1], have_d ? ridx[2] : 0, have_d, trials, seed, res);
  if (k < 0) return fail(ctx, VEQ_E_UNSUPPORTED, "libmpfr.so.6 not available for witnesses");
  return finish(k);
}

int veq_decide_batch(veq_ctx *ctx, uint64_t n, const uint32_t *f, const uint32_t *g, const uint64_t *seeds,
                     uint64_t trials, uint32_t n_threads, uint32_t *kinds) {
  if (!ctx || (n && (!f || !g || !seeds || !kinds))) return VEQ_E_ARG;
  if (!n) return VEQ_OK;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const auto t0 = std::chrono::steady_clock::now();
  // every difference in one launch
  uint32_t *df = nullptr, *dg = nullptr, *dd = nullptr;
  { int r_ = ws_get(ctx, 29, (void **)&df, n * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 30, (void **)&dg, n * 4); if (r_) return r_; }
  { int r_ = ws_get(ctx, 31, (void **)&dd, n * 4); if (r_) return r_; }
  CK(cudaMemcpyAsync(df, f, n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dg, g, n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(ctx->pool_used, 0, 8, s));
  const uint64_t chunk = std::min<uint64_t>(1ull << 20, std::max<uint64_t>(16ull << 10, ctx->pool_cap / (4 * n)));
  k_canon_sub_many<<<blocks(n, 128), 128, 0, s>>>(ctx->T, df, dg, dd, n, ctx->pool, ctx->pool_used, ctx->pool_cap,
                                                   chunk);
  CK(cudaGetLastError());
  std::vector<uint32_t> d(n);
  CK(cudaMemcpyAsync(d.data(), dd, n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (int er = check_error_flag(ctx)) return er;
  // one DAG for all of them (shared subterms exported once)
  std::vector<uint32_t> roots, ridx;
  roots.reserve(3 * n);
  for (uint64_t i = 0; i < n; i++) {
    roots.push_back(f[i]);
    roots.push_back(g[i]);
    roots.push_back(d[i] == ~0u || d[i] == ~1u ? f[i] : d[i]);
  }
  static const bool prof = getenv("VEQ_PROF") && getenv("VEQ_PROF")[0] == '1';
  const auto t1 = std::chrono::steady_clock::now();
  veqdec::Dag dag;
  if (int r = export_to_dag(ctx, roots, dag, ridx)) return r;
  const auto t2 = std::chrono::steady_clock::now();
  // host decisions: independent per VC, on a thread pool
  unsigned nt = n_threads ? n_threads : std::max(1u, std::thread::hardware_concurrency());
  nt = (unsigned)std::min<uint64_t>(nt, n);
  std::atomic<uint64_t> next{0};
  std::atomic<int> bad{0};
  auto work = [&]() {
    for (;;) {
      const uint64_t i = next.fetch_add(1);
      if (i >= n) return;
      if (f[i] == g[i]) {
        kinds[i] = VEQ_EQUAL;
        continue;
      }
      veqdec::Result res;
      const bool have_d = d[i] != ~0u && d[i] != ~1u;
      if (!have_d) res.reason = no_diff_reason(d[i]);
      int k;
      try {
        k = decide_on_dag(dag, ridx[3 * i], ridx[3 * i + 1], ridx[3 * i + 2], have_d, trials, seeds[i], res, false);
      } catch (...) {
        k = -2;
      }
      if (k < 0) bad.store(k);
      kinds[i] = k < 0 ? VEQ_UNKNOWN : (uint32_t)k;
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; t++) pool.emplace_back(work);
  work();
  for (auto &t : pool) t.join();
  if (prof) {
    const auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[veq decide_batch] n %llu dag nodes %zu | canon+d2h %.1f export %.1f decide %.1f ms on %u threads\n",
            (unsigned long long)n, dag.nodes.size(), ms(t0, t1), ms(t1, t2), ms(t2, t3), nt);
  }
  if (bad.load() == -1) return fail(ctx, VEQ_E_UNSUPPORTED, "libmpfr.so.6 not available for witnesses");
  if (bad.load() == -2) return fail(ctx, VEQ_E_UNSUPPORTED, "veq_decide_batch: host decision failed");
  return VEQ_OK;
}

int veq_verdict_counters(veq_ctx *ctx, uint64_t out[4]) {
  if (!ctx || !out) return VEQ_E_ARG;
  out[0] = ctx->last_equal;
  out[1] = ctx->last_vcs;
  out[2] = ctx->last_faults;
  out[3] = ctx->last_missing;
  return VEQ_OK;
}

}  // extern "C"
