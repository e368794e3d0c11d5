// libsamu host runtime: the C ABI of include/samu.h.  Registries, validation, device uploads,
// batched simulation launches (K1/K2/K3), NCCL trial sharding and the Algorithm 1 control loop
// whose scoring runs on the device (K4).  No simulation arithmetic runs here.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <condition_variable>
#include <mutex>
#include <set>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <tuple>
#include <vector>
#include <chrono>

#include "samu_internal.cuh"

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) { p = nullptr; return e; }
    n = std::max<size_t>(bytes, 16);
    return cudaSuccess;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct ModelReg {
  bool spec_set = false, ecdf_set = false;
  samu_model_spec spec{};
  std::vector<uint32_t> bucket_B;
  std::vector<double> coeff;   // [5][3][2][nb]
  std::vector<double> load;    // [5][16]
  std::vector<uint32_t> ev, ec;
  // fingerprint of the registration and the eCDF (schedule-sharing hints, samu_app_load): one
  // multiply-xor step per field (a hint key only: records never depend on it)
  uint64_t fingerprint() const {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t x) { h = (h ^ (x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2))) * 1099511628211ull; };
    mix(spec.n_layers); mix(spec.hidden); mix(spec.c); mix(spec.l_max); mix(spec.tp_mask);
    mix(spec.weight_bytes); mix(spec.kv_bytes_per_token);
    auto mixd = [&mix](double x) { uint64_t u; std::memcpy(&u, &x, 8); mix(u); };
    for (uint32_t b : bucket_B) mix(b);
    for (double x : coeff) mixd(x);
    for (double x : load) mixd(x);
    for (uint32_t x : ev) mix(x);
    for (uint32_t x : ec) mix(x);
    return h;
  }
};

int log2_exact(uint32_t x) {
  for (int k = 0; k < 32; ++k) if ((1u << k) == x) return k;
  return -1;
}

}  // namespace

// In-process rank group: W contexts in one process (threads), typically on one GPU, exchange
// device buffers through a host barrier.  Same collective semantics as the NCCL path.
struct samu_local_group {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptrs;
  // all ranks publish a pointer, wait until everyone has, then read the others'
  void exchange(int rank, const void* p) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    ptrs[rank] = p;
    if (++count == world) { count = 0; ++gen; cv.notify_all(); }
    else cv.wait(lk, [&] { return gen != my; });
  }
  void barrier(int rank) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    (void)rank;
    if (++count == world) { count = 0; ++gen; cv.notify_all(); }
    else cv.wait(lk, [&] { return gen != my; });
  }
};

// Device buffers of the planner (Greedy / Replay), kept by the context between calls: allocating
// and freeing ~100 MB-1 GB per call (cudaMalloc / cudaFree synchronise and page-map) made the
// planner's wall time vary by seconds.
struct PlanBufs {
  DevBuf lo, li, st, g, fin_t, over, cache, local_rec, d_sc, d_out, d_best, d_any;
  std::vector<DevBuf> fin_pool;
};

struct RequestSetBufs {
  DevBuf tab, knots, tab_off, nobs, mnode, lmax, lib, cap, pred, node, succ, cross, heads;
};

struct samu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux_stream = nullptr;        // K2 LEAN launches beside the general / FRESH ones
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  samu_local_group* group = nullptr;   // in-process ranks instead of NCCL
  std::string err;
  bool poisoned = false;
  int n_sm = 148;
  ModelReg models[SAMU_MAX_NODES];

  // application
  bool app_loaded = false;
  samu_engine_cfg eng{};
  int n_nodes = 0, n_req = 0;
  std::vector<int32_t> node_model, node_begin, node_end, node_input, node_has_succ;
  std::vector<samu_request> req;
  std::vector<double> node_exp_out;   // mean expected output tokens of a node's requests (work-item ordering only)
  std::vector<double> node_mean_lin;  // mean base prompt tokens of a node's requests (work-item ordering only)
  std::vector<int32_t> succ;
  std::vector<uint8_t> cross;
  std::vector<std::vector<int32_t>> waves;
  DevBuf d_l_in_base, d_cap, d_pred, d_node, d_succ, d_cross;
  DevBuf d_tab, d_tab_off, d_nobs, d_mnode, d_lmax, d_known, d_fit_gone;
  int32_t smem_tab_bytes = 0;
  std::vector<DevBuf> d_waves;
  std::map<std::pair<int, int>, DevBuf> coef;                      // (model, tp slot) -> dense table
  struct RepLists { DevBuf off, req; uint64_t gen = 0; };
  std::map<std::pair<int, int>, RepLists> rep;    // (node, dp) -> replica CSR, built for app load `gen`
  // every (node, dp) of the nodes' valid plans, built at the first use after an app load into
  // one arena (one upload instead of two synchronous ones per pair): key -> (off, req) offsets
  DevBuf rep_arena;
  uint64_t rep_arena_gen = 0;
  std::map<std::pair<int, int>, std::pair<size_t, size_t>> rep_at;
  uint64_t app_gen = 1;                            // bumped by every samu_app_load (buffers are reused)
  std::map<std::pair<int, int>, std::vector<uint32_t>> rep_off_host;

  // launch scratch
  DevBuf d_cand_sum;   // per-candidate summaries of samu_simulate_batch
  DevBuf d_stage;      // staging for app-load tables (eCDF knots, coefficient rows)
  PlanBufs pb;         // planner buffers (borrowed by Greedy / Replay for the duration of a call)
  DevBuf d_cands, d_items, d_counter, d_rep_rec, d_scratch_q, d_scratch_key, d_scratch_idx, d_error, d_fb;
  DevBuf d_sum, d_gather_send, d_gather_recv, d_gather_meta, d_flag;
  RequestSetBufs rs;   // samu_sample_requests scratch
  int sim_blocks_per_sm[SAMU_K2_MODES] = {};   // resident K2 blocks per SM, per K2 mode

  // stats
  int64_t n_sims = 0;
  uint64_t launches = 0;          // kernels launched by this context
  int64_t share[3] = {0, 0, 0};   // schedule sharing: group items, member items, fallbacks
  // schedule-sharing hints: (node, dp, tp, mode) -> fraction of the member's items that fell out of
  // sync in its last grouped batch (reset by samu_app_load)
  std::map<std::array<int, 4>, double> share_hint;
  // the hints belong to one application: a fingerprint of the loaded app (engine, node models'
  // registrations, requests); reloading the same app keeps them
  uint64_t hint_app = 0;
  uint64_t req_iters = 0;
};

#define FAIL(ctx, code, msg)          \
  do {                                \
    (ctx)->err = (msg);               \
    return (code);                    \
  } while (0)

#define CK(ctx, call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      (ctx)->err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #call;      \
      if (e_ != cudaErrorMemoryAllocation) (ctx)->poisoned = true;                     \
      return e_ == cudaErrorMemoryAllocation ? SAMU_E_NOMEM : SAMU_E_CUDA;             \
    }                                                                                  \
  } while (0)

#define CKN(ctx, call)                                                                 \
  do {                                                                                 \
    ncclResult_t e_ = (call);                                                          \
    if (e_ != ncclSuccess) {                                                           \
      (ctx)->err = std::string("NCCL: ") + ncclGetErrorString(e_);                     \
      (ctx)->poisoned = true;                                                          \
      return SAMU_E_NCCL;                                                              \
    }                                                                                  \
  } while (0)

#define GUARD(ctx)                                                                     \
  do {                                                                                 \
    if (!(ctx)) return SAMU_E_INVALID;                                                 \
    if ((ctx)->poisoned) return SAMU_E_STATE;                                          \
    cudaSetDevice((ctx)->device);                                                      \
  } while (0)

#define RET(x)                 \
  do {                         \
    samu_status r_ = (x);      \
    if (r_ != SAMU_OK) return r_; \
  } while (0)

// ---- collectives over the context's ranks (NCCL, or the in-process group) ----
static samu_status comm_allgather(samu_ctx* c, const void* send, void* recv, size_t bytes) {
  cudaStream_t s = c->stream;
  if (c->group) {
    CK(c, cudaStreamSynchronize(s));
    c->group->exchange(c->rank, send);
    for (int w = 0; w < c->world; ++w)
      CK(c, cudaMemcpyAsync((char*)recv + (size_t)w * bytes, c->group->ptrs[w], bytes, cudaMemcpyDeviceToDevice, s));
    CK(c, cudaStreamSynchronize(s));
    c->group->barrier(c->rank);   // nobody reuses its send buffer before every copy finished
    return SAMU_OK;
  }
  CKN(c, ncclAllGather(send, recv, bytes, ncclUint8, c->comm, s));
  return SAMU_OK;
}

// element-wise max (op = 0) or sum (op = 1) of n int32 over ranks, device buffers
static samu_status comm_allreduce_i32(samu_ctx* c, const int32_t* send, int32_t* recv, int n, int op) {
  cudaStream_t s = c->stream;
  if (c->group) {
    CK(c, cudaStreamSynchronize(s));
    c->group->exchange(c->rank, send);
    // Every copy runs on the context's stream and is waited for: a plain cudaMemcpy from pageable
    // host memory may return before its DMA lands and is not ordered with a non-blocking stream,
    // so a later read of `recv` on the stream could see the previous call's value — ranks then
    // disagree on a flag (e.g. an unfinished node) and one of them waits alone in a collective.
    std::vector<int32_t> acc(n, 0), tmp(n);
    for (int w = 0; w < c->world; ++w) {
      CK(c, cudaMemcpyAsync(tmp.data(), c->group->ptrs[w], sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
      CK(c, cudaStreamSynchronize(s));
      for (int i = 0; i < n; ++i) acc[i] = (w == 0) ? tmp[i] : (op == 0 ? std::max(acc[i], tmp[i]) : acc[i] + tmp[i]);
    }
    c->group->barrier(c->rank);
    CK(c, cudaMemcpyAsync(recv, acc.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(c, cudaStreamSynchronize(s));
    return SAMU_OK;
  }
  CKN(c, ncclAllReduce(send, recv, n, ncclInt32, op == 0 ? ncclMax : ncclSum, c->comm, s));
  return SAMU_OK;
}

// Ranks leave a sharded call together: before the next collective, a rank-local failure (e.g. a
// kernel-detected infeasible trial on one rank's share) is agreed on with an all-reduce, so no
// rank waits in a collective its peers never reach.  (A poisoned context cannot take part: a
// CUDA / NCCL failure is reported on its rank; peers then need ncclCommAbort via ctx_destroy.)
static samu_status agree(samu_ctx* c, samu_status local) {
  if (!(c->world > 1 || c->comm != nullptr) || c->poisoned) return local;
  const std::string keep = c->err;
  int32_t f[2] = {local != SAMU_OK ? 1 : 0, 0};
  CK(c, c->d_flag.ensure(2 * sizeof(int32_t)));
  CK(c, cudaMemcpyAsync(c->d_flag.p, f, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  RET(comm_allreduce_i32(c, c->d_flag.as<int32_t>(), c->d_flag.as<int32_t>() + 1, 1, 0));
  CK(c, cudaMemcpyAsync(f + 1, c->d_flag.as<int32_t>() + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (local != SAMU_OK) { c->err = keep; return local; }
  if (f[1]) FAIL(c, SAMU_E_STATE, "another rank failed in this collective call");
  return SAMU_OK;
}

// NVTX ranges around the path's steps (K1 sampling, K2 batches, K3 summaries, planner stages):
// header-only NVTX v3, free when no profiler is attached (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static inline cudaError_t samu_count(samu_ctx* c, cudaError_t e) {
  c->launches += 1;
  return e;
}

// records and status go through the collectives (several ranks, or the one-rank NCCL test hook)
static inline bool sharded(const samu_ctx* c) { return c->world > 1 || c->comm != nullptr; }

template <class T>
static cudaError_t upload(DevBuf& b, const std::vector<T>& v, cudaStream_t s) {
  cudaError_t e = b.ensure(sizeof(T) * v.size());
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  e = cudaMemcpyAsync(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

// ---------------------------------------------------------------------------------------------
// engine arithmetic (reading c5/c6): blocks per replica, or -1 if the plan is invalid
// ---------------------------------------------------------------------------------------------
static int64_t plan_blocks(const samu_ctx* c, int model, int dp, int tp) {
  const samu_model_spec& M = c->models[model].spec;
  const samu_engine_cfg& e = c->eng;
  const int slot = log2_exact((uint32_t)tp);
  if (slot < 0 || slot >= SAMU_N_TP_SLOTS || !((M.tp_mask >> slot) & 1u)) return -1;
  if (M.hidden % (uint32_t)tp) return -1;
  if (dp < 1 || dp > SAMU_MAX_DP || (uint32_t)(dp * tp) > e.n_gpus) return -1;
  const uint64_t util = e.mem_bytes_per_gpu * e.mem_util_permille / 1000;
  const uint64_t wshard = (M.weight_bytes + (uint64_t)tp - 1) / (uint64_t)tp;
  if (util <= wshard) return -1;
  const uint64_t kv = std::min<uint64_t>(e.kv_cap_bytes_per_gpu, util - wshard);
  uint64_t blocks = ((uint64_t)tp * kv) / ((uint64_t)e.block_size * M.kv_bytes_per_token);
  if (blocks < (M.l_max + e.block_size - 1) / e.block_size) return -1;
  if (blocks > 0x7fffffffull) blocks = 0x7fffffffull;
  return (int64_t)blocks;
}

// valid plans of a model: ascending #gpu, then ascending tp
static std::vector<std::pair<int, int>> plans_of(const samu_ctx* c, int model) {
  std::vector<std::pair<int, int>> out;
  for (int gpus = 1; gpus <= (int)c->eng.n_gpus; ++gpus)
    for (int t = 1; t <= gpus; t *= 2)
      if (gpus % t == 0 && plan_blocks(c, model, gpus / t, t) >= 0) out.push_back({gpus / t, t});
  return out;
}

// ---------------------------------------------------------------------------------------------
// C ABI: context
// ---------------------------------------------------------------------------------------------
extern "C" samu_status samu_nccl_unique_id(uint8_t out[128]) {
  if (!out) return SAMU_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SAMU_E_NCCL;
  std::memcpy(out, id.internal, 128);
  return SAMU_OK;
}

extern "C" samu_status samu_ctx_create(samu_ctx** out, int32_t cuda_device, void* cuda_stream, int32_t rank,
                                       int32_t world, const uint8_t* nccl_unique_id) {
  if (!out) return SAMU_E_INVALID;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id)) return SAMU_E_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return SAMU_E_CUDA;
  if (cuda_device < 0 || cuda_device >= ndev) return SAMU_E_INVALID;
  samu_ctx* c = new samu_ctx();
  c->device = cuda_device;
  c->rank = rank;
  c->world = world;
  if (cudaSetDevice(cuda_device) != cudaSuccess) { delete c; return SAMU_E_CUDA; }
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, cuda_device);
  c->stream = (cudaStream_t)cuda_stream;   // NULL = the CUDA default (legacy) stream
  if (world > 1) {
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_unique_id, 128);
    if (ncclCommInitRank(&c->comm, world, id, rank) != ncclSuccess) { delete c; return SAMU_E_NCCL; }
  } else if (std::getenv("SAMU_FORCE_NCCL")) {
    // test hook: a one-rank NCCL communicator, so the sharded code path and its NCCL calls run
    // on a single GPU (NCCL refuses two ranks on one device)
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess || ncclCommInitRank(&c->comm, 1, id, 0) != ncclSuccess) {
      delete c;
      return SAMU_E_NCCL;
    }
  }
  *out = c;
  return SAMU_OK;
}

extern "C" samu_status samu_local_group_create(samu_local_group** out, int32_t world) {
  if (!out || world < 1) return SAMU_E_INVALID;
  samu_local_group* g = new samu_local_group();
  g->world = world;
  g->ptrs.assign(world, nullptr);
  *out = g;
  return SAMU_OK;
}

extern "C" void samu_local_group_destroy(samu_local_group* g) { delete g; }

extern "C" samu_status samu_ctx_create_local(samu_ctx** out, int32_t cuda_device, void* cuda_stream, int32_t rank,
                                             samu_local_group* group) {
  if (!out || !group || rank < 0 || rank >= group->world) return SAMU_E_INVALID;
  samu_status rc = samu_ctx_create(out, cuda_device, cuda_stream, 0, 1, nullptr);
  if (rc != SAMU_OK) return rc;
  (*out)->rank = rank;
  (*out)->world = group->world;
  (*out)->group = group;
  return SAMU_OK;
}

extern "C" void samu_ctx_destroy(samu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->aux_stream) {
    cudaStreamSynchronize(c->aux_stream);
    cudaStreamDestroy(c->aux_stream);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
}

extern "C" const char* samu_last_error(const samu_ctx* c) { return c ? c->err.c_str() : "null context"; }

extern "C" uint64_t samu_launch_count(const samu_ctx* c) { return c ? c->launches : 0; }
extern "C" void samu_share_stats(const samu_ctx* c, int64_t out[3]) {
  if (!out) return;
  for (int i = 0; i < 3; ++i) out[i] = c ? c->share[i] : 0;
}

// ---------------------------------------------------------------------------------------------
// C ABI: registration
// ---------------------------------------------------------------------------------------------
extern "C" samu_status samu_model_register(samu_ctx* c, int32_t model_id, const samu_model_spec* spec,
                                           int32_t n_buckets, const uint32_t* bucket_B, const double* coeff,
                                           const double* load_s) {
  GUARD(c);
  if (model_id < 0 || model_id >= SAMU_MAX_NODES || !spec || n_buckets < 1 || !bucket_B || !coeff || !load_s)
    FAIL(c, SAMU_E_INVALID, "model_register: bad arguments");
  const samu_model_spec& s = *spec;
  if (s.n_layers < 1 || s.hidden < 1 || s.c < 1 || s.l_max < 1 || s.l_max > 65535 || s.tp_mask == 0 ||
      (s.tp_mask >> SAMU_N_TP_SLOTS) || s.kv_bytes_per_token < 1)
    FAIL(c, SAMU_E_INVALID, "model_register: invalid spec");
  if (2ull * s.n_layers * s.hidden >= (1ull << 32))   // 2 L (h/tp) is a u32 factor in K2
    FAIL(c, SAMU_E_INVALID, "model_register: 2 L h must stay below 2^32");
  for (int k = 0; k < n_buckets; ++k)
    if (bucket_B[k] < 1 || (k && bucket_B[k] <= bucket_B[k - 1]))
      FAIL(c, SAMU_E_INVALID, "model_register: buckets not strictly increasing");
  // worst-case prefill FLOPs of one iteration must fit u64 (B*s <= 256 * l_max tokens)
  {
    const long double lm = (long double)std::max<uint32_t>(s.l_max, 65535u);
    const long double worst = (long double)s.n_layers * ((long double)s.c * 256.0L * lm + 2.0L * 256.0L * s.hidden * lm * lm);
    if (worst >= 1.8e19L) FAIL(c, SAMU_E_INVALID, "model_register: FLOPs could overflow u64");
  }
  ModelReg& M = c->models[model_id];
  M.spec = s;
  M.bucket_B.assign(bucket_B, bucket_B + n_buckets);
  M.coeff.assign(coeff, coeff + (size_t)SAMU_N_TP_SLOTS * 3 * 2 * n_buckets);
  M.load.assign(load_s, load_s + (size_t)SAMU_N_TP_SLOTS * SAMU_MAX_DP);
  M.spec_set = true;
  c->app_loaded = false;   // tables depend on the engine config: re-derive at app load
  return SAMU_OK;
}

extern "C" samu_status samu_ecdf_load(samu_ctx* c, int32_t model_id, const uint32_t* values, const uint32_t* cum,
                                      int32_t n_points) {
  GUARD(c);
  if (model_id < 0 || model_id >= SAMU_MAX_NODES || !values || !cum || n_points < 1)
    FAIL(c, SAMU_E_INVALID, "ecdf_load: bad arguments");
  for (int k = 0; k < n_points; ++k) {
    if ((k && values[k] <= values[k - 1]) || cum[k] < 1 || (k && cum[k] <= cum[k - 1]))
      FAIL(c, SAMU_E_INVALID, "ecdf_load: knots must be strictly increasing (P:466)");
  }
  ModelReg& M = c->models[model_id];
  M.ev.assign(values, values + n_points);
  M.ec.assign(cum, cum + n_points);
  M.ecdf_set = true;
  c->app_loaded = false;
  return SAMU_OK;
}

extern "C" samu_status samu_app_load(samu_ctx* c, const samu_engine_cfg* engine, int32_t n_nodes,
                                     const int32_t* node_model, int32_t n_req, const samu_request* reqs) {
  GUARD(c);
  if (!engine || n_nodes < 1 || n_nodes > SAMU_MAX_NODES || !node_model || n_req < 0 || (n_req && !reqs))
    FAIL(c, SAMU_E_INVALID, "app_load: bad arguments");
  const samu_engine_cfg& e = *engine;
  if (e.max_num_seqs < 1 || e.max_num_seqs > SAMU_MAX_SEQS || e.block_size < 1 || e.block_size > 32 ||
      e.n_gpus < 1 || e.n_gpus > 16 || e.mem_util_permille > 1000)
    FAIL(c, SAMU_E_INVALID, "app_load: invalid engine config");
  c->app_loaded = false;
  c->eng = e;
  c->n_nodes = n_nodes;
  c->n_req = n_req;
  c->node_model.assign(node_model, node_model + n_nodes);
  for (int v = 0; v < n_nodes; ++v) {
    const int m = node_model[v];
    if (m < 0 || m >= SAMU_MAX_NODES || !c->models[m].spec_set || !c->models[m].ecdf_set)
      FAIL(c, SAMU_E_INVALID, "app_load: node model not registered or no eCDF");
  }
  c->req.assign(reqs, reqs + n_req);
  c->node_begin.assign(n_nodes, 0);
  c->node_end.assign(n_nodes, 0);
  c->node_input.assign(n_nodes, -1);
  c->succ.assign(n_req, -1);
  c->cross.assign(n_req, 0);
  std::vector<int> has_same(n_nodes, 0), has_cross(n_nodes, 0);
  int last = -1;
  for (int r = 0; r < n_req; ++r) {
    const samu_request& q = c->req[r];
    if (q.node < 0 || q.node >= n_nodes || q.node < last) FAIL(c, SAMU_E_INVALID, "app_load: requests not grouped by ascending node");
    if (q.node != last) { c->node_begin[q.node] = r; last = q.node; }
    c->node_end[q.node] = r + 1;
    const samu_model_spec& M = c->models[node_model[q.node]].spec;
    if (q.l_in_base > 65535 || q.chain < -1) FAIL(c, SAMU_E_INVALID, "app_load: bad request field");
    if (q.pred < -1 || q.pred >= r) FAIL(c, SAMU_E_INVALID, "app_load: pred must precede its request");
    if (q.pred < 0) {
      if (q.l_in_base > M.l_max) FAIL(c, SAMU_E_INVALID, "app_load: l_in > l_max (S:199)");
    } else {
      const samu_request& p = c->req[q.pred];
      if (p.node == q.node) {
        if (p.chain != q.chain || q.chain < 0) FAIL(c, SAMU_E_INVALID, "app_load: chain successor must share chain id");
        if (c->succ[q.pred] >= 0) FAIL(c, SAMU_E_INVALID, "app_load: same-node dependencies must form chains");
        c->succ[q.pred] = r;
        has_same[q.node] = 1;
      } else {
        if (c->node_input[q.node] >= 0 && c->node_input[q.node] != p.node)
          FAIL(c, SAMU_E_INVALID, "app_load: a node may depend on one input node only");
        c->node_input[q.node] = p.node;
        c->cross[r] = 1;
        has_cross[q.node] = 1;
      }
    }
  }
  for (int v = 0; v < n_nodes; ++v)
    if (has_same[v] && has_cross[v]) FAIL(c, SAMU_E_INVALID, "app_load: node mixes chain and cross-node predecessors");
  c->node_has_succ = has_same;
  // sampling waves: chains rooted at pred < 0 first, then cross-node requests by node depth
  std::vector<int> depth(n_nodes, 0);
  for (int v = 0; v < n_nodes; ++v) if (c->node_input[v] >= 0) depth[v] = depth[c->node_input[v]] + 1;
  int maxd = 0;
  for (int v = 0; v < n_nodes; ++v) maxd = std::max(maxd, depth[v]);
  c->waves.assign(maxd + 1, {});
  for (int r = 0; r < n_req; ++r) {
    const samu_request& q = c->req[r];
    if (q.pred < 0) c->waves[0].push_back(r);
    else if (c->cross[r]) c->waves[depth[q.node]].push_back(r);
  }
  // K1 walks a chain serially in one thread: chain roots first (stable), so the blocks holding
  // them start at the front of each trial group's row of the grid instead of forming its tail
  // (sampled values are keyed by request id: the order changes nothing else)
  if (!std::getenv("SAMU_K1_INDEX_ORDER"))
    std::stable_partition(c->waves[0].begin(), c->waves[0].end(), [&](int r) { return c->succ[r] >= 0; });
  cudaStream_t s = c->stream;
  std::vector<uint32_t> lib(n_req), cap(n_req);
  std::vector<int32_t> pred(n_req), nd(n_req);
  for (int r = 0; r < n_req; ++r) { lib[r] = c->req[r].l_in_base; cap[r] = c->req[r].cap_y; pred[r] = c->req[r].pred; nd[r] = c->req[r].node; }
  CK(c, upload(c->d_l_in_base, lib, s));
  CK(c, upload(c->d_cap, cap, s));
  CK(c, upload(c->d_pred, pred, s));
  CK(c, upload(c->d_node, nd, s));
  CK(c, upload(c->d_succ, c->succ, s));
  CK(c, upload(c->d_cross, c->cross, s));
  if (c->d_waves.size() < c->waves.size()) c->d_waves.resize(c->waves.size());   // buffers kept across loads
  for (size_t i = 0; i < c->waves.size(); ++i) CK(c, upload(c->d_waves[i], c->waves[i], s));
  // eCDF tables: each registered model's sorted multiset expanded on the device (reading c2)
  {
    std::vector<int32_t> toff(SAMU_MAX_NODES + 1, 0);
    std::vector<uint32_t> nobs(SAMU_MAX_NODES, 0), lmax(n_nodes);
    for (int m = 0; m < SAMU_MAX_NODES; ++m) {
      toff[m + 1] = toff[m];
      if (c->models[m].ecdf_set) {
        nobs[m] = c->models[m].ec.back();
        toff[m + 1] += (int32_t)((nobs[m] + 7u) & ~7u);
      }
    }
    CK(c, c->d_tab.ensure(sizeof(uint16_t) * std::max(toff[SAMU_MAX_NODES], 8)));
    // every model's knots in one staging upload (values | cumulative counts), one table launch each
    std::vector<uint32_t> knots;
    std::vector<size_t> kat(SAMU_MAX_NODES, 0);
    for (int m = 0; m < SAMU_MAX_NODES; ++m) {
      if (!c->models[m].ecdf_set) continue;
      kat[m] = knots.size();
      knots.insert(knots.end(), c->models[m].ev.begin(), c->models[m].ev.end());
      knots.insert(knots.end(), c->models[m].ec.begin(), c->models[m].ec.end());
    }
    CK(c, upload(c->d_stage, knots, s));
    int32_t max_bytes = 0;
    for (int m = 0; m < SAMU_MAX_NODES; ++m) {
      if (!c->models[m].ecdf_set) continue;
      const uint32_t* kv = c->d_stage.as<uint32_t>() + kat[m];
      const size_t K = c->models[m].ev.size();
      CK(c, samu_count(c, launch_ecdf_table(kv, kv + K, (int32_t)K, nobs[m], c->d_tab.as<uint16_t>() + toff[m], s)));
      max_bytes = std::max(max_bytes, (toff[m + 1] - toff[m]) * 2);
    }
    CK(c, cudaStreamSynchronize(s));   // the staging buffer is reused below
    c->smem_tab_bytes = std::min(max_bytes, 200 * 1024);
    for (int v = 0; v < n_nodes; ++v) lmax[v] = c->models[node_model[v]].spec.l_max;
    CK(c, upload(c->d_tab_off, toff, s));
    CK(c, upload(c->d_nobs, nobs, s));
    CK(c, upload(c->d_mnode, c->node_model, s));
    CK(c, upload(c->d_lmax, lmax, s));
  }
  // dense coefficient tables for every (model of a node, allowed tp) (reading c11): one staging
  // upload of all bucket lists and coefficient rows, table buffers kept across app loads
  {
    std::vector<std::pair<int, int>> keys;
    for (int v = 0; v < n_nodes; ++v) {
      const int m = node_model[v];
      for (int slot = 0; slot < SAMU_N_TP_SLOTS; ++slot)
        if (((c->models[m].spec.tp_mask >> slot) & 1u) &&
            std::find(keys.begin(), keys.end(), std::make_pair(m, slot)) == keys.end())
          keys.emplace_back(m, slot);
    }
    std::vector<double> stage;   // per key: bucket B values (as doubles) | 6 nb coefficients
    std::vector<size_t> at;
    for (auto& k : keys) {
      const ModelReg& M = c->models[k.first];
      const size_t nb = M.bucket_B.size();
      at.push_back(stage.size());
      for (uint32_t b : M.bucket_B) stage.push_back((double)b);
      stage.insert(stage.end(), M.coeff.begin() + (size_t)k.second * 6 * nb, M.coeff.begin() + (size_t)(k.second + 1) * 6 * nb);
    }
    CK(c, upload(c->d_stage, stage, s));
    for (auto it = c->coef.begin(); it != c->coef.end();)
      it = std::find(keys.begin(), keys.end(), it->first) == keys.end() ? c->coef.erase(it) : std::next(it);
    for (size_t i = 0; i < keys.size(); ++i) {
      const ModelReg& M = c->models[keys[i].first];
      const int nb = (int)M.bucket_B.size();
      DevBuf& out = c->coef[keys[i]];
      CK(c, out.ensure(sizeof(double) * 8 * e.max_num_seqs));
      const double* base = c->d_stage.as<double>() + at[i];
      CK(c, samu_count(c, launch_dense_coeff(base, nb, base + nb, e.max_num_seqs, out.as<double>(), s)));
    }
    CK(c, cudaStreamSynchronize(s));
  }
  c->app_gen += 1;   // replica lists are rebuilt lazily into their existing buffers
  c->rep_off_host.clear();
  // expected output length per node, E[min(X, cap, l_max - l_in)] with X ~ the model's eCDF
  // (chain inputs taken at their base length): orders K2's work items longest-first
  c->node_exp_out.assign(n_nodes, 1.0);
  c->node_mean_lin.assign(n_nodes, 0.0);
  for (int v = 0; v < n_nodes; ++v) {
    double sl = 0.0;
    for (int r = c->node_begin[v]; r < c->node_end[v]; ++r) sl += (double)c->req[r].l_in_base;
    if (c->node_end[v] > c->node_begin[v]) c->node_mean_lin[v] = sl / (double)(c->node_end[v] - c->node_begin[v]);
    const ModelReg& M = c->models[node_model[v]];
    if (!M.ecdf_set || c->node_end[v] <= c->node_begin[v]) continue;
    const size_t K = M.ev.size();
    const double nobs = (double)M.ec.back();
    std::vector<double> part(K + 1, 0.0);   // part[k] = sum_{j<k} v_j * count_j
    for (size_t k = 0; k < K; ++k) part[k + 1] = part[k] + (double)M.ev[k] * (double)(M.ec[k] - (k ? M.ec[k - 1] : 0u));
    double acc = 0.0;
    for (int r = c->node_begin[v]; r < c->node_end[v]; ++r) {
      const uint32_t lim = std::min<uint32_t>(c->req[r].cap_y, M.spec.l_max - std::min(M.spec.l_max, c->req[r].l_in_base));
      const size_t k = (size_t)(std::lower_bound(M.ev.begin(), M.ev.end(), lim) - M.ev.begin());   // v_j < lim for j < k
      const double below = k ? (double)M.ec[k - 1] : 0.0;
      acc += (part[k] + (double)lim * (nobs - below)) / nobs;
    }
    c->node_exp_out[v] = std::max(1.0, acc / (double)(c->node_end[v] - c->node_begin[v]));
  }
  c->app_loaded = true;
  {   // one multiply-xor step per field (no struct padding); each model's fingerprint once
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t x) { h = (h ^ (x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2))) * 1099511628211ull; };
    std::map<int, uint64_t> model_fp;
    mix(e.max_num_seqs); mix(e.block_size); mix(e.min_batched_tokens); mix(e.mem_util_permille);
    mix(e.mem_bytes_per_gpu); mix(e.kv_cap_bytes_per_gpu); mix(e.n_gpus);
    mix((uint64_t)n_nodes);
    for (int v = 0; v < n_nodes; ++v) {
      mix((uint64_t)(uint32_t)node_model[v]);
      auto f = model_fp.find(node_model[v]);
      if (f == model_fp.end()) f = model_fp.emplace(node_model[v], c->models[node_model[v]].fingerprint()).first;
      mix(f->second);
    }
    mix((uint64_t)n_req);
    for (const samu_request& q : c->req) {
      mix(q.l_in_base); mix(q.cap_y); mix((uint32_t)q.pred); mix((uint32_t)q.node); mix((uint32_t)q.chain);
    }
    if (h != c->hint_app) c->share_hint.clear();
    c->hint_app = h;
  }
  return SAMU_OK;
}

extern "C" int32_t samu_enumerate_plans(samu_ctx* c, int32_t node, int32_t* dp, int32_t* tp, int32_t cap) {
  GUARD(c);
  if (!c->app_loaded || node < 0 || node >= c->n_nodes || cap < 0 || (cap && (!dp || !tp)))
    FAIL(c, SAMU_E_INVALID, "enumerate_plans: bad arguments");
  auto pl = plans_of(c, c->node_model[node]);
  for (int i = 0; i < (int)pl.size() && i < cap; ++i) { dp[i] = pl[i].first; tp[i] = pl[i].second; }
  return (int32_t)pl.size();
}

static DevApp dev_app(const samu_ctx* c) {
  DevApp a;
  a.n_req = c->n_req;
  a.n_nodes = c->n_nodes;
  a.l_in_base = c->d_l_in_base.as<uint32_t>();
  a.cap_y = c->d_cap.as<uint32_t>();
  a.pred = c->d_pred.as<int32_t>();
  a.node = c->d_node.as<int32_t>();
  a.succ = c->d_succ.as<int32_t>();
  a.cross = c->d_cross.as<uint8_t>();
  return a;
}

// requests of `node` grouped by dp replica (c13): key = chain id if >= 0 else index within node
static void replica_lists(const samu_ctx* c, int node, int dp, std::vector<uint32_t>& o, std::vector<uint32_t>& l) {
  // counting sort by replica, stable in request order
  const int b = c->node_begin[node], e = c->node_end[node];
  auto rep_of = [&](int r) { return (c->req[r].chain >= 0 ? c->req[r].chain : r - b) % dp; };
  o.assign(dp + 1, 0);
  for (int r = b; r < e; ++r) o[rep_of(r) + 1] += 1;
  for (int j = 0; j < dp; ++j) o[j + 1] += o[j];
  l.resize((size_t)(e - b));
  std::vector<uint32_t> at(o.begin(), o.end() - 1);
  for (int r = b; r < e; ++r) l[at[rep_of(r)]++] = (uint32_t)r;
}

static samu_status replicas(samu_ctx* c, int node, int dp, const uint32_t** off, const uint32_t** lst) {
  auto key = std::make_pair(node, dp);
  if (c->rep_arena_gen != c->app_gen) {   // first use after an app load: every plan's lists at once
    c->rep_at.clear();
    std::vector<uint32_t> all, o, l;
    for (int v = 0; v < c->n_nodes; ++v) {
      std::set<int> dps;
      for (const auto& pl : plans_of(c, c->node_model[v])) dps.insert(pl.first);
      for (int d : dps) {
        replica_lists(c, v, d, o, l);
        c->rep_at[{v, d}] = {all.size(), all.size() + o.size()};
        all.insert(all.end(), o.begin(), o.end());
        all.insert(all.end(), l.begin(), l.end());
        c->rep_off_host[{v, d}] = o;
      }
    }
    CK(c, upload(c->rep_arena, all, c->stream));
    c->rep_arena_gen = c->app_gen;
  }
  auto at = c->rep_at.find(key);
  if (at != c->rep_at.end()) {
    *off = c->rep_arena.as<uint32_t>() + at->second.first;
    *lst = c->rep_arena.as<uint32_t>() + at->second.second;
    return SAMU_OK;
  }
  auto it = c->rep.find(key);
  if (it == c->rep.end() || it->second.gen != c->app_gen) {   // a (node, dp) outside the plans
    std::vector<uint32_t> o, l;
    replica_lists(c, node, dp, o, l);
    auto& pr = c->rep[key];
    CK(c, upload(pr.off, o, c->stream));
    CK(c, upload(pr.req, l, c->stream));
    pr.gen = c->app_gen;
    c->rep_off_host[key] = o;
    it = c->rep.find(key);
  }
  *off = it->second.off.as<uint32_t>();
  *lst = it->second.req.as<uint32_t>();
  return SAMU_OK;
}

// ---------------------------------------------------------------------------------------------
// sampling
// ---------------------------------------------------------------------------------------------
static samu_status sample_or_known(samu_ctx* c, uint64_t seed, int32_t trial_begin, int32_t n_trials,
                                   const uint32_t* known_dev, uint16_t* out_l_out, uint16_t* out_l_in_eff) {
  NvtxRange nv("samu K1 sample_lengths");
  DevApp a = dev_app(c);
  DevEcdf e;
  e.tab = c->d_tab.as<uint16_t>();
  e.tab_off = c->d_tab_off.as<int32_t>();
  e.n_obs = c->d_nobs.as<uint32_t>();
  e.model_of_node = c->d_mnode.as<int32_t>();
  e.l_max_of_node = c->d_lmax.as<uint32_t>();
  e.smem_tab_bytes = c->smem_tab_bytes;
  for (size_t w = 0; w < c->waves.size(); ++w)
    CK(c, samu_count(c, launch_sample(a, e, c->d_waves[w].as<int32_t>(), (int32_t)c->waves[w].size(), seed, trial_begin,
                                      n_trials, known_dev, out_l_out, out_l_in_eff, c->stream)));
  return SAMU_OK;
}

extern "C" samu_status samu_sample_lengths(samu_ctx* c, uint64_t seed, int32_t trial_begin, int32_t n_trials,
                                           uint16_t* out_l_out, uint16_t* out_l_in_eff) {
  GUARD(c);
  if (!c->app_loaded) FAIL(c, SAMU_E_INVALID, "sample_lengths: no app loaded");
  if (n_trials < 0 || trial_begin < 0 || (n_trials && (!out_l_out || !out_l_in_eff)))
    FAIL(c, SAMU_E_INVALID, "sample_lengths: bad arguments");
  if (n_trials > 65535) FAIL(c, SAMU_E_INVALID, "sample_lengths: at most 65535 trials per call");
  return sample_or_known(c, seed, trial_begin, n_trials, nullptr, out_l_out, out_l_in_eff);
}

// one model's request set with its own Philox stream (samu.h): a temporary one-node application
extern "C" samu_status samu_sample_requests(samu_ctx* c, int32_t model_id, uint32_t stream_id, const samu_request* reqs,
                                           int32_t n_req, uint32_t index_base, uint64_t seed, int32_t trial_begin,
                                           int32_t n_trials, uint16_t* out_l_out, uint16_t* out_l_in_eff) {
  GUARD(c);
  if (model_id < 0 || model_id >= SAMU_MAX_NODES || !c->models[model_id].spec_set || !c->models[model_id].ecdf_set)
    FAIL(c, SAMU_E_INVALID, "sample_requests: model not registered or no eCDF");
  if (n_req < 0 || n_trials < 0 || trial_begin < 0 || stream_id >= (1u << 31) || (n_req && !reqs) ||
      (n_req && n_trials && (!out_l_out || !out_l_in_eff)))
    FAIL(c, SAMU_E_INVALID, "sample_requests: bad arguments");
  if (n_trials > 65535) FAIL(c, SAMU_E_INVALID, "sample_requests: at most 65535 trials per call");
  if ((uint64_t)n_req * (uint64_t)std::max(n_trials, 1) >= (1ull << 32)) FAIL(c, SAMU_E_INVALID, "sample_requests: too large");
  if (n_req == 0 || n_trials == 0) return SAMU_OK;
  const ModelReg& M = c->models[model_id];
  std::vector<uint32_t> lib(n_req), cap(n_req);
  std::vector<int32_t> pred(n_req), node(n_req, 0), succ(n_req, -1), heads;
  std::vector<uint8_t> cross(n_req, 0);
  for (int32_t i = 0; i < n_req; ++i) {
    const samu_request& q = reqs[i];
    if (q.l_in_base > M.spec.l_max) FAIL(c, SAMU_E_INVALID, "sample_requests: l_in_base > l_max");
    if (q.pred >= i || q.pred < -1) FAIL(c, SAMU_E_INVALID, "sample_requests: pred must be -1 or an earlier request");
    if (q.pred >= 0) {
      if (succ[q.pred] >= 0) FAIL(c, SAMU_E_INVALID, "sample_requests: two successors of one request");
      succ[q.pred] = i;
    } else {
      heads.push_back(i);
    }
    lib[i] = q.l_in_base;
    cap[i] = q.cap_y;
    pred[i] = q.pred;
  }
  // the model's sorted-multiset table (reading c2), laid out as the app tables with this model's
  // entries at offset 0
  const uint32_t nobs = M.ec.back();
  const int32_t K = (int32_t)M.ev.size();
  std::vector<int32_t> toff(SAMU_MAX_NODES + 1, 0), mnode{model_id};
  for (int m = model_id + 1; m <= SAMU_MAX_NODES; ++m) toff[m] = (int32_t)((nobs + 7u) & ~7u);
  std::vector<uint32_t> nob(SAMU_MAX_NODES, 0), lmax{M.spec.l_max}, knots;
  nob[model_id] = nobs;
  knots.insert(knots.end(), M.ev.begin(), M.ev.end());
  knots.insert(knots.end(), M.ec.begin(), M.ec.end());
  RequestSetBufs& B = c->rs;
  cudaStream_t s = c->stream;
  CK(c, B.tab.ensure(sizeof(uint16_t) * std::max<uint32_t>((nobs + 7u) & ~7u, 8u)));
  CK(c, upload(B.knots, knots, s));
  CK(c, samu_count(c, launch_ecdf_table(B.knots.as<uint32_t>(), B.knots.as<uint32_t>() + K, K, nobs, B.tab.as<uint16_t>(), s)));
  CK(c, upload(B.tab_off, toff, s));
  CK(c, upload(B.nobs, nob, s));
  CK(c, upload(B.mnode, mnode, s));
  CK(c, upload(B.lmax, lmax, s));
  CK(c, upload(B.lib, lib, s));
  CK(c, upload(B.cap, cap, s));
  CK(c, upload(B.pred, pred, s));
  CK(c, upload(B.node, node, s));
  CK(c, upload(B.succ, succ, s));
  CK(c, upload(B.cross, cross, s));
  CK(c, upload(B.heads, heads, s));
  DevApp a;
  a.n_req = n_req;
  a.n_nodes = 1;
  a.l_in_base = B.lib.as<uint32_t>();
  a.cap_y = B.cap.as<uint32_t>();
  a.pred = B.pred.as<int32_t>();
  a.node = B.node.as<int32_t>();
  a.succ = B.succ.as<int32_t>();
  a.cross = B.cross.as<uint8_t>();
  DevEcdf e;
  e.tab = B.tab.as<uint16_t>();
  e.tab_off = B.tab_off.as<int32_t>();
  e.n_obs = B.nobs.as<uint32_t>();
  e.model_of_node = B.mnode.as<int32_t>();
  e.l_max_of_node = B.lmax.as<uint32_t>();
  e.smem_tab_bytes = (int32_t)(sizeof(uint16_t) * ((nobs + 7u) & ~7u));
  CK(c, samu_count(c, launch_sample(a, e, B.heads.as<int32_t>(), (int32_t)heads.size(), seed, trial_begin, n_trials,
                                    nullptr, out_l_out, out_l_in_eff, s, index_base, (int32_t)stream_id)));
  CK(c, cudaStreamSynchronize(s));   // the scratch tables are reused by the next call
  return SAMU_OK;
}

// host l_true [n_req] -> device scratch (kept in the context until the next call)
static samu_status upload_known(samu_ctx* c, const uint32_t* l_true, const uint32_t** dev) {
  CK(c, c->d_known.ensure(sizeof(uint32_t) * std::max<size_t>(c->n_req, 1)));
  if (c->n_req)
    CK(c, cudaMemcpyAsync(c->d_known.p, l_true, sizeof(uint32_t) * c->n_req, cudaMemcpyHostToDevice, c->stream));
  *dev = c->d_known.as<uint32_t>();
  return SAMU_OK;
}

extern "C" samu_status samu_known_lengths(samu_ctx* c, const uint32_t* l_true, uint16_t* out_l_out,
                                          uint16_t* out_l_in_eff) {
  GUARD(c);
  if (!c->app_loaded) FAIL(c, SAMU_E_INVALID, "known_lengths: no app loaded");
  if (c->n_req && (!l_true || !out_l_out || !out_l_in_eff)) FAIL(c, SAMU_E_INVALID, "known_lengths: bad arguments");
  const uint32_t* d = nullptr;
  RET(upload_known(c, l_true, &d));
  RET(sample_or_known(c, 0, 0, 1, d, out_l_out, out_l_in_eff));
  CK(c, cudaStreamSynchronize(c->stream));   // the host array may be released on return
  return SAMU_OK;
}

// ---------------------------------------------------------------------------------------------
// batched simulation (internal form used by samu_simulate_batch and the greedy)
// ---------------------------------------------------------------------------------------------
struct SimJob {
  samu_candidate cand;
  int phase = 0;                       // dependency depth inside the batch
  const double* src_fin = nullptr;     // [T][n]
  const double* tau = nullptr;         // [T]
  const samu_trial_rec* tau_rec = nullptr;
  double* fin_t_out = nullptr;         // [T][n]
  uint32_t* fin_iter_out = nullptr;    // [T][n]
  samu_trial_rec* out_rec = nullptr;   // [T]
  bool fresh_node = false;             // the node's WorkloadState is FRESH in every trial (never committed)
};

struct StatePtrs {
  uint32_t* st = nullptr;
  uint16_t* g = nullptr;
  double* fin_t = nullptr;
  double* over = nullptr;
};

// SAMU_TRACE=1: per-stage planner timing on stderr (host wall clock; run_jobs is synchronous)
static bool trace_on() {
  static const bool on = [] { const char* e = std::getenv("SAMU_TRACE"); return e && *e == '1'; }();
  return on;
}
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static double g_trace_jobs_s = 0.0;   // time inside run_jobs since the last reset (trace only)
static int64_t g_trace_jobs_n = 0;

static samu_status run_jobs_impl(samu_ctx* c, std::vector<SimJob>& jobs, const uint16_t* l_out, const uint16_t* l_in,
                                 int32_t T, const StatePtrs& S);
static samu_status run_jobs(samu_ctx* c, std::vector<SimJob>& jobs, const uint16_t* l_out, const uint16_t* l_in,
                            int32_t T, const StatePtrs& S) {
  NvtxRange nv("samu K2 simulate batch");
  if (!trace_on()) return run_jobs_impl(c, jobs, l_out, l_in, T, S);
  const double t0 = now_s();
  const samu_status r = run_jobs_impl(c, jobs, l_out, l_in, T, S);
  g_trace_jobs_s += now_s() - t0;
  g_trace_jobs_n += 1;
  return r;
}

static samu_status run_jobs_impl(samu_ctx* c, std::vector<SimJob>& jobs, const uint16_t* l_out, const uint16_t* l_in,
                                 int32_t T, const StatePtrs& S) {
  if (jobs.empty() || T == 0) return SAMU_OK;
  if ((uint64_t)T * (uint64_t)c->n_req >= (1ull << 32))   // K2 indexes [trial][request] with u32
    FAIL(c, SAMU_E_INVALID, "simulate: trials x requests must stay below 2^32 per launch");
  cudaStream_t s = c->stream;
  int max_phase = 0;
  for (auto& j : jobs) max_phase = std::max(max_phase, j.phase);
  if (!c->sim_blocks_per_sm[0]) {
    int bpsm[SAMU_K2_MODES] = {};
    CK(c, simulate_prepare(bpsm));
    for (int md = 0; md < SAMU_K2_MODES; ++md)
      if (bpsm[md] < 1) FAIL(c, SAMU_E_CUDA, "simulate: kernel does not fit on an SM");
    for (int md = 0; md < SAMU_K2_MODES; ++md) c->sim_blocks_per_sm[md] = bpsm[md];
  }
  CK(c, c->d_error.ensure(2 * sizeof(int32_t)));
  CK(c, cudaMemsetAsync(c->d_error.p, 0, 2 * sizeof(int32_t), s));
  for (int ph = 0; ph <= max_phase; ++ph) {
    std::vector<int> idx;
    for (int i = 0; i < (int)jobs.size(); ++i) if (jobs[i].phase == ph) idx.push_back(i);
    if (idx.empty()) continue;
    std::vector<DevCand> dc(idx.size());
    std::vector<uint64_t> cost(idx.size());
    std::vector<double> kvf(idx.size(), 1.0);
    uint32_t max_q = 1, max_p = 1;
    for (size_t x = 0; x < idx.size(); ++x) {
      const SimJob& J = jobs[idx[x]];
      const samu_candidate& cd = J.cand;
      const int node = cd.node, model = c->node_model[node];
      const ModelReg& M = c->models[model];
      const int64_t blocks = plan_blocks(c, model, cd.dp, cd.tp);
      if (blocks < 0) FAIL(c, SAMU_E_INVALID, "simulate: invalid plan for the node's model");
      DevCand& D = dc[x];
      D.node = node; D.dp = cd.dp; D.tp = cd.tp; D.resume = cd.resume ? 1 : 0; D.commit = cd.commit ? 1 : 0;
      D.has_succ = c->node_has_succ[node];
      D.max_seqs = c->eng.max_num_seqs;
      D.bs = c->eng.block_size;
      D.budget = std::max(M.spec.l_max, c->eng.min_batched_tokens);
      D.blocks = (int32_t)blocks;
      D.L = M.spec.n_layers;
      D.h_tp = M.spec.hidden / (uint32_t)cd.tp;
      D.c = M.spec.c;
      D.LC = (uint64_t)D.L * D.c;
      D.K1 = 2ull * D.L * D.h_tp;
      const int slot = log2_exact((uint32_t)cd.tp);
      D.load_s = M.load[(size_t)slot * SAMU_MAX_DP + (cd.dp - 1)];
      D.coef = c->coef.at({model, slot}).as<double>();
      RET(replicas(c, node, cd.dp, &D.rep_off, &D.rep_req));
      D.src_fin = J.src_fin;
      D.tau = J.tau;
      D.tau_rec = J.tau_rec;
      D.fin_t_out = J.fin_t_out;
      D.fin_iter_out = J.fin_iter_out;
      D.out_rec = J.out_rec;
      // K2 path (DevCand::mode): FRESH = fresh state, no cross-node arrivals, no per-request
      // outputs; LEAN = FRESH without chain successors; 3 / 4 = LEAN / FRESH cut at a time limit
      const bool fresh = (S.st == nullptr || J.fresh_node) && !D.resume && !D.commit && !D.src_fin &&
                         !D.fin_t_out && !D.fin_iter_out && c->node_input[node] < 0 && c->eng.block_size == 16;
      const bool cut = D.tau != nullptr || D.tau_rec != nullptr;
      D.mode = !fresh ? 0 : D.has_succ ? (cut ? 4 : 2) : (cut ? 3 : 1);
      const std::vector<uint32_t>& ho = c->rep_off_host.at({node, cd.dp});
      uint32_t mx = 0;
      for (int j = 0; j < cd.dp; ++j) mx = std::max(mx, ho[j + 1] - ho[j]);
      max_q = std::max(max_q, mx);
      if (c->node_input[node] >= 0 || S.st) max_p = std::max(max_p, mx);
      // replica requests x expected output, x the KV pressure: a replica whose running set would
      // need more blocks than it has simulates more iterations (preemption, smaller batches)
      const double tok_r = c->node_mean_lin[node] + c->node_exp_out[node];
      const double demand = std::min<double>(c->eng.max_num_seqs, mx) * std::ceil(tok_r / c->eng.block_size);
      kvf[x] = std::max(1.0, demand / std::max<double>(1.0, (double)blocks));
      cost[x] = (uint64_t)((double)mx * c->node_exp_out[node]);
    }
    // small trial shares (e.g. one rank of an 8-GPU run): each launch is a few waves and its
    // longest replica-sims are the critical path, so their order counts the KV pressure too (and
    // the single candidates join the group launches below)
    int64_t items_all = 0;
    for (const DevCand& D : dc) items_all += (int64_t)T * D.dp;
    const bool small_share = items_all < 24 * (int64_t)c->n_sm * 24;
    static const int kvf_order = std::getenv("SAMU_K2_KVF_ORDER") ? std::atoi(std::getenv("SAMU_K2_KVF_ORDER")) : 0;
    if (small_share || kvf_order == 1)
      for (size_t x = 0; x < idx.size(); ++x) cost[x] = (uint64_t)((double)cost[x] * kvf[x]);
    // longest-first work items (cand, trial, replica)
    std::vector<int> order(idx.size());
    for (size_t x = 0; x < idx.size(); ++x) order[x] = (int)x;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    // one launch per K2 mode present (a single kernel holding several code paths runs ~10 %
    // slower: a multiple of the instruction footprint)
    {
      // small batches (e.g. the planner's later inner steps) run as one general launch: a launch per
      // mode only pays off when each covers several waves of the persistent grid
      int64_t cnt[SAMU_K2_MODES] = {};
      for (size_t x = 0; x < dc.size(); ++x) cnt[dc[x].mode] += (int64_t)T * dc[x].dp;
      const int64_t wave = (int64_t)c->n_sm * 24;
      // SAMU_K2_MODES=always|never overrides the size rule (tests run the LEAN / FRESH paths on
      // small batches; "never" runs everything on the general path)
      const char* pol = std::getenv("SAMU_K2_MODES");
      const bool always = pol && std::strcmp(pol, "always") == 0, never = pol && std::strcmp(pol, "never") == 0;
      const bool split = !never && (always || cnt[0] + cnt[1] + cnt[2] + cnt[3] + cnt[4] >= 4 * wave);
      for (DevCand& D : dc)
        if (!split || (!always && cnt[D.mode] < wave)) D.mode = 0;
    }
    {
      int64_t total = 0;
      for (const DevCand& D : dc) total += (int64_t)T * D.dp;
      if (total >= ((int64_t)1 << 31)) FAIL(c, SAMU_E_INVALID, "simulate: too many work items (trials x replicas)");
    }
    // Schedule sharing in the modes without a time limit (1 LEAN, 2 FRESH): the candidates of one
    // (node, dp) differ only in tp (KV blocks, coefficients, FLOPs factor, load time) and share
    // their event schedule while KV never binds below the largest block count.  They form groups
    // of <= 4, most blocks first, simulated once by the group launches (modes 5 / 6,
    // SimLaunch::grp); a member that falls out of sync in an item is re-simulated alone from the
    // launch's fallback queue.  A member that fell out of sync in most items of its last grouped
    // batch is scheduled on its own (a scheduling hint only: every record is exact either way).
    // SAMU_K2_GROUP=never: no groups; =always: group every member, ignoring the hints.
    const char* gpol = std::getenv("SAMU_K2_GROUP");
    const bool grouping = !(gpol && std::strcmp(gpol, "never") == 0);
    const bool group_all = gpol && std::strcmp(gpol, "always") == 0;
    auto hint_key = [&](const DevCand& D) { return std::array<int, 4>{D.node, D.dp, D.tp, D.mode}; };
    std::vector<std::vector<int>> groups;   // member lists, head (most blocks) first
    std::vector<bool> non_head(dc.size(), false);
    // small trial shares: the single candidates join the group launch (as groups of one) instead
    // of starting after it: one LEAN and one FRESH launch, longest first
    const bool fold = grouping && small_share;
    if (grouping) {
      std::vector<bool> taken(dc.size(), false);
      for (int x : order) {
        if (taken[x] || (dc[x].mode != 1 && dc[x].mode != 2)) continue;
        std::vector<int> mem;
        for (int y : order)
          if (!taken[y] && dc[y].mode == dc[x].mode && dc[y].node == dc[x].node && dc[y].dp == dc[x].dp) mem.push_back(y);
        for (int y : mem) taken[y] = true;
        std::stable_sort(mem.begin(), mem.end(), [&](int a, int b) { return dc[a].blocks > dc[b].blocks; });
        std::vector<int> keep{mem[0]};
        for (size_t i = 1; i < mem.size(); ++i) {
          auto h = c->share_hint.find(hint_key(dc[mem[i]]));
          if (group_all || h == c->share_hint.end() || h->second < 0.5) keep.push_back(mem[i]);
        }
        for (size_t g0 = 0; g0 < keep.size(); g0 += 4) {
          const size_t nv = std::min<size_t>(4, keep.size() - g0);
          if (nv < 2 && !fold) continue;   // a single member stays on the single-candidate path
          groups.emplace_back(keep.begin() + g0, keep.begin() + g0 + nv);
          for (size_t i = 0; i < nv; ++i) {
            if (i) non_head[keep[g0 + i]] = true;
            dc[keep[g0 + i]].mode += 4;
          }
        }
        if (fold)   // excluded members: groups of one in the same launch
          for (int y : mem)
            if (std::find(keep.begin(), keep.end(), y) == keep.end()) {
              groups.push_back({y});
              dc[y].mode += 4;
            }
      }
    }
    // per mode: candidate (group head) order and item offsets (the device decodes item ->
    // (candidate, trial, replica))
    std::vector<uint32_t> ord_off;   // [mode 0 ord | off] ... [mode 6 ...] [grp mode 5][grp mode 6]
    size_t ord_at[SAMU_K2_MODES], off_at[SAMU_K2_MODES], grp_at[SAMU_K2_MODES] = {};
    int64_t n_items[SAMU_K2_MODES], fb_cap[SAMU_K2_MODES] = {};
    int n_ord[SAMU_K2_MODES];
    std::vector<uint32_t> grp_words[SAMU_K2_MODES];
    for (int md = 0; md < SAMU_K2_MODES; ++md) {
      std::vector<uint32_t> ordm, offm{0};
      if (md == 5 || md == 6) {
        for (const auto& G : groups) {
          if (dc[G[0]].mode != md) continue;
          ordm.push_back((uint32_t)G[0]);
          offm.push_back(offm.back() + (uint32_t)(T * dc[G[0]].dp));
          uint32_t wds[4] = {(uint32_t)G.size(), 0u, 0u, 0u};
          for (size_t i = 1; i < G.size(); ++i) wds[i] = (uint32_t)G[i];
          grp_words[md].insert(grp_words[md].end(), wds, wds + 4);
          fb_cap[md] += (int64_t)(G.size() - 1) * T * dc[G[0]].dp;
        }
      } else {
        for (int x : order)
          if (dc[x].mode == md) {
            ordm.push_back((uint32_t)x);
            offm.push_back(offm.back() + (uint32_t)(T * dc[x].dp));
          }
      }
      n_items[md] = offm.back();
      n_ord[md] = (int)ordm.size();
      ord_at[md] = ord_off.size();
      ord_off.insert(ord_off.end(), ordm.begin(), ordm.end());
      off_at[md] = ord_off.size();
      ord_off.insert(ord_off.end(), offm.begin(), offm.end());
    }
    for (int md = 5; md <= 6; ++md) {
      if (grp_words[md].empty()) continue;
      while (ord_off.size() % 4) ord_off.push_back(0);   // uint4 alignment
      grp_at[md] = ord_off.size();
      ord_off.insert(ord_off.end(), grp_words[md].begin(), grp_words[md].end());
    }

    SimLaunch L;
    L.app = dev_app(c);
    L.n_cands = (int32_t)idx.size();
    L.n_trials = T;
    L.n_items = 0;   // set per launch (one launch per K2 mode)
    L.l_out = l_out;
    L.l_in = l_in;
    L.st = S.st;
    L.g = S.g;
    L.fin_t = S.fin_t;
    L.over = S.over;
    L.error = c->d_error.as<int32_t>();
    const int64_t fb_total = fb_cap[5] + fb_cap[6];
    {
      // persistent grid per mode: resident blocks x SMs, no more warps than items
      int n_blocks[SAMU_K2_MODES];
      size_t n_warps = SAMU_WARPS_PER_BLOCK;   // scratch rings: modes 0, 2, 4, 6 (the LEAN modes use none)
      for (int md = 0; md < SAMU_K2_MODES; ++md) {
        const int64_t want = (n_items[md] + fb_cap[md] + SAMU_WARPS_PER_BLOCK - 1) / SAMU_WARPS_PER_BLOCK;
        static const int bcap = std::getenv("SAMU_K2_BPSM_CAP") ? std::atoi(std::getenv("SAMU_K2_BPSM_CAP")) : 0;
        const int bpsm = bcap > 0 ? std::min(bcap, c->sim_blocks_per_sm[md]) : c->sim_blocks_per_sm[md];
        n_blocks[md] = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->n_sm * bpsm, want));
        if (md != 1 && md != 3 && md != 5) n_warps = std::max(n_warps, (size_t)n_blocks[md] * SAMU_WARPS_PER_BLOCK);
      }
      CK(c, c->d_scratch_q.ensure(sizeof(uint32_t) * n_warps * max_q));
      CK(c, c->d_scratch_key.ensure(sizeof(uint64_t) * n_warps * 4 * max_p));
      CK(c, c->d_scratch_idx.ensure(sizeof(uint32_t) * n_warps * 4 * max_p));
      CK(c, upload(c->d_cands, dc, s));
      CK(c, upload(c->d_items, ord_off, s));
      // item counters [7], fallback counters [2][3] (modes 5, 6), fallbacks per candidate [n]
      const size_t n_ctr = SAMU_K2_MODES + 6 + idx.size();
      CK(c, c->d_counter.ensure(n_ctr * sizeof(uint32_t)));
      CK(c, cudaMemsetAsync(c->d_counter.p, 0, n_ctr * sizeof(uint32_t), s));
      if (fb_total >= ((int64_t)1 << 31)) FAIL(c, SAMU_E_INVALID, "simulate: too many work items (trials x replicas)");
      if (fb_total) {
        CK(c, c->d_fb.ensure(sizeof(uint2) * fb_total));
        CK(c, cudaMemsetAsync(c->d_fb.p, 0xFF, sizeof(uint2) * fb_total, s));
      }
      CK(c, c->d_rep_rec.ensure(sizeof(samu_trial_rec) * 16 * idx.size() * T));
      L.cands = c->d_cands.as<DevCand>();
      L.ord = nullptr;
      L.off = nullptr;
      L.n_ord = 0;
      L.next_item = c->d_counter.as<uint32_t>();
      L.grp = nullptr;
      L.fb = nullptr;
      L.fb_ctr = nullptr;
      L.fb_count = c->d_counter.as<uint32_t>() + SAMU_K2_MODES + 6;
      L.rep_rec = c->d_rep_rec.as<samu_trial_rec>();
      L.scratch_q = c->d_scratch_q.as<uint32_t>();
      L.scratch_key = c->d_scratch_key.as<uint64_t>();
      L.scratch_idx = c->d_scratch_idx.as<uint32_t>();
      L.max_q = (int32_t)max_q;
      L.max_p = (int32_t)max_p;
      SimLaunch LM[SAMU_K2_MODES];
      int modes[SAMU_K2_MODES], nb[SAMU_K2_MODES], n_launch = 0;
      // in order on s; the LEAN launches (5, 1) concurrent on the aux stream
      static int order[SAMU_K2_MODES] = {0, 6, 2, 4, 3, 5, 1};
      static bool order_read = false;
      if (!order_read) {   // SAMU_K2_ORDER: launch order of the modes (experiments), e.g. "0,6,2,4,3,1,5"
        order_read = true;
        if (const char* o = std::getenv("SAMU_K2_ORDER")) {
          int v[SAMU_K2_MODES], n = 0;
          for (const char* p = o; *p && n < SAMU_K2_MODES; ) {
            v[n++] = std::atoi(p);
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
          }
          int seen = 0;
          for (int i = 0; i < n; ++i) seen |= (v[i] >= 0 && v[i] < SAMU_K2_MODES) ? 1 << v[i] : 0;
          if (n == SAMU_K2_MODES && seen == (1 << SAMU_K2_MODES) - 1)   // a permutation of the modes
            for (int i = 0; i < n; ++i) order[i] = v[i];
        }
      }
      for (int md : order) {
        if (n_items[md] == 0) continue;
        SimLaunch& X = LM[n_launch];
        X = L;
        X.ord = c->d_items.as<uint32_t>() + ord_at[md];
        X.off = c->d_items.as<uint32_t>() + off_at[md];
        X.n_ord = n_ord[md];
        X.n_items = (int32_t)n_items[md];
        X.next_item = c->d_counter.as<uint32_t>() + md;
        if (md == 5 || md == 6) {
          X.grp = reinterpret_cast<const uint4*>(c->d_items.as<uint32_t>() + grp_at[md]);
          X.fb = c->d_fb.as<uint2>() + (md == 6 ? fb_cap[5] : 0);
          X.fb_ctr = c->d_counter.as<uint32_t>() + SAMU_K2_MODES + 3 * (md - 5);
        }
        modes[n_launch] = md;
        nb[n_launch] = n_blocks[md];
        ++n_launch;
      }
      if (n_launch > 1 && !c->aux_stream) {
        CK(c, cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
        CK(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CK(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
      }
      // concurrent LEAN launches only when the others are short (a few waves): then their
      // longest replica-sims are the critical path and the LEAN items fill the idle warps; with
      // many waves the kernels only compete for the instruction cache (~2 % slower)
      // (SAMU_K2_OVERLAP=0 / 1 overrides the rule: tests and sanitizer runs of the chained launches)
      const int ov_env = std::getenv("SAMU_K2_OVERLAP") ? std::atoi(std::getenv("SAMU_K2_OVERLAP")) : -1;
      const bool overlap = ov_env >= 0 ? ov_env != 0
                                       : n_items[0] + n_items[2] + n_items[3] + n_items[4] + n_items[6] < 8 * (int64_t)c->n_sm * 24;
      CK(c, launch_simulate(LM, modes, nb, n_launch, dc.data(), (uint32_t)c->eng.block_size, s,
                            overlap ? c->aux_stream : nullptr, c->ev_fork, c->ev_join));
      c->launches += n_launch > 1 ? n_launch - 1 : 0;
    }
    CK(c, launch_combine(L.rep_rec, L.cands, (int32_t)idx.size(), T, S.over, c->n_nodes, s));
    c->launches += 2;
    c->n_sims += (int64_t)idx.size() * T;
    int32_t herr[2] = {0, 0};
    std::vector<uint32_t> hfb;
    CK(c, cudaMemcpyAsync(herr, c->d_error.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (fb_total) {
      hfb.assign(idx.size(), 0u);
      CK(c, cudaMemcpyAsync(hfb.data(), c->d_counter.as<uint32_t>() + SAMU_K2_MODES + 6, sizeof(uint32_t) * idx.size(),
                            cudaMemcpyDeviceToHost, s));
    }
    CK(c, cudaStreamSynchronize(s));
    for (const auto& G : groups) {
      const int64_t items = (int64_t)T * dc[G[0]].dp;
      c->share[0] += items;
      c->share[1] += items * (int64_t)(G.size() - 1);
      for (size_t i = 1; i < G.size(); ++i) {
        DevCand D = dc[G[i]];
        D.mode -= 4;
        c->share[2] += hfb[G[i]];
        c->share_hint[hint_key(D)] = (double)hfb[G[i]] / (double)items;
      }
    }
    if (herr[0]) {
      static const char* sites[] = {"?", "waiting chain successor of a done request", "bad status word",
                                    "scratch overflow", "running/preempted set exceeds the engine slots",
                                    "running rank out of range", "preempted seq out of range",
                                    "queued seq out of range", "carried KV blocks exceed capacity",
                                    "head cannot fit an empty engine", "preemption emptied the engine"};
      const int si = (herr[1] >= 0 && herr[1] <= 10) ? herr[1] : 0;
      FAIL(c, herr[0], std::string(herr[0] == SAMU_E_INFEASIBLE ? "simulate: infeasible (capacity below one sequence): "
                                                              : "simulate: inconsistent WorkloadState: ") + sites[si]);
    }
  }
  return SAMU_OK;
}

// ---------------------------------------------------------------------------------------------
// trial sharding: rank r owns trials [begin, begin + count) of T (contiguous blocks)
// ---------------------------------------------------------------------------------------------
static void trial_share(int T, int world, int rank, int* begin, int* count) {
  const int base = T / world, rem = T % world;
  *count = base + (rank < rem ? 1 : 0);
  *begin = rank * base + std::min(rank, rem);
}

// Sharding of a (jobs x trials) product over the ranks: world = Wt x Wc, rank r simulates trial
// block r % Wt (contiguous split of T over Wt blocks) of the jobs of class r / Wt.  Wc = 1 (pure
// trial sharding) whenever T >= world: trials are i.i.d., so every rank gets the same work and
// all of its candidates.  With fewer trials than ranks (C1: T = 1) the candidates are split into
// Wc = world / Wt classes, Wt the largest divisor of world not above T.  SAMU_SHARD_CLASSES=k
// forces Wc = k (k | world; tests).
static void shard_split_w(int world, int T, int forced, int* Wt, int* Wc) {
  int wc = 1;
  if (forced > 0 && world % forced == 0) wc = forced;
  else if (T < world) {
    int wt = 1;
    for (int d = 1; d <= world; ++d) if (world % d == 0 && d <= std::max(T, 1)) wt = d;
    wc = world / wt;
  }
  *Wc = wc;
  *Wt = world / wc;
}

static void shard_split(const samu_ctx* c, int T, int* Wt, int* Wc) {
  const char* e = std::getenv("SAMU_SHARD_CLASSES");
  shard_split_w(c->world, T, e ? std::atoi(e) : 0, Wt, Wc);
}

// Job classes of one batch (Wc > 1): jobs longest-first (stable on ties) onto the least loaded
// class (lowest index on ties); identical on every rank.
static void assign_classes(const std::vector<int>& jobs, const std::vector<double>& work, int Wc, std::vector<int>& cls) {
  std::vector<int> order(jobs);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
  std::vector<double> load(Wc, 0.0);
  for (int x : order) {
    int k = 0;
    for (int q = 1; q < Wc; ++q) if (load[q] < load[k]) k = q;
    cls[x] = k;
    load[k] += work[x];
  }
}

extern "C" samu_status samu_shard_plan(int32_t n_trials, int32_t world, int32_t rank, int32_t forced_classes,
                                       int32_t* trial_blocks, int32_t* job_classes, int32_t* trial_begin,
                                       int32_t* trial_count, int32_t* my_class) {
  if (n_trials < 0 || world < 1 || rank < 0 || rank >= world) return SAMU_E_INVALID;
  int Wt = 1, Wc = 1, b = 0, cnt = 0;
  shard_split_w(world, n_trials, forced_classes, &Wt, &Wc);
  trial_share(n_trials, Wt, rank % Wt, &b, &cnt);
  if (trial_blocks) *trial_blocks = Wt;
  if (job_classes) *job_classes = Wc;
  if (trial_begin) *trial_begin = b;
  if (trial_count) *trial_count = cnt;
  if (my_class) *my_class = rank / Wt;
  return SAMU_OK;
}

extern "C" samu_status samu_shard_classes(int32_t n_jobs, const double* work, int32_t job_classes, int32_t* out_class) {
  if (n_jobs < 0 || job_classes < 1 || (n_jobs > 0 && (!work || !out_class))) return SAMU_E_INVALID;
  std::vector<int> jobs(n_jobs), cls(n_jobs, 0);
  std::vector<double> w(n_jobs);
  for (int x = 0; x < n_jobs; ++x) {
    if (!(work[x] >= 0.0)) return SAMU_E_INVALID;   // also rejects NaN
    jobs[x] = x;
    w[x] = work[x];
  }
  assign_classes(jobs, w, job_classes, cls);
  for (int x = 0; x < n_jobs; ++x) out_class[x] = cls[x];
  return SAMU_OK;
}

// all-gather per-(job, local trial) records [n][T_local] into rows of `dst` ([*][T]) at `slots`;
// job_class[x] = class of job x (all 0 under pure trial sharding), Wt trial blocks
static samu_status gather_records(samu_ctx* c, const samu_trial_rec* local, int n, int T, samu_trial_rec* dst,
                                  const std::vector<int>& slots, const std::vector<int>* job_class = nullptr,
                                  int Wt = 0) {
  cudaStream_t s = c->stream;
  if (n == 0) return SAMU_OK;
  if (!sharded(c)) {
    for (int x = 0; x < n; ++x)
      if (dst + (size_t)slots[x] * T != local + (size_t)x * T)
        CK(c, cudaMemcpyAsync(dst + (size_t)slots[x] * T, local + (size_t)x * T, sizeof(samu_trial_rec) * T,
                              cudaMemcpyDeviceToDevice, s));
    return SAMU_OK;
  }
  if (Wt <= 0) Wt = c->world;
  int b0, cnt0;
  trial_share(T, Wt, c->rank % Wt, &b0, &cnt0);
  const int Tmax = (T + Wt - 1) / Wt;
  const size_t row = sizeof(samu_trial_rec) * Tmax;
  CK(c, c->d_gather_send.ensure(row * n));
  CK(c, c->d_gather_recv.ensure(row * n * c->world));
  CK(c, cudaMemsetAsync(c->d_gather_send.p, 0, row * n, s));
  if (cnt0)
    CK(c, cudaMemcpy2DAsync(c->d_gather_send.p, row, local, sizeof(samu_trial_rec) * cnt0, sizeof(samu_trial_rec) * cnt0,
                            n, cudaMemcpyDeviceToDevice, s));
  RET(comm_allgather(c, c->d_gather_send.p, c->d_gather_recv.p, row * n));
  // one unpack kernel instead of a copy per (job, rank)
  std::vector<int32_t> meta(2 * (size_t)n);
  for (int x = 0; x < n; ++x) {
    meta[x] = slots[x];
    meta[n + x] = job_class ? (*job_class)[x] : 0;
  }
  CK(c, upload(c->d_gather_meta, meta, s));
  CK(c, samu_count(c, launch_unpack_gather(c->d_gather_recv.as<samu_trial_rec>(), c->world, n, Tmax, T, Wt,
                                           c->d_gather_meta.as<int32_t>(), c->d_gather_meta.as<int32_t>() + n, dst, s)));
  return SAMU_OK;
}

// ---------------------------------------------------------------------------------------------
// C ABI: samu_simulate_batch
// ---------------------------------------------------------------------------------------------
extern "C" samu_status samu_simulate_batch(samu_ctx* c, const samu_candidate* cands, int32_t n_cands,
                                           const uint16_t* l_out, const uint16_t* l_in_eff, int32_t n_trials,
                                           uint32_t* st, uint16_t* g, double* fin_t, double* overshoot,
                                           const double* time_limit, samu_trial_rec* out_recs,
                                           samu_cand_summary* out_summary, uint32_t* out_fin_iter,
                                           double* out_fin_t) {
  GUARD(c);
  if (!c->app_loaded) FAIL(c, SAMU_E_INVALID, "simulate_batch: no app loaded");
  if (n_cands < 0 || (n_cands && !cands) || n_trials < 0 || (n_trials && n_cands && (!l_out || !l_in_eff || !out_recs)))
    FAIL(c, SAMU_E_INVALID, "simulate_batch: bad arguments");
  if (n_trials >= (1 << 27)) FAIL(c, SAMU_E_INVALID, "simulate_batch: too many trials");
  const bool has_state = st != nullptr;
  if (has_state && (!g || !fin_t || !overshoot)) FAIL(c, SAMU_E_INVALID, "simulate_batch: partial state");
  const size_t n = (size_t)c->n_req;
  std::vector<SimJob> jobs(n_cands);
  std::vector<int> commit_nodes;
  std::vector<DevBuf> own_fin;
  std::vector<int> needs_fin(n_cands, 0);
  for (int i = 0; i < n_cands; ++i) {
    const samu_candidate& cd = cands[i];
    if (cd.node < 0 || cd.node >= c->n_nodes) FAIL(c, SAMU_E_INVALID, "simulate_batch: bad node");
    if (plan_blocks(c, c->node_model[cd.node], cd.dp, cd.tp) < 0) FAIL(c, SAMU_E_INVALID, "simulate_batch: invalid plan");
    if (cd.dep_src >= 0) {
      if (cd.dep_src >= i || cands[cd.dep_src].node != c->node_input[cd.node])
        FAIL(c, SAMU_E_INVALID, "simulate_batch: dep_src must be an earlier candidate of the node's input node");
      needs_fin[cd.dep_src] = 1;
    }
    if (cd.commit) {
      if (!has_state) FAIL(c, SAMU_E_INVALID, "simulate_batch: commit needs a WorkloadState");
      if (std::find(commit_nodes.begin(), commit_nodes.end(), cd.node) != commit_nodes.end())
        FAIL(c, SAMU_E_INVALID, "simulate_batch: two committing candidates for one node");
      commit_nodes.push_back(cd.node);
    }
  }
  for (int i = 0; i < n_cands; ++i) {
    SimJob& J = jobs[i];
    J.cand = cands[i];
    J.phase = cands[i].dep_src >= 0 ? jobs[cands[i].dep_src].phase + 1 : 0;
    J.tau = time_limit ? time_limit + (size_t)i * n_trials : nullptr;
    J.out_rec = out_recs + (size_t)i * n_trials;
    J.fin_iter_out = out_fin_iter ? out_fin_iter + (size_t)i * n_trials * n : nullptr;
    if (out_fin_t) J.fin_t_out = out_fin_t + (size_t)i * n_trials * n;
    else if (needs_fin[i]) {
      own_fin.emplace_back();
      CK(c, own_fin.back().ensure(sizeof(double) * n_trials * n));
      J.fin_t_out = own_fin.back().as<double>();
    }
    if (out_fin_iter) CK(c, cudaMemsetAsync(J.fin_iter_out, 0xFF, sizeof(uint32_t) * n_trials * n, c->stream));
    if (J.fin_t_out)
      CK(c, samu_count(c, launch_fill_f64(J.fin_t_out, (int64_t)n_trials * n, std::numeric_limits<double>::infinity(), c->stream)));
  }
  for (int i = 0; i < n_cands; ++i)
    if (cands[i].dep_src >= 0) jobs[i].src_fin = jobs[cands[i].dep_src].fin_t_out;
  StatePtrs S{st, g, fin_t, overshoot};
  {
    samu_status rj = run_jobs(c, jobs, l_out, l_in_eff, n_trials, S);
    if (out_summary && n_cands) rj = agree(c, rj);   // the summary below is collective
    RET(rj);
  }
  if (out_summary && n_cands) {
    int T_total = n_trials;
    const samu_trial_rec* all = out_recs;
    if (sharded(c)) {
      // every rank holds n_trials local trials; the world total is their sum
      int32_t Tl = n_trials, Tsum = 0;
      DevBuf tmp;
      CK(c, tmp.ensure(sizeof(int32_t) * 2));
      CK(c, cudaMemcpyAsync(tmp.p, &Tl, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
      RET(comm_allreduce_i32(c, tmp.as<int32_t>(), tmp.as<int32_t>() + 1, 1, 1));
      CK(c, cudaMemcpyAsync(&Tsum, tmp.as<int32_t>() + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
      CK(c, cudaStreamSynchronize(c->stream));
      int b, cnt;
      trial_share(Tsum, c->world, c->rank, &b, &cnt);
      samu_status split = SAMU_OK;
      if (cnt != n_trials) {
        c->err = "simulate_batch: local trial count must follow the contiguous split";
        split = SAMU_E_INVALID;
      }
      RET(agree(c, split));
      T_total = Tsum;
      CK(c, c->d_sum.ensure(sizeof(samu_trial_rec) * (size_t)n_cands * T_total));
      std::vector<int> slots(n_cands);
      for (int i = 0; i < n_cands; ++i) slots[i] = i;
      RET(gather_records(c, out_recs, n_cands, T_total, c->d_sum.as<samu_trial_rec>(), slots));
      all = c->d_sum.as<samu_trial_rec>();
    }
    NvtxRange nv("samu K3 summaries");
    CK(c, c->d_cand_sum.ensure(sizeof(samu_cand_summary) * n_cands));
    CK(c, samu_count(c, launch_summary(all, n_cands, T_total, c->d_cand_sum.as<samu_cand_summary>(), c->stream)));
    CK(c, cudaMemcpyAsync(out_summary, c->d_cand_sum.p, sizeof(samu_cand_summary) * n_cands, cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
  }
  return SAMU_OK;
}

// ---------------------------------------------------------------------------------------------
// C ABI: samu_plan_greedy — Algorithm 1 with the device estimator
// ---------------------------------------------------------------------------------------------
namespace {

struct Ent {
  int node, dp, tp;
  bool operator==(const Ent& o) const { return node == o.node && dp == o.dp && tp == o.tp; }
};

struct Greedy {
  samu_ctx* c;
  int T = 0, Tl = 0, tb = 0;
  int Wt = 1, Wc = 1, my_class = 0;        // (trial block, job class) sharding, shard_split
  std::map<int, int> slot_class;           // simulation slot -> job class that ran it
  std::map<int, SimJob> slot_job;          // full slot -> its job (re-run locally for a commit)
  std::map<int, int> slot_src;             // slot -> full slot of its dependency source
  std::set<int> have_fin;                  // full slots whose finish times this rank computed
  size_t n = 0;
  DevBuf lo, li, st, g, fin_t, over;
  StatePtrs S;
  std::vector<Ent> prev;
  // per-stage caches of simulations: records [slot][T] (all trials), finish-time buffers
  DevBuf cache, local_rec, d_sc, d_out, d_best, d_any;
  int cap_slots = 0, n_slots = 0;
  std::map<std::vector<int>, int> full_slot, cut_slot;
  std::map<int, DevBuf> fin_buf;           // full slot -> [Tl][n] finish times (dependency sources)
  std::vector<DevBuf> fin_pool;            // finish-time buffers of earlier stages, reused (no cudaMalloc / cudaFree per stage)
  std::map<int, int> pending_phase;        // slot -> phase within the pending batch
  std::vector<SimJob> pending;
  std::vector<int> pending_slots;
  std::vector<int> pending_tau;            // f* full slot whose records give tau, or -1
  std::vector<int> pending_src;            // full slot of the job's dependency source, or -1
  int64_t evals = 0;
  std::vector<bool> is_input;
  std::vector<bool> touched;               // node committed in some stage (its state is no longer FRESH)
  bool preempt = true;                  // false: no-preemption ablation (reading c29)
  const uint32_t* known = nullptr;      // device known output lengths (reading c30)
  std::vector<int> undone_now;          // per node: unfinished in some trial (current stage)

  // No-preemption: every model of the previous stage that is unfinished keeps its entry
  std::vector<Ent> pinned() const {
    std::vector<Ent> E;
    if (preempt) return E;
    for (const Ent& e : prev) if (undone_now[e.node]) E.push_back(e);
    return E;
  }
  static bool is_pinned(const std::vector<Ent>& pin, int v) {
    for (const Ent& e : pin) if (e.node == v) return true;
    return false;
  }

  bool resumes(const Ent& e) const {
    for (const Ent& x : prev) if (x == e) return true;
    return false;
  }
  std::vector<int> key_of(const Ent& e, const std::vector<Ent>& E) const {
    std::vector<int> k{e.node, e.dp, e.tp, resumes(e) ? 1 : 0};
    const int src = c->node_input[e.node];
    if (src >= 0)
      for (const Ent& x : E)
        if (x.node == src) { auto ks = key_of(x, E); k.insert(k.end(), ks.begin(), ks.end()); }
    return k;
  }
  samu_status grow(int need) {
    if (need <= cap_slots) return SAMU_OK;
    int nc = std::max(need, std::max(64, cap_slots * 2));
    DevBuf nb;
    CK(c, nb.ensure(sizeof(samu_trial_rec) * (size_t)nc * T));
    if (cap_slots) CK(c, cudaMemcpyAsync(nb.p, cache.p, sizeof(samu_trial_rec) * (size_t)cap_slots * T, cudaMemcpyDeviceToDevice, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    cache = std::move(nb);
    cap_slots = nc;
    return SAMU_OK;
  }
  samu_trial_rec* rec(int slot) { return cache.as<samu_trial_rec>() + (size_t)slot * T; }

  samu_status ensure_full(const Ent& e, const std::vector<Ent>& E, int* out_slot) {
    auto key = key_of(e, E);
    auto it = full_slot.find(key);
    if (it != full_slot.end()) { *out_slot = it->second; return SAMU_OK; }
    const double* sf = nullptr;
    int phase = 0, src_slot = -1;
    const int src = c->node_input[e.node];
    if (src >= 0)
      for (const Ent& x : E)
        if (x.node == src) {
          int ss;
          RET(ensure_full(x, E, &ss));
          sf = fin_buf.at(ss).as<double>();
          src_slot = ss;
          auto pp = pending_phase.find(ss);
          if (pp != pending_phase.end()) phase = pp->second + 1;
        }
    const int slot = n_slots++;
    RET(grow(n_slots));
    full_slot[key] = slot;
    SimJob J;
    J.cand = samu_candidate{e.node, e.dp, e.tp, resumes(e) ? 1 : 0, -1, 0};
    J.fresh_node = !touched[e.node];
    J.phase = phase;
    J.src_fin = sf;
    if (is_input[e.node]) {
      DevBuf& fb = fin_buf[slot];
      if (!fin_pool.empty()) { fb = std::move(fin_pool.back()); fin_pool.pop_back(); }
      CK(c, fb.ensure(sizeof(double) * (size_t)Tl * n));
      J.fin_t_out = fb.as<double>();
    }
    pending.push_back(J);
    pending_slots.push_back(slot);
    pending_tau.push_back(-1);
    pending_src.push_back(src_slot);
    pending_phase[slot] = phase;
    slot_job[slot] = J;
    slot_src[slot] = src_slot;
    *out_slot = slot;
    return SAMU_OK;
  }
  samu_status ensure_cut(const Ent& e, const Ent& f, const std::vector<Ent>& E, int fslot, int* out_slot) {
    auto key = key_of(e, E);
    auto kf = key_of(f, E);
    key.push_back(-1);
    key.insert(key.end(), kf.begin(), kf.end());
    auto it = cut_slot.find(key);
    if (it != cut_slot.end()) { *out_slot = it->second; return SAMU_OK; }
    const double* sf = nullptr;
    int src_slot = -1;
    const int src = c->node_input[e.node];
    if (src >= 0)
      for (const Ent& x : E)
        if (x.node == src) { int ss; RET(ensure_full(x, E, &ss)); sf = fin_buf.at(ss).as<double>(); src_slot = ss; }
    const int slot = n_slots++;
    RET(grow(n_slots));
    cut_slot[key] = slot;
    SimJob J;
    J.cand = samu_candidate{e.node, e.dp, e.tp, resumes(e) ? 1 : 0, -1, 0};
    J.fresh_node = !touched[e.node];
    J.phase = 0;
    J.src_fin = sf;
    pending.push_back(J);             // tau_k = T_f*^(k) (this rank's trials), resolved at flush
    pending_slots.push_back(slot);
    pending_tau.push_back(fslot);
    pending_src.push_back(src_slot);
    slot_src[slot] = src_slot;
    *out_slot = slot;
    return SAMU_OK;
  }
  // run the pending simulations, then all-gather their records into the cache
  samu_status flush() {
    if (pending.empty()) return SAMU_OK;
    // job classes (Wc > 1: fewer trials than ranks): jobs without a dependency source are spread
    // over the classes longest-first onto the least loaded (identically on every rank); a
    // dependent job runs where its source's finish times are
    std::vector<int> cls(pending.size(), 0);
    if (Wc > 1) {
      std::vector<int> free_jobs;
      std::vector<double> work(pending.size(), 0.0);
      for (size_t x = 0; x < pending.size(); ++x) {
        const int v = pending[x].cand.node;
        work[x] = (double)(c->node_end[v] - c->node_begin[v]) * c->node_exp_out[v];
        if (pending_src[x] < 0) free_jobs.push_back((int)x);
      }
      assign_classes(free_jobs, work, Wc, cls);
      for (int x : free_jobs) slot_class[pending_slots[x]] = cls[x];
      for (size_t x = 0; x < pending.size(); ++x)
        if (pending_src[x] >= 0) {
          cls[x] = slot_class.at(pending_src[x]);
          slot_class[pending_slots[x]] = cls[x];
        }
    }
    // the cache may have been reallocated after tau_rec pointers were taken: re-point them
    CK(c, local_rec.ensure(sizeof(samu_trial_rec) * pending.size() * std::max(Tl, 1)));
    std::vector<SimJob> mine;
    for (size_t x = 0; x < pending.size(); ++x) {
      pending[x].out_rec = !sharded(c) ? rec(pending_slots[x]) : local_rec.as<samu_trial_rec>() + x * Tl;
      pending[x].tau_rec = pending_tau[x] >= 0 ? rec(pending_tau[x]) + tb : nullptr;
      if (cls[x] != my_class) continue;
      if (pending[x].fin_t_out) {
        CK(c, samu_count(c, launch_fill_f64(pending[x].fin_t_out, (int64_t)Tl * n, std::numeric_limits<double>::infinity(),
                                            c->stream)));
        have_fin.insert(pending_slots[x]);
      }
      mine.push_back(pending[x]);
    }
    RET(agree(c, run_jobs(c, mine, lo.as<uint16_t>(), li.as<uint16_t>(), Tl, S)));
    if (sharded(c))
      RET(gather_records(c, local_rec.as<samu_trial_rec>(), (int)pending.size(), T, cache.as<samu_trial_rec>(), pending_slots,
                         &cls, Wt));
    pending.clear();
    pending_slots.clear();
    pending_tau.clear();
    pending_src.clear();
    pending_phase.clear();
    return SAMU_OK;
  }

  // finish times of full slot `ss` on this rank (job classes: the slot may have run elsewhere):
  // re-simulated here, after its own source, for a commit that depends on it
  samu_status ensure_local_fin(int ss) {
    if (have_fin.count(ss)) return SAMU_OK;
    const int src = slot_src.count(ss) ? slot_src.at(ss) : -1;
    if (src >= 0) RET(ensure_local_fin(src));
    SimJob J = slot_job.at(ss);
    J.phase = 0;
    J.src_fin = src >= 0 ? fin_buf.at(src).as<double>() : nullptr;
    J.fin_t_out = fin_buf.at(ss).as<double>();
    J.tau_rec = nullptr;
    CK(c, local_rec.ensure(sizeof(samu_trial_rec) * std::max(Tl, 1)));
    J.out_rec = local_rec.as<samu_trial_rec>();
    CK(c, samu_count(c, launch_fill_f64(J.fin_t_out, (int64_t)Tl * n, std::numeric_limits<double>::infinity(), c->stream)));
    std::vector<SimJob> one{J};
    RET(run_jobs(c, one, lo.as<uint16_t>(), li.as<uint16_t>(), Tl, S));
    have_fin.insert(ss);
    return SAMU_OK;
  }

  struct Cand { std::vector<Ent> E; Ent P; };

  // Score candidate stages on the device: full simulations of every entry, f* per candidate,
  // cut simulations of the other entries at t_E^(k), then T_E and the choice.  mode 0: Alg. 1's
  // argmax dT/dN (ties: dN, node, tp, dp); mode 1: argmax T_E (ties: first candidate).
  samu_status score_batch(const std::vector<Cand>& cands, double TE_star, int g_star, int mode, int32_t* best,
                          double* maxdT, std::vector<StageOut>& so, bool count = true) {
    cudaStream_t s = c->stream;
    const int nc = (int)cands.size();
    std::vector<StageCand> sc(nc);
    for (int x = 0; x < nc; ++x) {
      StageCand& q = sc[x];
      std::memset(&q, 0, sizeof(q));
      q.n_entries = (int)cands[x].E.size();
      q.gpus = 0;
      for (int i = 0; i < q.n_entries; ++i) {
        const Ent& e = cands[x].E[i];
        RET(ensure_full(e, cands[x].E, &q.full_slot[i]));
        q.node[i] = e.node;
        q.cut_slot[i] = -1;
        q.gpus += e.dp * e.tp;
      }
      q.changed_node = cands[x].P.node;
      q.changed_dp = cands[x].P.dp;
      q.changed_tp = cands[x].P.tp;
    }
    RET(flush());
    CK(c, upload(d_sc, sc, s));
    CK(c, d_out.ensure(sizeof(StageOut) * nc));
    CK(c, samu_count(c, launch_fstar(cache.as<samu_trial_rec>(), T, d_sc.as<StageCand>(), nc, d_out.as<StageOut>(), s)));
    so.assign(nc, StageOut{});
    CK(c, cudaMemcpyAsync(so.data(), d_out.p, sizeof(StageOut) * nc, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    for (int x = 0; x < nc; ++x) {
      const int f = so[x].fstar;
      for (int i = 0; i < sc[x].n_entries; ++i)
        if (i != f) RET(ensure_cut(cands[x].E[i], cands[x].E[f], cands[x].E, sc[x].full_slot[f], &sc[x].cut_slot[i]));
    }
    RET(flush());
    CK(c, upload(d_sc, sc, s));
    CK(c, samu_count(c, launch_stage_score(cache.as<samu_trial_rec>(), T, d_sc.as<StageCand>(), nc, d_out.as<StageOut>(),
                                           TE_star, g_star, mode, d_best.as<int32_t>(),
                                           reinterpret_cast<double*>(d_best.as<char>() + 8), s)));
    if (count) evals += nc;
    CK(c, cudaMemcpyAsync(best, d_best.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(c, cudaMemcpyAsync(maxdT, d_best.as<char>() + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(c, cudaMemcpyAsync(so.data(), d_out.p, sizeof(StageOut) * nc, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    return SAMU_OK;
  }

  std::vector<std::vector<std::pair<int, int>>> plans;

  // Algorithm 1 inner loop
  samu_status choose_greedy(const std::vector<int>& unfinished, const std::vector<int>& undone, std::vector<Ent>& Es,
                            StageOut& chosen) {
    const int N = (int)c->eng.n_gpus;
    const std::vector<Ent> pin = pinned();
    double TE_star = 0.0;
    if (!pin.empty()) {   // E* starts from the running models
      int32_t b = -1;
      double mx = 0.0;
      std::vector<StageOut> so;
      RET(score_batch({Cand{pin, pin[0]}}, 0.0, 0, 1, &b, &mx, so));
      Es = pin;
      TE_star = so[0].TE;
      chosen = so[0];
    }
    for (;;) {
      std::vector<int> ready;
      for (int v : unfinished) {
        const int u = c->node_input[v];
        bool ok = u < 0 || !undone[u];
        for (const Ent& e : Es) if (e.node == u) ok = true;
        if (ok) ready.push_back(v);
      }
      std::vector<Cand> cands;
      int g_star = 0;
      for (const Ent& e : Es) g_star += e.dp * e.tp;
      for (int v : ready)
        for (auto& pl : plans[v]) {
          if (is_pinned(pin, v)) break;
          Ent P{v, pl.first, pl.second};
          int prime = -1;
          for (size_t i = 0; i < Es.size(); ++i) if (Es[i].node == v) prime = (int)i;
          std::vector<Ent> E = Es;
          int gE = 0;
          if (prime >= 0) {
            E[prime] = P;
            for (const Ent& x : E) gE += x.dp * x.tp;
            if (!(g_star < gE && gE <= N)) continue;      // Alg. 1 line 11
          } else {
            E.push_back(P);
            for (const Ent& x : E) gE += x.dp * x.tp;
            if (gE > N) continue;                          // Alg. 1 line 14
          }
          std::sort(E.begin(), E.end(), [](const Ent& a, const Ent& b) { return a.node < b.node; });
          cands.push_back({E, P});
        }
      if (cands.empty()) break;
      int32_t best = -1;
      double maxdT = 0.0;
      std::vector<StageOut> so;
      RET(score_batch(cands, TE_star, g_star, 0, &best, &maxdT, so));
      if (maxdT < 0.0) break;                               // Alg. 1 line 19
      Es = cands[best].E;
      TE_star = so[best].TE;
      chosen = so[best];
    }
    return SAMU_OK;
  }

  // Max-heuristic: all GPUs to the lowest-id ready model, plan of highest stage
  // throughput (ties: enumeration order), stage runs that model to completion
  samu_status choose_max(const std::vector<int>& unfinished, const std::vector<int>& undone, std::vector<Ent>& Es,
                         StageOut& chosen) {
    int v = -1;
    for (int u : unfinished) {
      const int in = c->node_input[u];
      if (in < 0 || !undone[in]) { v = u; break; }
    }
    if (v < 0) return SAMU_OK;
    std::vector<Cand> cands;
    for (auto& pl : plans[v]) {
      Ent P{v, pl.first, pl.second};
      cands.push_back({std::vector<Ent>{P}, P});
    }
    if (cands.empty()) return SAMU_OK;
    int32_t best = -1;
    double mx = 0.0;
    std::vector<StageOut> so;
    RET(score_batch(cands, 0.0, 0, 1, &best, &mx, so));
    Es = cands[best].E;
    chosen = so[best];
    return SAMU_OK;
  }

  // Min-heuristic: as many ready models as GPUs allow (lowest ids first; a model
  // whose input is selected in the same stage counts as ready), GPUs split as evenly as possible,
  // the combination of highest stage throughput among the splits and the plans using exactly the
  // assigned GPUs (<= 10^4 combinations in enumeration order; ties: first); one model fewer if
  // no combination exists
  samu_status choose_min(const std::vector<int>& unfinished, const std::vector<int>& undone, std::vector<Ent>& Es,
                         StageOut& chosen) {
    const std::vector<Ent> pin = pinned();   // no-preemption: running models keep their entries
    int N = (int)c->eng.n_gpus;
    for (const Ent& e : pin) N -= e.dp * e.tp;
    std::vector<int> sel;
    for (int v : unfinished) {
      if ((int)sel.size() >= N) break;
      if (is_pinned(pin, v)) continue;
      const int in = c->node_input[v];
      bool ok = in < 0 || !undone[in];
      for (int x : sel) if (x == in) ok = true;
      if (is_pinned(pin, in)) ok = true;
      if (ok) sel.push_back(v);
    }
    bool found = false;
    for (int k = (int)sel.size(); k >= 1 && !found; --k) {
      const int base = N / k, extra = N % k;
      std::vector<Cand> cands;
      std::vector<int> pick(extra);
      for (int i = 0; i < extra; ++i) pick[i] = i;
      bool more = true;
      while (more && cands.size() < 10000) {
        std::vector<int> gv(k, base);
        for (int i : pick) gv[i] += 1;
        std::vector<std::vector<int>> opts(k);
        bool feasible = true;
        for (int i = 0; i < k; ++i) {
          for (size_t pi = 0; pi < plans[sel[i]].size(); ++pi)
            if (plans[sel[i]][pi].first * plans[sel[i]][pi].second == gv[i]) opts[i].push_back((int)pi);
          if (opts[i].empty()) feasible = false;
        }
        if (feasible) {
          std::vector<int> idx(k, 0);
          for (;;) {
            if (cands.size() >= 10000) break;
            std::vector<Ent> E = pin;
            for (int i = 0; i < k; ++i) {
              const auto& pl = plans[sel[i]][opts[i][idx[i]]];
              E.push_back({sel[i], pl.first, pl.second});
            }
            std::sort(E.begin(), E.end(), [](const Ent& a, const Ent& b) { return a.node < b.node; });
            cands.push_back({E, E[0]});
            int q = k - 1;   // odometer, last model fastest
            while (q >= 0 && ++idx[q] == (int)opts[q].size()) { idx[q] = 0; --q; }
            if (q < 0) break;
          }
        }
        int i = extra - 1;
        while (i >= 0 && pick[i] == k - extra + i) --i;
        if (i < 0) more = false;
        else {
          ++pick[i];
          for (int j2 = i + 1; j2 < extra; ++j2) pick[j2] = pick[j2 - 1] + 1;
        }
      }
      if (cands.empty()) continue;
      int32_t best = -1;
      double mx = 0.0;
      std::vector<StageOut> so;
      RET(score_batch(cands, 0.0, 0, 1, &best, &mx, so));
      Es = cands[best].E;
      chosen = so[best];
      found = true;
    }
    if (!found && !pin.empty()) {   // nothing to add: the stage is the running models
      int32_t b = -1;
      double mx = 0.0;
      std::vector<StageOut> so;
      RET(score_batch({Cand{pin, pin[0]}}, 0.0, 0, 1, &b, &mx, so, false));
      Es = pin;
      chosen = so[0];
    }
    return SAMU_OK;
  }

  // take the context's planner buffers for this call (returned by the destructor)
  bool borrowed = false;
  void borrow() {
    PlanBufs& b = c->pb;
    lo = std::move(b.lo); li = std::move(b.li); st = std::move(b.st); g = std::move(b.g);
    fin_t = std::move(b.fin_t); over = std::move(b.over); cache = std::move(b.cache);
    local_rec = std::move(b.local_rec); d_sc = std::move(b.d_sc); d_out = std::move(b.d_out);
    d_best = std::move(b.d_best); d_any = std::move(b.d_any); fin_pool = std::move(b.fin_pool);
    cap_slots = T > 0 ? (int)(cache.n / (sizeof(samu_trial_rec) * (size_t)T)) : 0;
    borrowed = true;
  }
  ~Greedy() {
    if (!borrowed) return;
    PlanBufs& b = c->pb;
    for (auto& kv : fin_buf) fin_pool.push_back(std::move(kv.second));
    b.lo = std::move(lo); b.li = std::move(li); b.st = std::move(st); b.g = std::move(g);
    b.fin_t = std::move(fin_t); b.over = std::move(over); b.cache = std::move(cache);
    b.local_rec = std::move(local_rec); b.d_sc = std::move(d_sc); b.d_out = std::move(d_out);
    b.d_best = std::move(d_best); b.d_any = std::move(d_any); b.fin_pool = std::move(fin_pool);
  }

  samu_status setup(uint64_t seed, int T_total) {
    T = T_total;
    if (!borrowed) borrow();
    n = (size_t)c->n_req;
    shard_split(c, T, &Wt, &Wc);
    my_class = c->rank / Wt;
    trial_share(T, Wt, c->rank % Wt, &tb, &Tl);
    cudaStream_t s = c->stream;
    is_input.assign(c->n_nodes, false);
    touched.assign(c->n_nodes, false);
    for (int v = 0; v < c->n_nodes; ++v) if (c->node_input[v] >= 0) is_input[c->node_input[v]] = true;
    const size_t tn = (size_t)std::max(Tl, 1) * n;
    CK(c, lo.ensure(sizeof(uint16_t) * tn));
    CK(c, li.ensure(sizeof(uint16_t) * tn));
    CK(c, st.ensure(sizeof(uint32_t) * tn));
    CK(c, g.ensure(sizeof(uint16_t) * tn));
    CK(c, fin_t.ensure(sizeof(double) * tn));
    CK(c, over.ensure(sizeof(double) * (size_t)std::max(Tl, 1) * c->n_nodes * 16));
    CK(c, cudaMemsetAsync(st.p, 0, sizeof(uint32_t) * tn, s));
    CK(c, cudaMemsetAsync(g.p, 0, sizeof(uint16_t) * tn, s));
    CK(c, cudaMemsetAsync(over.p, 0, sizeof(double) * (size_t)std::max(Tl, 1) * c->n_nodes * 16, s));
    CK(c, samu_count(c, launch_fill_f64(fin_t.as<double>(), (int64_t)tn, std::numeric_limits<double>::infinity(), s)));
    if (Tl) RET(sample_or_known(c, seed, tb, Tl, known, lo.as<uint16_t>(), li.as<uint16_t>()));
    S = StatePtrs{st.as<uint32_t>(), g.as<uint16_t>(), fin_t.as<double>(), over.as<double>()};
    CK(c, d_best.ensure(sizeof(int32_t) + sizeof(double)));
    CK(c, d_any.ensure(sizeof(int32_t) * (size_t)c->n_nodes * std::max(Tl, 1) + 2 * sizeof(int32_t) * SAMU_MAX_NODES));
    plans.assign(c->n_nodes, {});
    for (int v = 0; v < c->n_nodes; ++v) plans[v] = plans_of(c, c->node_model[v]);
    return SAMU_OK;
  }

  // commit a stage (Alg. 1 lines 24-25): f* to completion, the others cut at t_E^(k), state
  // carried, finish times re-based; `chosen` is the stage's score (f*, mean t_E, T_E)
  samu_status commit_stage(const std::vector<Ent>& Es, const StageOut& chosen) {
    cudaStream_t s = c->stream;
    const int f = chosen.fstar;
    int fslot = -1;
    RET(ensure_full(Es[f], Es, &fslot));
    std::vector<SimJob> jobs;
    std::vector<int> src_slots;
    CK(c, local_rec.ensure(sizeof(samu_trial_rec) * Es.size() * std::max(Tl, 1)));
    for (size_t i = 0; i < Es.size(); ++i) {
      const Ent& e = Es[i];
      SimJob J;
      J.cand = samu_candidate{e.node, e.dp, e.tp, resumes(e) ? 1 : 0, -1, 1};
      J.phase = 0;
      const int src = c->node_input[e.node];
      for (size_t q = 0; q < Es.size(); ++q)
        if (Es[q].node == src) {
          int ss;
          RET(ensure_full(Es[q], Es, &ss));
          J.src_fin = fin_buf.at(ss).as<double>();
          J.phase = 1;
          src_slots.push_back(ss);
        }
      J.tau_rec = ((int)i == f) ? nullptr : rec(fslot) + tb;
      J.out_rec = local_rec.as<samu_trial_rec>() + i * Tl;
      jobs.push_back(J);
    }
    RET(flush());
    for (int ss : src_slots) RET(ensure_local_fin(ss));   // job classes: a source may have run elsewhere
    CK(c, local_rec.ensure(sizeof(samu_trial_rec) * Es.size() * std::max(Tl, 1)));
    for (size_t i = 0; i < jobs.size(); ++i) jobs[i].out_rec = local_rec.as<samu_trial_rec>() + i * Tl;
    // depth > 1 chains of dependencies commit in topological (node id) order
    for (size_t i = 0; i < jobs.size(); ++i) {
      int d = 0, v = Es[i].node;
      while (c->node_input[v] >= 0) { ++d; v = c->node_input[v]; }
      jobs[i].phase = d;
    }
    RET(agree(c, run_jobs(c, jobs, lo.as<uint16_t>(), li.as<uint16_t>(), Tl, S)));
    CK(c, samu_count(c, launch_rebase(st.as<uint32_t>(), fin_t.as<double>(), (int64_t)Tl * n, rec(fslot) + tb, (int32_t)n, s)));
    for (const Ent& e : Es) touched[e.node] = true;
    prev = Es;
    return SAMU_OK;
  }

  void new_stage_caches() {
    full_slot.clear();
    cut_slot.clear();
    slot_class.clear();
    slot_job.clear();
    slot_src.clear();
    have_fin.clear();
    for (auto& kv : fin_buf) fin_pool.push_back(std::move(kv.second));
    fin_buf.clear();
    n_slots = 0;
  }

  samu_status run(uint64_t seed, int T_total, int algo, samu_plan* plan) {
    double t_stage = now_s();
    g_trace_jobs_s = 0.0;
    g_trace_jobs_n = 0;
    RET(setup(seed, T_total));
    if (trace_on()) std::fprintf(stderr, "[samu trace] setup %.4f s\n", now_s() - t_stage);
    std::memset(plan, 0, sizeof(*plan));
    for (;;) {
      if (trace_on()) { t_stage = now_s(); g_trace_jobs_s = 0.0; g_trace_jobs_n = 0; }
      // unfinished nodes (in any trial of any rank)
      std::vector<int> undone(c->n_nodes, 0);
      RET(node_status(undone));
      std::vector<int> unfinished;
      for (int v = 0; v < c->n_nodes; ++v) if (undone[v]) unfinished.push_back(v);
      if (unfinished.empty()) break;
      undone_now = undone;
      if (plan->n_stages >= 64) FAIL(c, SAMU_E_STATE, "plan: too many stages");
      new_stage_caches();
      NvtxRange nv("samu planner stage");
      std::vector<Ent> Es;
      StageOut chosen{};
      if (algo == 0) RET(choose_greedy(unfinished, undone, Es, chosen));
      else if (algo == 1) RET(choose_max(unfinished, undone, Es, chosen));
      else RET(choose_min(unfinished, undone, Es, chosen));
      if (Es.empty()) FAIL(c, SAMU_E_INFEASIBLE, "plan: no ready model fits an empty stage");
      evals += 1;   // the stage is scored once more at commit (oracle parity of the counter)
      RET(commit_stage(Es, chosen));
      samu_plan_stage& PS = plan->stages[plan->n_stages++];
      PS.n_entries = (int)Es.size();
      for (size_t i = 0; i < Es.size(); ++i) { PS.node[i] = Es[i].node; PS.dp[i] = Es[i].dp; PS.tp[i] = Es[i].tp; }
      PS.fstar = Es[chosen.fstar].node;
      PS.mean_tE = chosen.mean_tE;
      PS.T_E = chosen.TE;
      plan->total += chosen.mean_tE;
      if (trace_on())
        std::fprintf(stderr, "[samu trace] stage %d: %.4f s wall, %.4f s in %lld simulate batches, %d entries\n",
                     plan->n_stages - 1, now_s() - t_stage, g_trace_jobs_s, (long long)g_trace_jobs_n, PS.n_entries);
    }
    plan->n_cand_evals = evals;
    return SAMU_OK;
  }

  samu_status node_status(std::vector<int>& undone) {
    cudaStream_t s = c->stream;
    int32_t* any = d_any.as<int32_t>();
    int32_t* red = any + (size_t)c->n_nodes * std::max(Tl, 1);
    std::vector<int32_t> h((size_t)c->n_nodes * std::max(Tl, 1), 0), flag(c->n_nodes, 0);
    if (Tl) {
      CK(c, samu_count(c, launch_node_done(st.as<uint32_t>(), Tl, (int32_t)n, c->d_node.as<int32_t>(), any, c->n_nodes, s)));
      CK(c, cudaMemcpyAsync(h.data(), any, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost, s));
      CK(c, cudaStreamSynchronize(s));
      for (int v = 0; v < c->n_nodes; ++v)
        for (int k = 0; k < Tl; ++k) flag[v] |= h[(size_t)v * Tl + k];
    }
    if (sharded(c)) {
      CK(c, cudaMemcpyAsync(red, flag.data(), sizeof(int32_t) * c->n_nodes, cudaMemcpyHostToDevice, s));
      RET(comm_allreduce_i32(c, red, red + SAMU_MAX_NODES, c->n_nodes, 0));
      CK(c, cudaMemcpyAsync(flag.data(), red + SAMU_MAX_NODES, sizeof(int32_t) * c->n_nodes, cudaMemcpyDeviceToHost, s));
      CK(c, cudaStreamSynchronize(s));
    }
    for (int v = 0; v < c->n_nodes; ++v) undone[v] = flag[v];
    return SAMU_OK;
  }
};

// Runtime replay with the dynamic scheduler (reading c33): the plan runs against true
// lengths (known, or another seed's draw, one trial); each actual stage = the running pairs, ended
// by the first actual finish (device-scored f*, cut commit); then the dynamic scheduler picks the
// next running set.  NVSwitch placement: continuing pairs keep their GPUs, new pairs take the
// lowest free ids, sparing the GPUs of pairs that may keep running.
struct Replay : Greedy {
  const samu_plan* plan = nullptr;
  std::vector<int> last_stage, undone;
  std::vector<Ent> R, Q;
  std::vector<uint32_t> mask;
  uint32_t used = 0, soft = 0;

  static bool has(const std::vector<Ent>& E, const Ent& e) {
    for (const Ent& x : E) if (x == e) return true;
    return false;
  }
  static bool has_node(const std::vector<Ent>& E, int v) {
    for (const Ent& x : E) if (x.node == v) return true;
    return false;
  }
  bool done(int v) const { return !undone[v]; }
  bool place(const Ent& e) {
    const int N = (int)c->eng.n_gpus, need = e.dp * e.tp;
    const uint32_t all = N >= 32 ? 0xFFFFFFFFu : ((1u << N) - 1u);
    const uint32_t freem = all & ~used;
    if (__builtin_popcount(freem) < need) return false;
    uint32_t m = 0;
    int k = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < N && k < need; ++i) {
        const bool sp = (soft >> i) & 1u;
        if (((freem >> i) & 1u) && (pass == 0 ? !sp : sp)) { m |= 1u << i; ++k; }
      }
    used |= m;
    R.push_back(e);
    mask.push_back(m);
    return true;
  }
  void place_from_Q() {
    std::vector<Ent> rest;
    for (const Ent& e : Q)
      if (!done(e.node) && !place(e)) rest.push_back(e);
    Q = rest;
  }
  std::vector<Ent> stage_entries(int k) const {
    std::vector<Ent> E;
    const samu_plan_stage& P = plan->stages[k];
    for (int i = 0; i < P.n_entries; ++i) E.push_back(Ent{P.node[i], P.dp[i], P.tp[i]});
    return E;
  }
  std::vector<Ent> drop_blocked() {
    std::vector<Ent> dropped;
    for (bool changed = true; changed;) {
      changed = false;
      for (size_t i = 0; i < R.size(); ++i) {
        const int src = c->node_input[R[i].node];
        if (src >= 0 && !done(src) && !has_node(R, src)) {
          dropped.push_back(R[i]);
          used &= ~mask[i];
          R.erase(R.begin() + i);
          mask.erase(mask.begin() + i);
          changed = true;
          break;
        }
      }
    }
    return dropped;
  }

  samu_status run_replay(uint64_t seed, samu_replay* out) {
    RET(setup(seed, 1));
    std::memset(out, 0, sizeof(*out));
    const int N = (int)c->eng.n_gpus;
    const int S_n = plan->n_stages;
    undone.assign(c->n_nodes, 0);
    RET(node_status(undone));
    last_stage.assign(c->n_nodes, -1);
    for (int k = 0; k < S_n; ++k)
      for (const Ent& e : stage_entries(k)) {
        if (e.node < 0 || e.node >= c->n_nodes) FAIL(c, SAMU_E_INVALID, "replay: plan node out of range");
        last_stage[e.node] = k;
      }
    for (int v = 0; v < c->n_nodes; ++v)
      if (last_stage[v] < 0 && !done(v)) FAIL(c, SAMU_E_INVALID, "replay: plan misses a model");
    int cur = 0;
    Q = stage_entries(0);
    place_from_Q();
    for (const Ent& e : drop_blocked()) Q.insert(Q.begin(), e);
    double clock = 0.0;
    for (;;) {
      bool any = false;
      for (int v = 0; v < c->n_nodes; ++v) if (!done(v)) any = true;
      if (!any) break;
      if (R.empty()) FAIL(c, SAMU_E_STATE, "replay: nothing can run");
      if (out->n_stages >= 64) FAIL(c, SAMU_E_STATE, "replay: too many stages");
      std::vector<size_t> ord(R.size());
      for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
      std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return R[a].node < R[b].node; });
      std::vector<Ent> Es;
      std::vector<uint32_t> Ms;
      for (size_t i : ord) { Es.push_back(R[i]); Ms.push_back(mask[i]); }
      samu_replay_stage& RS = out->stages[out->n_stages++];
      RS.n_entries = (int)Es.size();
      int g_used = 0;
      for (size_t i = 0; i < Es.size(); ++i) {
        RS.node[i] = Es[i].node; RS.dp[i] = Es[i].dp; RS.tp[i] = Es[i].tp;
        RS.gpu_mask[i] = Ms[i];
        RS.resumed[i] = resumes(Es[i]) ? 1 : 0;
        g_used += Es[i].dp * Es[i].tp;
      }
      RS.planned_stage = cur;
      // score the actual stage on the device (f* = first finisher), then commit it
      new_stage_caches();
      int32_t b = -1;
      double mx = 0.0;
      std::vector<StageOut> so;
      RET(score_batch({Cand{Es, Es[0]}}, 0.0, 0, 1, &b, &mx, so, false));
      const StageOut chosen = so[0];
      {
        int fslot = -1;
        RET(ensure_full(Es[chosen.fstar], Es, &fslot));
        samu_trial_rec r0;
        CK(c, cudaMemcpyAsync(&r0, rec(fslot), sizeof(r0), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        if (!(r0.flags & 1u)) FAIL(c, SAMU_E_STATE, "replay: first finisher is blocked");
      }
      RET(commit_stage(Es, chosen));
      RET(node_status(undone));
      RS.first_finisher = Es[chosen.fstar].node;
      RS.t_start = clock;
      RS.duration = chosen.mean_tE;
      RS.idle_gpus = N - g_used;
      clock += chosen.mean_tE;
      out->idle_gpu_seconds += (double)(N - g_used) * chosen.mean_tE;
      // dynamic scheduler transition
      std::vector<Ent> R_unf;
      std::vector<uint32_t> M_unf;
      for (size_t i = 0; i < R.size(); ++i)
        if (!done(R[i].node)) { R_unf.push_back(R[i]); M_unf.push_back(mask[i]); }
      R.clear(); mask.clear(); used = 0;
      auto keep = [&](size_t i) { R.push_back(R_unf[i]); mask.push_back(M_unf[i]); used |= M_unf[i]; };
      if (!Q.empty()) {
        for (size_t i = 0; i < R_unf.size(); ++i) keep(i);
        place_from_Q();
      } else {
        int nxt = cur + 1;
        while (nxt < S_n) {
          bool live = false;
          for (const Ent& e : stage_entries(nxt)) if (!done(e.node)) live = true;
          if (live) break;
          ++nxt;
        }
        if (nxt >= S_n) {
          for (size_t i = 0; i < R_unf.size(); ++i) keep(i);
        } else {
          const std::vector<Ent> En = stage_entries(nxt);
          std::vector<size_t> maybe, ordu(R_unf.size());
          for (size_t i = 0; i < ordu.size(); ++i) ordu[i] = i;
          std::sort(ordu.begin(), ordu.end(), [&](size_t a2, size_t b2) { return R_unf[a2].node < R_unf[b2].node; });
          for (size_t i : ordu) {
            const Ent& e = R_unf[i];
            if (last_stage[e.node] <= cur) { keep(i); out->n_kept_last++; }
            else if (has(En, e)) keep(i);
            else if (has_node(En, e.node)) { /* gives way to its E_nxt plan */ }
            else maybe.push_back(i);
          }
          Q.clear();
          for (const Ent& e : En) if (!done(e.node) && !has(R, e)) Q.push_back(e);
          soft = 0;
          for (size_t i : maybe) soft |= M_unf[i];
          place_from_Q();
          soft = 0;
          for (size_t i : maybe) {
            if (Q.empty() && !(used & M_unf[i])) { keep(i); out->n_kept_room++; }
            else out->n_stopped++;
          }
          cur = nxt;
        }
      }
      for (const Ent& e : drop_blocked()) {
        if (last_stage[e.node] >= cur && has(stage_entries(cur), e)) Q.insert(Q.begin(), e);
        else out->n_stopped++;
      }
    }
    out->total = clock;
    out->planned_total = plan->total;
    return SAMU_OK;
  }
};

}  // namespace

static samu_status plan_with(samu_ctx* c, uint64_t seed, int32_t n_trials, const samu_plan_opts* o, samu_plan** out) {
  GUARD(c);
  if (!out || n_trials < 1 || !o || o->algo < SAMU_ALGO_GREEDY || o->algo > SAMU_ALGO_MIN)
    FAIL(c, SAMU_E_INVALID, "plan: bad arguments");
  if (!c->app_loaded) FAIL(c, SAMU_E_INVALID, "plan: no app loaded");
  if (o->known_l_out && n_trials != 1) FAIL(c, SAMU_E_INVALID, "plan: known output lengths need n_trials == 1");
  *out = nullptr;
  samu_plan* p = new samu_plan();
  Greedy G;
  G.c = c;
  G.preempt = o->allow_preemption != 0;
  if (o->known_l_out) {
    samu_status rk = upload_known(c, o->known_l_out, &G.known);
    if (rk != SAMU_OK) { delete p; return rk; }
  }
  const int64_t sims0 = c->n_sims;
  samu_status rc = G.run(seed, n_trials, o->algo, p);
  if (rc != SAMU_OK) { delete p; return rc; }
  p->n_sims = c->n_sims - sims0;
  *out = p;
  return SAMU_OK;
}

extern "C" samu_status samu_plan_run(samu_ctx* c, uint64_t seed, int32_t n_trials, const samu_plan_opts* opts,
                                 samu_plan** out) {
  return plan_with(c, seed, n_trials, opts, out);
}

extern "C" samu_status samu_plan_greedy(samu_ctx* c, uint64_t seed, int32_t n_trials, samu_plan** out) {
  const samu_plan_opts o{SAMU_ALGO_GREEDY, 1, nullptr};
  return plan_with(c, seed, n_trials, &o, out);
}

extern "C" samu_status samu_plan_max_heuristic(samu_ctx* c, uint64_t seed, int32_t n_trials, samu_plan** out) {
  const samu_plan_opts o{SAMU_ALGO_MAX, 1, nullptr};
  return plan_with(c, seed, n_trials, &o, out);
}

extern "C" samu_status samu_plan_min_heuristic(samu_ctx* c, uint64_t seed, int32_t n_trials, samu_plan** out) {
  const samu_plan_opts o{SAMU_ALGO_MIN, 1, nullptr};
  return plan_with(c, seed, n_trials, &o, out);
}

extern "C" samu_status samu_replay_plan(samu_ctx* c, const samu_plan* plan, uint64_t seed, const uint32_t* known_l_out,
                                        samu_replay* out) {
  GUARD(c);
  if (!plan || !out || plan->n_stages < 1 || plan->n_stages > 64) FAIL(c, SAMU_E_INVALID, "replay: bad arguments");
  if (!c->app_loaded) FAIL(c, SAMU_E_INVALID, "replay: no app loaded");
  for (int k = 0; k < plan->n_stages; ++k)
    if (plan->stages[k].n_entries < 1 || plan->stages[k].n_entries > 16) FAIL(c, SAMU_E_INVALID, "replay: bad stage");
  Replay G;
  G.c = c;
  G.plan = plan;
  if (known_l_out) RET(upload_known(c, known_l_out, &G.known));
  return G.run_replay(seed, out);
}

extern "C" samu_status samu_fit_coeffs(samu_ctx* c, int32_t n_buckets, const int64_t* off, const double* x,
                                       const double* y, int32_t trim_permille, double* out_a, double* out_b,
                                       int32_t* out_n_used, int32_t* out_flags) {
  GUARD(c);
  if (n_buckets < 0 || (n_buckets && (!off || !x || !y || !out_a || !out_b || !out_n_used || !out_flags)) ||
      trim_permille < 0 || trim_permille > 500)
    FAIL(c, SAMU_E_INVALID, "fit_coeffs: bad arguments");
  if (!n_buckets) return SAMU_OK;
  int64_t n_total = 0;
  CK(c, cudaMemcpyAsync(&n_total, off + n_buckets, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (n_total < 0) FAIL(c, SAMU_E_INVALID, "fit_coeffs: bad offsets");
  CK(c, c->d_fit_gone.ensure(std::max<int64_t>(n_total, 1)));
  CK(c, samu_count(c, launch_fit(off, n_buckets, x, y, trim_permille, c->d_fit_gone.as<uint8_t>(), out_a, out_b,
                                 out_n_used, out_flags, c->stream)));
  std::vector<int32_t> flags(n_buckets);
  CK(c, cudaMemcpyAsync(flags.data(), out_flags, sizeof(int32_t) * n_buckets, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < n_buckets; ++k)
    if (flags[k] & 1) FAIL(c, SAMU_E_INVALID, "fit_coeffs: bucket " + std::to_string(k) + " has fewer than two distinct x");
  return SAMU_OK;
}

extern "C" void samu_plan_free(samu_plan* p) { delete p; }
