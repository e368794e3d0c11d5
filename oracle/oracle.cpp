// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C++17, fp64, -ffp-contract=off.
//
// What it computes (PAPER.md = P:<line>; readings = DESIGN.md §3 / SURVEY.md §8(c)):
//   sampler        P:465-469  l_out = min(X, y, l_max - l_in), X ~ F_out (eCDF of 10,000 lengths)
//   simulator      P:472-476  FCFS continuous batching, iteration by iteration
//   FLOPs          P:301-306  Eq. prefill / Eq. decode
//   latency        P:480-489  t = t_comp + t_prep + t_samp, each a[B]*x + b[B]
//   total          P:491-496  sum of per-iteration latencies + model loading time
//   stage metrics  P:401-422  t_E = min over models (preemption), T_E = FLOPs_E / t_E
//   greedy         P:542-595  Algorithm 1
// Everything is written as the plain definition: the sampler expands the eCDF into its sorted
// multiset and indexes it; the simulator walks every running request every iteration; the
// planner re-simulates every candidate.  No blocking, fusion or reordering.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <string>
#include <thread>
#include <atomic>
#include <tuple>
#include <vector>

typedef unsigned __int128 u128;

static thread_local std::string g_err;
static void set_err(const std::string& s) { g_err = s; }
extern "C" const char* or_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11; Random123).  Reading c1: the paper names no RNG
// (S:211 uses a hash); the north star fixes a counter-based Philox.
// ---------------------------------------------------------------------------------------------
extern "C" void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// ---------------------------------------------------------------------------------------------
// Problem (validated copy of the application)
// ---------------------------------------------------------------------------------------------
struct Model {
  uint32_t L, h, l_max, tp_mask;
  uint64_t c, weight_bytes, kv_bytes_per_token;
  std::vector<uint32_t> bucket_B;
  std::vector<double> coeff;   // [5][3][2][nb]
  std::vector<double> load;    // [5][16]
  std::vector<uint32_t> multiset;  // the eCDF's sorted multiset of n observed lengths
};

struct Req { uint32_t l_in_base, cap_y; int32_t pred, node, chain; };

struct or_problem {
  or_engine eng;
  std::vector<Model> models;
  std::vector<int> node_model;
  std::vector<Req> req;
  std::vector<int> node_begin, node_end;
  std::vector<std::vector<int>> succ_same;  // same-node successors of each request (index order)
  std::vector<int> node_input;              // the one other node this node's requests depend on, or -1
};

static int log2_exact(uint32_t x) {
  for (int k = 0; k < 32; ++k) if ((1u << k) == x) return k;
  return -1;
}

extern "C" or_problem* or_problem_create(const or_app* a) {
  if (!a) { set_err("null app"); return nullptr; }
  or_problem* p = new or_problem();
  p->eng = a->engine;
  const or_engine& e = p->eng;
  if (e.max_num_seqs < 1 || e.max_num_seqs > OR_MAX_SEQS || e.block_size < 1 || e.n_gpus < 1 ||
      e.n_gpus > 16 || e.mem_util_permille > 1000) {
    set_err("invalid engine config"); delete p; return nullptr;
  }
  for (int m = 0; m < a->n_models; ++m) {
    const or_model& s = a->models[m];
    Model M;
    M.L = s.L; M.h = s.h; M.c = s.c; M.l_max = s.l_max; M.tp_mask = s.tp_mask;
    M.weight_bytes = s.weight_bytes; M.kv_bytes_per_token = s.kv_bytes_per_token;
    if (s.L < 1 || s.h < 1 || s.c < 1 || s.l_max < 1 || s.l_max > 65535 || s.tp_mask == 0 ||
        (s.tp_mask >> OR_N_TP_SLOTS) != 0 || s.kv_bytes_per_token < 1 || s.n_buckets < 1 ||
        s.ecdf_k < 1) {
      set_err("invalid model spec " + std::to_string(m)); delete p; return nullptr;
    }
    for (int k = 0; k < s.n_buckets; ++k) {
      if (s.bucket_B[k] < 1 || (k > 0 && s.bucket_B[k] <= s.bucket_B[k - 1])) {
        set_err("buckets not strictly increasing"); delete p; return nullptr;
      }
      M.bucket_B.push_back(s.bucket_B[k]);
    }
    M.coeff.assign(s.coeff, s.coeff + (size_t)OR_N_TP_SLOTS * 3 * 2 * s.n_buckets);
    M.load.assign(s.load, s.load + (size_t)OR_N_TP_SLOTS * OR_MAX_DP);
    // eCDF: knots (value, cumulative count), strictly increasing; expand the multiset.
    uint32_t prev_v = 0, prev_c = 0;
    for (int k = 0; k < s.ecdf_k; ++k) {
      uint32_t v = s.ecdf_values[k], c = s.ecdf_cum[k];
      if ((k > 0 && v <= prev_v) || c <= prev_c) {
        set_err("eCDF knots not strictly increasing"); delete p; return nullptr;
      }
      for (uint32_t j = prev_c; j < c; ++j) M.multiset.push_back(v);
      prev_v = v; prev_c = c;
    }
    p->models.push_back(std::move(M));
  }
  for (int n = 0; n < a->n_nodes; ++n) {
    int m = a->node_model[n];
    if (m < 0 || m >= a->n_models) { set_err("node model out of range"); delete p; return nullptr; }
    p->node_model.push_back(m);
  }
  p->node_begin.assign(a->n_nodes, 0);
  p->node_end.assign(a->n_nodes, 0);
  p->node_input.assign(a->n_nodes, -1);
  std::vector<int> has_same(a->n_nodes, 0), has_cross(a->n_nodes, 0);
  p->succ_same.assign(a->n_req, {});
  int last_node = -1;
  for (int r = 0; r < a->n_req; ++r) {
    Req q{a->l_in_base[r], a->cap_y[r], a->pred[r], a->node[r], a->chain[r]};
    if (q.node < 0 || q.node >= a->n_nodes || q.node < last_node) {
      set_err("requests must be grouped by ascending node"); delete p; return nullptr;
    }
    if (q.node != last_node) { p->node_begin[q.node] = r; last_node = q.node; }
    p->node_end[q.node] = r + 1;
    const Model& M = p->models[p->node_model[q.node]];
    if (q.l_in_base > 65535 || q.chain < -1) { set_err("bad request field"); delete p; return nullptr; }
    if (q.pred >= r || q.pred < -1) { set_err("pred must precede its request"); delete p; return nullptr; }
    if (q.pred == -1) {
      if (q.l_in_base > M.l_max) {   // l_in > l_max cannot be served
        set_err("root request with l_in > l_max"); delete p; return nullptr;
      }
    } else {
      const Req& pr = p->req[q.pred];
      if (pr.node == q.node) {
        if (pr.chain != q.chain || q.chain < 0) { set_err("chain successor must share chain id"); delete p; return nullptr; }
        has_same[q.node] = 1;
        p->succ_same[q.pred].push_back(r);
      } else {
        if (p->node_input[q.node] != -1 && p->node_input[q.node] != pr.node) {
          set_err("a node may depend on one input node only"); delete p; return nullptr;
        }
        p->node_input[q.node] = pr.node;
        has_cross[q.node] = 1;
      }
    }
    p->req.push_back(q);
  }
  for (int n = 0; n < a->n_nodes; ++n)
    if (has_same[n] && has_cross[n]) { set_err("node mixes chain and cross-node predecessors"); delete p; return nullptr; }
  return p;
}

extern "C" void or_problem_destroy(or_problem* p) { delete p; }

// ---------------------------------------------------------------------------------------------
// Sampler.  Reading c2: X = the t-th (0-based) element of the eCDF's sorted
// multiset with t = floor(u * n / 2^32).  Reading c3: chain / evaluator inputs add the
// predecessor's generated tokens max(l_out, 1), truncated to l_max.
// ---------------------------------------------------------------------------------------------
extern "C" uint32_t or_ecdf_inverse(const or_problem* p, int32_t model, uint32_t u) {
  const std::vector<uint32_t>& ms = p->models[model].multiset;
  uint64_t n = ms.size();
  uint64_t t = ((uint64_t)u * n) >> 32;
  return ms[t];
}

extern "C" int32_t or_sample_lengths(const or_problem* p, uint64_t seed, int32_t trial_begin, int32_t n_trials,
                                     uint16_t* l_out, uint16_t* l_in_eff) {
  const int n = (int)p->req.size();
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int k = 0; k < n_trials; ++k) {
    uint16_t* lo = l_out + (size_t)k * n;
    uint16_t* li = l_in_eff + (size_t)k * n;
    for (int r = 0; r < n; ++r) {
      const Req& q = p->req[r];
      const Model& M = p->models[p->node_model[q.node]];
      uint32_t ctr[4] = {(uint32_t)r >> 2, (uint32_t)(trial_begin + k), (uint32_t)q.node, 0u};
      uint32_t w[4];
      or_philox4x32_10(ctr, key, w);
      uint32_t u = w[r & 3];
      uint32_t X = or_ecdf_inverse(p, p->node_model[q.node], u);
      uint32_t lin = q.l_in_base;
      if (q.pred >= 0) lin += std::max<uint32_t>(lo[q.pred], 1u);
      lin = std::min(lin, M.l_max);
      uint32_t out = std::min(std::min(X, q.cap_y), M.l_max - lin);
      lo[r] = (uint16_t)out;
      li[r] = (uint16_t)lin;
    }
  }
  return OR_OK;
}

// Known output lengths ("replace the output lengths generated by the output sampler
// in the cost model with the real output lengths"; reading c30): l_true[r] takes the place of the
// sampled X, with the same clamps (cap, l_max - l_in) and the same chained prompt arithmetic.
extern "C" int32_t or_known_lengths(const or_problem* p, const uint32_t* l_true, uint16_t* l_out, uint16_t* l_in_eff) {
  const int n = (int)p->req.size();
  for (int r = 0; r < n; ++r) {
    const Req& q = p->req[r];
    const Model& M = p->models[p->node_model[q.node]];
    uint32_t lin = q.l_in_base;
    if (q.pred >= 0) lin += std::max<uint32_t>(l_out[q.pred], 1u);
    lin = std::min(lin, M.l_max);
    uint32_t out = std::min(std::min(l_true[r], q.cap_y), M.l_max - lin);
    l_out[r] = (uint16_t)out;
    l_in_eff[r] = (uint16_t)lin;
  }
  return OR_OK;
}

// ---------------------------------------------------------------------------------------------
// Cost model pieces
// ---------------------------------------------------------------------------------------------
// Eq. prefill FLOPs: L (c B s + 2 B h s^2 / tp).  tp | h, so h/tp is exact (c12).
extern "C" uint64_t or_flops_prefill(uint32_t L, uint64_t c, uint32_t h, uint32_t tp, uint64_t B, uint64_t s) {
  u128 v = (u128)L * ((u128)c * B * s + (u128)2 * B * (h / tp) * s * s);
  return (uint64_t)v;
}
// Eq. decode FLOPs: L (c B + 2 h S / tp).
extern "C" uint64_t or_flops_decode(uint32_t L, uint64_t c, uint32_t h, uint32_t tp, uint64_t B, uint64_t S) {
  u128 v = (u128)L * ((u128)c * B + (u128)2 * (h / tp) * S);
  return (uint64_t)v;
}

// Eq. per-iter cost: t = t_comp + t_prep + t_samp, each a_phase[B] x_phase + b_phase[B],
// x = FLOPs, B*s, S.  Reading c24: each phase term is one correctly rounded fused multiply-add,
// summed left to right.
extern "C" double or_iter_latency(const double* a3, const double* b3, uint64_t flops, uint64_t Bs, uint64_t S) {
  double t_comp = std::fma(a3[0], (double)flops, b3[0]);
  double t_prep = std::fma(a3[1], (double)Bs, b3[1]);
  double t_samp = std::fma(a3[2], (double)S, b3[2]);
  return (t_comp + t_prep) + t_samp;
}

// Reading c11: coefficients of an unprofiled B are linearly interpolated between the nearest
// profiled buckets (clamped outside), v = v0 + (v1 - v0) * ((B - B0) / (B1 - B0)).
extern "C" int32_t or_dense_coeff(const or_problem* p, int32_t model, int32_t tp, double* a, double* b) {
  const Model& M = p->models[model];
  int slot = log2_exact((uint32_t)tp);
  if (slot < 0 || slot >= OR_N_TP_SLOTS || !((M.tp_mask >> slot) & 1)) return OR_E_INVALID;
  const int nb = (int)M.bucket_B.size();
  const int ms = (int)p->eng.max_num_seqs;
  for (int ph = 0; ph < 3; ++ph) {
    const double* ca = &M.coeff[(((size_t)slot * 3 + ph) * 2 + 0) * nb];
    const double* cb = &M.coeff[(((size_t)slot * 3 + ph) * 2 + 1) * nb];
    for (int B = 1; B <= ms; ++B) {
      double va, vb;
      if ((uint32_t)B <= M.bucket_B[0]) { va = ca[0]; vb = cb[0]; }
      else if ((uint32_t)B >= M.bucket_B[nb - 1]) { va = ca[nb - 1]; vb = cb[nb - 1]; }
      else {
        int k = 0;
        while (!((uint32_t)B >= M.bucket_B[k] && (uint32_t)B < M.bucket_B[k + 1])) ++k;
        double w = (double)(B - (int)M.bucket_B[k]) / (double)(M.bucket_B[k + 1] - M.bucket_B[k]);
        va = ca[k] + (ca[k + 1] - ca[k]) * w;
        vb = cb[k] + (cb[k + 1] - cb[k]) * w;
      }
      a[ph * ms + (B - 1)] = va;
      b[ph * ms + (B - 1)] = vb;
    }
  }
  return OR_OK;
}

// Plan validity and KV blocks per replica (reading c5):
//   util = floor(mem * permille / 1000); usable = util - ceil(weights / tp) (must be > 0);
//   kv = min(kv_cap, usable) per GPU; blocks = floor(tp * kv / (bs * kv_bytes_per_token)).
//   valid iff tp allowed, tp | h, 1 <= dp <= 16, dp*tp <= N, blocks >= ceil(l_max / bs).
extern "C" int64_t or_plan_blocks(const or_problem* p, int32_t model, int32_t dp, int32_t tp) {
  const Model& M = p->models[model];
  const or_engine& e = p->eng;
  int slot = log2_exact((uint32_t)tp);
  if (slot < 0 || slot >= OR_N_TP_SLOTS || !((M.tp_mask >> slot) & 1)) return -1;
  if (M.h % (uint32_t)tp != 0) return -1;
  if (dp < 1 || dp > OR_MAX_DP || (uint32_t)(dp * tp) > e.n_gpus) return -1;
  uint64_t util = e.mem_bytes_per_gpu * e.mem_util_permille / 1000;
  uint64_t wshard = (M.weight_bytes + (uint64_t)tp - 1) / (uint64_t)tp;
  if (util <= wshard) return -1;
  uint64_t usable = util - wshard;
  uint64_t kv = std::min<uint64_t>(e.kv_cap_bytes_per_gpu, usable);
  uint64_t blocks = ((uint64_t)tp * kv) / ((uint64_t)e.block_size * M.kv_bytes_per_token);
  uint64_t need = (M.l_max + e.block_size - 1) / e.block_size;
  if (blocks < need) return -1;
  if (blocks > (uint64_t)0x7fffffff) blocks = 0x7fffffff;
  return (int64_t)blocks;
}

// Valid plans in order of ascending GPU count, then ascending tp.
extern "C" int32_t or_enumerate_plans(const or_problem* p, int32_t model, int32_t* dp, int32_t* tp, int32_t cap) {
  int cnt = 0;
  for (int gpus = 1; gpus <= (int)p->eng.n_gpus; ++gpus)
    for (int t = 1; t <= gpus; t *= 2) {
      if (gpus % t) continue;
      int d = gpus / t;
      if (or_plan_blocks(p, model, d, t) < 0) continue;
      if (cnt < cap) { dp[cnt] = d; tp[cnt] = t; }
      ++cnt;
    }
  return cnt;
}

// ---------------------------------------------------------------------------------------------
// Simulator: one dp replica of one candidate in one trial (ORACLE-SIM in
// SURVEY.md §8(c) with readings c3-c9, c13, c15, c18, c19).
// ---------------------------------------------------------------------------------------------
static inline uint32_t st_status(uint32_t w) { return w >> 28; }
static inline uint32_t st_rank(uint32_t w) { return w & 0x0FFFFFFFu; }
static inline uint32_t st_make(uint32_t s, uint32_t r) { return (s << 28) | (r & 0x0FFFFFFFu); }
static inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

struct SimCtx {
  const or_problem* p;
  int node, model, dp, tp;
  bool resume;
  uint32_t bs, max_seqs, budget;
  int64_t blocks;
  std::vector<double> a, b;    // dense [3][max_seqs]
  // per-trial views
  const uint16_t* l_out;
  const uint16_t* l_in;
  uint32_t* st;      // may be null (fresh)
  uint16_t* g_st;
  double* fin_t;     // carried finish times (stage clock), may be null
  double* over;      // [16] for this node, may be null
  const double* src_fin;
  double tau;
  bool commit;
  uint32_t* out_fin_iter;
  double* out_fin_t;
  // optional per-iteration trace (or_trace_replica): descriptors and the running set after each
  std::vector<or_iter_desc>* trace = nullptr;
  std::vector<std::pair<uint32_t, uint32_t>>* trace_run = nullptr;
  std::vector<int64_t>* trace_off = nullptr;
};

struct RepOut { double t_end; u128 flops; uint64_t req_iters; uint32_t iters; bool done; bool cut; int err; };

enum Grp { PRE = 0, HEAD = 1, QUEUED = 2 };
struct WEnt { int r; int grp; };

static RepOut sim_replica(SimCtx& C, const std::vector<int>& reqs, double t0, int replica) {
  const or_problem* p = C.p;
  const Model& M = p->models[C.model];
  RepOut out{t0, 0, 0, 0, false, false, OR_OK};
  // generated tokens per request, indexed by position within the node
  const int nb0 = p->node_begin[C.node];
  std::vector<uint32_t> gv(p->node_end[C.node] - nb0, 0);
  auto G = [&](int r) -> uint32_t& { return gv[r - nb0]; };
  std::deque<WEnt> W;              // waiting queue: [PRE ...][HEAD ...][QUEUED ...]
  std::vector<int> R;              // running, admission order
  std::vector<std::pair<double, int>> pending;  // cross-node requests by (ready, index)
  int64_t F = C.blocks;
  auto lout_eff = [&](int r) -> uint32_t { return std::max<uint32_t>(C.l_out[r], 1u); };

  // ---- initial state from the carried WorkloadState (c18) ----
  std::vector<std::pair<uint32_t, int>> running0, pre0, queued0;
  std::vector<int> heads;
  for (int r : reqs) {
    uint32_t w = C.st ? C.st[r] : st_make(OR_ST_FRESH, 0);
    uint32_t s = st_status(w);
    G(r) = C.g_st ? C.g_st[r] : 0;
    if (s == OR_ST_DONE) continue;
    if (s == OR_ST_RUNNING) running0.push_back({st_rank(w), r});
    else if (s == OR_ST_PREEMPTED) pre0.push_back({st_rank(w), r});
    else if (s == OR_ST_QUEUED) queued0.push_back({st_rank(w), r});
    else if (s == OR_ST_FRESH) {
      const Req& q = p->req[r];
      if (q.pred < 0) heads.push_back(r);
      else if (p->req[q.pred].node == C.node) {
        // chain successor: waits for its predecessor's release in this simulation
        uint32_t ps = C.st ? st_status(C.st[q.pred]) : OR_ST_FRESH;
        if (ps == OR_ST_DONE) { out.err = OR_E_STATE; return out; }
      } else {
        double ready;
        uint32_t ps = C.st ? st_status(C.st[q.pred]) : OR_ST_FRESH;
        if (ps == OR_ST_DONE && C.fin_t) ready = C.fin_t[q.pred];
        else if (C.src_fin) ready = C.src_fin[q.pred];
        else ready = std::numeric_limits<double>::infinity();
        pending.push_back({ready, r});
      }
    } else { out.err = OR_E_STATE; return out; }
  }
  std::sort(running0.begin(), running0.end());
  std::sort(pre0.begin(), pre0.end());
  std::sort(queued0.begin(), queued0.end());
  std::sort(pending.begin(), pending.end());
  if (C.resume) {
    for (auto& x : running0) {
      R.push_back(x.second);
      F -= (int64_t)cdiv(C.l_in[x.second] + G(x.second) - 1, C.bs);   // KV holds l_in + g - 1 tokens
    }
    if (F < 0) { out.err = OR_E_STATE; return out; }
  } else {
    // re-planned / newly loaded: everything partially decoded is recomputed, running
    // requests first (as if preempted last-admitted first), then the earlier preempted ones.
    for (auto& x : running0) W.push_back({x.second, PRE});
  }
  for (auto& x : pre0) W.push_back({x.second, PRE});
  for (int r : heads) W.push_back({r, HEAD});
  for (auto& x : queued0) W.push_back({x.second, QUEUED});
  size_t pend_i = 0;

  double t = t0;
  uint32_t iter = 0;
  for (;;) {
    // (1) time limit: iterations whose start < tau have all run (c15)
    if (t >= C.tau) { out.cut = true; break; }
    // (0) pending cross-node requests that are ready join the back of W in (ready, index) order
    while (pend_i < pending.size() && pending[pend_i].first <= t) {
      W.push_back({pending[pend_i].second, QUEUED});
      ++pend_i;
    }
    // (2) idle
    if (R.empty() && W.empty()) {
      if (pend_i < pending.size() && pending[pend_i].first != std::numeric_limits<double>::infinity()) {
        t = pending[pend_i].first;
        continue;
      }
      break;
    }
    // (3) admission: strict FCFS prefix of W (c8)
    std::vector<int> A;
    uint64_t tok = 0;
    int64_t blk = 0;
    while (!W.empty()) {
      int w = W.front().r;
      uint64_t pl = (uint64_t)C.l_in[w] + G(w);
      int64_t nb = (int64_t)cdiv(pl, C.bs);
      if (R.size() + A.size() + 1 > C.max_seqs) break;
      if (tok + pl > C.budget) break;
      if (blk + nb > F) break;
      A.push_back(w);
      tok += pl;
      blk += nb;
      W.pop_front();
    }
    uint64_t it_flops, B, s, S;
    std::vector<int> finished;
    uint32_t n_victims = 0;
    if (!A.empty()) {
      // (4) prefill iteration: prompt (+ already generated tokens when recomputing) of every
      // admitted request; it emits one token each (c4)
      F -= blk;
      B = A.size();
      s = 0; S = 0;
      for (int w : A) { uint64_t pl = (uint64_t)C.l_in[w] + G(w); s = std::max(s, pl); S += pl; }
      it_flops = or_flops_prefill(M.L, M.c, M.h, (uint32_t)C.tp, B, s);
      for (int w : A) {
        uint64_t pl = (uint64_t)C.l_in[w] + G(w);
        G(w) += 1;
        if (G(w) >= lout_eff(w)) { finished.push_back(w); F += (int64_t)cdiv(pl, C.bs); }
        else R.push_back(w);
      }
    } else {
      if (R.empty()) { out.err = OR_E_INFEASIBLE; return out; }   // head cannot fit an empty engine
      // (5) decode iteration: every running request feeds its last token (c9: l = l_in + g)
      int64_t need = 0;
      for (int r : R) { uint64_t l = (uint64_t)C.l_in[r] + G(r); if ((l - 1) % C.bs == 0) ++need; }
      while (need > F) {   // recompute preemption of the last admitted request (c7)
        int v = R.back();
        uint64_t l = (uint64_t)C.l_in[v] + G(v);
        F += (int64_t)cdiv(l - 1, C.bs);
        if ((l - 1) % C.bs == 0) --need;
        R.pop_back();
        W.push_front({v, PRE});
        ++n_victims;
        if (R.empty()) { out.err = OR_E_INFEASIBLE; return out; }
      }
      F -= need;
      B = R.size(); s = 0; S = 0;
      for (int r : R) { uint64_t l = (uint64_t)C.l_in[r] + G(r); s = std::max(s, l); S += l; }
      it_flops = or_flops_decode(M.L, M.c, M.h, (uint32_t)C.tp, B, S);
      std::vector<int> keep;
      for (int r : R) {
        uint64_t l = (uint64_t)C.l_in[r] + G(r);
        G(r) += 1;
        if (G(r) >= lout_eff(r)) { finished.push_back(r); F += (int64_t)cdiv(l, C.bs); }
        else keep.push_back(r);
      }
      R.swap(keep);
    }
    // (6) cost
    const double* a3 = nullptr;
    double av[3], bv[3];
    for (int ph = 0; ph < 3; ++ph) { av[ph] = C.a[ph * C.max_seqs + (B - 1)]; bv[ph] = C.b[ph * C.max_seqs + (B - 1)]; }
    a3 = av;
    double lat = or_iter_latency(a3, bv, it_flops, B * s, S);
    const double t_start = t;
    t = t + lat;
    out.flops += it_flops;
    out.req_iters += B;
    std::sort(finished.begin(), finished.end());
    std::vector<int> released;
    for (int r : finished) {
      if (C.out_fin_iter) C.out_fin_iter[r] = iter;
      if (C.out_fin_t) C.out_fin_t[r] = t;
      if (C.commit) { C.st[r] = st_make(OR_ST_DONE, 0); C.fin_t[r] = t; }
      for (int sr : p->succ_same[r]) released.push_back(sr);
    }
    std::sort(released.begin(), released.end());
    for (int sr : released) W.push_back({sr, QUEUED});   // ready at t, (t, index) order (c19)
    if (C.trace) {
      or_iter_desc d;
      d.t_start = t_start; d.lat = lat; d.flops = it_flops; d.s = s; d.S = S; d.free_blocks = F;
      d.kind = A.empty() ? 1u : 0u; d.B = (uint32_t)B; d.n_preempted = n_victims;
      d.n_finished = (uint32_t)finished.size();
      C.trace->push_back(d);
      for (int r : R) C.trace_run->push_back({(uint32_t)r, G(r)});
      C.trace_off->push_back((int64_t)C.trace_run->size());
    }
    ++iter;
  }
  out.t_end = t;
  out.iters = iter;
  out.done = R.empty() && W.empty() && pend_i == pending.size();
  if (C.commit) {
    // write back the end state (Alg. 1 line 25, "Update model workloads in G")
    for (int r : reqs) if (st_status(C.st[r]) != OR_ST_DONE) C.g_st[r] = (uint16_t)G(r);
    for (size_t i = 0; i < R.size(); ++i) C.st[R[i]] = st_make(OR_ST_RUNNING, (uint32_t)i);
    uint32_t npre = 0, nq = 0;
    for (const WEnt& w : W) {
      if (w.grp == PRE) C.st[w.r] = st_make(OR_ST_PREEMPTED, npre++);
      else if (w.grp == QUEUED) C.st[w.r] = st_make(OR_ST_QUEUED, nq++);
      else C.st[w.r] = st_make(OR_ST_FRESH, 0);
    }
    // reading c18: a cut replica's clock overshoots tau by the in-flight iteration (or load)
    C.over[replica] = (out.done || !out.cut) ? 0.0 : (t - C.tau);
  }
  return out;
}

static int sim_candidate_trial(const or_problem* p, const or_cand& cand, SimCtx& C, or_rec* rec) {
  C.p = p;
  C.node = cand.node;
  C.model = p->node_model[cand.node];
  C.dp = cand.dp;
  C.tp = cand.tp;
  C.resume = cand.resume != 0;
  const Model& M = p->models[C.model];
  // requests of this node, statically round-robined to dp replicas by request index within the
  // node, chains by chain id (c13)
  std::vector<std::vector<int>> rep(cand.dp);
  bool all_done = true;
  for (int r = p->node_begin[cand.node]; r < p->node_end[cand.node]; ++r) {
    const Req& q = p->req[r];
    int key = q.chain >= 0 ? q.chain : (r - p->node_begin[cand.node]);
    rep[key % cand.dp].push_back(r);
    if (!C.st || st_status(C.st[r]) != OR_ST_DONE) all_done = false;
  }
  std::memset(rec, 0, sizeof(*rec));
  if (all_done) {   // finished model: T = 0, no load charged (c16)
    rec->t_end = 0.0;
    rec->flags = 1;
    if (C.commit) for (int j = 0; j < 16; ++j) C.over[j] = 0.0;
    return OR_OK;
  }
  u128 fl = 0;
  bool done = true, cut = false;
  double tmax = -std::numeric_limits<double>::infinity();
  for (int j = 0; j < cand.dp; ++j) {
    // stage clock start: loading time for a newly started / re-planned model, the
    // carried overshoot for a model that keeps its plan (c18)
    int slot = log2_exact((uint32_t)cand.tp);
    double t0 = C.resume ? (C.over ? C.over[j] : 0.0) : M.load[(size_t)slot * OR_MAX_DP + (cand.dp - 1)];
    RepOut o = sim_replica(C, rep[j], t0, j);
    if (o.err) return o.err;
    tmax = std::max(tmax, o.t_end);
    fl += o.flops;
    rec->req_iters += o.req_iters;
    rec->iters += o.iters;
    done = done && o.done;
    cut = cut || o.cut;
  }
  if (C.commit) for (int j = cand.dp; j < 16; ++j) C.over[j] = 0.0;
  rec->t_end = tmax;   // model result: max over dp replicas
  rec->flops_lo = (uint64_t)fl;
  rec->flops_hi = (uint64_t)(fl >> 64);
  rec->flags = (done ? 1u : 0u) | (cut ? 2u : 0u);
  return OR_OK;
}

static int prepare_ctx(const or_problem* p, const or_cand& cand, SimCtx& C) {
  int model = p->node_model[cand.node];
  int64_t blocks = or_plan_blocks(p, model, cand.dp, cand.tp);
  if (blocks < 0) return OR_E_INVALID;
  C.blocks = blocks;
  C.bs = p->eng.block_size;
  C.max_seqs = p->eng.max_num_seqs;
  C.budget = std::max(p->models[model].l_max, p->eng.min_batched_tokens);   // c6
  C.a.assign(3 * C.max_seqs, 0.0);
  C.b.assign(3 * C.max_seqs, 0.0);
  return or_dense_coeff(p, model, cand.tp, C.a.data(), C.b.data());
}

extern "C" int32_t or_simulate(const or_problem* p, const or_cand* cand, int32_t n_trials,
                               const uint16_t* l_out, const uint16_t* l_in_eff,
                               uint32_t* st, uint16_t* g, double* fin_t, double* overshoot,
                               const double* tau, const double* src_fin_t, int32_t commit,
                               or_rec* out_rec, uint32_t* out_fin_iter, double* out_fin_t) {
  if (cand->node < 0 || cand->node >= (int)p->node_model.size()) { set_err("bad node"); return OR_E_INVALID; }
  if (commit && (!st || !g || !fin_t || !overshoot)) { set_err("commit needs state"); return OR_E_INVALID; }
  SimCtx C;
  int rc = prepare_ctx(p, *cand, C);
  if (rc) { set_err("invalid plan for model"); return rc; }
  const size_t n = p->req.size();
  const size_t nn = p->node_model.size();
  for (int k = 0; k < n_trials; ++k) {
    C.l_out = l_out + k * n;
    C.l_in = l_in_eff + k * n;
    C.st = st ? st + k * n : nullptr;
    C.g_st = g ? g + k * n : nullptr;
    C.fin_t = fin_t ? fin_t + k * n : nullptr;
    C.over = overshoot ? overshoot + (k * nn + cand->node) * 16 : nullptr;
    C.src_fin = src_fin_t ? src_fin_t + k * n : nullptr;
    C.tau = tau ? tau[k] : std::numeric_limits<double>::infinity();
    C.commit = commit != 0;
    C.out_fin_iter = out_fin_iter ? out_fin_iter + k * n : nullptr;
    C.out_fin_t = out_fin_t ? out_fin_t + k * n : nullptr;
    rc = sim_candidate_trial(p, *cand, C, &out_rec[k]);
    if (rc) { set_err(rc == OR_E_INFEASIBLE ? "infeasible: capacity below one sequence" : "state error"); return rc; }
  }
  return OR_OK;
}

extern "C" int32_t or_simulate_many(const or_problem* p, int32_t n_cands, const or_cand* cands, int32_t n_trials,
                                    const uint16_t* l_out, const uint16_t* l_in_eff, int32_t n_threads,
                                    or_rec* out_rec) {
  std::atomic<int64_t> next(0);
  std::atomic<int> err(0);
  const int64_t total = (int64_t)n_cands * n_trials;
  const size_t n = p->req.size();
  auto work = [&]() {
    for (;;) {
      int64_t w = next.fetch_add(1);
      if (w >= total || err.load()) return;
      int c = (int)(w / n_trials), k = (int)(w % n_trials);
      SimCtx C;
      if (prepare_ctx(p, cands[c], C)) { err = OR_E_INVALID; return; }
      C.l_out = l_out + k * n; C.l_in = l_in_eff + k * n;
      C.st = nullptr; C.g_st = nullptr; C.fin_t = nullptr; C.over = nullptr; C.src_fin = nullptr;
      C.tau = std::numeric_limits<double>::infinity(); C.commit = false;
      C.out_fin_iter = nullptr; C.out_fin_t = nullptr;
      int rc = sim_candidate_trial(p, cands[c], C, &out_rec[(size_t)c * n_trials + k]);
      if (rc) { err = rc; return; }
    }
  };
  std::vector<std::thread> th;
  for (int i = 0; i < std::max(1, n_threads); ++i) th.emplace_back(work);
  for (auto& x : th) x.join();
  return err.load();
}

// Per-iteration trace of one fresh replica-sim: the same sim_replica, with the trace hook.
extern "C" int32_t or_trace_replica(const or_problem* p, const or_cand* cand, const uint16_t* l_out, const uint16_t* l_in,
                                    int32_t replica, int64_t cap_desc, or_iter_desc* out_desc, int64_t cap_run,
                                    uint32_t* run_req, uint32_t* run_g, int64_t* run_off, int64_t* n_desc, int64_t* n_run) {
  if (cand->node < 0 || cand->node >= (int)p->node_model.size() || replica < 0 || replica >= cand->dp) {
    set_err("trace: bad candidate or replica");
    return OR_E_INVALID;
  }
  SimCtx C;
  if (prepare_ctx(p, *cand, C)) { set_err("trace: invalid plan for model"); return OR_E_INVALID; }
  C.p = p; C.node = cand->node; C.model = p->node_model[cand->node]; C.dp = cand->dp; C.tp = cand->tp;
  C.resume = false;
  C.l_out = l_out; C.l_in = l_in;
  C.st = nullptr; C.g_st = nullptr; C.fin_t = nullptr; C.over = nullptr; C.src_fin = nullptr;
  C.tau = std::numeric_limits<double>::infinity(); C.commit = false;
  C.out_fin_iter = nullptr; C.out_fin_t = nullptr;
  std::vector<or_iter_desc> tr;
  std::vector<std::pair<uint32_t, uint32_t>> run;
  std::vector<int64_t> off{0};
  C.trace = &tr; C.trace_run = &run; C.trace_off = &off;
  // the replica's requests (c13), as in sim_candidate_trial
  std::vector<int> reqs;
  for (int r = p->node_begin[cand->node]; r < p->node_end[cand->node]; ++r) {
    const Req& q = p->req[r];
    const int key = q.chain >= 0 ? q.chain : (r - p->node_begin[cand->node]);
    if (key % cand->dp == replica) reqs.push_back(r);
  }
  const Model& M = p->models[C.model];
  const double t0 = M.load[(size_t)log2_exact((uint32_t)cand->tp) * OR_MAX_DP + (cand->dp - 1)];
  RepOut o = sim_replica(C, reqs, t0, replica);
  if (o.err) { set_err("trace: simulation error"); return o.err; }
  *n_desc = (int64_t)tr.size();
  *n_run = (int64_t)run.size();
  if ((int64_t)tr.size() > cap_desc || (int64_t)run.size() > cap_run || !out_desc || !run_req || !run_g || !run_off) {
    set_err("trace: capacity too small");   // (a size query passes null buffers)
    return OR_E_INVALID;
  }
  for (size_t i = 0; i < tr.size(); ++i) out_desc[i] = tr[i];
  for (size_t i = 0; i < run.size(); ++i) { run_req[i] = run[i].first; run_g[i] = run[i].second; }
  for (size_t i = 0; i < off.size(); ++i) run_off[i] = off[i];
  return OR_OK;
}

// Per-candidate trial summaries (north star: "a segmented reduction to per-candidate mean and
// percentile latency"; reading c17), written as the definitions: mean = left-to-right fp64 sum
// of the trial totals in trial order / T; the p-th percentile = the nearest-rank order statistic
// sorted[ceil(p T / 100) - 1]; mean FLOPs = dbl(exact u128 sum) / T; mean request-iterations
// = dbl(exact u64 sum) / T.
static double u128_dbl(u128 x) {   // c17: dbl(hi) * 2^64 + dbl(lo), each step RN
  return (double)(uint64_t)(x >> 64) * 18446744073709551616.0 + (double)(uint64_t)x;
}

extern "C" int32_t or_summarise(int32_t n_cands, int32_t n_trials, const or_rec* recs, or_summary* out) {
  if (n_cands < 0 || n_trials < 1 || !recs || !out) { set_err("summarise: bad arguments"); return OR_E_INVALID; }
  for (int c = 0; c < n_cands; ++c) {
    const or_rec* r = recs + (size_t)c * n_trials;
    double sum = 0.0;
    u128 fl = 0;
    uint64_t ri = 0;
    std::vector<double> v(n_trials);
    for (int k = 0; k < n_trials; ++k) {
      sum = sum + r[k].t_end;
      fl += ((u128)r[k].flops_hi << 64) | r[k].flops_lo;
      ri += r[k].req_iters;
      v[k] = r[k].t_end;
    }
    std::sort(v.begin(), v.end());
    auto rank = [&](int pct) {   // ceil(pct * T / 100) - 1, at least 0
      const int64_t q = ((int64_t)pct * n_trials + 99) / 100;
      return v[(size_t)std::max<int64_t>(q - 1, 0)];
    };
    out[c].mean_t = sum / (double)n_trials;
    out[c].p50_t = rank(50);
    out[c].p90_t = rank(90);
    out[c].p99_t = rank(99);
    out[c].mean_flops = u128_dbl(fl) / (double)n_trials;
    out[c].mean_req_iters = (double)ri / (double)n_trials;
  }
  return OR_OK;
}

// ---------------------------------------------------------------------------------------------
// Greedy search (Algorithm 1; text P:585-595) with stage metrics.
// Reading c16 for T trials (exactly the paper at T = 1):
//   T_i^(k)  end clock of entry i in trial k (incl. load), 0 if its model is done in trial k
//   f*       argmin_i mean_k T_i^(k) (tie: lower node id);  t_E^(k) = T_f*^(k)
//   FLOPs_E^(k) = sum_i FLOPs of entry i's iterations that start before t_E^(k)   (c15)
//   T_E      = dbl(sum_k FLOPs_E^(k)) / (sum_k t_E^(k))  (0 if the denominator is 0)
//   argmax dT/dN, ties: smaller dN, lower node id, smaller tp, smaller dp; break if no
//   candidate or max dT < 0; commit: f* runs to completion, the others are cut at
//   t_E^(k) with their state carried; resume iff the same (node, plan) was in the previous stage.
// ---------------------------------------------------------------------------------------------
struct Entry { int node, dp, tp; };
static bool operator==(const Entry& a, const Entry& b) { return a.node == b.node && a.dp == b.dp && a.tp == b.tp; }

static double u128_to_double(u128 x) {   // c17: dbl(hi) * 2^64 + dbl(lo)
  return (double)(uint64_t)(x >> 64) * 18446744073709551616.0 + (double)(uint64_t)x;
}

struct Greedy {
  const or_problem* p;
  int T;
  size_t n, nn;
  std::vector<uint16_t> l_out, l_in;
  std::vector<uint32_t> st;
  std::vector<uint16_t> g;
  std::vector<double> fin_t, over;
  std::vector<Entry> prev;   // previous committed stage
  int64_t evals = 0;
  bool preempt = true;              // false: the no-preemption ablation (reading c29)
  const uint32_t* known = nullptr;  // known output lengths (reading c30)

  bool done_in(int node, int k) const {
    for (int r = p->node_begin[node]; r < p->node_end[node]; ++r)
      if (st_status(st[k * n + r]) != OR_ST_DONE) return false;
    return true;
  }
  bool done_all(int node) const {
    for (int k = 0; k < T; ++k) if (!done_in(node, k)) return false;
    return true;
  }
  bool resumes(const Entry& e) const {
    for (const Entry& x : prev) if (x == e) return true;
    return false;
  }
  // full simulation of entry e in candidate stage E (its dependency source, if any, in E)
  struct Full { std::vector<or_rec> rec; std::vector<double> fin; };
  std::map<std::vector<int>, Full> full_cache;
  std::map<std::vector<int>, std::vector<or_rec>> cut_cache;

  std::vector<int> key_of(const Entry& e, const std::vector<Entry>& E) const {
    std::vector<int> k{e.node, e.dp, e.tp, resumes(e) ? 1 : 0};
    int src = p->node_input[e.node];
    if (src >= 0) for (const Entry& x : E) if (x.node == src) {
      std::vector<int> ks = key_of(x, E);
      k.insert(k.end(), ks.begin(), ks.end());
    }
    return k;
  }
  const double* src_fin_of(const Entry& e, const std::vector<Entry>& E) {
    int src = p->node_input[e.node];
    if (src >= 0) for (const Entry& x : E) if (x.node == src) return full(x, E).fin.data();
    return nullptr;
  }
  Full& full(const Entry& e, const std::vector<Entry>& E) {
    std::vector<int> key = key_of(e, E);
    auto it = full_cache.find(key);
    if (it != full_cache.end()) return it->second;
    const double* sf = src_fin_of(e, E);
    Full f;
    f.rec.resize(T);
    f.fin.assign((size_t)T * n, std::numeric_limits<double>::infinity());
    or_cand c{e.node, e.dp, e.tp, resumes(e) ? 1 : 0};
    std::vector<uint32_t> st2 = st;
    std::vector<uint16_t> g2 = g;
    std::vector<double> ft2 = fin_t, ov2 = over;
    int rc = or_simulate(p, &c, T, l_out.data(), l_in.data(), st2.data(), g2.data(), ft2.data(), ov2.data(),
                         nullptr, sf, 0, f.rec.data(), nullptr, f.fin.data());
    if (rc) throw rc;
    return full_cache.emplace(key, std::move(f)).first->second;
  }
  const std::vector<or_rec>& cut(const Entry& e, const Entry& fs, const std::vector<Entry>& E,
                                 const std::vector<double>& tau) {
    std::vector<int> key = key_of(e, E);
    std::vector<int> kf = key_of(fs, E);
    key.push_back(-1);
    key.insert(key.end(), kf.begin(), kf.end());
    auto it = cut_cache.find(key);
    if (it != cut_cache.end()) return it->second;
    const double* sf = src_fin_of(e, E);
    std::vector<or_rec> rec(T);
    or_cand c{e.node, e.dp, e.tp, resumes(e) ? 1 : 0};
    std::vector<uint32_t> st2 = st;
    std::vector<uint16_t> g2 = g;
    std::vector<double> ft2 = fin_t, ov2 = over;
    int rc = or_simulate(p, &c, T, l_out.data(), l_in.data(), st2.data(), g2.data(), ft2.data(), ov2.data(),
                         tau.data(), sf, 0, rec.data(), nullptr, nullptr);
    if (rc) throw rc;
    return cut_cache.emplace(key, std::move(rec)).first->second;
  }

  struct Score { double TE; int fstar; std::vector<double> tE; double mean_tE; };
  Score score(const std::vector<Entry>& E) {
    ++evals;
    Score sc{0.0, -1, std::vector<double>(T, 0.0), 0.0};
    if (E.empty()) return sc;
    // f* = argmin of mean T_i (tie: lower node id; E is kept sorted by node id)
    int best = -1;
    double best_mean = 0.0;
    for (size_t i = 0; i < E.size(); ++i) {
      const Full& f = full(E[i], E);
      double sum = 0.0;
      for (int k = 0; k < T; ++k) sum += f.rec[k].t_end;
      double mean = sum / (double)T;
      if (best < 0 || mean < best_mean) { best = (int)i; best_mean = mean; }
    }
    sc.fstar = best;
    const Full& ff = full(E[best], E);
    u128 fl = 0;
    double den = 0.0;
    for (int k = 0; k < T; ++k) {
      sc.tE[k] = ff.rec[k].t_end;
      den += sc.tE[k];
      fl += ((u128)ff.rec[k].flops_hi << 64) | ff.rec[k].flops_lo;
    }
    for (size_t i = 0; i < E.size(); ++i) {
      if ((int)i == best) continue;
      const std::vector<or_rec>& rc = cut(E[i], E[best], E, sc.tE);
      for (int k = 0; k < T; ++k) fl += ((u128)rc[k].flops_hi << 64) | rc[k].flops_lo;
    }
    double sum = 0.0;
    for (int k = 0; k < T; ++k) sum += sc.tE[k];
    sc.mean_tE = sum / (double)T;
    sc.TE = den == 0.0 ? 0.0 : u128_to_double(fl) / den;
    return sc;
  }

  static int gpus(const std::vector<Entry>& E) {
    int s = 0;
    for (const Entry& e : E) s += e.dp * e.tp;
    return s;
  }

  std::vector<std::vector<int>> plans_dp, plans_tp;

  void init(uint64_t seed) {
    l_out.assign((size_t)T * n, 0);
    l_in.assign((size_t)T * n, 0);
    if (known) or_known_lengths(p, known, l_out.data(), l_in.data());
    else or_sample_lengths(p, seed, 0, T, l_out.data(), l_in.data());
    st.assign((size_t)T * n, st_make(OR_ST_FRESH, 0));
    g.assign((size_t)T * n, 0);
    fin_t.assign((size_t)T * n, std::numeric_limits<double>::infinity());
    over.assign((size_t)T * nn * 16, 0.0);
    plans_dp.assign(nn, {});
    plans_tp.assign(nn, {});
    for (size_t v = 0; v < nn; ++v) {
      int cnt = or_enumerate_plans(p, p->node_model[v], nullptr, nullptr, 0);
      plans_dp[v].resize(cnt); plans_tp[v].resize(cnt);
      or_enumerate_plans(p, p->node_model[v], plans_dp[v].data(), plans_tp[v].data(), cnt);
    }
  }

  // commit a chosen stage (Alg. 1 lines 24-25): f* to completion, the others cut at t_E^(k)
  int commit_stage(const std::vector<Entry>& Es, Score& sc) {
    sc = score(Es);
    for (size_t i = 0; i < Es.size(); ++i) {   // topological order = ascending node id
      const Entry& e = Es[i];
      const double* sf = src_fin_of(e, Es);
      std::vector<or_rec> rec(T);
      or_cand c{e.node, e.dp, e.tp, resumes(e) ? 1 : 0};
      int rc = or_simulate(p, &c, T, l_out.data(), l_in.data(), st.data(), g.data(), fin_t.data(), over.data(),
                           (int)i == sc.fstar ? nullptr : sc.tE.data(), sf, 1, rec.data(), nullptr, nullptr);
      if (rc) return rc;
    }
    for (int k = 0; k < T; ++k)   // carried finish times re-based to the next stage's clock
      for (size_t r = 0; r < n; ++r)
        if (st_status(st[k * n + r]) == OR_ST_DONE) fin_t[k * n + r] = fin_t[k * n + r] - sc.tE[k];
    prev = Es;
    full_cache.clear();
    cut_cache.clear();
    return OR_OK;
  }
  int commit(const std::vector<Entry>& Es, or_plan* out) {
    Score sc;
    int rc = commit_stage(Es, sc);
    if (rc) return rc;
    or_stage& S = out->stages[out->n_stages++];
    S.n_entries = (int)Es.size();
    for (size_t i = 0; i < Es.size(); ++i) { S.node[i] = Es[i].node; S.dp[i] = Es[i].dp; S.tp[i] = Es[i].tp; }
    S.fstar = Es[sc.fstar].node;
    S.mean_tE = sc.mean_tE;
    S.T_E = sc.TE;
    out->total += sc.mean_tE;
    return OR_OK;
  }

  // No-preemption: "the execution plan of a model would not be changed once chosen and a
  // running model would not be stopped once started" -- every model of the previous stage that is
  // unfinished keeps its entry (reading c29)
  std::vector<Entry> pinned() const {
    std::vector<Entry> E;
    if (preempt) return E;
    for (const Entry& e : prev) if (!done_all(e.node)) E.push_back(e);
    return E;
  }
  bool is_pinned(const std::vector<Entry>& pin, int v) const {
    for (const Entry& e : pin) if (e.node == v) return true;
    return false;
  }

  // Algorithm 1 inner loop: the stage E* for the current workload
  int choose_greedy(const std::vector<int>& unfinished, std::vector<Entry>& Es) {
    const int N = (int)p->eng.n_gpus;
    const std::vector<Entry> pin = pinned();
    Score s_star{0.0, -1, std::vector<double>(T, 0.0), 0.0};
    if (!pin.empty()) { Es = pin; s_star = score(Es); }   // E* starts from the running models
    for (;;) {
      // ready models: unfinished, and their input node finished or selected in E* (Alg.1 l.5)
      std::vector<int> ready;
      for (int v : unfinished) {
        int u = p->node_input[v];
        bool ok = (u < 0) || done_all(u);
        for (const Entry& e : Es) if (e.node == u) ok = true;
        if (ok) ready.push_back(v);
      }
      struct Cand { std::vector<Entry> E; Entry P; };
      std::vector<Cand> cands;
      const int g_star = gpus(Es);
      for (int v : ready) {
        if (is_pinned(pin, v)) continue;
        for (size_t pi = 0; pi < plans_dp[v].size(); ++pi) {
          Entry P{v, plans_dp[v][pi], plans_tp[v][pi]};
          int prime = -1;
          for (size_t i = 0; i < Es.size(); ++i) if (Es[i].node == v) prime = (int)i;
          std::vector<Entry> E = Es;
          if (prime >= 0) {
            E[prime] = P;
            int gE = gpus(E);
            if (!(g_star < gE && gE <= N)) continue;   // Alg. 1 line 11
          } else {
            E.push_back(P);
            if (gpus(E) > N) continue;                  // Alg. 1 line 14
          }
          std::sort(E.begin(), E.end(), [](const Entry& a, const Entry& b) { return a.node < b.node; });
          cands.push_back({E, P});
        }
      }
      if (cands.empty()) break;
      double maxdT = -std::numeric_limits<double>::infinity();
      int bi = -1;
      double br = 0.0;
      int bN = 0;
      Score bs{};
      for (size_t ci = 0; ci < cands.size(); ++ci) {
        Score sc = score(cands[ci].E);
        double dT = sc.TE - s_star.TE;
        int dN = gpus(cands[ci].E) - g_star;
        double ratio = dT / (double)dN;
        maxdT = std::max(maxdT, dT);
        bool better = false;
        if (bi < 0) better = true;
        else if (ratio > br) better = true;
        else if (ratio == br) {
          const Entry& a = cands[ci].P;
          const Entry& b = cands[bi].P;
          better = std::make_tuple(dN, a.node, a.tp, a.dp) < std::make_tuple(bN, b.node, b.tp, b.dp);
        }
        if (better) { bi = (int)ci; br = ratio; bN = dN; bs = sc; }
      }
      if (maxdT < 0.0) break;                           // Alg. 1 line 19
      Es = cands[bi].E;
      s_star = bs;
    }
    return OR_OK;
  }

  // Max-heuristic: all GPUs to one model at a time — the lowest-id ready
  // model — with the plan of highest stage throughput (ties: enumeration order, i.e. fewer GPUs,
  // then smaller tp); the stage runs that model to completion
  int choose_max(const std::vector<int>& unfinished, std::vector<Entry>& Es) {
    int v = -1;
    for (int u : unfinished) {
      int in = p->node_input[u];
      if (in < 0 || done_all(in)) { v = u; break; }
    }
    if (v < 0) return OR_OK;
    double bT = 0.0;
    for (size_t pi = 0; pi < plans_dp[v].size(); ++pi) {
      std::vector<Entry> E{{v, plans_dp[v][pi], plans_tp[v][pi]}};
      Score sc = score(E);
      if (Es.empty() || sc.TE > bT) { Es = E; bT = sc.TE; }
    }
    return OR_OK;
  }

  // Min-heuristic: as many ready models as GPUs allow (lowest node ids first; a
  // model whose input is selected in the same stage counts as ready), GPUs split as evenly as
  // possible (floor(N/k) each, N mod k of them one more); among those splits and the plans that
  // use exactly the assigned GPUs, the combination of highest stage throughput (at most 10^4
  // combinations in enumeration order; ties: first); if no combination exists, one model fewer
  // No-preemption (reading c29): the running models keep their entries; the free GPUs are split
  // the same way among the other ready models.
  int choose_min(const std::vector<int>& unfinished, std::vector<Entry>& Es) {
    const std::vector<Entry> pin = pinned();
    const int N = (int)p->eng.n_gpus - gpus(pin);
    std::vector<int> sel;
    for (int v : unfinished) {
      if ((int)sel.size() >= N) break;
      if (is_pinned(pin, v)) continue;
      int in = p->node_input[v];
      bool ok = in < 0 || done_all(in);
      for (int x : sel) if (x == in) ok = true;
      for (const Entry& e : pin) if (e.node == in) ok = true;
      if (ok) sel.push_back(v);
    }
    Es.clear();
    bool found = false;
    for (int k = (int)sel.size(); k >= 1 && !found; --k) {
      const int base = N / k, extra = N % k;
      double bT = 0.0;
      long count = 0;
      std::vector<int> pick(extra);
      for (int i = 0; i < extra; ++i) pick[i] = i;
      bool more_subsets = true;
      while (more_subsets && count < 10000) {
        std::vector<int> gv(k, base);
        for (int i : pick) gv[i] += 1;
        // plans of exactly gv[i] GPUs per selected model
        std::vector<std::vector<int>> opts(k);
        bool feasible = true;
        for (int i = 0; i < k; ++i) {
          int v = sel[i];
          for (size_t pi = 0; pi < plans_dp[v].size(); ++pi)
            if (plans_dp[v][pi] * plans_tp[v][pi] == gv[i]) opts[i].push_back((int)pi);
          if (opts[i].empty()) feasible = false;
        }
        if (feasible) {
          std::vector<int> idx(k, 0);
          for (;;) {
            if (count >= 10000) break;
            ++count;
            std::vector<Entry> E = pin;
            for (int i = 0; i < k; ++i) {
              int v = sel[i], pi = opts[i][idx[i]];
              E.push_back({v, plans_dp[v][pi], plans_tp[v][pi]});
            }
            std::sort(E.begin(), E.end(), [](const Entry& a, const Entry& b) { return a.node < b.node; });
            Score sc = score(E);
            if (!found || sc.TE > bT) { Es = E; bT = sc.TE; found = true; }
            int q = k - 1;   // odometer, last model fastest
            while (q >= 0 && ++idx[q] == (int)opts[q].size()) { idx[q] = 0; --q; }
            if (q < 0) break;
          }
        }
        // next subset of `extra` positions in lexicographic order
        int i = extra - 1;
        while (i >= 0 && pick[i] == k - extra + i) --i;
        if (i < 0) more_subsets = false;
        else {
          ++pick[i];
          for (int j2 = i + 1; j2 < extra; ++j2) pick[j2] = pick[j2 - 1] + 1;
        }
      }
    }
    if (!found) Es = pin;
    return OR_OK;
  }

  int run(uint64_t seed, int algo, or_plan* out) {
    init(seed);
    std::memset(out, 0, sizeof(*out));
    for (;;) {
      std::vector<int> unfinished;
      for (size_t v = 0; v < nn; ++v) if (!done_all((int)v)) unfinished.push_back((int)v);
      if (unfinished.empty()) break;
      if (out->n_stages >= 64) { set_err("too many stages"); return OR_E_STATE; }
      full_cache.clear();
      cut_cache.clear();
      std::vector<Entry> Es;
      int rc = algo == 0 ? choose_greedy(unfinished, Es) : (algo == 1 ? choose_max(unfinished, Es) : choose_min(unfinished, Es));
      if (rc) return rc;
      if (Es.empty()) { set_err("no ready model fits an empty stage"); return OR_E_INFEASIBLE; }
      rc = commit(Es, out);
      if (rc) return rc;
    }
    out->n_cand_evals = evals;
    return OR_OK;
  }
};

static int32_t plan_with(const or_problem* p, uint64_t seed, int32_t n_trials, int algo, or_plan* out,
                         int preempt = 1, const uint32_t* known = nullptr) {
  if (known && n_trials != 1) { set_err("known lengths: one trial"); return OR_E_INVALID; }
  Greedy G;
  G.p = p;
  G.T = n_trials;
  G.preempt = preempt != 0;
  G.known = known;
  G.n = p->req.size();
  G.nn = p->node_model.size();
  try {
    return G.run(seed, algo, out);
  } catch (int rc) {
    set_err("simulation error in planner");
    return rc;
  }
}

extern "C" int32_t or_plan_max_heuristic(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out) {
  return plan_with(p, seed, n_trials, 1, out);
}

extern "C" int32_t or_plan_min_heuristic(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out) {
  return plan_with(p, seed, n_trials, 2, out);
}

extern "C" int32_t or_plan_greedy(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out) {
  return plan_with(p, seed, n_trials, 0, out);
}

extern "C" int32_t or_plan_run(const or_problem* p, uint64_t seed, int32_t n_trials, int32_t algo, int32_t allow_preemption,
                           const uint32_t* known_l_out, or_plan* out) {
  if (algo < 0 || algo > 2) { set_err("bad algo"); return OR_E_INVALID; }
  return plan_with(p, seed, n_trials, algo, out, allow_preemption, known_l_out);
}

// ---------------------------------------------------------------------------------------------
// Runtime replay with the dynamic scheduler (reading c33).  The plan is executed
// against "true" lengths (known, or a differently seeded draw): the actual stage is the set of
// running (model, plan) pairs; it lasts until the first model actually finishes (same f* / cut
// commit as the planner, one trial).  At that event stage `cur` ends and the next planned stage
// nxt is scheduled:
//   - an unfinished running (M, P) keeps running if E_cur is the last stage M is planned in, or
//     if (M, P) is in E_nxt;
//   - if M is in E_nxt with another plan, (M, P) gives way (M reloads with its E_nxt plan);
//   - E_nxt's pairs are placed first (first fit in entry order); the other running pairs then
//     keep running, in node order, only if every E_nxt pair was placed and GPUs remain;
//     otherwise they are stopped (state carried, reloaded when next scheduled);
//   - E_nxt's pairs that do not fit wait (no stage after nxt is considered until they are placed
//     or their models finish), and are placed at later finish events as GPUs free up;
//   - a pair whose input model is unfinished and not running is not started (it waits / stops).
// Placement on NVSwitch is trivial: a continuing pair keeps its GPUs, a new pair takes the
// lowest free GPU ids; reload costs follow reading c18 (resume iff the same pair ran in the
// previous actual stage).
// ---------------------------------------------------------------------------------------------
struct Replay : Greedy {
  const or_plan* plan = nullptr;
  std::vector<int> last_stage;      // last planned stage index containing each node
  std::vector<Entry> R, Q;
  std::vector<uint32_t> mask;       // GPU mask of each pair in R
  uint32_t used = 0;
  uint32_t soft = 0;                // GPUs of running pairs that may keep running: taken last

  static bool has(const std::vector<Entry>& E, const Entry& e) {
    for (const Entry& x : E) if (x == e) return true;
    return false;
  }
  static bool has_node(const std::vector<Entry>& E, int v) {
    for (const Entry& x : E) if (x.node == v) return true;
    return false;
  }
  bool place(const Entry& e) {      // lowest free GPU ids, sparing `soft` ones while possible
    const int N = (int)p->eng.n_gpus, need = e.dp * e.tp;
    int freeg = 0;
    for (int i = 0; i < N; ++i) if (!(used >> i & 1u)) ++freeg;
    if (freeg < need) return false;
    uint32_t m = 0;
    int k = 0;
    for (int i = 0; i < N && k < need; ++i)
      if (!(used >> i & 1u) && !(soft >> i & 1u)) { m |= 1u << i; ++k; }
    for (int i = 0; i < N && k < need; ++i)
      if (!(used >> i & 1u) && (soft >> i & 1u)) { m |= 1u << i; ++k; }
    used |= m;
    R.push_back(e);
    mask.push_back(m);
    return true;
  }
  void place_from_Q() {
    std::vector<Entry> rest;
    for (const Entry& e : Q) if (done_all(e.node) || !place(e)) { if (!done_all(e.node)) rest.push_back(e); }
    Q = rest;
  }
  std::vector<Entry> stage_entries(int k) const {
    std::vector<Entry> E;
    const or_stage& S = plan->stages[k];
    for (int i = 0; i < S.n_entries; ++i) E.push_back({S.node[i], S.dp[i], S.tp[i]});
    return E;
  }
  // drop pairs whose input model is unfinished and not running (fixpoint); returns dropped ones
  std::vector<Entry> drop_blocked() {
    std::vector<Entry> dropped;
    for (bool changed = true; changed;) {
      changed = false;
      for (size_t i = 0; i < R.size(); ++i) {
        const int src = p->node_input[R[i].node];
        if (src >= 0 && !done_all(src) && !has_node(R, src)) {
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

  int run_replay(uint64_t seed, or_replay* out) {
    init(seed);
    std::memset(out, 0, sizeof(*out));
    const int N = (int)p->eng.n_gpus;
    const int S_n = plan->n_stages;
    if (S_n < 1) { set_err("replay: empty plan"); return OR_E_INVALID; }
    last_stage.assign(nn, -1);
    for (int k = 0; k < S_n; ++k)
      for (const Entry& e : stage_entries(k)) last_stage[e.node] = k;
    for (size_t v = 0; v < nn; ++v)
      if (last_stage[v] < 0 && !done_all((int)v)) { set_err("replay: plan misses a model"); return OR_E_INVALID; }
    int cur = 0;
    Q = stage_entries(0);
    place_from_Q();
    for (const Entry& e : drop_blocked()) Q.insert(Q.begin(), e);
    double clock = 0.0;
    for (;;) {
      bool any = false;
      for (size_t v = 0; v < nn; ++v) if (!done_all((int)v)) any = true;
      if (!any) break;
      if (R.empty()) { set_err("replay: nothing can run"); return OR_E_STATE; }
      if (out->n_stages >= 64) { set_err("replay: too many stages"); return OR_E_STATE; }
      // the actual stage: running pairs in node order
      std::vector<size_t> ord(R.size());
      for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
      std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return R[a].node < R[b].node; });
      std::vector<Entry> Es;
      std::vector<uint32_t> Ms;
      for (size_t i : ord) { Es.push_back(R[i]); Ms.push_back(mask[i]); }
      or_replay_stage& RS = out->stages[out->n_stages++];
      RS.n_entries = (int)Es.size();
      int g_used = 0;
      for (size_t i = 0; i < Es.size(); ++i) {
        RS.node[i] = Es[i].node; RS.dp[i] = Es[i].dp; RS.tp[i] = Es[i].tp;
        RS.gpu_mask[i] = Ms[i];
        RS.resumed[i] = resumes(Es[i]) ? 1 : 0;
        g_used += Es[i].dp * Es[i].tp;
      }
      RS.planned_stage = cur;
      Score sc;
      {
        // the first actual finisher must really finish (all its requests done)
        Score probe = score(Es);
        const Full& ff = full(Es[probe.fstar], Es);
        if (!(ff.rec[0].flags & 1u)) { set_err("replay: first finisher is blocked"); return OR_E_STATE; }
      }
      int rc = commit_stage(Es, sc);
      if (rc) return rc;
      RS.first_finisher = Es[sc.fstar].node;
      RS.t_start = clock;
      RS.duration = sc.tE[0];
      RS.idle_gpus = N - g_used;
      clock += sc.tE[0];
      out->idle_gpu_seconds += (double)(N - g_used) * sc.tE[0];
      // transition (dynamic scheduler)
      std::vector<Entry> R_unf;
      std::vector<uint32_t> M_unf;
      for (size_t i = 0; i < R.size(); ++i)
        if (!done_all(R[i].node)) { R_unf.push_back(R[i]); M_unf.push_back(mask[i]); }
      R.clear(); mask.clear(); used = 0;
      auto keep = [&](size_t i) { R.push_back(R_unf[i]); mask.push_back(M_unf[i]); used |= M_unf[i]; };
      if (!Q.empty()) {          // stage cur is still being scheduled
        for (size_t i = 0; i < R_unf.size(); ++i) keep(i);
        place_from_Q();
      } else {
        int nxt = cur + 1;
        while (nxt < S_n) {
          bool live = false;
          for (const Entry& e : stage_entries(nxt)) if (!done_all(e.node)) live = true;
          if (live) break;
          ++nxt;
        }
        if (nxt >= S_n) {
          for (size_t i = 0; i < R_unf.size(); ++i) keep(i);
        } else {
          const std::vector<Entry> En = stage_entries(nxt);
          std::vector<size_t> maybe;
          std::vector<size_t> ordu(R_unf.size());
          for (size_t i = 0; i < ordu.size(); ++i) ordu[i] = i;
          std::sort(ordu.begin(), ordu.end(), [&](size_t a, size_t b) { return R_unf[a].node < R_unf[b].node; });
          for (size_t i : ordu) {
            const Entry& e = R_unf[i];
            if (last_stage[e.node] <= cur) { keep(i); out->n_kept_last++; }
            else if (has(En, e)) keep(i);
            else if (has_node(En, e.node)) { /* gives way to its E_nxt plan */ }
            else maybe.push_back(i);
          }
          Q.clear();
          for (const Entry& e : En) if (!done_all(e.node) && !has(R, e)) Q.push_back(e);
          soft = 0;
          for (size_t i : maybe) soft |= M_unf[i];
          place_from_Q();
          soft = 0;
          for (size_t i : maybe) {
            // keeps running (on its own GPUs: moving would be a reload) only if the whole of
            // E_nxt is placed and its GPUs are still free
            if (Q.empty() && !(used & M_unf[i])) { keep(i); out->n_kept_room++; }
            else out->n_stopped++;
          }
          cur = nxt;
        }
      }
      for (const Entry& e : drop_blocked()) {
        if (last_stage[e.node] >= cur && has(stage_entries(cur), e)) Q.insert(Q.begin(), e);
        else out->n_stopped++;
      }
    }
    out->total = clock;
    out->planned_total = plan->total;
    return OR_OK;
  }
};

extern "C" int32_t or_replay_plan(const or_problem* p, const or_plan* plan, uint64_t seed, const uint32_t* known_l_out,
                                  or_replay* out) {
  if (!plan || !out) { set_err("replay: bad arguments"); return OR_E_INVALID; }
  Replay G;
  G.p = p;
  G.T = 1;
  G.known = known_l_out;
  G.n = p->req.size();
  G.nn = p->node_model.size();
  G.plan = plan;
  try {
    return G.run_replay(seed, out);
  } catch (int rc) {
    set_err("simulation error in replay");
    return rc;
  }
}

// ---------------------------------------------------------------------------------------------
// Per-iteration cost-model coefficients ("We profile the per-iteration computation
// with different inference workloads to compute the constants"; reading c34).  For each bucket
// (model, tp, phase, B) the least-squares line latency = a x + b over its samples (x = FLOPs,
// B s or S): means, then centred sums Sxx = sum (x - mx)^2, Sxy = sum (x - mx)(y - my), a =
// Sxy / Sxx, b = my - a mx; a < 0 is clamped to 0 with b = my.  Noise points (P: Fig. 5, "we
// can ignore them"): after a first fit the floor(n * trim_permille / 1000) samples of largest
// |residual| (ties: lower sample index first) are dropped and the line is refitted.  A bucket
// with fewer than two distinct x (before or after trimming) is an error.
// ---------------------------------------------------------------------------------------------
static int fit_line(const std::vector<double>& X, const std::vector<double>& Y, double* a, double* b, int* clamped) {
  const size_t n = X.size();
  if (n < 2) return 1;
  double xmin = X[0], xmax = X[0];
  for (double v : X) { xmin = std::min(xmin, v); xmax = std::max(xmax, v); }
  if (!(xmin < xmax)) return 1;
  double sx = 0.0, sy = 0.0;
  for (size_t i = 0; i < n; ++i) { sx += X[i]; sy += Y[i]; }
  const double mx = sx / (double)n, my = sy / (double)n;
  double sxx = 0.0, sxy = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double dx = X[i] - mx, dy = Y[i] - my;
    sxx += dx * dx;
    sxy += dx * dy;
  }
  double A = sxy / sxx;
  double B = my - A * mx;
  *clamped = 0;
  if (A < 0.0) { A = 0.0; B = my; *clamped = 1; }
  *a = A;
  *b = B;
  return 0;
}

extern "C" int32_t or_fit_coeffs(int32_t n_buckets, const int64_t* off, const double* x, const double* y,
                                 int32_t trim_permille, double* out_a, double* out_b, int32_t* out_n_used,
                                 int32_t* out_flags) {
  if (n_buckets < 0 || !off || trim_permille < 0 || trim_permille > 500) { set_err("fit: bad arguments"); return OR_E_INVALID; }
  int bad = -1;
  for (int k = 0; k < n_buckets; ++k) {
    std::vector<double> X(x + off[k], x + off[k + 1]), Y(y + off[k], y + off[k + 1]);
    double a = 0.0, b = 0.0;
    int cl = 0;
    int32_t flags = 0;
    if (fit_line(X, Y, &a, &b, &cl)) flags |= 1;
    else {
      const size_t n = X.size();
      const size_t drop = (size_t)((int64_t)n * trim_permille / 1000);
      if (drop > 0) {
        std::vector<std::pair<double, size_t>> r(n);
        for (size_t i = 0; i < n; ++i) r[i] = {std::fabs(Y[i] - (a * X[i] + b)), i};
        std::sort(r.begin(), r.end(), [](const std::pair<double, size_t>& p, const std::pair<double, size_t>& q) {
          if (p.first != q.first) return p.first > q.first;
          return p.second < q.second;
        });
        std::vector<char> gone(n, 0);
        for (size_t i = 0; i < drop; ++i) gone[r[i].second] = 1;
        std::vector<double> X2, Y2;
        for (size_t i = 0; i < n; ++i) if (!gone[i]) { X2.push_back(X[i]); Y2.push_back(Y[i]); }
        if (fit_line(X2, Y2, &a, &b, &cl)) flags |= 1;
        out_n_used[k] = (int32_t)X2.size();
      } else {
        out_n_used[k] = (int32_t)n;
      }
    }
    if (flags & 1) { a = 0.0; b = 0.0; out_n_used[k] = 0; if (bad < 0) bad = k; }
    if (cl && !(flags & 1)) flags |= 2;
    out_a[k] = a;
    out_b[k] = b;
    out_flags[k] = flags;
  }
  if (bad >= 0) { set_err("fit: bucket " + std::to_string(bad) + " has fewer than two distinct x"); return OR_E_INVALID; }
  return OR_OK;
}
