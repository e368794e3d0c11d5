// K3 / K4: per-(candidate, trial) combine over dp replicas, per-candidate trial summaries
// (mean, nearest-rank percentiles; reading c17), stage scoring for Algorithm 1 (f*, T_E,
// dT/dN argmax, reading c16), finish-time re-basing and done flags.
// Every reduction over trials runs in trial order on one thread, so results are independent of
// how trials were sharded across GPUs.
#include "samu_internal.cuh"

#include <algorithm>
#include <cstdlib>

#include <math_constants.h>

namespace {

__device__ __forceinline__ double u128_to_double(uint64_t hi, uint64_t lo) {   // c17
  return __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

__device__ __forceinline__ void add128(uint64_t& hi, uint64_t& lo, uint64_t bhi, uint64_t blo) {
  const uint64_t l = lo + blo;
  hi += bhi + (l < lo ? 1ull : 0ull);
  lo = l;
}

// model result per trial: max over replicas of the end clock, sums of the rest;
// a model whose requests were all done before the call has T = 0 and no load (c28)
__global__ void k_combine(const samu_trial_rec* __restrict__ rep, const DevCand* __restrict__ cands, int32_t n_cands,
                          int32_t T, double* over, int32_t n_nodes) {
  const int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n_cands * T) return;
  const int32_t c = x / T, k = x % T;
  const DevCand& C = cands[c];
  const samu_trial_rec* r = rep + (size_t)x * 16;
  bool all = true;
  for (int j = 0; j < C.dp; ++j) all = all && (r[j].flags & 4u);
  samu_trial_rec o;
  double* ov = (C.commit && over) ? over + ((size_t)k * n_nodes + C.node) * 16 : nullptr;
  if (all) {
    o.t_end = 0.0; o.flops_lo = 0; o.flops_hi = 0; o.req_iters = 0; o.iters = 0; o.flags = 1u;
    if (ov) for (int j = 0; j < 16; ++j) ov[j] = 0.0;
  } else {
    double t = -CUDART_INF;
    uint64_t hi = 0, lo = 0, ri = 0;
    uint32_t it = 0, done = 1u, cut = 0u;
    for (int j = 0; j < C.dp; ++j) {
      t = fmax(t, r[j].t_end);
      add128(hi, lo, r[j].flops_hi, r[j].flops_lo);
      ri += r[j].req_iters;
      it += r[j].iters;
      done &= r[j].flags & 1u;
      cut |= (r[j].flags >> 1) & 1u;
    }
    o.t_end = t; o.flops_lo = lo; o.flops_hi = hi; o.req_iters = ri; o.iters = it; o.flags = done | (cut << 1);
    if (ov) for (int j = C.dp; j < 16; ++j) ov[j] = 0.0;
  }
  C.out_rec[k] = o;
}

// per-candidate summary over T trials: sequential mean, nearest-rank percentiles via an
// in-shared-memory bitonic sort (T <= 8192; more trials: k_summary_select)
__global__ void k_summary(const samu_trial_rec* __restrict__ recs, int32_t T, samu_cand_summary* __restrict__ out) {
  extern __shared__ double sv[];
  const int32_t c = blockIdx.x;
  const samu_trial_rec* r = recs + (size_t)c * T;
  int32_t P2 = 1;
  while (P2 < T) P2 <<= 1;
  for (int32_t i = threadIdx.x; i < P2; i += blockDim.x) sv[i] = i < T ? r[i].t_end : CUDART_INF;
  __syncthreads();
  for (int32_t size = 2; size <= P2; size <<= 1)
    for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int32_t i = threadIdx.x; i < P2; i += blockDim.x) {
        const int32_t jx = i ^ stride;
        if (jx > i) {
          const bool up = (i & size) == 0;
          const double a = sv[i], b = sv[jx];
          if ((a > b) == up) { sv[i] = b; sv[jx] = a; }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) {
    double s = 0.0;
    uint64_t hi = 0, lo = 0;
    uint64_t ri = 0;
    for (int32_t k = 0; k < T; ++k) {
      s = __dadd_rn(s, r[k].t_end);
      add128(hi, lo, r[k].flops_hi, r[k].flops_lo);
      ri += r[k].req_iters;
    }
    samu_cand_summary o;
    o.mean_t = __ddiv_rn(s, (double)T);
    auto pct = [&](int32_t p) { return sv[max(0, (p * T + 99) / 100 - 1)]; };
    o.p50_t = pct(50);
    o.p90_t = pct(90);
    o.p99_t = pct(99);
    o.mean_flops = __ddiv_rn(u128_to_double(hi, lo), (double)T);
    o.mean_req_iters = __ddiv_rn(__ull2double_rn(ri), (double)T);
    out[c] = o;
  }
}

// T > 8192 trials: the same summary, the nearest-rank order statistics found by an MSB radix
// select over the order-preserving 64-bit keys of t_end (8 passes of 8 bits per percentile, a
// 256-bin shared histogram), so any trial count fits
__device__ __forceinline__ uint64_t order_key(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_double(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_summary_select(const samu_trial_rec* __restrict__ recs, int32_t T, samu_cand_summary* __restrict__ out) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_rank;
  const int32_t c = blockIdx.x;
  const samu_trial_rec* r = recs + (size_t)c * T;
  double pv[3];
  const int32_t pcts[3] = {50, 90, 99};
  for (int q = 0; q < 3; ++q) {
    const int64_t nr = ((int64_t)pcts[q] * T + 99) / 100;     // nearest rank, 1-based
    uint32_t rank = (uint32_t)(nr > 0 ? nr - 1 : 0);
    uint64_t prefix = 0;
    for (int pass = 0; pass < 8; ++pass) {
      const int sh = 56 - 8 * pass;
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
        const uint64_t key = order_key(r[k].t_end);
        if (pass == 0 || (key >> (sh + 8)) == (prefix >> (sh + 8))) atomicAdd(&hist[(key >> sh) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t acc = 0;
        int b = 0;
        for (; b < 255; ++b) {
          if (acc + hist[b] > rank) break;
          acc += hist[b];
        }
        s_rank = rank - acc;
        s_prefix = prefix | ((uint64_t)b << sh);
      }
      __syncthreads();
      prefix = s_prefix;
      rank = s_rank;
      __syncthreads();
    }
    pv[q] = key_double(prefix);
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    uint64_t hi = 0, lo = 0;
    uint64_t ri = 0;
    for (int32_t k = 0; k < T; ++k) {
      s = __dadd_rn(s, r[k].t_end);
      add128(hi, lo, r[k].flops_hi, r[k].flops_lo);
      ri += r[k].req_iters;
    }
    samu_cand_summary o;
    o.mean_t = __ddiv_rn(s, (double)T);
    o.p50_t = pv[0];
    o.p90_t = pv[1];
    o.p99_t = pv[2];
    o.mean_flops = __ddiv_rn(u128_to_double(hi, lo), (double)T);
    o.mean_req_iters = __ddiv_rn(__ull2double_rn(ri), (double)T);
    out[c] = o;
  }
}

// fill n doubles with v (finish-time buffers start at +inf: never finished)
__global__ void k_fill_f64(double* __restrict__ p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// carried finish times re-based to the next stage's clock: fin_t -= t_E^(k) for done requests
__global__ void k_rebase(const uint32_t* __restrict__ st, double* __restrict__ fin_t, int64_t total,
                         const samu_trial_rec* __restrict__ fstar, int32_t n) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= total) return;
  if ((st[x] >> 28) == SAMU_ST_DONE) fin_t[x] = __dsub_rn(fin_t[x], fstar[x / n].t_end);
}

__global__ void k_node_done(const uint32_t* __restrict__ st, int32_t T, int32_t n, const int32_t* __restrict__ node,
                            int32_t* out, int32_t n_nodes) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= (int64_t)T * n) return;
  const int32_t r = (int32_t)(x % n), k = (int32_t)(x / n);
  if ((st[x] >> 28) != SAMU_ST_DONE) out[(size_t)node[r] * T + k] = 1;
}

// f* = argmin_i mean_k T_i^(k) (ties: lower node id = earlier entry) (c16)
__global__ void k_fstar(const samu_trial_rec* __restrict__ cache, int32_t T, const StageCand* __restrict__ sc,
                        int32_t n, StageOut* __restrict__ out) {
  const int32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const StageCand& S = sc[x];
  int32_t best = -1;
  double bm = 0.0;
  for (int32_t i = 0; i < S.n_entries; ++i) {
    const samu_trial_rec* r = cache + (size_t)S.full_slot[i] * T;
    double s = 0.0;
    for (int32_t k = 0; k < T; ++k) s = __dadd_rn(s, r[k].t_end);
    const double mean = __ddiv_rn(s, (double)T);
    if (best < 0 || mean < bm) { best = i; bm = mean; }
  }
  out[x].fstar = best;
}

// T_E = dbl(sum_k FLOPs_E^(k)) / sum_k t_E^(k) (c15, c16), then dT/dN argmax with ties broken by
// smaller dN, lower node id, smaller tp, smaller dp; also max dT (Alg. 1 line 19)
__global__ void k_stage_score(const samu_trial_rec* __restrict__ cache, int32_t T, const StageCand* __restrict__ sc,
                              int32_t n, StageOut* __restrict__ out, double TE_star, int32_t gpus_star,
                              int32_t mode, int32_t* best, double* max_dT) {
  for (int32_t x = threadIdx.x; x < n; x += blockDim.x) {
    const StageCand& S = sc[x];
    const int32_t f = out[x].fstar;
    const samu_trial_rec* rf = cache + (size_t)S.full_slot[f] * T;
    uint64_t hi = 0, lo = 0;
    double den = 0.0;
    for (int32_t k = 0; k < T; ++k) {
      den = __dadd_rn(den, rf[k].t_end);
      add128(hi, lo, rf[k].flops_hi, rf[k].flops_lo);
    }
    for (int32_t i = 0; i < S.n_entries; ++i) {
      if (i == f) continue;
      const samu_trial_rec* rc = cache + (size_t)S.cut_slot[i] * T;
      for (int32_t k = 0; k < T; ++k) add128(hi, lo, rc[k].flops_hi, rc[k].flops_lo);
    }
    out[x].mean_tE = __ddiv_rn(den, (double)T);
    out[x].TE = den == 0.0 ? 0.0 : __ddiv_rn(u128_to_double(hi, lo), den);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t bi = -1, bN = 0;
    double br = 0.0, mx = -CUDART_INF;
    for (int32_t x = 0; x < n; ++x) {
      const StageCand& S = sc[x];
      const double dT = __dsub_rn(out[x].TE, TE_star);
      const int32_t dN = S.gpus - gpus_star;
      const double ratio = __ddiv_rn(dT, (double)dN);
      mx = fmax(mx, dT);
      bool better = false;
      if (mode == 1) {   // competitors: highest stage throughput, first candidate on ties
        if (bi < 0 || out[x].TE > br) { bi = x; br = out[x].TE; }
        continue;
      }
      if (bi < 0 || ratio > br) better = true;
      else if (ratio == br) {
        const StageCand& B = sc[bi];
        if (dN != bN) better = dN < bN;
        else if (S.changed_node != B.changed_node) better = S.changed_node < B.changed_node;
        else if (S.changed_tp != B.changed_tp) better = S.changed_tp < B.changed_tp;
        else better = S.changed_dp < B.changed_dp;
      }
      if (better) { bi = x; br = ratio; bN = dN; }
    }
    *best = bi;
    *max_dT = mx;
  }
}

// all-gathered record blocks [world][n][Tmax] -> rows slots[x] of dst [*][T], trial order.  Rank w
// holds trial block w % Wt (contiguous split of T over Wt blocks) of the jobs of class w / Wt.
__global__ void k_unpack_gather(const samu_trial_rec* __restrict__ recv, int32_t world, int32_t n, int32_t Tmax,
                                int32_t T, int32_t Wt, const int32_t* __restrict__ slots,
                                const int32_t* __restrict__ job_class, samu_trial_rec* __restrict__ dst) {
  const int64_t total = (int64_t)world * n * Tmax;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = (int32_t)(i % Tmax);
    const int32_t x = (int32_t)((i / Tmax) % n);
    const int32_t w = (int32_t)(i / ((int64_t)n * Tmax));
    if (job_class[x] != w / Wt) continue;
    const int32_t blk = w % Wt, base = T / Wt, rem = T % Wt;
    const int32_t cnt = base + (blk < rem ? 1 : 0), b0 = blk * base + min(blk, rem);
    if (k < cnt) dst[(size_t)slots[x] * T + b0 + k] = recv[i];
  }
}

}  // namespace

cudaError_t launch_unpack_gather(const samu_trial_rec* recv, int32_t world, int32_t n, int32_t Tmax, int32_t T,
                                 int32_t Wt, const int32_t* slots, const int32_t* job_class, samu_trial_rec* dst,
                                 cudaStream_t s) {
  const int64_t total = (int64_t)world * n * Tmax;
  if (total <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  k_unpack_gather<<<(unsigned)blocks, 256, 0, s>>>(recv, world, n, Tmax, T, Wt, slots, job_class, dst);
  return cudaGetLastError();
}

cudaError_t launch_combine(const samu_trial_rec* rep_rec, const DevCand* cands, int32_t n_cands, int32_t n_trials,
                           double* over, int32_t n_nodes, cudaStream_t s) {
  const int32_t tot = n_cands * n_trials;
  if (!tot) return cudaSuccess;
  k_combine<<<(tot + 127) / 128, 128, 0, s>>>(rep_rec, cands, n_cands, n_trials, over, n_nodes);
  return cudaGetLastError();
}

cudaError_t launch_summary(const samu_trial_rec* recs, int32_t n_cands, int32_t n_trials, samu_cand_summary* out,
                           cudaStream_t s) {
  if (n_cands <= 0 || n_trials <= 0) return cudaSuccess;
  int32_t P2 = 1;
  while (P2 < n_trials) P2 <<= 1;
  if (P2 > 8192 || std::getenv("SAMU_SUMMARY_SELECT")) {   // (the env var forces this path in tests)
    k_summary_select<<<n_cands, 256, 0, s>>>(recs, n_trials, out);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(double) * P2;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_summary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_summary<<<n_cands, 256, smem, s>>>(recs, n_trials, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_f64(double* p, int64_t n, double v, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_fill_f64<<<(unsigned)blocks, 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}

cudaError_t launch_rebase(uint32_t* st, double* fin_t, int64_t n_total, const samu_trial_rec* fstar_rec, int32_t n_req,
                          cudaStream_t s) {
  if (!n_total) return cudaSuccess;
  k_rebase<<<(unsigned)((n_total + 255) / 256), 256, 0, s>>>(st, fin_t, n_total, fstar_rec, n_req);
  return cudaGetLastError();
}

cudaError_t launch_node_done(const uint32_t* st, int32_t n_trials, int32_t n_req, const int32_t* node,
                             int32_t* out_any_undone, int32_t n_nodes, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out_any_undone, 0, sizeof(int32_t) * n_nodes * n_trials, s);
  if (e != cudaSuccess) return e;
  const int64_t tot = (int64_t)n_trials * n_req;
  if (!tot) return cudaSuccess;
  k_node_done<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(st, n_trials, n_req, node, out_any_undone, n_nodes);
  return cudaGetLastError();
}

cudaError_t launch_fstar(const samu_trial_rec* cache, int32_t T, const StageCand* sc, int32_t n, StageOut* out,
                         cudaStream_t s) {
  if (!n) return cudaSuccess;
  k_fstar<<<(n + 63) / 64, 64, 0, s>>>(cache, T, sc, n, out);
  return cudaGetLastError();
}

cudaError_t launch_stage_score(const samu_trial_rec* cache, int32_t T, const StageCand* sc, int32_t n, StageOut* out,
                               double TE_star, int32_t gpus_star, int32_t mode, int32_t* best, double* max_dT,
                               cudaStream_t s) {
  k_stage_score<<<1, 256, 0, s>>>(cache, T, sc, n, out, TE_star, gpus_star, mode, best, max_dT);
  return cudaGetLastError();
}
