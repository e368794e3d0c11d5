// K1: counter-based output-length sampler (readings c1-c3) + the dense per-B
// coefficient table (reading c11).
//
// One thread per (trial, request sequence).  A sequence is a chain root followed by its
// same-node successors (fused self-loop) — the successor's prompt needs its
// predecessor's sampled output — or one cross-node request (evaluator) in a
// later wave.  Every draw is Philox4x32-10 keyed by (seed) with counter (r >> 2, trial, node, 0):
// no state, so any trial range on any rank reproduces the same lengths.
#include "samu_internal.cuh"

namespace {

__device__ __forceinline__ uint32_t philox_word(uint32_t r, uint32_t trial, uint32_t node, uint32_t k0,
                                                uint32_t k1) {
  uint32_t c0 = r >> 2, c1 = trial, c2 = node, c3 = 0u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    if (i) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  const uint32_t w = r & 3u;
  return w == 0 ? c0 : (w == 1 ? c1 : (w == 2 ? c2 : c3));
}

// X = value of the first knot whose cumulative count exceeds t = floor(u n / 2^32) (c2)
__device__ __forceinline__ uint32_t ecdf_draw(const uint32_t* __restrict__ values, const uint32_t* __restrict__ cum,
                                              int32_t K, uint32_t u) {
  const uint32_t n = __ldg(cum + K - 1);
  const uint32_t t = __umulhi(u, n);
  int32_t lo = 0, hi = K - 1;   // invariant: cum[hi] > t
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (__ldg(cum + mid) > t) hi = mid; else lo = mid + 1;
  }
  return __ldg(values + lo);
}

__global__ void __launch_bounds__(256) k_sample_lengths(DevApp app, DevEcdf e, const int32_t* __restrict__ seq_head,
                                                        int32_t n_seq, uint32_t k0, uint32_t k1, int32_t trial_begin,
                                                        uint16_t* __restrict__ l_out, uint16_t* __restrict__ l_in) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seq) return;
  const int32_t k = blockIdx.y;
  const size_t base = (size_t)k * app.n_req;
  int32_t r = __ldg(seq_head + s);
  uint32_t prev_out = 0;
  bool first = true;
  while (r >= 0) {
    const int32_t nd = __ldg(app.node + r);
    const int32_t m = __ldg(e.model_of_node + nd);
    const uint32_t l_max = __ldg(e.l_max_of_node + nd);
    const int32_t off = __ldg(e.off + m);
    const int32_t K = __ldg(e.off + m + 1) - off;
    const uint32_t u = philox_word((uint32_t)r, (uint32_t)(trial_begin + k), (uint32_t)nd, k0, k1);
    const uint32_t X = ecdf_draw(e.values + off, e.cum + off, K, u);
    uint32_t lin = __ldg(app.l_in_base + r);
    const int32_t p = __ldg(app.pred + r);
    if (p >= 0) {
      const uint32_t po = first ? (uint32_t)l_out[base + p] : prev_out;   // cross-node: earlier wave
      lin += po > 1u ? po : 1u;
    }
    lin = min(lin, l_max);
    const uint32_t out = min(min(X, __ldg(app.cap_y + r)), l_max - lin);
    l_out[base + r] = (uint16_t)out;
    l_in[base + r] = (uint16_t)lin;
    prev_out = out;
    first = false;
    r = __ldg(app.succ + r);
  }
}

// v = v0 + (v1 - v0) * ((B - B0) / (B1 - B0)), clamped outside the profiled buckets (c11).
__global__ void k_dense_coeff(const uint32_t* __restrict__ bucket_B, int32_t nb, const double* __restrict__ coeff,
                              uint32_t max_seqs, double* __restrict__ out) {
  const int32_t B = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int32_t pa = blockIdx.y;   // phase * 2 + (a|b)
  if (B > (int32_t)max_seqs) return;
  const double* v = coeff + (size_t)pa * nb;
  double r;
  if ((uint32_t)B <= bucket_B[0]) r = v[0];
  else if ((uint32_t)B >= bucket_B[nb - 1]) r = v[nb - 1];
  else {
    int32_t k = 0;
    while (!((uint32_t)B >= bucket_B[k] && (uint32_t)B < bucket_B[k + 1])) ++k;
    const double w = __ddiv_rn((double)(B - (int32_t)bucket_B[k]), (double)(bucket_B[k + 1] - bucket_B[k]));
    r = __dadd_rn(v[k], __dmul_rn(__dsub_rn(v[k + 1], v[k]), w));
  }
  out[(size_t)pa * max_seqs + (B - 1)] = r;
}

}  // namespace

cudaError_t launch_sample(const DevApp& app, const DevEcdf& e, const int32_t* seq_head, int32_t n_seq,
                          uint64_t seed, int32_t trial_begin, int32_t n_trials, uint16_t* l_out,
                          uint16_t* l_in, cudaStream_t s) {
  if (n_seq == 0 || n_trials == 0) return cudaSuccess;
  dim3 grid((n_seq + 255) / 256, n_trials);
  k_sample_lengths<<<grid, 256, 0, s>>>(app, e, seq_head, n_seq, (uint32_t)seed, (uint32_t)(seed >> 32),
                                        trial_begin, l_out, l_in);
  return cudaGetLastError();
}

cudaError_t launch_dense_coeff(const uint32_t* bucket_B, int32_t nb, const double* coeff_slot, uint32_t max_seqs,
                               double* out, cudaStream_t s) {
  dim3 grid((max_seqs + 127) / 128, 6);
  k_dense_coeff<<<grid, 128, 0, s>>>(bucket_B, nb, coeff_slot, max_seqs, out);
  return cudaGetLastError();
}
