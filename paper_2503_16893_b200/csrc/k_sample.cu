// K1: counter-based output-length sampler (readings c1-c3) + the dense per-B
// coefficient table (reading c11).
//
// Every draw is Philox4x32-10 keyed by (seed) with counter (r >> 2, trial, node, 0): no state,
// so any trial range on any rank reproduces the same lengths.  The inverse eCDF is one lookup:
// at app load each model's eCDF is expanded on the device into its sorted multiset, a u16 table
// of n entries (the t-th element for t = floor(u n / 2^32), reading c2; values clamp at 65535,
// above any l_max).  A block handles a chunk of request sequences for a group of trials: its
// model's table is staged into shared memory with one TMA bulk copy (cp.async.bulk + mbarrier)
// and the chunk's request fields once, then every thread draws for its sequence across the
// trials.  A sequence is a chain root followed by its same-node successors (their prompt needs
// the predecessor's sampled output) or one cross-node request in a later wave
// (evaluator).
#include "samu_internal.cuh"

namespace {

constexpr int K1_THREADS = 256;
constexpr int K1_TRIALS_PER_BLOCK = 8;

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(K1_THREADS) k_sample_lengths(DevApp app, DevEcdf e, const int32_t* __restrict__ seq_head,
                                                               int32_t n_seq, uint32_t k0, uint32_t k1, int32_t trial_begin,
                                                               int32_t n_trials, const uint32_t* __restrict__ known,
                                                               uint16_t* __restrict__ l_out, uint16_t* __restrict__ l_in,
                                                               uint32_t r_base, int32_t stream) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t s_lib[K1_THREADS], s_cap[K1_THREADS];
  __shared__ int32_t s_pred[K1_THREADS], s_node[K1_THREADS];
  uint16_t* tab = reinterpret_cast<uint16_t*>(sm);

  const int32_t s0 = blockIdx.x * K1_THREADS;
  const int32_t s = s0 + threadIdx.x;
  const bool valid = s < n_seq;
  // stage the chunk's request fields (one coalesced read, reused across the trial group)
  const int32_t r0 = valid ? __ldg(seq_head + s) : -1;
  if (valid) {
    s_lib[threadIdx.x] = __ldg(app.l_in_base + r0);
    s_cap[threadIdx.x] = __ldg(app.cap_y + r0);
    s_pred[threadIdx.x] = __ldg(app.pred + r0);
    s_node[threadIdx.x] = __ldg(app.node + r0);
  }
  // the block's model = the model of its first sequence; its table goes to smem via TMA
  const int32_t first_node = __ldg(app.node + __ldg(seq_head + s0));
  const int32_t bm = __ldg(e.model_of_node + first_node);
  const int32_t tab_off = __ldg(e.tab_off + bm);
  const uint32_t tab_n = (uint32_t)(__ldg(e.tab_off + bm + 1) - tab_off);   // padded to 8 entries
  const uint32_t bytes = tab_n * 2u;
  const bool staged = bytes <= (uint32_t)e.smem_tab_bytes;
  if (staged && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(tab)),
        "l"(e.tab + tab_off), "r"(bytes), "r"(smem_u32(&bar))
        : "memory");
  }
  __syncthreads();
  if (staged) {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    }
  }
  if (!valid) return;

  const int32_t kend = min(n_trials, (int32_t)(blockIdx.y + 1) * K1_TRIALS_PER_BLOCK);
  for (int32_t k = blockIdx.y * K1_TRIALS_PER_BLOCK; k < kend; ++k) {
    const size_t base = (size_t)k * app.n_req;
    int32_t r = r0;
    uint32_t prev_out = 0;
    bool first = true;
    while (r >= 0) {
      const int32_t nd = first ? s_node[threadIdx.x] : __ldg(app.node + r);
      const int32_t m = __ldg(e.model_of_node + nd);
      const uint32_t l_max = __ldg(e.l_max_of_node + nd);
      uint32_t X;
      if (known) {   // known output lengths in place of the draw (reading c30)
        X = __ldg(known + r);
      } else {
        // counter (request id, trial, stream): stream = node id (stream >= 0: a request set's own
        // stream id, request ids offset by r_base; samu_sample_requests)
        const uint32_t u = philox_word((uint32_t)r + r_base, (uint32_t)(trial_begin + k),
                                       stream >= 0 ? (uint32_t)stream : (uint32_t)nd, k0, k1);
        // inverse eCDF (c2): the t-th element of the sorted multiset, t = floor(u n / 2^32)
        const uint32_t t = __umulhi(u, __ldg(e.n_obs + m));
        X = (staged && m == bm) ? (uint32_t)tab[t] : (uint32_t)__ldg(e.tab + __ldg(e.tab_off + m) + t);
      }
      uint32_t lin = first ? s_lib[threadIdx.x] : __ldg(app.l_in_base + r);
      const int32_t p = first ? s_pred[threadIdx.x] : __ldg(app.pred + r);
      if (p >= 0) {
        const uint32_t po = first ? (uint32_t)l_out[base + p] : prev_out;   // cross-node: earlier wave
        lin += po > 1u ? po : 1u;
      }
      lin = min(lin, l_max);
      const uint32_t cap = first ? s_cap[threadIdx.x] : __ldg(app.cap_y + r);
      const uint32_t out = min(min(X, cap), l_max - lin);
      l_out[base + r] = (uint16_t)out;
      l_in[base + r] = (uint16_t)lin;
      prev_out = out;
      first = false;
      r = __ldg(app.succ + r);
    }
  }
}

// expand model eCDF knots into the sorted multiset table: tab[t] = value of the first knot with
// cum > t (clamped to 65535), one thread per table entry
__global__ void k_ecdf_table(const uint32_t* __restrict__ values, const uint32_t* __restrict__ cum, int32_t K,
                             uint32_t n, uint16_t* __restrict__ tab) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int32_t lo = 0, hi = K - 1;   // invariant: cum[hi] > t
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cum[mid] > t) hi = mid; else lo = mid + 1;
  }
  tab[t] = (uint16_t)min(values[lo], 65535u);
}

// v = v0 + (v1 - v0) * ((B - B0) / (B1 - B0)), clamped outside the profiled buckets (c11).
__global__ void k_dense_coeff(const double* __restrict__ bucket_B, int32_t nb, const double* __restrict__ coeff,
                              uint32_t max_seqs, double* __restrict__ out) {
  const int32_t B = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int32_t pa = blockIdx.y;   // phase * 2 + (a|b)
  if (B > (int32_t)max_seqs) return;
  const double* v = coeff + (size_t)pa * nb;
  // bucket B values arrive as exact doubles (one staging buffer with the coefficients)
  auto bk = [&](int32_t i) { return (uint32_t)bucket_B[i]; };
  double r;
  if ((uint32_t)B <= bk(0)) r = v[0];
  else if ((uint32_t)B >= bk(nb - 1)) r = v[nb - 1];
  else {
    int32_t k = 0;
    while (!((uint32_t)B >= bk(k) && (uint32_t)B < bk(k + 1))) ++k;
    const double w = __ddiv_rn((double)(B - (int32_t)bk(k)), (double)(bk(k + 1) - bk(k)));
    r = __dadd_rn(v[k], __dmul_rn(__dsub_rn(v[k + 1], v[k]), w));
  }
  out[(size_t)(B - 1) * 8 + pa] = r;   // [B][a_c b_c a_p b_p a_s b_s pad pad]: 3 x 16-byte loads per B
}

}  // namespace

cudaError_t launch_sample(const DevApp& app, const DevEcdf& e, const int32_t* seq_head, int32_t n_seq,
                          uint64_t seed, int32_t trial_begin, int32_t n_trials, const uint32_t* known,
                          uint16_t* l_out, uint16_t* l_in, cudaStream_t s, uint32_t r_base, int32_t stream) {
  if (n_seq == 0 || n_trials == 0) return cudaSuccess;
  cudaError_t err = cudaFuncSetAttribute(k_sample_lengths, cudaFuncAttributeMaxDynamicSharedMemorySize, e.smem_tab_bytes);
  if (err != cudaSuccess) return err;
  dim3 grid((n_seq + K1_THREADS - 1) / K1_THREADS, (n_trials + K1_TRIALS_PER_BLOCK - 1) / K1_TRIALS_PER_BLOCK);
  k_sample_lengths<<<grid, K1_THREADS, e.smem_tab_bytes, s>>>(app, e, seq_head, n_seq, (uint32_t)seed,
                                                              (uint32_t)(seed >> 32), trial_begin, n_trials, known, l_out, l_in,
                                                              r_base, stream);
  return cudaGetLastError();
}

cudaError_t launch_ecdf_table(const uint32_t* values, const uint32_t* cum, int32_t K, uint32_t n, uint16_t* tab,
                              cudaStream_t s) {
  k_ecdf_table<<<(n + 255) / 256, 256, 0, s>>>(values, cum, K, n, tab);
  return cudaGetLastError();
}

cudaError_t launch_dense_coeff(const double* bucket_B, int32_t nb, const double* coeff_slot, uint32_t max_seqs,
                               double* out, cudaStream_t s) {
  dim3 grid((max_seqs + 127) / 128, 6);
  k_dense_coeff<<<grid, 128, 0, s>>>(bucket_B, nb, coeff_slot, max_seqs, out);
  return cudaGetLastError();
}
