// K4: per-iteration cost-model coefficient fit (reading c34).
//
// One CTA per bucket (model, tp, phase, B); samples of bucket k are [off[k], off[k+1]).  The
// CTA fits latency = a x + b by least squares with centred sums (two passes over the bucket:
// means, then Sxx and Sxy), clamps a < 0 to a = 0 / b = mean y, and, when trimming, drops the
// floor(n * trim / 1000) samples of largest |residual| (ties: lower sample index first): an
// 8-pass MSB radix select over the residual bit patterns (non-negative doubles order like their
// bits) finds the cut value v, samples above v go, and among those equal to v the lowest
// indices go (ordered block scan); then the line is refitted on the rest.  Reductions run in a
// fixed order (per-thread strided partial sums, then a fixed tree), so results are
// deterministic; they differ from a sequential sum only by rounding (compared at 1e-9 rel).
#include "samu_internal.cuh"

#include <math_constants.h>

namespace {

constexpr int KF_THREADS = 256;
constexpr int KF_WARPS = KF_THREADS / 32;

struct Red {
  double v[KF_WARPS][4];
};

// block-wide sum of up to 4 doubles (fixed order), result broadcast to every thread
__device__ __forceinline__ void block_sum4(double (&a)[4], Red& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[j] = __dadd_rn(a[j], __shfl_down_sync(0xFFFFFFFFu, a[j], o));
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < 4; ++j) sm.v[w][j] = a[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double s = sm.v[0][j];
    for (int q = 1; q < KF_WARPS; ++q) s = __dadd_rn(s, sm.v[q][j]);
    a[j] = s;
  }
}

__device__ __forceinline__ double block_min(double v, Red& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xFFFFFFFFu, v, o));
  __syncthreads();
  if (lane == 0) sm.v[w][0] = v;
  __syncthreads();
  double r = sm.v[0][0];
  for (int q = 1; q < KF_WARPS; ++q) r = fmin(r, sm.v[q][0]);
  return r;
}

__device__ __forceinline__ double block_max(double v, Red& sm) {
  return -block_min(-v, sm);
}

// fit over the samples of [b0, b1) with gone[i] == 0; returns false if < 2 distinct x
__device__ bool fit_line(const double* __restrict__ x, const double* __restrict__ y, const uint8_t* __restrict__ gone,
                         int64_t b0, int64_t b1, Red& sm, double* a_out, double* b_out, bool* clamped, int64_t* used) {
  double lo = CUDART_INF, hi = -CUDART_INF;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = b0 + threadIdx.x; i < b1; i += KF_THREADS) {
    if (gone && gone[i]) continue;
    const double xi = x[i];
    lo = fmin(lo, xi);
    hi = fmax(hi, xi);
    s[0] = __dadd_rn(s[0], xi);
    s[1] = __dadd_rn(s[1], y[i]);
    s[2] = __dadd_rn(s[2], 1.0);
  }
  lo = block_min(lo, sm);
  hi = block_max(hi, sm);
  block_sum4(s, sm);
  const int64_t n = (int64_t)s[2];
  *used = n;
  if (n < 2 || !(lo < hi)) return false;
  const double mx = __ddiv_rn(s[0], (double)n), my = __ddiv_rn(s[1], (double)n);
  double t[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = b0 + threadIdx.x; i < b1; i += KF_THREADS) {
    if (gone && gone[i]) continue;
    const double dx = __dsub_rn(x[i], mx), dy = __dsub_rn(y[i], my);
    t[0] = __dadd_rn(t[0], __dmul_rn(dx, dx));
    t[1] = __dadd_rn(t[1], __dmul_rn(dx, dy));
  }
  block_sum4(t, sm);
  double A = __ddiv_rn(t[1], t[0]);
  double B = __dsub_rn(my, __dmul_rn(A, mx));
  *clamped = false;
  if (A < 0.0) { A = 0.0; B = my; *clamped = true; }
  *a_out = A;
  *b_out = B;
  return true;
}

__device__ __forceinline__ uint64_t resid_bits(double xi, double yi, double a, double b) {
  return (uint64_t)__double_as_longlong(fabs(__dsub_rn(yi, __dadd_rn(__dmul_rn(a, xi), b))));
}

__global__ void __launch_bounds__(KF_THREADS) k_fit(const int64_t* __restrict__ off, const double* __restrict__ x,
                                                    const double* __restrict__ y, int32_t trim_permille,
                                                    uint8_t* __restrict__ gone, double* __restrict__ out_a,
                                                    double* __restrict__ out_b, int32_t* __restrict__ out_n_used,
                                                    int32_t* __restrict__ out_flags) {
  __shared__ Red sm;
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_need;
  __shared__ int64_t s_eq_base;
  const int k = blockIdx.x;
  const int64_t b0 = off[k], b1 = off[k + 1], n = b1 - b0;
  double a = 0.0, b = 0.0;
  bool clamped = false;
  int64_t used = 0;
  int32_t flags = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += KF_THREADS) gone[i] = 0;
  __syncthreads();
  if (!fit_line(x, y, nullptr, b0, b1, sm, &a, &b, &clamped, &used)) {
    flags |= 1;
  } else {
    const int64_t drop = n * (int64_t)trim_permille / 1000;
    if (drop > 0) {
      // radix select: the drop-th largest residual bit pattern v
      if (threadIdx.x == 0) { s_prefix = 0; s_need = drop; }
      __syncthreads();
      for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        const uint64_t hmask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (int d = threadIdx.x; d < 256; d += KF_THREADS) hist[d] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += KF_THREADS) {
          const uint64_t key = resid_bits(x[i], y[i], a, b);
          if ((key & hmask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int64_t need = s_need;
          int d = 255;
          for (; d > 0; --d) {
            if ((int64_t)hist[d] >= need) break;
            need -= hist[d];
          }
          s_need = need;   // rank of v among keys with this digit prefix (1-based, from the top)
          s_prefix = prefix | ((uint64_t)d << shift);
        }
        __syncthreads();
      }
      const uint64_t v = s_prefix;
      const int64_t take_eq = s_need;   // keys equal to v to drop (lowest indices first)
      // keys > v go; among keys == v, the first take_eq in sample order go (ordered scan)
      if (threadIdx.x == 0) s_eq_base = 0;
      __syncthreads();
      for (int64_t c0 = b0; c0 < b1; c0 += KF_THREADS) {
        const int64_t i = c0 + threadIdx.x;
        uint64_t key = 0;
        bool eq = false;
        if (i < b1) {
          key = resid_bits(x[i], y[i], a, b);
          eq = key == v;
          if (key > v) gone[i] = 1;
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, eq);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        __shared__ uint32_t wcnt[KF_WARPS];
        if (lane == 0) wcnt[w] = __popc(bal);
        __syncthreads();
        int64_t before = s_eq_base;
        for (int q = 0; q < w; ++q) before += wcnt[q];
        before += __popc(bal & ((1u << lane) - 1u));
        if (eq && before < take_eq) gone[i] = 1;
        __syncthreads();
        if (threadIdx.x == 0) {
          int64_t tot = 0;
          for (int q = 0; q < KF_WARPS; ++q) tot += wcnt[q];
          s_eq_base += tot;
        }
        __syncthreads();
      }
      if (!fit_line(x, y, gone, b0, b1, sm, &a, &b, &clamped, &used)) flags |= 1;
    }
  }
  if (threadIdx.x == 0) {
    if (flags & 1) { a = 0.0; b = 0.0; used = 0; }
    if (clamped && !(flags & 1)) flags |= 2;
    out_a[k] = a;
    out_b[k] = b;
    out_n_used[k] = (int32_t)used;
    out_flags[k] = flags;
  }
}

}  // namespace

cudaError_t launch_fit(const int64_t* off, int32_t n_buckets, const double* x, const double* y, int32_t trim_permille,
                       uint8_t* gone, double* out_a, double* out_b, int32_t* out_n_used, int32_t* out_flags,
                       cudaStream_t s) {
  if (!n_buckets) return cudaSuccess;
  k_fit<<<n_buckets, KF_THREADS, 0, s>>>(off, x, y, trim_permille, gone, out_a, out_b, out_n_used, out_flags);
  return cudaGetLastError();
}
