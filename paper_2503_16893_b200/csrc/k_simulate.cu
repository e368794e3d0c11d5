// K2: iteration-level continuous-batching simulation (readings c3-c9,
// c13, c15, c18, c19, c23-c25), one warp per (candidate, trial, dp replica).
//
// Design (B200-first, not a translation of the per-request oracle loop):
//  * persistent grid, one work item per warp, pulled from an atomic counter; items are decoded on
//    the device from the launch's longest-first candidate order and item offsets (replica-sims
//    differ ~100x in length);
//  * instantiations per block size, one launch each (MODE): LEAN (fresh state, independent
//    requests: the queue is the replica list), FRESH (fresh state with chain successors), both
//    also with a time limit (cut simulations), and the general one (carried state, commit,
//    resume, cross-node arrivals, finish records); candidate descriptors are read from the
//    constant bank;
//  * the running set lives in shared memory: 256 slots, lane L owns slots L + 32 j (bank-conflict
//    free), with the lane's occupancy bits in a register; a 32-entry register window, circular
//    over the lanes, caches the head of the waiting queue;
//  * between events every running request advances one token per decode, so a "decode run" has
//    fixed B while S and B*s grow by B per iteration and the KV-block need of decode d follows
//    from a histogram over the request phases (l - 1 - d) mod bs fixed at admission.  The run
//    evaluates the contract's per-iteration latency sum in fp64 — every iteration is visited
//    (c23), in 32- / 64-iteration chunks summed in parallel yet bit-identically to the
//    sequential adds (binade-local rounding + warp scan, sequential walk on ties) — while FLOPs
//    (folded into u128 once per item), request-iterations and block counts are exact integer
//    closed forms;
//  * events (admission = prefill iteration, finish, preemption) are warp-cooperative: admission
//    is a warp REDUX / prefix-scan over the next 32 queue heads (tokens, KV blocks), retirement
//    a transposed slot scan + ballot / REDUX reductions, preemption a max over packed
//    (admission rank, slot) keys.
#include "samu_internal.cuh"

#include <math_constants.h>

#include <cstdlib>
#include <mutex>

#ifndef SAMU_K2_MULTI_EAGER   // 1: refill the window after every multi-request admission round
#define SAMU_K2_MULTI_EAGER 0
#endif
#ifndef SAMU_K2_CHUNK_GRP   // schedule-sharing launches: chunk runs longer than this x the group size
#define SAMU_K2_CHUNK_GRP 5
#endif
#ifndef SAMU_K2_CHUNK_MIN
#define SAMU_K2_CHUNK_MIN 4   // decode runs longer than this take the lane-parallel chunk sums
#endif

#ifdef SAMU_K2_STATS   // debug build only: event counters (scripts/k2_stats.py)
__device__ unsigned long long g_k2_stats[32];
#define K2STAT(i, v) do { if (lane == 0) atomicAdd(&g_k2_stats[i], (unsigned long long)(v)); } while (0)
extern "C" int samu_debug_k2_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_k2_stats, sizeof(g_k2_stats)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[32] = {0};
    if (cudaMemcpyToSymbol(g_k2_stats, z, sizeof(z)) != cudaSuccess) return -1;
  }
  return 0;
}
#else
#define K2STAT(i, v) do { } while (0)
#endif

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr int SLOTS = 256;

// K2 modes (DevCand::mode) whose items never hold per-request outputs or successors: the smaller
// shared block and the LEAN launch bounds
__host__ __device__ constexpr bool is_lean(int mode) { return mode == 1 || mode == 3 || mode == 5; }

// SMALL (LEAN launches): no finish / release lists, 2 KB less, so 28 warps fit an SM; GRP
// (schedule-sharing launches, modes 5 / 6): the group members' tables
template <bool SMALL, bool GRP>
struct WarpSmT {
  uint32_t s_req[SLOTS];     // request id of an occupied slot
  int2 s_fo[SLOTS];          // (decode index at which it finishes, l - d)
  uint32_t s_meta[SLOTS];    // admission rank << 5 | phase  (phase = (o - 1) mod bs)
  uint32_t stk_req[SLOTS];   // preempted stack, top = front of W
  uint32_t stk_pr[SLOTS];    // its prompt tokens p = l_in + g (bits 31..16) and tokens still to generate (15..0)
  uint32_t tmp[SMALL ? 1 : SLOTS];    // finished requests of the current iteration / radix histogram
  uint32_t hist[32];         // running requests per phase
  // admission exchange / retirement lane tables, and the per-iteration costs of a decode-run
  // chunk (lane j = iteration j): never live in the same event, so they share their storage
  union {
    struct {
      uint32_t adm_req[32], adm_meta[32];
    };
    double cbuf[32];
  };
  int2 adm_fo[32];
  const double* vcoef[GRP ? 32 : 1];   // schedule sharing: lane v's member's dense coefficients and
  uint32_t vK1[GRP ? 32 : 1];          // 2 L (h/tp), candidate index, and the group size
  uint32_t vci[GRP ? 32 : 1];
  uint32_t nv;
  int32_t minF;              // minimum free KV blocks so far (INT_MIN once a preemption happened)
  // warp-uniform state off the hot path (kept out of registers); every lane writes the same
  // value and reads back its own write, so no synchronisation is needed
  double tau, next_ready;    // time limit, ready time of the next pending cross-node arrival
  const uint64_t* pk;        // pending arrivals sorted by (ready time, index): keys / requests
  const uint32_t* pi;
  uint32_t pend_ptr, n_pend, n_heads;
  int32_t site;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// inclusive scan within segments of WIDTH lanes (lanes below WIDTH: the first segment)
template <int WIDTH>
__device__ __forceinline__ uint32_t seg_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < WIDTH; o <<= 1) {
    const uint32_t n = __shfl_up_sync(FULL, v, o, WIDTH);
    if ((lane & (WIDTH - 1)) >= o) v += n;
  }
  return v;
}

__device__ __forceinline__ uint64_t dkey(double x) {   // order-preserving double -> u64
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double kdouble(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

// block-size arithmetic; the kernel is instantiated for the default block size 16 (reading c5)
// as a compile-time constant, for other powers of two (BSK = 0) and for the general case (-1)
template <int BSK>
struct Bs {
  uint32_t v_, mask_, shift_;
  __device__ __forceinline__ uint32_t v() const { return BSK > 0 ? (uint32_t)BSK : v_; }
  __device__ __forceinline__ uint32_t mask() const { return BSK > 0 ? (uint32_t)BSK - 1u : mask_; }
  __device__ __forceinline__ uint32_t shift() const { return BSK > 0 ? (uint32_t)__builtin_ctz(BSK > 0 ? BSK : 1) : shift_; }
  __device__ __forceinline__ uint32_t mod(uint32_t x) const { return BSK >= 0 ? (x & mask()) : x % v_; }
  __device__ __forceinline__ uint32_t div(uint32_t x) const { return BSK >= 0 ? (x >> shift()) : x / v_; }
  __device__ __forceinline__ uint32_t cdiv(uint32_t x) const { return div(x + v() - 1); }
  __device__ __forceinline__ uint32_t posmod(int32_t a) const {
    if (BSK >= 0) return (uint32_t)a & mask();
    const int32_t r = a % (int32_t)v_;
    return (uint32_t)(r < 0 ? r + (int32_t)v_ : r);
  }
};

// Eq. per-iter cost, reading c24: ((fma_c + fma_p) + fma_s), exact integer -> RN
__device__ __forceinline__ double iter_cost(const double* __restrict__ coef, uint32_t B, uint64_t F, uint32_t Bs_,
                                            uint32_t S) {
  const double2* cb = reinterpret_cast<const double2*>(coef + (size_t)(B - 1) * 8);   // dense [B][8] (c11)
  const double2 c = __ldg(cb), p = __ldg(cb + 1), q = __ldg(cb + 2);
  const double tc = __fma_rn(c.x, __ull2double_rn(F), c.y);
  const double tp = __fma_rn(p.x, __uint2double_rn(Bs_), p.y);
  const double ts = __fma_rn(q.x, __uint2double_rn(S), q.y);
  return __dadd_rn(__dadd_rn(tc, tp), ts);
}

__device__ __forceinline__ void set_error(int32_t* e, int32_t code, int32_t site) {
  if (atomicCAS(e, 0, code) == 0) e[1] = site;
}

struct Sim {
  // warp-uniform scalar state
  double t, stop;   // stop = min(tau, next ready time of a pending arrival)
  // FLOPs of the completed iterations = L c * a1 + 2 L (h/tp) * a2 (exact, folded into u128 at
  // the end): a1 = sum of decode B + prefill B s, a2 = sum of decode S + prefill B s^2.  With the
  // closed-form request-iterations (REQIT_CF) a1 holds only the prefill terms B (s - 1): the
  // decode B sum is reqit minus the prefills' B
  uint64_t a1, a2, reqit;
  uint32_t iter, d, needidx, B, S, next_fin, next_rank;   // iter: prefill iterations (decodes: d)
  int32_t F, maxO;
  uint32_t stack_cnt, q_head, q_tail, n_front;
  int32_t err;
};


// Stable LSD radix sort of n (key, idx) pairs by the 64-bit key (8 passes of 8 bits, passes where
// every key shares the digit are skipped), one warp, 256-bin histogram in shared memory.
// Returns the buffer holding the sorted keys; *out_idx the matching indices.
__device__ const uint64_t* warp_radix_sort(uint64_t* ka, uint32_t* ia, uint64_t* kb, uint32_t* ib, uint32_t n,
                                           uint32_t* hist, int lane, uint32_t** out_idx) {
  for (int pass = 0; pass < 8; ++pass) {
    const int sh = pass * 8;
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) atomicAdd(&hist[(ka[i] >> sh) & 255u], 1u);
    __syncwarp();
    uint32_t loc[8], sum = 0;
    bool one_bin = false;
#pragma unroll
    for (int b = 0; b < 8; ++b) { loc[b] = hist[lane * 8 + b]; sum += loc[b]; one_bin |= loc[b] == n; }
    if (__any_sync(FULL, one_bin)) { __syncwarp(); continue; }
    const uint32_t incl = warp_incl_scan(sum, lane);
    uint32_t run = incl - sum;
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 8; ++b) { hist[lane * 8 + b] = run; run += loc[b]; }
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t i = base + lane;
      const bool v = i < n;
      const uint32_t act = __ballot_sync(FULL, v);
      if (v) {
        const uint64_t key = ka[i];
        const uint32_t dg = (uint32_t)(key >> sh) & 255u;
        const uint32_t peers = __match_any_sync(act, dg);
        const uint32_t pos = hist[dg] + __popc(peers & lanemask_lt());
        kb[pos] = key;
        ib[pos] = ia[i];
        __syncwarp(act);
        if ((peers & lanemask_lt()) == 0) hist[dg] += __popc(peers);
      }
      __syncwarp();
    }
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint32_t* ti = ia; ia = ib; ib = ti;
  }
  __syncwarp();
  *out_idx = ia;
  return ka;
}

// Decode-run latency sums in 32-iteration chunks (64 in the FRESH modes), evaluated in parallel
// and bit-identically to the sequential adds (see the exact binade form below; c23, c24): lane j
// evaluates iteration done_it + j (the x of every iteration are exact integers, so their
// conversions equal the sequential increments).  t = clock (updated), coef / K1 = the member's
// dense coefficients and 2 L (h/tp); B, K0 = L c B, S0, smax0 = the run's first S and s.
// Returns the iterations done (m_run, or fewer when t reached stop_t).
template <int MODE>
__device__ __forceinline__ uint32_t run_chunks(double& t, const double* __restrict__ coef, const uint32_t K1,
                                               const uint32_t B, const uint64_t K0, const uint32_t S0,
                                               const uint32_t smax0, const uint32_t m_run, const double stop_t,
                                               const int lane, double* cbuf) {
  // modes 1 / 2: no time limit and no arrivals, stop_t = +inf; in the exact-sum chunks a
  // partial sum that is not below it is not below 2^(e+1) either (already a fallback)
  constexpr bool NOSTOP = MODE == 1 || MODE == 2 || MODE == 5 || MODE == 6;
  const double2* cb = reinterpret_cast<const double2*>(coef + (size_t)(B - 1) * 8);
  const double2 cc = __ldg(cb), cp = __ldg(cb + 1), cs = __ldg(cb + 2);
  const double ac = cc.x, bc = cc.y, ap = cp.x, bp = cp.y, as_ = cs.x, bs_ = cs.y;
  uint32_t done_it = 0;
    bool stopped = false;
    // FRESH (chain summariser: long runs of small B): 64 iterations per scan (lane j:
    // iterations 2j and 2j + 1), the same exact binade form (only in that instantiation:
    // elsewhere the extra live values cost more than the saved scans)
    // (without a stop time the last pass may be partial: 33..64 iterations, the unused ones cost
    // exactly 0 and leave every partial sum unchanged)
#ifdef SAMU_K2_NO_CHUNK64P
    constexpr uint32_t MIN64 = 64u;
#else
    constexpr uint32_t MIN64 = NOSTOP ? 33u : 64u;
#endif
    while ((MODE == 2 || MODE == 4 || MODE == 6) && !stopped && m_run - done_it >= MIN64) {
      const uint64_t eb = (uint64_t)__double_as_longlong(t) & 0x7FF0000000000000ull;
      if (!(t > 0.0 && eb >= (64ull << 52) && eb < (0x7F0ull << 52))) break;
      const uint32_t cnt64 = NOSTOP ? min(64u, m_run - done_it) : 64u;
      const uint32_t ja = done_it + 2u * (uint32_t)lane;
      const uint32_t Sa = S0 + B * ja, Sb = Sa + B;
      const double c0v = __dadd_rn(__dadd_rn(__fma_rn(ac, __ull2double_rn(K0 + (uint64_t)K1 * Sa), bc),
                                             __fma_rn(ap, __uint2double_rn(B * (smax0 + ja)), bp)),
                                   __fma_rn(as_, __uint2double_rn(Sa), bs_));
      const double c1v = __dadd_rn(__dadd_rn(__fma_rn(ac, __ull2double_rn(K0 + (uint64_t)K1 * Sb), bc),
                                             __fma_rn(ap, __uint2double_rn(B * (smax0 + ja + 1u)), bp)),
                                   __fma_rn(as_, __uint2double_rn(Sb), bs_));
      const double c0 = (!NOSTOP || 2u * (uint32_t)lane < cnt64) ? c0v : 0.0;
      const double c1 = (!NOSTOP || 2u * (uint32_t)lane + 1u < cnt64) ? c1v : 0.0;
      const double r0 = __dsub_rn(__dadd_rn(t, c0), t), r1 = __dsub_rn(__dadd_rn(t, c1), t);
      const double e0 = __dsub_rn(c0, r0), e1 = __dsub_rn(c1, r1);
      const double halfu = __longlong_as_double((long long)(eb - (53ull << 52)));
      const double top = __longlong_as_double((long long)(eb + (1ull << 52)));
      const double rp = __dadd_rn(r0, r1);
      double psum = rp;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double nb2 = __shfl_up_sync(FULL, psum, o);
        if (lane >= o) psum = __dadd_rn(psum, nb2);
      }
      const double acc_b = __dadd_rn(t, psum);                              // after 2j + 1
      const double acc_a = __dadd_rn(t, __dadd_rn(__dsub_rn(psum, rp), r0));   // after 2j
      const bool stop_a = !NOSTOP && !(acc_a < stop_t);
      const uint32_t bstop = NOSTOP ? 0u : __ballot_sync(FULL, stop_a || !(acc_b < stop_t));
      const uint32_t L = bstop ? (uint32_t)(__ffs(bstop) - 1) : 31u;
      const bool chk_b = (uint32_t)lane < L || ((uint32_t)lane == L && !stop_a);
      const bool bad = (uint32_t)lane <= L &&
                       (c0 < 0.0 || fabs(e0) == halfu || !(acc_a < top) ||
                        (chk_b && (c1 < 0.0 || fabs(e1) == halfu || !(acc_b < top))));
      if (__any_sync(FULL, bad)) break;   // the 32-iteration chunks below take over
      if (bstop) {
        const bool sa = __shfl_sync(FULL, stop_a, L);
        t = sa ? __shfl_sync(FULL, acc_a, L) : __shfl_sync(FULL, acc_b, L);
        done_it += 2u * L + (sa ? 1u : 2u);
        stopped = true;
      } else {
        t = __shfl_sync(FULL, acc_b, 31);
        done_it += cnt64;
      }
    }
    while (done_it < m_run && !stopped) {
      const uint32_t cnt = min(32u, m_run - done_it);
      double cj = 0.0;
      if ((uint32_t)lane < cnt) {
        // S_j and B (s + j) stay below 256 * l_max < 2^24 (kernel limits)
        const uint32_t jj = done_it + (uint32_t)lane;
        const uint32_t S_j = S0 + B * jj;
        const double xc = __ull2double_rn(K0 + (uint64_t)K1 * S_j);
        const double xp = __uint2double_rn(B * (smax0 + jj));
        const double xs = __uint2double_rn(S_j);
        cj = __dadd_rn(__dadd_rn(__fma_rn(ac, xc, bc), __fma_rn(ap, xp, bp)), __fma_rn(as_, xs, bs_));
      }
      // Exact parallel form of the sequential sum (same doubles as the one-by-one adds):
      // while every partial sum stays in t's binade [2^e, 2^(e+1)) (ulp u), each add
      // RN(acc + c) = acc + round_u(c), where round_u(c) = RN(t + c) - t (exact), unless c
      // sits exactly half-way between multiples of u (a tie, whose even-rounding depends
      // on acc): the partial sums are then t + prefix sums of the round_u(c), all
      // multiples of u below 2^(e+1), hence exact in any order (a warp scan).  Chunks with
      // a negative cost, a tie or a binade crossing take the sequential walk below.
      {
        const uint64_t eb = (uint64_t)__double_as_longlong(t) & 0x7FF0000000000000ull;
        const bool tok = t > 0.0 && eb >= (64ull << 52) && eb < (0x7F0ull << 52);
        if (tok) {
          const double s = __dadd_rn(t, cj);
          const double r = __dsub_rn(s, t);
          const double err = __dsub_rn(cj, r);   // exact (Fast2Sum, t >= c when in binade)
          const double halfu = __longlong_as_double((long long)(eb - (53ull << 52)));
          const double top = __longlong_as_double((long long)(eb + (1ull << 52)));   // 2^(e+1)
          double psum = r;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double nb2 = __shfl_up_sync(FULL, psum, o);
            if (lane >= o) psum = __dadd_rn(psum, nb2);
          }
          const double acc_j = __dadd_rn(t, psum);   // partial sum after iteration lane
          const bool in = (uint32_t)lane < cnt;
          const uint32_t bstop = NOSTOP ? 0u : __ballot_sync(FULL, in && !(acc_j < stop_t));
          const uint32_t upto = bstop ? (uint32_t)(__ffs(bstop) - 1) : cnt - 1;   // last lane used
          const bool bad = (uint32_t)lane <= upto && (cj < 0.0 || fabs(err) == halfu || !(acc_j < top));
          if (!__any_sync(FULL, bad)) {
            t = __shfl_sync(FULL, acc_j, upto);
            done_it += upto + 1;
            stopped = bstop != 0;
            continue;
          }
        }
      }
      cbuf[lane] = cj;
      const bool mono = __all_sync(FULL, !(cj < 0.0));
      __syncwarp();
      double acc = t;
#pragma unroll 8
      for (uint32_t q2 = 0; q2 < cnt; ++q2) acc = __dadd_rn(acc, cbuf[q2]);
      if (mono && acc < stop_t) {
        t = acc;
        done_it += cnt;
      } else {   // the chunk reaches stop_t (or costs are not monotone): step and check
        acc = t;
        uint32_t q2 = 0;
        do {
          acc = __dadd_rn(acc, cbuf[q2]);
          ++q2;
        } while (q2 < cnt && acc < stop_t);
        t = acc;
        done_it += q2;
        stopped = acc >= stop_t;
      }
      __syncwarp();
    }
  return done_it;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Candidate descriptors of a launch with <= SAMU_K2_CONST_CANDS candidates live in the constant
// bank: a field read is one register-indexed LDC (warp-uniform index) instead of an address
// rebuild + L1 load each time register pressure forces the compiler to re-read it.
#define SAMU_K2_CONST_CANDS 400
static_assert(sizeof(DevCand) * SAMU_K2_CONST_CANDS <= 64 * 1024, "candidate table exceeds the constant bank");
__constant__ DevCand c_cands[SAMU_K2_CONST_CANDS];

// One work item (candidate, trial, replica): the whole simulation of one replica-sim.
// MODE (DevCand::mode; 3 / 4 = LEAN / FRESH with a time limit tau, i.e. cut simulations): 0 general; 2 FRESH: fresh state, no cross-node arrivals, no time limit,
// no per-request outputs (chain successors allowed) — the event loop carries no commit / cut /
// arrival machinery; 1 LEAN: FRESH without chain successors (e.g. the first greedy step of
// ensembling / routing nodes) — the queue is then the replica's request list itself.  Fewer live
// registers: ~10 % faster on those items.
template <int BSK, bool CONSTC, int MODE>
__device__ __forceinline__ void sim_item(const SimLaunch& P, WarpSmT<is_lean(MODE), (MODE == 5 || MODE == 6)>& W, const int lane, uint32_t* q, uint64_t* pkey,
                                         uint32_t* pidx, const uint32_t ci, const uint32_t rel, const uint4 grp) {
  constexpr bool LEAN = is_lean(MODE), FRESH = MODE != 0, CUT = MODE == 3 || MODE == 4;
  constexpr bool GRP = MODE == 5 || MODE == 6;   // schedule sharing across a (node, dp) group's tp variants
  // Request-iterations in closed form: without a time limit every request of the replica runs to
  // completion, and every iteration it takes part in emits one of its tokens (recompute prefills
  // included, c7), so the sum over iterations of B is the sum of the replica's max(l_out, 1)
#ifdef SAMU_K2_REQIT_LIVE
  constexpr bool REQIT_CF = false;
#else
  constexpr bool REQIT_CF = MODE == 1 || MODE == 2 || MODE == 5 || MODE == 6;
#endif
  // compact small batches (one request per lane: slot 0 only): the chain summariser's KV-bound
  // FRESH items run at B ~ 10-20; the LEAN launches' batches are large (the checks cost more there)
#ifdef SAMU_K2_NO_COMPACT
  constexpr bool COMPACT = false;
#else
  constexpr bool COMPACT = !LEAN;
#endif
  // the host runs a candidate on the FRESH paths (modes 2, 4, 6) only when its node has chain
  // successors (DevCand::has_succ): no constant-bank read for it there
  constexpr bool SUCC = MODE == 2 || MODE == 4 || MODE == 6;
  // ... and without per-request outputs a running request's id is needed only to find its chain
  // successor when it finishes: on those paths the window, the slots, the preempted stack and the
  // finisher list carry the successor's id (-1: none) instead, loaded beside the request's lengths
  // when it enters the window, so a finish releases its successor without a dependent global load
#ifdef SAMU_K2_NO_SUCC_SLOT
  constexpr bool SUCC_SLOT = false;
#else
  constexpr bool SUCC_SLOT = SUCC;
#endif
  // lazy window refills (see the loop top)
#ifdef SAMU_K2_EAGER_WIN
  constexpr bool LAZYW = false;
#else
  constexpr bool LAZYW = true;
#endif
  const DevApp& A = P.app;
  const int n = A.n_req;
    const DevCand& C = CONSTC ? c_cands[ci] : P.cands[ci];
    const uint32_t dpc = (uint32_t)C.dp;
    const uint32_t k = rel / dpc, j = rel - k * dpc;
    const size_t tb = (size_t)k * n;
    // sampled lengths of this trial, indexed with 32-bit offsets from the kernel parameters (the
    // host guarantees local trials x requests < 2^32): one add + one wide multiply per load
    const uint32_t tb32 = (uint32_t)k * (uint32_t)n;
#define LO_(r) P.l_out[tb32 + (uint32_t)(r)]
#define LI_(r) P.l_in[tb32 + (uint32_t)(r)]
    uint32_t* st = P.st ? P.st + tb : nullptr;
    uint16_t* gst = P.g ? P.g + tb : nullptr;
    double* ft = P.fin_t ? P.fin_t + tb : nullptr;
    const double* sfin = C.src_fin ? C.src_fin + tb : nullptr;
    double* fto = C.fin_t_out ? C.fin_t_out + tb : nullptr;
    uint32_t* fio = C.fin_iter_out ? C.fin_iter_out + tb : nullptr;
    double* over = P.over ? P.over + ((size_t)k * A.n_nodes + C.node) * 16 : nullptr;
    const uint32_t r0 = C.rep_off[j], r1 = C.rep_off[j + 1];
    const uint32_t ms = C.max_seqs;
    Bs<BSK> bs;
    bs.v_ = C.bs;
    bs.mask_ = C.bs - 1;
    bs.shift_ = __ffs(C.bs) - 1;
    const bool commit = !FRESH && C.commit && st;
    // waiting-queue reads: the replica's request list (LEAN: never appended to) or the scratch ring
    const uint32_t* qr = LEAN ? C.rep_req + r0 : q;

    Sim m;
    m.t = C.resume ? (over ? over[j] : 0.0) : C.load_s;
    // schedule sharing (GRP): the group is simulated once with the head's KV blocks; lane v
    // carries the clock (and cost coefficients) of member min(v, nv - 1), every integer of the
    // schedule is shared.  Member v's schedule equals the head's iff no preemption happened and
    // the peak block use never exceeded its own count: min F >= blocks_head - blocks_v.
    if (GRP) {
      W.minF = C.blocks;
      uint32_t my_ci = ci;
      if (grp.x > 1) {
        const uint32_t v = min((uint32_t)lane, grp.x - 1);
        my_ci = v == 0 ? ci : v == 1 ? grp.y : v == 2 ? grp.z : grp.w;
      }
      const DevCand& Cl = CONSTC ? c_cands[my_ci] : P.cands[my_ci];
      m.t = Cl.load_s;
      W.vcoef[lane] = Cl.coef;
      W.vK1[lane] = (uint32_t)Cl.K1;
      W.vci[lane] = my_ci;
      W.nv = grp.x;
    }
    double tau = (FRESH && !CUT) ? CUDART_INF : C.tau ? C.tau[k] : (C.tau_rec ? C.tau_rec[k].t_end : CUDART_INF);
    m.a1 = m.a2 = m.reqit = 0;
    m.iter = 0; m.d = 0; m.needidx = 0; m.B = 0; m.S = 0; m.next_rank = 0;
    m.F = C.blocks; m.maxO = INT_MIN; m.next_fin = FULL;
    m.stack_cnt = 0; m.q_head = 0; m.q_tail = 0; m.n_front = 0;
    uint32_t n_heads = 0, n_pend = 0;
    m.err = 0;
    int32_t site = 0;
    uint32_t occ = 0;   // this lane's occupied slots (bit j = slot lane + 32 j)

    W.hist[lane] = 0;
    __syncwarp();

    // ---- initial state from the carried WorkloadState (c18, c27) ----
    // W = [preempted stack (smem, new preemptions)] + queue: [front: recomputed running (reload)
    // and earlier-preempted requests][never-started heads, index order][queued / arrived]
    uint64_t* skey = pkey + 2 * (size_t)P.max_p;   // carried-entry sort buffers
    uint32_t* sidx = pidx + 2 * (size_t)P.max_p;
    uint32_t n_run = 0, n_pre = 0, n_q = 0, n_cls = 0;
    bool all_done = true;
    if (LEAN) {
      n_heads = r1 - r0;
      all_done = r1 == r0;
    } else {
    for (uint32_t base = r0; base < r1; base += 32) {
      const uint32_t idx = base + lane;
      const bool valid = idx < r1;
      const uint32_t r = valid ? __ldg(C.rep_req + idx) : 0u;
      const uint32_t w = (valid && st) ? st[r] : 0u;
      const uint32_t s = w >> 28, rk = w & 0x0FFFFFFFu;
      const int32_t pr = valid ? __ldg(A.pred + r) : -1;
      const bool cross = valid && pr >= 0 && __ldg(A.cross + r);
      const bool fresh = valid && s == SAMU_ST_FRESH;
      const bool head = fresh && pr < 0;
      const bool pend = fresh && cross;
      const bool succ_wait = fresh && pr >= 0 && !cross;
      if (succ_wait && st && (st[pr] >> 28) == SAMU_ST_DONE) { m.err = SAMU_E_STATE; site = 1; }
      if (valid && s > SAMU_ST_DONE) { m.err = SAMU_E_STATE; site = 2; }
      const uint32_t bh = __ballot_sync(FULL, head);
      // fresh state (no state, or a never-committed node on the FRESH paths): no front region
      if (head && (!st || FRESH)) q[n_heads + __popc(bh & lanemask_lt())] = r;
      n_heads += __popc(bh);
      // carried entries: class 0 running (reload) | 1 preempted | 3 queued | 4 running (resume)
      uint32_t cls = 7;
      if (valid && s == SAMU_ST_RUNNING) cls = C.resume ? 4u : 0u;
      else if (valid && s == SAMU_ST_PREEMPTED) cls = 1u;
      else if (valid && s == SAMU_ST_QUEUED) cls = 3u;
      const uint32_t bc = __ballot_sync(FULL, cls != 7);
      if (cls != 7) {
        const uint32_t pos = n_cls + __popc(bc & lanemask_lt());
        if (pos < (uint32_t)P.max_p) { skey[pos] = ((uint64_t)cls << 60) | ((uint64_t)rk << 32) | r; sidx[pos] = r; }
      }
      n_cls += __popc(bc);
      const uint32_t bp = __ballot_sync(FULL, pend);
      if (pend) {
        double ready;
        if (st && (st[pr] >> 28) == SAMU_ST_DONE && ft) ready = ft[pr];
        else if (sfin) ready = sfin[pr];
        else ready = CUDART_INF;
        const uint32_t pos = n_pend + __popc(bp & lanemask_lt());
        if (pos < (uint32_t)P.max_p) { pkey[pos] = dkey(ready); pidx[pos] = r; }
      }
      n_pend += __popc(bp);
      if (bc) {
        n_run += __popc(__ballot_sync(FULL, valid && s == SAMU_ST_RUNNING));
        n_pre += __popc(__ballot_sync(FULL, valid && s == SAMU_ST_PREEMPTED));
        n_q += __popc(__ballot_sync(FULL, valid && s == SAMU_ST_QUEUED));
      }
      if (__ballot_sync(FULL, valid && s != SAMU_ST_DONE)) all_done = false;
    }
    }
    site = (int32_t)__reduce_max_sync(FULL, (uint32_t)site);
    m.err = __reduce_max_sync(FULL, (uint32_t)(-m.err)) ? SAMU_E_STATE : 0;
    m.n_front = C.resume ? n_pre : n_run + n_pre;
    if (!LEAN && (n_pend > (uint32_t)P.max_p || n_cls > (uint32_t)P.max_p ||
                  m.n_front + n_heads + n_q > (uint32_t)P.max_q)) { m.err = SAMU_E_STATE; site = 3; }
    if (C.resume && n_run > ms) { m.err = SAMU_E_STATE; site = 4; }
    m.q_tail = m.n_front + n_heads + n_q;
    if (!FRESH && !m.err && st) {
      // heads after the front region, in index order
      uint32_t nh = 0;
      for (uint32_t base = r0; base < r1; base += 32) {
        const uint32_t idx = base + lane;
        const bool valid = idx < r1;
        const uint32_t r = valid ? __ldg(C.rep_req + idx) : 0u;
        const bool head = valid && (st[r] >> 28) == SAMU_ST_FRESH && __ldg(A.pred + r) < 0;
        const uint32_t bh = __ballot_sync(FULL, head);
        if (head) q[m.n_front + nh + __popc(bh & lanemask_lt())] = r;
        nh += __popc(bh);
      }
      if (n_cls) {
        // carried entries in (class, rank / seq, index) order (the oracle's sorted pairs)
        uint32_t* sorted_idx;
        warp_radix_sort(skey, sidx, skey + P.max_p, sidx + P.max_p, n_cls, W.tmp, lane, &sorted_idx);
        int32_t used = 0;
        uint32_t S0 = 0;
        const uint32_t q_base = m.n_front + n_heads;
        for (uint32_t i = lane; i < n_cls; i += 32) {
          const uint32_t r = sorted_idx[i];
          if (i < m.n_front) q[i] = r;
          else if (i < m.n_front + n_q) q[q_base + (i - m.n_front)] = r;
          else {   // resume: running requests keep their admission order in slots 0..B-1
            const uint32_t jx = i - m.n_front - n_q;
            const uint32_t g = gst[r];
            const uint32_t lin = LI_(r);
            const uint32_t Lr = max((uint32_t)LO_(r), 1u);
            const int32_t o = (int32_t)(lin + g);
            const uint32_t ph = bs.posmod(o - 1);
            if (g >= Lr || g == 0) { m.err = SAMU_E_STATE; site = 5; }
            W.s_req[jx] = r;
            W.s_fo[jx] = make_int2((int32_t)(Lr - g), o);
            W.s_meta[jx] = (jx << 5) | ph;
            atomicAdd(&W.hist[ph], 1u);
            used += (int32_t)bs.cdiv(lin + g - 1);
            S0 += lin + g;
          }
        }
        used = (int32_t)__reduce_add_sync(FULL, (uint32_t)used);
        S0 = __reduce_add_sync(FULL, S0);
        site = (int32_t)__reduce_max_sync(FULL, (uint32_t)site);
        m.err = __reduce_max_sync(FULL, (uint32_t)(-m.err)) ? SAMU_E_STATE : 0;
        if (C.resume) {
          m.B = n_run;
          m.S = S0;
          m.F -= used;
          m.next_rank = n_run;
          if (m.F < 0) { m.err = SAMU_E_STATE; site = 8; }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if ((uint32_t)(lane + 32 * jj) < n_run) occ |= 1u << jj;
        }
      }
    }
    __syncwarp();

    // ---- pending cross-node arrivals in (ready, index) order: stable LSD radix sort ----
    const uint64_t* pk = pkey;
    const uint32_t* pi = pidx;
    if (!FRESH && !m.err && n_pend > 1) {
      uint32_t* si;
      pk = warp_radix_sort(pkey, pidx, pkey + P.max_p, pidx + P.max_p, n_pend, W.tmp, lane, &si);
      pi = si;
    }
    const double next_ready0 = n_pend ? kdouble(pk[0]) : CUDART_INF;
    __syncwarp();   // lane 0 writes the warp's cold state; every later reader is behind a __syncwarp
    if (lane == 0) {
      W.tau = tau;
      W.next_ready = next_ready0;
      W.pk = pk;
      W.pi = pi;
      W.pend_ptr = 0;
      W.n_pend = n_pend;
      W.n_heads = n_heads;
      W.site = site;
    }
    __syncwarp();
    m.stop = fmin(tau, next_ready0);
    const uint32_t K1 = (uint32_t)C.K1;   // 2 L (h/tp) (< 2^32, checked by the host)
    // this lane's member (GRP: read from the warp's shared block, off the register budget)
#define K1_l (GRP ? W.vK1[lane] : K1)
#define coef_l (GRP ? W.vcoef[lane] : C.coef)
    const uint64_t LC = C.LC;   // L c
    // phase whose requests need a new KV block at the next decode: -d mod bs (phase = (l - 1 - d)
    // mod bs, fixed at admission); kept in a register only for the general block size
#define NEEDIDX (BSK >= 0 ? ((0u - m.d) & bs.mask()) : m.needidx)
    const bool need_rel = LEAN ? false : FRESH ? (SUCC || (bool)C.has_succ) : (fio || fto || commit || C.has_succ);
    bool cut = false;
    // per-lane summaries of this lane's slots: min finish index, max (l - d)
    uint32_t lminf = FULL;
    int32_t lmaxo = INT_MIN;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
      if ((occ >> jj) & 1u) {
        const int2 fo = W.s_fo[lane + 32 * jj];
        lminf = min(lminf, (uint32_t)fo.x);
        lmaxo = max(lmaxo, fo.y);
      }
    m.next_fin = __reduce_min_sync(FULL, lminf);
    m.maxO = __reduce_max_sync(FULL, lmaxo);
    // window: register cache of the first wn (<= 32) entries of W, circular over the lanes
    // (position i in lane (wb + i) mod 32, so admitting a prefix just advances wb and the admitted
    // requests enter the running set from their own lanes, spread round-robin over all lanes):
    // request, prompt tokens p = l_in + g, tokens still to generate incl. the prefill's (L - g).
    // Entries from the preempted stack carry (p, L - g) from shared memory (no global loads).
    uint32_t w_r = 0, w_p = 0, w_rem = 0, wn = 0, wb = 0;
    // load window position pos of W (stack top first, then the queue) into this lane
#define WIN_LOAD(pos)                                                                          \
    do {                                                                                       \
      if ((pos) < m.stack_cnt) {                                                               \
        const uint32_t si_ = m.stack_cnt - 1 - (pos);                                          \
        w_r = W.stk_req[si_];                                                                  \
        const uint32_t pr_ = W.stk_pr[si_];                                                    \
        w_p = pr_ >> 16;                                                                       \
        w_rem = pr_ & 0xFFFFu;                                                                 \
      } else {                                                                                 \
        const uint32_t qp_ = m.q_head + (pos) - m.stack_cnt;                                   \
        const uint32_t r_ = qr[qp_];                                                           \
        /* recompute front (reload) keeps its tokens */                                        \
        const uint32_t g_ = (!FRESH && qp_ < m.n_front) ? (uint32_t)gst[r_] : 0u;              \
        w_r = SUCC_SLOT ? (uint32_t)__ldg(A.succ + r_) : r_;                                   \
        w_p = LI_(r_) + g_;                                                                    \
        w_rem = max((uint32_t)LO_(r_), 1u) - g_;                                               \
      }                                                                                        \
    } while (0)

    K2STAT(0, 1);
    // ---- main loop (c25) ----
    // (every error site inside the loop breaks out of it: the error code is not a loop condition)
#ifdef SAMU_K2_ERR_LOOP
    while (!m.err) {
#else
    if (!m.err) for (;;) {
#endif
      K2STAT(1, 1);
      if (CUT && m.t >= m.stop) { cut = true; break; }   // no arrivals in these modes: stop = tau
      if (!FRESH && m.t >= m.stop) {   // stop time or a pending arrival reached
        const double tau_w = W.tau;
        if (m.t >= tau_w) { cut = true; break; }
        // pending cross-node arrivals with ready <= t join the back of W
        const uint32_t n_pend_w = W.n_pend;
        const uint64_t* pk_w = W.pk;
        uint32_t pend_ptr = W.pend_ptr;
        double next_ready = W.next_ready;
        while (pend_ptr < n_pend_w && next_ready <= m.t) {
          const uint32_t i = pend_ptr + lane;
          const bool ok = i < n_pend_w && kdouble(pk_w[i]) <= m.t;
          const uint32_t b = __ballot_sync(FULL, ok);
          const uint32_t cnt = (b == FULL) ? 32u : (uint32_t)(__ffs(~b) - 1);
          if ((uint32_t)lane < cnt) q[m.q_tail + lane] = W.pi[i];
          m.q_tail += cnt;
          pend_ptr += cnt;
          next_ready = pend_ptr < n_pend_w ? kdouble(pk_w[pend_ptr]) : CUDART_INF;
        }
        __syncwarp();
        if (lane == 0) { W.pend_ptr = pend_ptr; W.next_ready = next_ready; }
        __syncwarp();
        m.stop = fmin(tau_w, next_ready);
      }
      const uint32_t wlen = m.stack_cnt + (m.q_tail - m.q_head);
      if (m.B == 0 && wlen == 0) {
        if (!FRESH && W.pend_ptr < W.n_pend && W.next_ready != CUDART_INF) { m.t = W.next_ready; continue; }
        break;
      }
      // refill the window so it holds min(32, |W|) entries (LAZYW: only once it holds fewer than
      // min(2, |W|): the head checks read its first two entries, the multi-request admission below
      // refills it in full first; a refill loads all missing entries in one pass)
      {
        const uint32_t want = min(32u, wlen);
        if (wn < (LAZYW ? min(2u, wlen) : want)) {
          const uint32_t pos = ((uint32_t)lane - wb) & 31u;
          if (pos >= wn && pos < want) WIN_LOAD(pos);
          wn = want;
        }
      }
      // does the head of W fit? (slots, token budget, blocks)
      const uint32_t hp = __shfl_sync(FULL, w_p, wb);
      const bool fits = wlen > 0 && m.B < ms && hp <= C.budget && (int32_t)bs.cdiv(hp) <= m.F;
      uint32_t n_fin = 0;
      bool go_decode = !fits;
      if (fits) {
        // ================= prefill iteration (c8): admit a strict FCFS prefix of W =========
        uint32_t k_adm = 0, tok = 0, smaxp = 0, S_add = 0, n_stay = 0;
        int32_t blk = 0, freed = 0;
        bool reduce_fo = true;   // per-lane finish / offset summaries changed in several lanes
        // Exactly the head enters when one slot is free, one request waits, or the first two do
        // not fit together (block-bound prefills, e.g. 2k-token chunks): the head fits (above), so
        // it is admitted alone with warp-uniform arithmetic, no reductions or scans.
        const uint32_t nb0 = bs.cdiv(hp);
        bool single = wn <= 1u || m.B + 1u >= ms;
        if (!single) {
          const uint32_t p1 = __shfl_sync(FULL, w_p, (wb + 1u) & 31u);
          single = hp + p1 > C.budget || (int32_t)(nb0 + bs.cdiv(p1)) > m.F;
        }
        if (single) {
          K2STAT(4, 1);
          const uint32_t rem0 = __shfl_sync(FULL, w_rem, wb);
          const uint32_t r0 = __shfl_sync(FULL, w_r, wb);
          k_adm = 1;
          tok = hp;
          smaxp = hp;
          blk = (int32_t)nb0;
          if (rem0 <= 1u) {   // done in its prefill
            n_fin = 1;
            freed = (int32_t)nb0;
            if (need_rel && lane == 0) W.tmp[0] = r0;
          } else {
            n_stay = 1;
            S_add = hp + 1;
            const int32_t s_o = (int32_t)(hp + 1) - (int32_t)m.d;
            const uint32_t s_fin = m.d + rem0 - 1;
            const uint32_t s_meta = (m.next_rank << 5) | bs.posmod((int32_t)hp - (int32_t)m.d);
            // into a free slot of the head's lane, else of the first lane with one (B < 256)
            // (COMPACT: prefer an empty lane, so a small batch keeps one request per lane and
            // retirement and victim search read one slot per lane)
            const uint32_t e0 = COMPACT ? __ballot_sync(FULL, occ == 0u) : 0u;
            const uint32_t fl = e0 ? e0 : __ballot_sync(FULL, occ != 0xFFu);
            const uint32_t tgt = ((fl >> wb) & 1u) ? wb : (uint32_t)(__ffs(fl) - 1);
            if ((uint32_t)lane == tgt) {
              const int jb = __ffs(~occ & 0xFFu) - 1;
              const int s = lane + 32 * jb;
              W.s_req[s] = r0;
              W.s_fo[s] = make_int2((int32_t)s_fin, s_o);
              W.s_meta[s] = s_meta;
              W.hist[s_meta & 31u] += 1u;
              occ |= 1u << jb;
              lminf = min(lminf, s_fin);
              lmaxo = max(lmaxo, s_o);
            }
            m.next_fin = min(m.next_fin, s_fin);
            m.maxO = max(m.maxO, s_o);
            reduce_fo = false;
            __syncwarp();
          }
          const uint32_t take = min(1u, m.stack_cnt);
          m.stack_cnt -= take;
          m.q_head += 1u - take;
          wb = (wb + 1u) & 31u;
          wn -= 1u;
          const uint32_t want = min(32u, m.stack_cnt + (m.q_tail - m.q_head));
          // (LAZYW: the merged decode check below reads the new head)
          if (wn < (LAZYW ? min(1u, want) : want)) {
            const uint32_t pos = ((uint32_t)lane - wb) & 31u;
            if (pos >= wn && pos < want) WIN_LOAD(pos);
            wn = want;
          }
        } else
        for (;;) {
          if (LAZYW) {   // the FCFS prefix may extend over the whole window: fill it
            const uint32_t want = min(32u, m.stack_cnt + (m.q_tail - m.q_head));
            if (wn < want) {
              const uint32_t pos = ((uint32_t)lane - wb) & 31u;
              if (pos >= wn && pos < want) WIN_LOAD(pos);
              wn = want;
            }
          }
          const uint32_t pos = ((uint32_t)lane - wb) & 31u;   // window position of this lane
          const bool valid = pos < wn;
          const uint32_t p = valid ? w_p : 0u;
          const uint32_t nb = valid ? bs.cdiv(p) : 0u;
          uint32_t mm, add_tok, add_blk;   // admitted count, tokens, blocks
          K2STAT(4, 1);
          const uint32_t slots = min(wn, ms - m.B - k_adm);
          if (slots <= 1u) {
            // at most the head can enter (one free slot or one waiting request): no scans
            const uint32_t p0 = __shfl_sync(FULL, p, wb);
            add_tok = p0;
            add_blk = bs.cdiv(p0);
            mm = (wn > 0 && m.B + k_adm < ms && tok + p0 <= C.budget && (int32_t)(blk + add_blk) <= m.F) ? 1u : 0u;
          } else if ((add_tok = __reduce_add_sync(FULL, pos < slots ? p : 0u)) + tok <= C.budget &&
                     (int32_t)((add_blk = __reduce_add_sync(FULL, pos < slots ? nb : 0u)) + blk) <= m.F) {
            // the first `slots` entries fit the token and block budgets together: only the slots
            // bind (the FCFS prefix is limited by them), no scans
            mm = slots;
          } else if (const uint32_t p01 = __shfl_sync(FULL, p, wb) + __shfl_sync(FULL, p, (wb + 1u) & 31u),
                                    b01 = __shfl_sync(FULL, nb, wb) + __shfl_sync(FULL, nb, (wb + 1u) & 31u);
                     tok + p01 > C.budget || (int32_t)(blk + b01) > m.F) {
            // the first two do not fit together (block-bound prefills, e.g. 2k-token chunks): at
            // most the head enters, no scans
            const uint32_t p0 = __shfl_sync(FULL, p, wb);
            add_tok = p0;
            add_blk = bs.cdiv(p0);
            mm = (tok + p0 <= C.budget && (int32_t)(blk + add_blk) <= m.F) ? 1u : 0u;
          } else {
            K2STAT(5, 1);
            // scans in window order: lane i takes position i
            const uint32_t src = ((uint32_t)lane + wb) & 31u;
            const uint32_t sp = warp_incl_scan(__shfl_sync(FULL, p, src), lane);
            const uint32_t sb = warp_incl_scan(__shfl_sync(FULL, nb, src), lane);
            const bool ok = (uint32_t)lane < wn && (m.B + k_adm + lane + 1 <= ms) && (tok + sp <= C.budget) &&
                            ((int32_t)(blk + sb) <= m.F);
            const uint32_t bal = __ballot_sync(FULL, ok);
            mm = (bal == FULL) ? 32u : (uint32_t)(__ffs(~bal) - 1);
            add_tok = __shfl_sync(FULL, sp, mm == 0 ? 0 : mm - 1);
            add_blk = __shfl_sync(FULL, sb, mm == 0 ? 0 : mm - 1);
          }
          if (mm == 0) break;
          const bool adm = pos < mm;
          const bool finish_now = adm && w_rem <= 1u;
          const bool stay = adm && !finish_now;
          const uint32_t bst = __ballot_sync(FULL, stay);
          const uint32_t bfn = __ballot_sync(FULL, finish_now);
          const uint32_t ns = __popc(bst);
          int32_t s_fin = 0, s_o = 0;
          uint32_t s_meta = 0;
          if (stay) {
            s_o = (int32_t)(p + 1) - (int32_t)m.d;
            s_fin = (int32_t)(m.d + w_rem - 1);
            s_meta = ((m.next_rank + k_adm + pos) << 5) | bs.posmod((int32_t)p - (int32_t)m.d);
            atomicAdd(&W.hist[s_meta & 31u], 1u);
          }
          if (finish_now && need_rel) W.tmp[n_fin + __popc(bfn & lanemask_lt())] = w_r;
          n_fin += __popc(bfn);
          if (bfn) {
            freed += (int32_t)__reduce_add_sync(FULL, finish_now ? nb : 0u);
            S_add += __reduce_add_sync(FULL, stay ? p + 1 : 0u);
          } else {
            S_add += add_tok + ns;   // every admitted request stays: sum of (p + 1)
          }
          smaxp = max(smaxp, __reduce_max_sync(FULL, adm ? p : 0u));
          // insert the stays into free slots: the a-th lane with a free slot takes the a-th stay
          if (ns) {
            const bool has_free = occ != 0xFFu;
            const uint32_t fl = __ballot_sync(FULL, has_free);
            if ((bst & ~fl) == 0) {
              // every staying lane has a free slot of its own: no exchange
              if (stay) {
                const int jb = __ffs(~occ & 0xFFu) - 1;
                const int s = lane + 32 * jb;
                W.s_req[s] = w_r;
                W.s_fo[s] = make_int2(s_fin, s_o);
                W.s_meta[s] = s_meta;
                occ |= 1u << jb;
                lminf = min(lminf, (uint32_t)s_fin);
                lmaxo = max(lmaxo, s_o);
              }
            } else if ((uint32_t)__popc(fl) >= ns) {
              // a-th stay lane -> a-th lane with a free slot, through a lane table in smem
              if (stay) W.adm_meta[__popc(bst & lanemask_lt())] = (uint32_t)lane;
              __syncwarp();
              const uint32_t a = __popc(fl & lanemask_lt());
              const bool take = has_free && a < ns;
              const uint32_t src = take ? W.adm_meta[a] : 0u;
              const uint32_t r_v = __shfl_sync(FULL, w_r, src);
              const int32_t f_v = __shfl_sync(FULL, s_fin, src);
              const int32_t o_v = __shfl_sync(FULL, s_o, src);
              const uint32_t m_v = __shfl_sync(FULL, s_meta, src);
              if (take) {
                const int jb = __ffs(~occ & 0xFFu) - 1;
                const int s = lane + 32 * jb;
                W.s_req[s] = r_v;
                W.s_fo[s] = make_int2(f_v, o_v);
                W.s_meta[s] = m_v;
                occ |= 1u << jb;
                lminf = min(lminf, (uint32_t)f_v);
                lmaxo = max(lmaxo, o_v);
              }
            } else {
              if (stay) {
                const uint32_t a = __popc(bst & lanemask_lt());
                W.adm_req[a] = w_r;
                W.adm_fo[a] = make_int2(s_fin, s_o);
                W.adm_meta[a] = s_meta;
              }
              __syncwarp();
              uint32_t fm = ~occ & 0xFFu;
              const uint32_t nf = __popc(fm);
              uint32_t a = warp_incl_scan(nf, lane) - nf;
              while (fm && a < ns) {
                const int jb = __ffs(fm) - 1;
                fm &= fm - 1;
                const int s = lane + 32 * jb;
                const int2 fo = W.adm_fo[a];
                W.s_req[s] = W.adm_req[a];
                W.s_fo[s] = fo;
                W.s_meta[s] = W.adm_meta[a];
                occ |= 1u << jb;
                lminf = min(lminf, (uint32_t)fo.x);
                lmaxo = max(lmaxo, fo.y);
                ++a;
              }
            }
            __syncwarp();
          }
          n_stay += ns;
          tok += add_tok;
          blk += (int32_t)add_blk;
          k_adm += mm;
          const uint32_t take = min(mm, m.stack_cnt);
          m.stack_cnt -= take;
          m.q_head += mm - take;
          // advance the window by mm and refill it (LAZYW: the next round fills it first; after the
          // last round the merged decode check reads the new head)
          wb = (wb + mm) & 31u;
          wn -= mm;
          const uint32_t wl2 = m.stack_cnt + (m.q_tail - m.q_head);
          const uint32_t want = min(32u, wl2);
          if (wn < ((LAZYW && !SAMU_K2_MULTI_EAGER) ? min(1u, want) : want)) {
            const uint32_t pos = ((uint32_t)lane - wb) & 31u;
            if (pos >= wn && pos < want) WIN_LOAD(pos);
            wn = want;
          }
          if (mm < 32) break;
        }
        m.F -= blk;
        if (GRP) W.minF = min(W.minF, m.F);
        K2STAT(2, 1);
        K2STAT(3, k_adm);
        // Eq. prefill FLOPs: L (c B s + 2 B h s^2 / tp)
        // = B s (L c + 2 L (h/tp) s): the same integer, fewer 64-bit products (B s < 2^24)
        const uint32_t Bs32 = k_adm * smaxp;
        const uint64_t fl = (LC + (uint64_t)K1_l * smaxp) * Bs32;
        const double lat = iter_cost(coef_l, k_adm, fl, Bs32, tok);
        m.t = __dadd_rn(m.t, lat);
        m.a1 += REQIT_CF ? Bs32 - k_adm : Bs32;   // (closed form: the decode part of a1 is reqit minus the prefills' B)
        m.a2 += (uint64_t)Bs32 * smaxp;
        if (!REQIT_CF) m.reqit += k_adm;
        m.iter += 1;
        m.F += freed;
        m.B += n_stay;
        m.S += S_add;
        m.next_rank += k_adm;
        if (n_stay && reduce_fo) {
          m.next_fin = __reduce_min_sync(FULL, lminf);
          m.maxO = __reduce_max_sync(FULL, lmaxo);
        }
        // Without a stop time or arrivals (modes 1, 2, 5, 6) the next iteration's choice needs
        // only the refilled window: when the new head does not fit, the decode follows in this
        // same pass (not when a successor released by this prefill could become the head)
#ifndef SAMU_K2_NO_MERGE
        if ((MODE == 1 || MODE == 2 || MODE == 5 || MODE == 6) && (LEAN || n_fin == 0) && m.B > 0) {
          const uint32_t wl3 = m.stack_cnt + (m.q_tail - m.q_head);
          const uint32_t hp3 = wl3 ? __shfl_sync(FULL, w_p, wb) : 0u;
          go_decode = !(wl3 > 0 && m.B < ms && hp3 <= C.budget && (int32_t)bs.cdiv(hp3) <= m.F);
        }
#endif
      }
      if (go_decode) {
        if (m.B == 0) { m.err = SAMU_E_INFEASIBLE; if (lane == 0) W.site = 9; break; }
        // ================= decode run (c9): uniform iterations until an event ===============
        const uint32_t need1 = W.hist[NEEDIDX];
        if (m.next_fin == m.d + 1 && (int32_t)need1 <= m.F) {
          K2STAT(6, 1);
          // one decode that retires requests and needs no preemption: the run below with
          // m_run = 1, without its search and closed forms (same arithmetic)
          const uint32_t B1 = m.B;
          const uint32_t smax = (uint32_t)((int32_t)m.d + m.maxO);
          const uint64_t fl = LC * B1 + (uint64_t)K1_l * m.S;
          m.t = __dadd_rn(m.t, iter_cost(coef_l, B1, fl, B1 * smax, m.S));
          if (!REQIT_CF) m.a1 += B1;
          m.a2 += m.S;
          if (!REQIT_CF) m.reqit += B1;
          m.F -= (int32_t)need1;
          if (GRP) W.minF = min(W.minF, m.F);
          m.S += B1;
          m.d += 1;
          if (BSK < 0) m.needidx = m.needidx == 0 ? bs.v() - 1 : m.needidx - 1;
        } else {
        K2STAT(7, 1);
        const uint32_t B = m.B;
        // no time limit and no arrivals in modes 1, 2, 5, 6: the stop time is a compile-time +inf
        const double stop_t = (MODE == 1 || MODE == 2 || MODE == 5 || MODE == 6) ? CUDART_INF : m.stop;
        // KV need of the run's decodes: histogram rotated to start at needidx, prefix sums
        const uint32_t m_fin = m.next_fin - m.d;
        uint32_t i_pre = 0x7fffffffu;   // first run iteration that must preempt
        uint32_t pre = 0, hv = 0;
        bool tight = true;
        if ((int32_t)need1 > m.F) {
          i_pre = 0;   // the first decode already preempts (KV thrash): no run, no search
        } else {
          hv = (uint32_t)lane < bs.v() ? W.hist[bs.mod(NEEDIDX + bs.v() - (uint32_t)lane)] : 0u;
          // each bs decodes need exactly B blocks: no search (and no scan) when the run cannot run out
          tight = (uint32_t)m.F < B * (bs.div(m_fin) + 1u);   // <= 256 * (65535 + 1): 32 bits
#ifndef SAMU_K2_NO_TIGHT2
          // (LEAN only: on the chain summariser's FRESH path most runs that fail the first test also
          // preempt, and the extra reduction measured slower)
          if (LEAN && tight) {
            // the exact need of the whole run (full cycles of B blocks + its first m_fin mod bs
            // phases) is non-decreasing in the decode count: no preemption if it fits
            const uint32_t rf = bs.mod(m_fin);
            tight = bs.div(m_fin) * B + __reduce_add_sync(FULL, (uint32_t)lane < rf ? hv : 0u) > (uint32_t)m.F;
          }
#endif
          if (tight) {
            // (only lanes below bs are read: a block size <= 16 needs a 16-lane scan)
            pre = (BSK > 0 && BSK <= 16) ? seg_incl_scan<16>(hv, lane) : warp_incl_scan(hv, lane);
            {
              const uint32_t F0 = (uint32_t)m.F;
              // q0 = F0 / B from an fp32 estimate corrected by the remainder (F0 < B (l_max / bs + 1)
              // here, so the estimate is within one of the quotient)
              uint32_t q0 = 0;
              int32_t rs = (int32_t)F0;
              if (F0 >= B) {   // (KV-bound runs mostly have fewer free blocks than requests)
                q0 = __float2uint_rz(__fdividef((float)F0, (float)B));
                rs = (int32_t)(F0 - q0 * B);
                while (rs < 0) { --q0; rs += (int32_t)B; }
                while (rs >= (int32_t)B) { ++q0; rs -= (int32_t)B; }
              }
              const uint32_t rem = (uint32_t)rs;
              const uint32_t bad = __ballot_sync(FULL, (uint32_t)lane < bs.v() && pre > rem);
              const uint64_t ip = (uint64_t)q0 * bs.v() + (uint32_t)(__ffs(bad) - 1);
              i_pre = ip > 0x7fffffffull ? 0x7fffffffu : (uint32_t)ip;
            }
          }
        }
        const uint32_t m_run = min(m_fin, i_pre);
        uint32_t done_it = 0;
        // run-length histogram (1, 2-4, 5-8, 9-16, 17-32, 33-64, 65-128, > 128), runs ending in a
        // preemption, runs that took the preemption search
        K2STAT(16 + (m_run <= 1 ? 0 : m_run <= 4 ? 1 : m_run <= 8 ? 2 : m_run <= 16 ? 3 : m_run <= 32 ? 4 : m_run <= 64 ? 5 : m_run <= 128 ? 6 : 7), 1);
        K2STAT(24, i_pre < m_fin ? 1 : 0);
        K2STAT(25, tight ? 1 : 0);
        if (m_run > 0) {
          const uint64_t K0 = LC * B;
          const uint32_t smax0 = (uint32_t)((int32_t)m.d + m.maxO);
          // (schedule sharing: the chunked sums run once per member while the iteration-by-
          // iteration path evaluates every member in its own lane at once, so the chunks pay off
          // only for runs ~nv times longer)
          const uint32_t chunk_min = GRP ? (uint32_t)SAMU_K2_CHUNK_GRP * W.nv : (uint32_t)SAMU_K2_CHUNK_MIN;
          if (m_run > chunk_min) {
            if (GRP) {
              // the chunked exact sums once per group member (lane v keeps member v's clock)
              const uint32_t nv = W.nv;
              for (uint32_t v = 0; v < nv; ++v) {
                const uint32_t civ = W.vci[v];
                const DevCand& Cv = CONSTC ? c_cands[civ] : P.cands[civ];
                double tv = __shfl_sync(FULL, m.t, v);
                done_it = run_chunks<MODE>(tv, Cv.coef, (uint32_t)Cv.K1, B, K0, m.S, smax0, m_run, stop_t, lane, W.cbuf);
                if ((uint32_t)lane == v) m.t = tv;
              }
            } else {
              double t = m.t;
              done_it = run_chunks<MODE>(t, C.coef, K1, B, K0, m.S, smax0, m_run, stop_t, lane, W.cbuf);
              m.t = t;
            }
          } else {
            // short runs: iteration by iteration (each lane its own member under GRP)
            const double2* cb = reinterpret_cast<const double2*>(coef_l + (size_t)(B - 1) * 8);
            const double2 cc = __ldg(cb), cp = __ldg(cb + 1), cs = __ldg(cb + 2);
            const double ac = cc.x, bc = cc.y, ap = cp.x, bp = cp.y, as_ = cs.x, bs_ = cs.y;
            double t = m.t;
            if (K0 + (uint64_t)K1_l * (m.S + B * (m_run - 1)) < (1ull << 53)) {
              // every x of the run is an integer below 2^53: exact fp64 increments == RN conversions
              double xc = (double)(K0 + (uint64_t)K1_l * m.S);
              const double dxc = (double)((uint64_t)K1_l * B), dB = (double)B;
              double xp = (double)(B * smax0), xs = (double)m.S;
              uint32_t jj = 0;
              do {
                const double tc = __fma_rn(ac, xc, bc);
                const double tp = __fma_rn(ap, xp, bp);
                const double ts = __fma_rn(as_, xs, bs_);
                t = __dadd_rn(t, __dadd_rn(__dadd_rn(tc, tp), ts));
                xc = __dadd_rn(xc, dxc);
                xp = __dadd_rn(xp, dB);
                xs = __dadd_rn(xs, dB);
                ++jj;
              } while (jj < m_run && t < stop_t);
              done_it = jj;
            } else {
              uint32_t jj = 0;
              do {
                const uint32_t S_j = m.S + B * jj;
                const double tc = __fma_rn(ac, __ull2double_rn(K0 + (uint64_t)K1_l * S_j), bc);
                const double tp = __fma_rn(ap, __uint2double_rn(B * (smax0 + jj)), bp);
                const double ts = __fma_rn(as_, __uint2double_rn(S_j), bs_);
                t = __dadd_rn(t, __dadd_rn(__dadd_rn(tc, tp), ts));
                ++jj;
              } while (jj < m_run && t < stop_t);
              done_it = jj;
            }
            m.t = t;
          }
          K2STAT(8, done_it);
          if (m_run > chunk_min) K2STAT(14, 1);
          // closed-form exact updates for the done_it iterations of the run
          // sum_j (K0 + K1 (S + B j)) = L c (B mm) + K1 (mm S + B mm (mm - 1) / 2); mm <= l_max < 2^16,
          // so mm (mm - 1) fits 32 bits and every product is one widening 32 x 32 multiply
          const uint32_t mm = done_it;
          const uint64_t Bmm = (uint64_t)B * mm;
          if (!REQIT_CF) m.a1 += Bmm;
          m.a2 += (uint64_t)mm * m.S + (uint64_t)B * ((mm * (mm - 1u)) >> 1);
          if (!REQIT_CF) m.reqit += Bmm;
          const uint32_t rr = bs.mod(done_it);
          const uint32_t need_rr = rr == 0 ? 0u
                                   : tight ? __shfl_sync(FULL, pre, rr - 1)
                                           : __reduce_add_sync(FULL, (uint32_t)lane < rr ? hv : 0u);
          const uint32_t need_sum = bs.div(done_it) * B + need_rr;
          m.F -= (int32_t)need_sum;
          if (GRP) W.minF = min(W.minF, m.F);
          m.S += B * done_it;
          m.d += done_it;
          if (BSK < 0) m.needidx = bs.mod(m.needidx + bs.v() - rr);
        }
        if (m.d != m.next_fin && done_it == i_pre && !(done_it > 0 && m.t >= stop_t)) {
          // ---- this decode must preempt (c7): recompute the last admitted requests ----
          uint32_t need = W.hist[NEEDIDX];
          if (GRP && (int32_t)need > m.F) W.minF = INT_MIN;
          while ((int32_t)need > m.F) {
            uint32_t vmeta;
            int ol, vs;
            if (m.next_rank < (1u << 23)) {
              // ranks are unique: key = (meta << 3 | j) + 1 names the slot of the lane's maximum
              uint32_t key = 0;
              if (COMPACT && __all_sync(FULL, occ <= 1u)) {   // compact: slot 0 only
                key = occ ? (W.s_meta[lane] << 3) + 1u : 0u;
              } else {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  const uint32_t kj = ((occ >> jj) & 1u) ? ((W.s_meta[lane + 32 * jj] << 3) | (uint32_t)jj) + 1u : 0u;
                  key = max(key, kj);
                }
              }
              const uint32_t vkey = __reduce_max_sync(FULL, key);
              ol = __ffs(__ballot_sync(FULL, key == vkey)) - 1;
              vs = ol + 32 * (int)((vkey - 1u) & 7u);
              vmeta = (vkey - 1u) >> 3;
            } else {
              uint32_t best = 0;
              int bslot = -1;
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const int s = lane + 32 * jj;
                if (((occ >> jj) & 1u) && (bslot < 0 || W.s_meta[s] > best)) { best = W.s_meta[s]; bslot = s; }
              }
              vmeta = __reduce_max_sync(FULL, bslot >= 0 ? best : 0u);
              const uint32_t own = __ballot_sync(FULL, bslot >= 0 && best == vmeta);
              ol = __ffs(own) - 1;
              vs = __shfl_sync(FULL, bslot, ol);
            }
            const uint32_t vr = W.s_req[vs];
            const int2 vfo = W.s_fo[vs];
            const uint32_t vph = vmeta & 31u;
            // recompute: prompt p = l_in + g = its current length l, still to generate (incl. the
            // recompute prefill's token) L - g = its finish index - d (> 0: it is not due now)
            const uint32_t l = (uint32_t)(vfo.y + (int32_t)m.d);
            const uint32_t vrem = (uint32_t)vfo.x - m.d;
            m.F += (int32_t)bs.cdiv(l - 1);
            if (vph == NEEDIDX) --need;
            __syncwarp();
            if (lane == ol) {
              occ &= ~(1u << (vs >> 5));
              W.hist[vph] -= 1;
              W.stk_req[m.stack_cnt] = vr;
              W.stk_pr[m.stack_cnt] = (l << 16) | vrem;
              // the lane's summaries change only if the victim held one of them
              if (occ == 0u) {
                lminf = FULL;
                lmaxo = INT_MIN;
              } else if ((uint32_t)vfo.x == lminf || vfo.y == lmaxo) {
                lminf = FULL;
                lmaxo = INT_MIN;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                  if ((occ >> jj) & 1u) {
                    const int2 fo = W.s_fo[lane + 32 * jj];
                    lminf = min(lminf, (uint32_t)fo.x);
                    lmaxo = max(lmaxo, fo.y);
                  }
              }
            }
            __syncwarp();
            // the victim is the new front of W: shift the window up by one
            wb = (wb - 1u) & 31u;   // a full window drops its last entry, the lane now at wb
            if ((uint32_t)lane == wb) { w_r = vr; w_p = l; w_rem = vrem; }
            wn = min(wn + 1, 32u);
            m.stack_cnt += 1;
            K2STAT(9, 1);
            m.B -= 1;
            m.S -= l;
            if (m.B == 0) { m.err = SAMU_E_INFEASIBLE; if (lane == 0) W.site = 10; break; }
          }
          if (m.err) break;
          m.next_fin = __reduce_min_sync(FULL, lminf);
          m.maxO = __reduce_max_sync(FULL, lmaxo);
          // the preempting decode iteration itself
          K2STAT(10, 1);
          const uint32_t B2 = m.B;
          const uint32_t smax = (uint32_t)((int32_t)m.d + m.maxO);
          m.F -= (int32_t)need;
          const uint64_t fl = LC * B2 + (uint64_t)K1_l * m.S;
          const double lat = iter_cost(coef_l, B2, fl, B2 * smax, m.S);
          m.t = __dadd_rn(m.t, lat);
          if (!REQIT_CF) m.a1 += B2;
          m.a2 += m.S;
          if (!REQIT_CF) m.reqit += B2;
          m.S += B2;
          m.d += 1;
          if (BSK < 0) m.needidx = m.needidx == 0 ? bs.v() - 1 : m.needidx - 1;
        }
        }
        if (m.d == m.next_fin) {
          // ---- retire the finishers (ballot / REDUX) ----
          const uint32_t inv = __ballot_sync(FULL, lminf == m.d);
          const uint32_t ninv = __popc(inv);
          K2STAT(11, 1);
          if (ninv <= 4) K2STAT(13, 1);
          uint32_t cnt_l = 0, sfin_l = 0;
          int32_t fr_l = 0;
          if (COMPACT && __all_sync(FULL, occ <= 1u)) {
            // compact: every lane holds at most its slot 0, whose finish index is lminf
            const bool fin = lminf == m.d;
            if (fin) {
              const uint32_t l_now = (uint32_t)(W.s_fo[lane].y + (int32_t)m.d);
              fr_l = (int32_t)bs.cdiv(l_now - 1);
              sfin_l = l_now;
              cnt_l = 1;
              atomicSub(&W.hist[W.s_meta[lane] & 31u], 1u);
              occ = 0;
              lminf = FULL;
              lmaxo = INT_MIN;
            }
            if (need_rel) {
              const uint32_t fb = __ballot_sync(FULL, fin);
              if (fin) W.tmp[__popc(fb & lanemask_lt())] = W.s_req[lane];
            }
          } else if (ninv <= 4) {
            // transposed scan: 8-lane group g reads the 8 slots of the g-th involved lane
            const int g = lane >> 3, jj = lane & 7;
            // one involved lane (common): its id is the ballot's only bit, no lane table
            uint32_t Lg;
            if (ninv == 1) {
              Lg = (uint32_t)(__ffs(inv) - 1);
            } else {
              if ((inv >> lane) & 1u) W.adm_req[__popc(inv & lanemask_lt())] = (uint32_t)lane;
              __syncwarp();
              Lg = (uint32_t)g < ninv ? W.adm_req[g] : 0u;
            }
            const uint32_t occ_g = __shfl_sync(FULL, occ, Lg);
            const bool has = (uint32_t)g < ninv && ((occ_g >> jj) & 1u);
            const int s = (int)Lg + 32 * jj;
            const int2 fo = has ? W.s_fo[s] : make_int2(0, 0);
            const bool fin = has && (uint32_t)fo.x == m.d;
            if (fin) {
              const uint32_t l_now = (uint32_t)(fo.y + (int32_t)m.d);
              fr_l = (int32_t)bs.cdiv(l_now - 1);
              sfin_l = l_now;
              cnt_l = 1;
              atomicSub(&W.hist[W.s_meta[s] & 31u], 1u);
            }
            const uint32_t fb = __ballot_sync(FULL, fin);
            if (need_rel && fin) W.tmp[__popc(fb & lanemask_lt())] = W.s_req[s];
            uint32_t mn = (has && !fin) ? (uint32_t)fo.x : FULL;
            int32_t mx = (has && !fin) ? fo.y : INT_MIN;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
              mn = min(mn, __shfl_xor_sync(FULL, mn, o));
              mx = max(mx, __shfl_xor_sync(FULL, mx, o));
            }
            // each involved lane takes its group's result
            const bool me = (inv >> lane) & 1u;
            const uint32_t gl = 8u * __popc(inv & lanemask_lt());
            const uint32_t mn_g = __shfl_sync(FULL, mn, me ? gl : 0u);
            const int32_t mx_g = __shfl_sync(FULL, mx, me ? gl : 0u);
            if (me) {
              lminf = mn_g;
              lmaxo = mx_g;
              occ &= ~((fb >> gl) & 0xFFu);
            }
          } else {
            uint32_t mn = FULL, cnt = 0, finm = 0;   // finm: this lane's finishing slots
            int32_t mx = INT_MIN;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              if ((occ >> jj) & 1u) {
                const int s = lane + 32 * jj;
                const int2 fo = W.s_fo[s];
                if ((uint32_t)fo.x == m.d) {
                  const uint32_t l_now = (uint32_t)(fo.y + (int32_t)m.d);
                  fr_l += (int32_t)bs.cdiv(l_now - 1);
                  sfin_l += l_now;
                  atomicSub(&W.hist[W.s_meta[s] & 31u], 1u);
                  occ &= ~(1u << jj);
                  finm |= 1u << jj;
                  ++cnt;
                } else {
                  mn = min(mn, (uint32_t)fo.x);
                  mx = max(mx, fo.y);
                }
              }
            }
            cnt_l = cnt;
            lminf = mn;
            lmaxo = mx;
            if (need_rel) {   // finished requests listed from their (not yet reused) slots
              uint32_t ex = warp_incl_scan(cnt, lane) - cnt;
              for (uint32_t f = finm; f; f &= f - 1) W.tmp[ex++] = W.s_req[lane + 32 * (__ffs(f) - 1)];
            }
          }
          if (BSK >= 16) {
            // freed blocks (<= 256 * ceil(65535 / 16) = 2^20) and the count (<= 256) in one word
            const uint32_t pk = __reduce_add_sync(FULL, ((uint32_t)fr_l << 9) | cnt_l);
            n_fin = pk & 0x1FFu;
            m.F += (int32_t)(pk >> 9);
          } else {
            n_fin = __reduce_add_sync(FULL, cnt_l);
            m.F += (int32_t)__reduce_add_sync(FULL, (uint32_t)fr_l);
          }
          K2STAT(12, n_fin);
          m.S -= __reduce_add_sync(FULL, sfin_l);
          m.B -= n_fin;
          m.next_fin = __reduce_min_sync(FULL, lminf);
          m.maxO = __reduce_max_sync(FULL, lmaxo);
          __syncwarp();
        }
      }
      // ---- finish records + chain successor release (c19), for this iteration's finishers ----
      if (!LEAN && n_fin && need_rel) {
        const uint32_t itx = m.iter + m.d - 1;   // iterations = prefills + decodes
        if (FRESH && n_fin == 1) {
          // one finisher (FRESH: no outputs): its successor, if any, joins the back of W
          const int32_t sr = SUCC_SLOT ? (int32_t)W.tmp[0] : (SUCC || C.has_succ) ? __ldg(A.succ + W.tmp[0]) : -1;
          if (sr >= 0) {
            if (lane == 0) q[m.q_tail] = (uint32_t)sr;
            m.q_tail += 1;
          }
          __syncwarp();
        } else if (n_fin <= 32) {
          // one finisher per lane; released successors ranked in registers (index order, c19)
          const bool v = (uint32_t)lane < n_fin;
          const uint32_t r = v ? W.tmp[lane] : 0u;
          int32_t sr = -1;
          if (v) {
            if (!FRESH) {
              if (!FRESH) {
                if (fio) fio[r] = itx;
                if (fto) fto[r] = m.t;
                if (commit) { st[r] = SAMU_ST_DONE << 28; ft[r] = m.t; }
              }
            }
            if (SUCC_SLOT) sr = (int32_t)r;
            else if (SUCC || C.has_succ) sr = __ldg(A.succ + r);
          }
          const uint32_t br = __ballot_sync(FULL, sr >= 0);
          if (br) {
            uint32_t rank = 0;
            for (uint32_t bb = br; bb; bb &= bb - 1) {   // rank among the released ids
              const int32_t x = __shfl_sync(FULL, sr, __ffs(bb) - 1);
              rank += (x < sr) ? 1u : 0u;
            }
            if (sr >= 0) q[m.q_tail + rank] = (uint32_t)sr;
            m.q_tail += __popc(br);
          }
          __syncwarp();   // the finisher list is rewritten by the next retirement
        } else {
          uint32_t nrel = 0;
          for (uint32_t base = 0; base < n_fin; base += 32) {
            const uint32_t i = base + lane;
            const bool v = i < n_fin;
            const uint32_t r = v ? W.tmp[i] : 0u;
            int32_t sr = -1;
            if (v) {
              if (!FRESH) {
                if (fio) fio[r] = itx;
                if (fto) fto[r] = m.t;
                if (commit) { st[r] = SAMU_ST_DONE << 28; ft[r] = m.t; }
              }
              if (SUCC_SLOT) sr = (int32_t)r;
              else if (SUCC || C.has_succ) sr = __ldg(A.succ + r);
            }
            // compacted in place: the k-th successor overwrites finisher slot <= k, already read
            // by every lane of this pass (the __syncwarp orders those reads before the writes)
            __syncwarp();
            const uint32_t br = __ballot_sync(FULL, sr >= 0);
            if (sr >= 0) W.tmp[nrel + __popc(br & lanemask_lt())] = (uint32_t)sr;
            nrel += __popc(br);
            __syncwarp();
          }
          if (nrel) {
            // append in index order: rank of each released id among the released set
            for (uint32_t i = lane; i < nrel; i += 32) {
              const uint32_t x = W.tmp[i];
              uint32_t rank = 0;
              for (uint32_t jj = 0; jj < nrel; ++jj) rank += W.tmp[jj] < x ? 1u : 0u;
              q[m.q_tail + rank] = x;
            }
            m.q_tail += nrel;
            __syncwarp();
          }
        }
      }
    }

    // ---- write back (commit) and the per-replica record ----
    const bool done = !m.err && m.B == 0 && m.stack_cnt == 0 && m.q_head == m.q_tail && W.pend_ptr == W.n_pend;
    if (m.err && lane == 0) set_error(P.error, m.err, W.site);
    if (commit && !m.err) {
      // running ranks renumbered 0..B-1 in admission order
      for (int s = lane; s < SLOTS; s += 32) W.tmp[s] = 0xFFFFFFFFu;
      __syncwarp();
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if ((occ >> jj) & 1u) W.tmp[lane + 32 * jj] = W.s_meta[lane + 32 * jj];
      __syncwarp();
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        if ((occ >> jj) & 1u) {
          const int s = lane + 32 * jj;
          const uint32_t rq = W.s_req[s];
          const uint32_t me = W.tmp[s];
          uint32_t rank = 0;
          for (int s2 = 0; s2 < SLOTS; ++s2) rank += W.tmp[s2] < me ? 1u : 0u;
          st[rq] = (SAMU_ST_RUNNING << 28) | rank;
          gst[rq] = (uint16_t)((uint32_t)(W.s_fo[s].y + (int32_t)m.d) - (uint32_t)LI_(rq));
        }
      }
      for (uint32_t i = lane; i < m.stack_cnt; i += 32) {
        const uint32_t rq = W.stk_req[i];
        st[rq] = (SAMU_ST_PREEMPTED << 28) | (m.stack_cnt - 1 - i);
        gst[rq] = (uint16_t)((W.stk_pr[i] >> 16) - (uint32_t)LI_(rq));
      }
      const uint32_t qbase = max(m.q_head, m.n_front + W.n_heads);
      for (uint32_t pos = m.q_head + lane; pos < m.q_tail; pos += 32) {
        const uint32_t rq = q[pos];
        if (pos < m.n_front) st[rq] = (SAMU_ST_PREEMPTED << 28) | (m.stack_cnt + pos - m.q_head);
        else if (pos < m.n_front + W.n_heads) gst[rq] = 0;
        else { st[rq] = (SAMU_ST_QUEUED << 28) | (pos - qbase); gst[rq] = 0; }
      }
      if (over && lane == 0) over[j] = (done || !cut) ? 0.0 : __dsub_rn(m.t, W.tau);
    }
    uint64_t reqit_cf = 0;
    if (REQIT_CF) {
      uint64_t sl = 0;
      for (uint32_t i = r0 + (uint32_t)lane; i < r1; i += 32) sl += max((uint32_t)LO_(__ldg(C.rep_req + i)), 1u);
      // in 24-bit digits (32 lanes x (2^24 - 1) fits a 32-bit reduction)
      reqit_cf = (uint64_t)__reduce_add_sync(FULL, (uint32_t)(sl & 0xFFFFFFu)) +
                 ((uint64_t)__reduce_add_sync(FULL, (uint32_t)((sl >> 24) & 0xFFFFFFu)) << 24) +
                 ((uint64_t)__reduce_add_sync(FULL, (uint32_t)(sl >> 48)) << 48);
    }
    // lane v < nv writes member v's record (lane 0 alone without groups), or queues the member's
    // item for a simulation of its own when its schedule would have differed from the head's
    const uint32_t nv = GRP ? W.nv : 1u;
    const uint32_t my_ci = GRP ? W.vci[lane] : ci;
    if ((uint32_t)lane < nv) {
      const bool in_sync = lane == 0 || W.minF >= C.blocks - (CONSTC ? c_cands[my_ci] : P.cands[my_ci]).blocks;
      if (in_sync) {
        samu_trial_rec rec;
        rec.t_end = m.t;
        {   // FLOPs = LC a1 + K1 a2 in u128
          const uint64_t a1 = REQIT_CF ? m.a1 + reqit_cf : m.a1;
          uint64_t lo = LC * a1, hi = __umul64hi(LC, a1);
          const uint64_t plo = (uint64_t)K1_l * m.a2, phi = __umul64hi((uint64_t)K1_l, m.a2);
          lo += plo;
          hi += phi + (lo < plo ? 1ull : 0ull);
          rec.flops_lo = lo;
          rec.flops_hi = hi;
        }
        rec.req_iters = REQIT_CF ? reqit_cf : m.reqit;
        rec.iters = m.iter + m.d;
        rec.flags = (done ? 1u : 0u) | (cut ? 2u : 0u) | (all_done ? 4u : 0u);
        P.rep_rec[((size_t)my_ci * P.n_trials + k) * 16 + j] = rec;
      } else if (GRP) {
        const uint32_t slot = atomicAdd(P.fb_ctr, 1u);
        atomicAdd(P.fb_count + my_ci, 1u);
        // one 64-bit store: a reader sees either the empty marker or the whole entry
        *reinterpret_cast<volatile unsigned long long*>(P.fb + slot) = (unsigned long long)my_ci | ((unsigned long long)rel << 32);
        __threadfence();
      }
    }
    __syncwarp();
}
#undef LO_
#undef LI_
#undef WIN_LOAD
#undef NEEDIDX
#undef K1_l
#undef coef_l

// Occupancy: 6 blocks of 4 warps per SM caps registers at 80 for 24 resident warps (C5 step
// 436 -> 418 ms against 5 blocks at 96 registers, once the cold state moved to shared memory;
// 7 blocks / 72 registers is slower, 16 warps at 128 registers slower still; see
// scripts/variants.sh).  SAMU_DEFINES overrides both.
#ifndef SAMU_K2_MINB
#define SAMU_K2_MINB 6
#endif
// FRESH launches without groups (modes 2, 4): their shared block fits 7 blocks too (28 warps at
// 72 registers: equal to 6 x 80 in round 1, -2 ms per C5 step once the window refills went lazy)
#ifndef SAMU_K2_MINB_FRESH
#define SAMU_K2_MINB_FRESH 7
#endif
// LEAN launches: 7 blocks (28 warps, 72 registers; the smaller shared block fits)
#ifndef SAMU_K2_MINB_LEAN
#define SAMU_K2_MINB_LEAN 7
#endif
// LEAN schedule-sharing launches (mode 5): the LEAN count unless overridden (experiments)
#ifndef SAMU_K2_MINB_GRP
#define SAMU_K2_MINB_GRP SAMU_K2_MINB_LEAN
#endif
// A launch holds only items of one MODE (DevCand::mode); the host issues one launch per mode
// present (one kernel holding several paths is slower: a multiple of the code footprint).
template <int BSK, bool CONSTC, int MODE>
// (the minimum block counts are per 4-warp block: the register caps stay the same for any block size)
__global__ void __launch_bounds__(32 * SAMU_WARPS_PER_BLOCK,
                                  (MODE == 5 ? SAMU_K2_MINB_GRP : is_lean(MODE) ? SAMU_K2_MINB_LEAN : (MODE == 2 || MODE == 4) ? SAMU_K2_MINB_FRESH
                                                                                    : SAMU_K2_MINB) * 4 / SAMU_WARPS_PER_BLOCK)
    k_simulate(SimLaunch P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // lane id kept in a register: an opaque copy cannot be rematerialised from SR_TID (an S2R
  // with ~20 cycles of latency) under register pressure (-1.3 % step time);
  int lane_v = threadIdx.x & 31;
  asm volatile("" : "+r"(lane_v));
  const int lane = lane_v;
  int warp_v = threadIdx.x >> 5;   // the same for the warp index, i.e. the warp's shared block (-3.3 %)
  asm volatile("" : "+r"(warp_v));
  const int warp = warp_v;
  WarpSmT<is_lean(MODE), (MODE == 5 || MODE == 6)>& W = reinterpret_cast<WarpSmT<is_lean(MODE), (MODE == 5 || MODE == 6)>*>(smem_raw)[warp];
  const int gw = blockIdx.x * SAMU_WARPS_PER_BLOCK + warp;
  uint32_t* q = P.scratch_q + (size_t)gw * P.max_q;
  uint64_t* pkey = P.scratch_key + (size_t)gw * 4 * P.max_p;
  uint32_t* pidx = P.scratch_idx + (size_t)gw * 4 * P.max_p;
  constexpr bool GRP = MODE == 5 || MODE == 6;
  const bool groups = GRP && P.grp != nullptr;
  for (;;) {
    // next work: a queued fallback item first (lane 0 claims it), else a static item.  A warp that
    // queued fallbacks comes back here after its item, so no queued entry is ever left without a
    // warp to claim it: nobody waits for the others to finish
    uint32_t kind = 1, item = 0, fb_ci = 0;
    if (lane == 0) {
      bool got = false;
      if (groups) {
        volatile uint32_t* ctr = P.fb_ctr;
        uint32_t f = ctr[1];
        while (f < ctr[0]) {
          const uint32_t old = atomicCAS(P.fb_ctr + 1, f, f + 1);
          if (old == f) { got = true; break; }
          f = old;
        }
        if (got) {   // allocated entries are written right after their allocation
          unsigned long long e;
          do { e = *reinterpret_cast<volatile unsigned long long*>(P.fb + f); } while ((uint32_t)e == SAMU_EMPTY);
          kind = 2; fb_ci = (uint32_t)e; item = (uint32_t)(e >> 32);
        }
      }
      if (!got) {
        item = atomicAdd(P.next_item, 1u);
        kind = item < (uint32_t)P.n_items ? 1u : 0u;
      }
    }
    kind = __shfl_sync(FULL, kind, 0);
    if (kind == 0) break;
    item = __shfl_sync(FULL, item, 0);
    uint32_t ci, rel;
    uint4 grp = make_uint4(1u, 0u, 0u, 0u);
    if (kind == 2) {   // fallback: a member simulated on its own (item = index within the candidate)
      ci = __shfl_sync(FULL, fb_ci, 0);
      rel = item;
    } else {
      // decode the item: candidate (group head) by binary search over the launch's offsets
      uint32_t lo_x = 0, hi_x = (uint32_t)P.n_ord;   // off[lo_x] <= item < off[hi_x]
      while (hi_x - lo_x > 1) {
        const uint32_t mid = (lo_x + hi_x) >> 1;
        if (__ldg(P.off + mid) <= item) lo_x = mid; else hi_x = mid;
      }
      ci = __ldg(P.ord + lo_x);
      rel = item - __ldg(P.off + lo_x);
      if (groups) grp = __ldg(P.grp + lo_x);
    }
    sim_item<BSK, CONSTC, MODE>(P, W, lane, q, pkey, pidx, ci, rel, grp);
  }
  // Programmatic dependent launch (launches of one batch in one stream): this warp has no more
  // work, so the next K2 launch may start its blocks on the SM resources this launch frees while
  // its last items run; that launch does not read this one's results.  Before exiting, a block
  // waits for the previous launch of the chain to complete, so the completion of the last launch
  // implies the completion of them all (the combine kernel after them is an ordinary launch).
  // Both are no-ops for a launch without the programmatic-serialization attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

int32_t simulate_smem_bytes(int mode) {
  const size_t b = mode == 5 ? sizeof(WarpSmT<true, true>) : mode == 6 ? sizeof(WarpSmT<false, true>)
                 : is_lean(mode) ? sizeof(WarpSmT<true, false>) : sizeof(WarpSmT<false, false>);
  return (int32_t)(b * SAMU_WARPS_PER_BLOCK);
}

template <int BSK, bool CONSTC, int MODE>
static cudaError_t prepare_one(int* bpsm_modes) {
  const int smem = simulate_smem_bytes(MODE);
  int* bpsm = bpsm_modes + MODE;
  cudaError_t e = cudaFuncSetAttribute(k_simulate<BSK, CONSTC, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int a = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_simulate<BSK, CONSTC, MODE>, 32 * SAMU_WARPS_PER_BLOCK, smem);
  *bpsm = *bpsm < a ? *bpsm : a;
  return e;
}

// resident blocks per SM for each K2 mode (the minimum over that mode's instantiations)
cudaError_t simulate_prepare(int blocks_per_sm[SAMU_K2_MODES]) {
  for (int md = 0; md < SAMU_K2_MODES; ++md) blocks_per_sm[md] = 1 << 30;
  cudaError_t e;
  if ((e = prepare_one<16, true, 0>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 1>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 2>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 3>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 4>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 5>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, true, 6>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 5>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 6>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 3>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 4>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 0>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 1>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<16, false, 2>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<0, true, 0>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<0, false, 0>(blocks_per_sm)) != cudaSuccess) return e;
  if ((e = prepare_one<-1, true, 0>(blocks_per_sm)) != cudaSuccess) return e;
  return prepare_one<-1, false, 0>(blocks_per_sm);
}

template <int BSK, bool CONSTC, int MODE>
static cudaError_t launch_one(const SimLaunch& L, int32_t n_blocks, int smem, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_blocks);
  cfg.blockDim = dim3(32 * SAMU_WARPS_PER_BLOCK);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_simulate<BSK, CONSTC, MODE>, L);
}

template <bool CONSTC>
static cudaError_t launch_variant(const SimLaunch& L, uint32_t block_size, int mode, int32_t n_blocks, int smem,
                                  cudaStream_t s, bool pdl) {
  if (block_size == 16 && mode == 1) return launch_one<16, CONSTC, 1>(L, n_blocks, smem, s, pdl);
  if (block_size == 16 && mode == 2) return launch_one<16, CONSTC, 2>(L, n_blocks, smem, s, pdl);
  if (block_size == 16 && mode == 3) return launch_one<16, CONSTC, 3>(L, n_blocks, smem, s, pdl);
  if (block_size == 16 && mode == 4) return launch_one<16, CONSTC, 4>(L, n_blocks, smem, s, pdl);
  if (block_size == 16 && mode == 5) return launch_one<16, CONSTC, 5>(L, n_blocks, smem, s, pdl);
  if (block_size == 16 && mode == 6) return launch_one<16, CONSTC, 6>(L, n_blocks, smem, s, pdl);
  if (block_size == 16) return launch_one<16, CONSTC, 0>(L, n_blocks, smem, s, pdl);
  if ((block_size & (block_size - 1)) == 0) return launch_one<0, CONSTC, 0>(L, n_blocks, smem, s, pdl);
  return launch_one<-1, CONSTC, 0>(L, n_blocks, smem, s, pdl);
}

// Launch the K2 kernels of one simulate batch, one per mode present (Ls[i] / modes[i] / n_blocks[i]).
// General and FRESH launches share the per-warp scratch and run in order on s; a LEAN launch uses
// no scratch and runs concurrently on s2 (forked after the table copy, joined back into s), so
// its items fill the SMs beside the long chain replica-sims of a FRESH launch instead of after
// them (the FRESH launch's longest item is its critical path at small trial shares).
cudaError_t launch_simulate(const SimLaunch* Ls, const int* modes, const int32_t* n_blocks, int n_launch,
                            const DevCand* host_cands, uint32_t block_size, cudaStream_t s, cudaStream_t s2,
                            cudaEvent_t ev_fork, cudaEvent_t ev_join) {
  if (n_launch == 0) return cudaSuccess;
  const bool constc = Ls[0].n_cands <= SAMU_K2_CONST_CANDS;
  // The constant table is one per device and process while contexts may launch on their own
  // streams: the copy waits for the previous table user (any stream) and this batch becomes the
  // next (host mutex: copy + launches + event record are one unit).
  static std::mutex mu;
  static cudaEvent_t last[64] = {};
  std::unique_lock<std::mutex> lock(mu, std::defer_lock);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (constc) {
    lock.lock();
    if (!last[dev] && (e = cudaEventCreateWithFlags(&last[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, last[dev], 0)) != cudaSuccess) return e;
    e = cudaMemcpyToSymbolAsync(c_cands, host_cands, sizeof(DevCand) * (size_t)Ls[0].n_cands, 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
  }
  // the LEAN launches without a time limit (modes 1 and 5) may run on the auxiliary stream
  int n_lean = 0, n_other = 0;
  for (int i = 0; i < n_launch; ++i) (modes[i] == 1 || modes[i] == 5 ? n_lean : n_other) += 1;
  const bool fork = n_lean > 0 && n_other > 0 && s2 != nullptr;
  if (fork) {   // s2 starts after the table copy (and everything before it on s)
    if ((e = cudaEventRecord(ev_fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s2, ev_fork, 0)) != cudaSuccess) return e;
  }
  // serialized launches (one stream): a launch may start beside the tail of the previous one
  // (programmatic dependent launch) unless both use the per-warp scratch rings, which are indexed
  // by the warp's position in its grid (the general / FRESH modes 0, 2, 4, 6)
  static const bool pdl_on = !std::getenv("SAMU_K2_PDL") || std::atoi(std::getenv("SAMU_K2_PDL")) != 0;
  auto scratch = [](int md) { return md == 0 || md == 2 || md == 4 || md == 6; };
  for (int i = 0; i < n_launch; ++i) {
    const bool on_aux = fork && (modes[i] == 1 || modes[i] == 5);
    const int smem = simulate_smem_bytes(modes[i]);
    cudaStream_t st = on_aux ? s2 : s;
    const bool pdl = pdl_on && !fork && i > 0 && !(scratch(modes[i]) && scratch(modes[i - 1]));
    e = constc ? launch_variant<true>(Ls[i], block_size, modes[i], n_blocks[i], smem, st, pdl)
               : launch_variant<false>(Ls[i], block_size, modes[i], n_blocks[i], smem, st, pdl);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (fork) {
    if ((e = cudaEventRecord(ev_join, s2)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, ev_join, 0)) != cudaSuccess) return e;
  }
  if (constc) return cudaEventRecord(last[dev], s);
  return cudaSuccess;
}
