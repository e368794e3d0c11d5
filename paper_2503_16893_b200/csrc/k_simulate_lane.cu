// K2L: iteration-level continuous-batching simulation, one LANE per (candidate, trial, dp
// replica) — same semantics as K2 (k_simulate.cu; readings c3-c9, c13,
// c15, c19, c23-c25), for batches that start from a fresh WorkloadState and have no cross-node
// arrivals (the first greedy inner step, every full / cut simulation of a fresh stage, the bench).
//
// Why lanes: in warp-per-simulation every scalar of the simulation (clock, B, S, latency chain,
// event bookkeeping) is executed redundantly by 32 lanes and each event costs hundreds of
// warp-instructions.  Here 32 simulations advance per warp-instruction:
//  * running set per lane: slots {o = l - d, request, admission rank | running bit} and a 4-ary
//    min-heap of (finish decode index, rank, slot) in a per-lane global scratch block (L1/L2
//    resident); preempted victims are deleted lazily (heap entries are validated by rank);
//  * the KV-block phase histogram (reading c9: need of decode d = #{phase == (-d) mod bs}) is kept
//    in registers as 9 bit-sliced counters over <= 32 bins, so the need of a decode, the need of a
//    whole run and the first decode that must preempt are popcounts;
//  * max(l - d) comes from a top-4 cache in registers, rebuilt by a slot scan only when emptied;
//  * decode runs are identical to K2 (fp64 latency per iteration, exact closed-form integer sums).
#include "samu_internal.cuh"

#include <math_constants.h>

namespace {

constexpr uint32_t FULLM = 0xFFFFFFFFu;
constexpr uint32_t RUNBIT = 0x80000000u;
constexpr int HCAP = 512;   // heap capacity (256 live + lazily deleted victims)

struct LaneMem {
  unsigned long long heap[HCAP];   // fin << 32 | (rank & 0xFFFFFF) << 8 | slot
  int32_t s_o[256];
  uint32_t s_req[256];
  uint32_t s_rank[256];            // admission rank | RUNBIT while running
  uint32_t stk_req[256];
  uint32_t stk_g[256];
  uint8_t free_list[256];
};

template <bool POW2>
struct BsL {
  uint32_t v, mask, shift;
  __device__ __forceinline__ uint32_t mod(uint32_t x) const { return POW2 ? (x & mask) : x % v; }
  __device__ __forceinline__ uint32_t div(uint32_t x) const { return POW2 ? (x >> shift) : x / v; }
  __device__ __forceinline__ uint32_t cdiv(uint32_t x) const { return div(x + v - 1); }
  __device__ __forceinline__ uint32_t posmod(int32_t a) const {
    if (POW2) return (uint32_t)a & mask;
    const int32_t r = a % (int32_t)v;
    return (uint32_t)(r < 0 ? r + (int32_t)v : r);
  }
};

// 9 bit-sliced counters (<= 511 per bin) over up to 32 phase bins
struct Hist {
  uint32_t s[9];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int k = 0; k < 9; ++k) s[k] = 0;
  }
  __device__ __forceinline__ void inc(uint32_t bin) {
    uint32_t c = 1u << bin;
#pragma unroll
    for (int k = 0; k < 9; ++k) { const uint32_t n = s[k] ^ c; c &= s[k]; s[k] = n; }
  }
  __device__ __forceinline__ void dec(uint32_t bin) {
    uint32_t b = 1u << bin;
#pragma unroll
    for (int k = 0; k < 9; ++k) { const uint32_t n = s[k] ^ b; b &= ~s[k]; s[k] = n; }
  }
  __device__ __forceinline__ uint32_t count(uint32_t m) const {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) r += (uint32_t)__popc(s[k] & m) << k;
    return r;
  }
};

// bins visited by the next `len` (< bs) decodes starting at needidx: needidx, needidx-1, ... (mod bs)
__device__ __forceinline__ uint32_t window_mask(uint32_t needidx, uint32_t len, uint32_t bs) {
  if (len == 0) return 0u;
  if (len >= bs) return bs == 32 ? FULLM : ((1u << bs) - 1u);
  // bins [needidx - len + 1, needidx] mod bs
  const int32_t lo = (int32_t)needidx - (int32_t)len + 1;
  uint32_t m;
  if (lo >= 0) m = ((len == 32 ? FULLM : ((1u << len) - 1u)) << lo);
  else {
    const uint32_t hi_part = (needidx + 1 == 32) ? FULLM : ((1u << (needidx + 1)) - 1u);
    const uint32_t wrap = (uint32_t)(-lo);   // bins bs - wrap .. bs - 1
    m = hi_part | (((1u << wrap) - 1u) << (bs - wrap));
  }
  return m;
}

__device__ __forceinline__ double lane_iter_cost(const double* __restrict__ coef, uint32_t ms, uint32_t B, uint64_t F,
                                                 uint32_t Bs_, uint32_t S) {
  const double* cb = coef + (B - 1);
  const double tc = __fma_rn(__ldg(cb), __ull2double_rn(F), __ldg(cb + ms));
  const double tp = __fma_rn(__ldg(cb + 2 * ms), __uint2double_rn(Bs_), __ldg(cb + 3 * ms));
  const double ts = __fma_rn(__ldg(cb + 4 * ms), __uint2double_rn(S), __ldg(cb + 5 * ms));
  return __dadd_rn(__dadd_rn(tc, tp), ts);
}

}  // namespace

// ---------------------------------------------------------------------------------------------
template <bool POW2>
__global__ void __launch_bounds__(128) k_simulate_lane(SimLaunch P, LaneMem* __restrict__ mem) {
  const uint32_t gl = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  LaneMem& M = mem[gl];
  const DevApp& A = P.app;
  const int n = A.n_req;
  bool have = false;
  uint32_t item = 0;

  for (;;) {
    // warp-aggregated work fetch: one atomic per warp for all lanes that need an item
    const uint32_t need = __ballot_sync(FULLM, !have);
    if (need) {
      uint32_t base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(P.next_item, (uint32_t)__popc(need));
      base = __shfl_sync(FULLM, base, leader);
      if (!have) {
        item = base + (uint32_t)__popc(need & ((1u << lane) - 1u));
        have = true;
      }
    }
    const bool live = have && item < (uint32_t)P.n_items;
    if (!__any_sync(FULLM, live)) break;
    if (!live) {   // this lane is out of work: idle while the others finish
      have = true;
      item = 0xFFFFFFFFu;
      continue;
    }

    const uint2 it = P.items[item];
    const uint32_t ci = it.x, k = it.y >> 4, j = it.y & 15u;
    const DevCand& C = P.cands[ci];
    const size_t tb = (size_t)k * n;
    const uint16_t* __restrict__ lo = P.l_out + tb;
    const uint16_t* __restrict__ li = P.l_in + tb;
    double* fto = C.fin_t_out ? C.fin_t_out + tb : nullptr;
    uint32_t* fio = C.fin_iter_out ? C.fin_iter_out + tb : nullptr;
    const uint32_t ms = C.max_seqs;
    BsL<POW2> bs;
    bs.v = C.bs;
    bs.mask = C.bs - 1;
    bs.shift = __ffs(C.bs) - 1;
    const uint64_t K1 = 2ull * C.L * C.h_tp;
    const uint64_t LC = (uint64_t)C.L * C.c;
    // W = [preempted stack] + [never-started heads of this replica, index order] + [released
    // chain successors in (release time, index) order, per-item tail region]
    const uint32_t* heads = C.head_req + C.head_off[j];
    uint32_t hd = 0;
    const uint32_t hd_end = C.head_off[j + 1] - C.head_off[j];
    uint32_t* tail = C.has_succ ? P.scratch_q + P.tail_off[item] : nullptr;
    uint32_t tl_head = 0, tl_tail = 0;

    double t = C.load_s;
    const double tau = C.tau ? C.tau[k] : (C.tau_rec ? C.tau_rec[k].t_end : CUDART_INF);
    uint64_t fl_lo = 0, fl_hi = 0, reqit = 0;
    uint32_t iters = 0, d = 0, needidx = 0, B = 0, S = 0, next_rank = 0, stack_cnt = 0, hn = 0;
    uint32_t nfree = 0, hw = 0;   // recycled slots / high-water mark of slots ever used
    int32_t F = C.blocks;
    Hist hist;
    hist.clear();
    // top-4 cache of o = l - d among running requests; invariant: every running o outside the
    // cache is <= min(cache) (the cache is rebuilt by a slot scan when it empties)
    int32_t top[4];
    uint32_t topslot[4];
    uint32_t ntop = 0;
    bool cut = false;
    int32_t err = 0;

    auto add_fl = [&](uint64_t f) {
      const uint64_t l2 = fl_lo + f;
      fl_hi += (l2 < fl_lo) ? 1ull : 0ull;
      fl_lo = l2;
    };
    // entry i of W: (request, p = l_in + g, tokens still to generate incl. the prefill's)
    auto peek = [&](uint32_t i, uint32_t& r, uint32_t& p, uint32_t& rem) -> bool {
      uint32_t g = 0;
      if (i < stack_cnt) { r = M.stk_req[stack_cnt - 1 - i]; g = M.stk_g[stack_cnt - 1 - i]; }
      else {
        i -= stack_cnt;
        if (hd + i < hd_end) r = __ldg(heads + hd + i);
        else {
          i -= hd_end - hd;
          if (tl_head + i < tl_tail) r = tail[tl_head + i];
          else return false;
        }
      }
      p = (uint32_t)li[r] + g;
      rem = max((uint32_t)lo[r], 1u) - g;
      return true;
    };
    auto pop_head = [&]() {
      if (stack_cnt) --stack_cnt;
      else if (hd < hd_end) ++hd;
      else ++tl_head;
    };
    auto heap_push = [&](unsigned long long key) {
      uint32_t i = hn++;
      while (i > 0) {
        const uint32_t pa = (i - 1) >> 2;
        const unsigned long long pk = M.heap[pa];
        if (pk <= key) break;
        M.heap[i] = pk;
        i = pa;
      }
      M.heap[i] = key;
    };
    auto heap_pop = [&]() {
      const unsigned long long last = M.heap[--hn];
      uint32_t i = 0;
      for (;;) {
        const uint32_t c0 = 4 * i + 1;
        if (c0 >= hn) break;
        uint32_t mc = c0;
        unsigned long long mk = M.heap[c0];
#pragma unroll
        for (int q = 1; q < 4; ++q) {
          if (c0 + q < hn) {
            const unsigned long long kq = M.heap[c0 + q];
            if (kq < mk) { mk = kq; mc = c0 + q; }
          }
        }
        if (mk >= last) break;
        M.heap[i] = mk;
        i = mc;
      }
      if (hn) M.heap[i] = last;
    };
    auto entry_live = [&](unsigned long long kk) -> bool {
      const uint32_t sr = M.s_rank[(uint32_t)(kk & 0xFFu)];
      return (sr & RUNBIT) && (sr & 0xFFFFFFu) == ((uint32_t)(kk >> 8) & 0xFFFFFFu);
    };
    // drop lazily-deleted (preempted) entries from the top of the heap
    auto heap_clean = [&]() {
      while (hn && !entry_live(M.heap[0])) heap_pop();
    };
    auto heap_compact = [&]() {   // remove every deleted entry and re-heapify (rare)
      uint32_t w2 = 0;
      for (uint32_t i = 0; i < hn; ++i) if (entry_live(M.heap[i])) M.heap[w2++] = M.heap[i];
      hn = 0;
      for (uint32_t i = 0; i < w2; ++i) heap_push(M.heap[i]);   // in-place: pushes read entries < i
    };
    auto top_insert = [&](int32_t o, uint32_t s, uint32_t running_before) {
      if (ntop == 0) {
        if (running_before == 0) { top[0] = o; topslot[0] = s; ntop = 1; }
        return;
      }
      uint32_t mi = 0;
      for (uint32_t q = 1; q < ntop; ++q) if (top[q] < top[mi]) mi = q;
      if (o <= top[mi]) return;
      if (ntop < 4) { top[ntop] = o; topslot[ntop] = s; ++ntop; }
      else { top[mi] = o; topslot[mi] = s; }
    };
    auto top_remove = [&](uint32_t s) {
      for (uint32_t q = 0; q < ntop; ++q)
        if (topslot[q] == s) { top[q] = top[ntop - 1]; topslot[q] = topslot[ntop - 1]; --ntop; break; }
    };
    auto top_rebuild = [&]() {   // full scan of the running slots (only when the cache empties)
      ntop = 0;
      for (uint32_t s = 0; s < hw; ++s) {
        if (!(M.s_rank[s] & RUNBIT)) continue;
        const int32_t o = M.s_o[s];
        if (ntop < 4) { top[ntop] = o; topslot[ntop] = s; ++ntop; }
        else {
          uint32_t mi = 0;
          for (uint32_t q = 1; q < 4; ++q) if (top[q] < top[mi]) mi = q;
          if (o > top[mi]) { top[mi] = o; topslot[mi] = s; }
        }
      }
    };
    auto max_o = [&]() -> int32_t {
      int32_t mx = INT_MIN;
      for (uint32_t q = 0; q < ntop; ++q) mx = max(mx, top[q]);
      return mx;
    };
    // a finished request: records + chain successor staged at the tail (c19)
    uint32_t nrel = 0;
    auto finished = [&](uint32_t r) {
      if (fio) fio[r] = iters - 1;
      if (fto) fto[r] = t;
      if (C.has_succ) {
        const int32_t sr = __ldg(A.succ + r);
        if (sr >= 0) tail[tl_tail + nrel++] = (uint32_t)sr;
      }
    };
    auto flush_rel = [&]() {   // released successors of one iteration join W in index order
      for (uint32_t a = 1; a < nrel; ++a) {
        const uint32_t x = tail[tl_tail + a];
        uint32_t b = a;
        while (b > 0 && tail[tl_tail + b - 1] > x) { tail[tl_tail + b] = tail[tl_tail + b - 1]; --b; }
        tail[tl_tail + b] = x;
      }
      tl_tail += nrel;
      nrel = 0;
    };

    // ---- main loop (c25) ----
    for (;;) {
      if (t >= tau) { cut = true; break; }
      uint32_t hr = 0, hp = 0, hrem = 0;
      const bool wnon = peek(0, hr, hp, hrem);
      if (B == 0 && !wnon) break;
      const bool fits = wnon && B < ms && hp <= C.budget && (int32_t)bs.cdiv(hp) <= F;
      if (fits) {
        // ===== prefill iteration (c8): strict FCFS prefix of W =====
        // pass 1: the admitted prefix and the iteration's (B, s, S)
        uint32_t k_adm = 0, tok = 0, smaxp = 0;
        int32_t blk = 0;
        {
          uint32_t r = hr, p = hp, rem = hrem;
          bool ok = true;
          while (ok) {
            const uint32_t nb = bs.cdiv(p);
            if (B + k_adm + 1 > ms || tok + p > C.budget || blk + (int32_t)nb > F) break;
            tok += p;
            blk += (int32_t)nb;
            smaxp = max(smaxp, p);
            ++k_adm;
            ok = peek(k_adm, r, p, rem);
          }
        }
        F -= blk;
        const uint64_t Bp = k_adm, sp64 = smaxp;
        const uint64_t fl = LC * Bp * sp64 + (uint64_t)C.L * 2ull * Bp * C.h_tp * sp64 * sp64;
        const double lat = lane_iter_cost(C.coef, ms, k_adm, fl, k_adm * smaxp, tok);
        t = __dadd_rn(t, lat);
        add_fl(fl);
        reqit += k_adm;
        iters += 1;
        // pass 2: pop the admitted requests; the prefill emits one token each
        const uint32_t B0 = B;
        for (uint32_t a = 0; a < k_adm; ++a) {
          uint32_t r, p, rem;
          peek(0, r, p, rem);
          pop_head();
          const uint32_t rank = next_rank + a;
          if (rem <= 1u) {   // finishes in this prefill (c3: at least one token)
            F += (int32_t)bs.cdiv(p);
            finished(r);
          } else {
            const uint32_t s = nfree ? (uint32_t)M.free_list[--nfree] : hw++;
            const int32_t o = (int32_t)(p + 1) - (int32_t)(d);
            M.s_o[s] = o;
            M.s_req[s] = r;
            M.s_rank[s] = (rank & 0xFFFFFFu) | RUNBIT;
            if (hn == HCAP) heap_compact();
            heap_push(((unsigned long long)(d + rem - 1) << 32) | ((unsigned long long)(rank & 0xFFFFFFu) << 8) | s);
            hist.inc(bs.posmod((int32_t)p - (int32_t)d));
            top_insert(o, s, B);
            S += p + 1;
            ++B;
          }
        }
        (void)B0;
        next_rank += k_adm;
        if (nrel) flush_rel();
      } else {
        if (B == 0) { err = SAMU_E_INFEASIBLE; break; }
        // ===== decode run (c9) =====
        heap_clean();
        const uint32_t next_fin = (uint32_t)(M.heap[0] >> 32);
        const uint32_t m_fin = next_fin - d;
        const double stop_t = tau;
        // first run iteration whose cumulative KV need exceeds F (bit-sliced histogram)
        uint32_t i_pre = 0x7fffffffu;
        if ((uint64_t)(uint32_t)F < (uint64_t)B * ((uint64_t)bs.div(m_fin) + 1)) {
          const uint32_t q0 = (uint32_t)F / B, rm = (uint32_t)F - q0 * B;
          // smallest len in [1, bs] with count(window(len)) > rm  (window(bs) counts B > rm)
          uint32_t lo_l = 1, hi_l = bs.v;
          while (lo_l < hi_l) {
            const uint32_t mid = (lo_l + hi_l) >> 1;
            if (hist.count(window_mask(needidx, mid, bs.v)) > rm) hi_l = mid; else lo_l = mid + 1;
          }
          const uint64_t ip = (uint64_t)q0 * bs.v + (lo_l - 1);
          i_pre = ip > 0x7fffffffull ? 0x7fffffffu : (uint32_t)ip;
        }
        const uint32_t m_run = min(m_fin, i_pre);
        uint32_t done_it = 0;
        if (m_run > 0) {
          const uint64_t K0 = LC * B;
          const uint32_t smax0 = (uint32_t)((int32_t)d + max_o());
          const double* cb = C.coef + (B - 1);
          const double ac = __ldg(cb), bc = __ldg(cb + ms), ap = __ldg(cb + 2 * ms), bp = __ldg(cb + 3 * ms);
          const double as_ = __ldg(cb + 4 * ms), bs_ = __ldg(cb + 5 * ms);
          const uint64_t f_last = K0 + K1 * ((uint64_t)S + (uint64_t)B * (m_run - 1));
          double tt = t;
          if (f_last < (1ull << 53)) {
            // every x of the run is an integer below 2^53: exact fp64 increments == RN conversions
            double xc = (double)(K0 + K1 * (uint64_t)S);
            const double dxc = (double)(K1 * B), dB = (double)B;
            double xp = (double)((uint64_t)B * smax0), xs = (double)S;
            uint32_t jj = 0;
            do {
              const double tc = __fma_rn(ac, xc, bc);
              const double tp = __fma_rn(ap, xp, bp);
              const double ts = __fma_rn(as_, xs, bs_);
              tt = __dadd_rn(tt, __dadd_rn(__dadd_rn(tc, tp), ts));
              xc = __dadd_rn(xc, dxc);
              xp = __dadd_rn(xp, dB);
              xs = __dadd_rn(xs, dB);
              ++jj;
            } while (jj < m_run && tt < stop_t);
            done_it = jj;
          } else {
            uint32_t jj = 0;
            do {
              const uint64_t S_j = (uint64_t)S + (uint64_t)B * jj;
              const double tc = __fma_rn(ac, __ull2double_rn(K0 + K1 * S_j), bc);
              const double tp = __fma_rn(ap, __ull2double_rn((uint64_t)B * (smax0 + jj)), bp);
              const double ts = __fma_rn(as_, __ull2double_rn(S_j), bs_);
              tt = __dadd_rn(tt, __dadd_rn(__dadd_rn(tc, tp), ts));
              ++jj;
            } while (jj < m_run && tt < stop_t);
            done_it = jj;
          }
          t = tt;
          const uint64_t mm = done_it;
          const uint64_t inner = mm * (uint64_t)S + (uint64_t)B * (mm * (mm - 1) / 2);
          if (f_last < (1ull << 53) && mm < 2048ull) add_fl(mm * K0 + K1 * inner);
          else {
            uint64_t lo64 = mm * K0, hi64 = __umul64hi(mm, K0);
            const uint64_t plo = K1 * inner, phi = __umul64hi(K1, inner);
            lo64 += plo;
            hi64 += phi + (lo64 < plo ? 1ull : 0ull);
            const uint64_t nlo = fl_lo + lo64;
            fl_hi += hi64 + (nlo < lo64 ? 1ull : 0ull);
            fl_lo = nlo;
          }
          reqit += (uint64_t)B * mm;
          iters += done_it;
          const uint32_t rr = bs.mod(done_it);
          const uint32_t need_sum = bs.div(done_it) * B + hist.count(window_mask(needidx, rr, bs.v));
          F -= (int32_t)need_sum;
          S += B * done_it;
          d += done_it;
          needidx = bs.mod(needidx + bs.v - rr);
        }
        if (d != next_fin && done_it == i_pre && !(done_it > 0 && t >= stop_t)) {
          // ---- this decode must preempt the last admitted requests (c7) ----
          uint32_t needd = hist.count(1u << needidx);
          while ((int32_t)needd > F) {
            uint32_t vs = 0, vrank = 0;
            bool found = false;
            for (uint32_t s = 0; s < hw; ++s) {
              const uint32_t sr = M.s_rank[s];
              if ((sr & RUNBIT) && (!found || (sr & 0xFFFFFFu) > vrank)) { vrank = sr & 0xFFFFFFu; vs = s; found = true; }
            }
            const int32_t vo = M.s_o[vs];
            const uint32_t vr = M.s_req[vs];
            const uint32_t l = (uint32_t)(vo + (int32_t)d);
            const uint32_t ph = bs.posmod(vo - 1);
            F += (int32_t)bs.cdiv(l - 1);
            if (ph == needidx) --needd;
            hist.dec(ph);
            M.s_rank[vs] = 0;                       // its heap entry is deleted lazily
            M.free_list[nfree++] = (uint8_t)vs;
            top_remove(vs);
            M.stk_req[stack_cnt] = vr;
            M.stk_g[stack_cnt] = l - (uint32_t)li[vr];
            ++stack_cnt;
            --B;
            S -= l;
            if (B == 0) { err = SAMU_E_INFEASIBLE; break; }
            if (ntop == 0) top_rebuild();
          }
          if (err) break;
          heap_clean();
          const uint32_t smax = (uint32_t)((int32_t)d + max_o());
          F -= (int32_t)needd;
          const uint64_t fl = LC * B + K1 * (uint64_t)S;
          const double lat = lane_iter_cost(C.coef, ms, B, fl, B * smax, S);
          t = __dadd_rn(t, lat);
          add_fl(fl);
          reqit += B;
          iters += 1;
          S += B;
          d += 1;
          needidx = needidx == 0 ? bs.v - 1 : needidx - 1;
        }
        // ---- retire the finishers of this decode ----
        heap_clean();
        while (hn && (uint32_t)(M.heap[0] >> 32) == d) {
          const unsigned long long kk = M.heap[0];
          heap_pop();
          const uint32_t s = (uint32_t)(kk & 0xFFu);
          const int32_t o = M.s_o[s];
          const uint32_t l_now = (uint32_t)(o + (int32_t)d);
          F += (int32_t)bs.cdiv(l_now - 1);
          S -= l_now;
          --B;
          hist.dec(bs.posmod(o - 1));
          M.s_rank[s] = 0;
          M.free_list[nfree++] = (uint8_t)s;
          top_remove(s);
          finished(M.s_req[s]);
          heap_clean();
        }
        if (nrel) flush_rel();
        if (ntop == 0 && B > 0) top_rebuild();
      }
    }

    // ---- per-replica record ----
    const bool done = !err && B == 0 && stack_cnt == 0 && hd == hd_end && tl_head == tl_tail;
    if (err) {
      if (atomicCAS(P.error, 0, err) == 0) P.error[1] = 20;
    }
    samu_trial_rec rec;
    rec.t_end = t;
    rec.flops_lo = fl_lo;
    rec.flops_hi = fl_hi;
    rec.req_iters = reqit;
    rec.iters = iters;
    rec.flags = (done ? 1u : 0u) | (cut ? 2u : 0u) | (hd_end == 0 ? 4u : 0u);
    P.rep_rec[((size_t)ci * P.n_trials + k) * 16 + j] = rec;
    have = false;
  }
}

size_t lane_mem_bytes() { return sizeof(LaneMem); }

cudaError_t lane_prepare(int* blocks_per_sm) {
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_simulate_lane<true>, 128, 0);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_simulate_lane<false>, 128, 0);
  *blocks_per_sm = a < b ? a : b;
  return e;
}

cudaError_t launch_simulate_lane(const SimLaunch& L, void* mem, int32_t n_blocks, bool pow2_block, cudaStream_t s) {
  if (pow2_block) k_simulate_lane<true><<<n_blocks, 128, 0, s>>>(L, reinterpret_cast<LaneMem*>(mem));
  else k_simulate_lane<false><<<n_blocks, 128, 0, s>>>(L, reinterpret_cast<LaneMem*>(mem));
  return cudaGetLastError();
}
