// Internal declarations shared by libsamu's translation units (product path only; the oracle
// under oracle/ shares nothing with this tree).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/samu.h"

#define SAMU_EMPTY 0xFFFFFFFFu
#ifndef SAMU_WARPS_PER_BLOCK
#define SAMU_WARPS_PER_BLOCK 4   // K2 block = 4 warps; 6 blocks / SM (80 registers): 24 warps per SM
#endif

// ------------------------------------------------------------------------------------------
// Application tables on the device (uploaded by samu_app_load)
// ------------------------------------------------------------------------------------------
struct DevApp {
  int32_t n_req, n_nodes;
  const uint32_t* l_in_base;   // [n]
  const uint32_t* cap_y;       // [n]
  const int32_t* pred;         // [n]
  const int32_t* node;         // [n]
  const int32_t* succ;         // [n] same-node chain successor or -1
  const uint8_t* cross;        // [n] 1 if pred is in another node
};

// eCDF tables for the sampler: per model the sorted multiset of its n observed lengths as a u16
// table (reading c2), packed, each model's table padded to 8 entries (16-byte TMA granularity)
struct DevEcdf {
  const uint16_t* tab;         // packed tables
  const int32_t* tab_off;      // [SAMU_MAX_NODES + 1] entry offsets
  const uint32_t* n_obs;       // [SAMU_MAX_NODES] n = cum[K-1]
  const int32_t* model_of_node;  // [n_nodes]
  const uint32_t* l_max_of_node; // [n_nodes]
  int32_t smem_tab_bytes;      // dynamic shared memory reserved for one staged table
};

// One candidate (node, plan) as the simulation kernel sees it.
struct DevCand {
  int32_t node, dp, tp, resume, commit, has_succ;
  int32_t mode;                // K2 path: 0 general, 2 FRESH (fresh state, no arrivals / cut / outputs), 1 LEAN (FRESH, no successors), 3 / 4 = LEAN / FRESH cut at tau, 5 / 6 = LEAN / FRESH schedule-sharing groups
  uint32_t max_seqs, bs, budget;
  int32_t blocks;              // KV blocks per replica (c5)
  uint32_t L, h_tp;            // layers, h / tp
  uint64_t c;                  // per-layer matmul weight elements
  uint64_t LC, K1;             // L c and 2 L (h/tp): FLOPs = LC B + K1 S (decode), B s (LC + K1 s) (prefill)
  double load_s;               // loading time of (model, dp, tp)
  const double* coef;          // dense [3 phases][2 (a,b)][max_seqs]
  const uint32_t* rep_off;     // [dp + 1]
  const uint32_t* rep_req;     // requests of the node grouped by replica, index order

  const double* src_fin;       // [T][n] finish times of the dependency source, or null
  const double* tau;           // [T] time limits or null
  const samu_trial_rec* tau_rec;  // [T] take tau_k = tau_rec[k].t_end (f* of a stage), or null
  double* fin_t_out;           // [T][n] or null
  uint32_t* fin_iter_out;      // [T][n] or null
  samu_trial_rec* out_rec;     // [T] per-(candidate, trial) records (after the replica combine)
};

struct SimLaunch {
  DevApp app;
  const DevCand* cands;
  int32_t n_cands;
  int32_t n_trials;
  // work items (candidate, trial, replica), longest candidates first: item i belongs to candidate
  // ord[x] for off[x] <= i < off[x + 1] (off[x + 1] - off[x] = trials x dp), then trial-major
  const uint32_t* ord;         // [n_ord] candidate indices
  const uint32_t* off;         // [n_ord + 1] item offsets
  int32_t n_ord;
  int32_t n_items;
  uint32_t* next_item;         // work counter
  const uint16_t* l_out;       // [T][n]
  const uint16_t* l_in;        // [T][n]
  uint32_t* st;                // [T][n] or null (fresh)
  uint16_t* g;
  double* fin_t;
  double* over;                // [T][n_nodes][16]
  samu_trial_rec* rep_rec;     // [n_cands][T][16]
  uint32_t* scratch_q;         // [n_warps][max_q]
  uint64_t* scratch_key;       // [n_warps][4][max_p]: pending sort (2) + carried-state sort (2)
  uint32_t* scratch_idx;       // [n_warps][4][max_p]
  int32_t max_q, max_p;
  int32_t* error;              // first error code (0 = ok), error site
  // Schedule sharing (K2 modes 5 / 6 = 1 / 2 with groups: fresh state, no time limit).  Candidates of one (node, dp)
  // that differ only in tp run one event schedule as long as KV blocks never bind below the
  // largest variant's count: ord entry x then heads a group, grp[x] = (members, 2nd, 3rd, 4th
  // candidate; fewer blocks), simulated once with per-lane clocks.  A member whose schedule
  // would differ in a (trial, replica) item goes to the fallback queue fb (candidate, item
  // within the candidate) and is simulated on its own in the same launch.  fb_ctr: [0]
  // allocated, [1] claimed.  grp == null: no groups.
  const uint4* grp;
  uint2* fb;
  uint32_t* fb_ctr;
  uint32_t* fb_count;          // [n_cands] fallback items per member candidate (scheduling hints)
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_sample(const DevApp& app, const DevEcdf& e, const int32_t* seq_head, int32_t n_seq,
                          uint64_t seed, int32_t trial_begin, int32_t n_trials, const uint32_t* known,
                          uint16_t* l_out, uint16_t* l_in, cudaStream_t s, uint32_t r_base = 0, int32_t stream = -1);
cudaError_t launch_ecdf_table(const uint32_t* values, const uint32_t* cum, int32_t K, uint32_t n, uint16_t* tab,
                              cudaStream_t s);
cudaError_t launch_dense_coeff(const double* bucket_B, int32_t nb, const double* coeff_slot,
                               uint32_t max_seqs, double* out, cudaStream_t s);
cudaError_t launch_simulate(const SimLaunch* Ls, const int* modes, const int32_t* n_blocks, int n_launch,
                            const DevCand* host_cands, uint32_t block_size, cudaStream_t s, cudaStream_t s2,
                            cudaEvent_t ev_fork, cudaEvent_t ev_join);
#define SAMU_K2_MODES 7   // 0 general, 1 LEAN, 2 FRESH, 3 / 4 LEAN / FRESH cut, 5 / 6 LEAN / FRESH schedule-sharing groups
cudaError_t simulate_prepare(int blocks_per_sm[SAMU_K2_MODES]);   // per K2 mode

int32_t simulate_smem_bytes(int mode);
cudaError_t launch_combine(const samu_trial_rec* rep_rec, const DevCand* cands, int32_t n_cands, int32_t n_trials,
                           double* over, int32_t n_nodes, cudaStream_t s);
cudaError_t launch_summary(const samu_trial_rec* recs, int32_t n_cands, int32_t n_trials,
                           samu_cand_summary* out, cudaStream_t s);
cudaError_t launch_unpack_gather(const samu_trial_rec* recv, int32_t world, int32_t n, int32_t Tmax, int32_t T,
                                 int32_t Wt, const int32_t* slots, const int32_t* job_class, samu_trial_rec* dst,
                                 cudaStream_t s);
cudaError_t launch_fill_f64(double* p, int64_t n, double v, cudaStream_t s);
cudaError_t launch_rebase(uint32_t* st, double* fin_t, int64_t n_total, const samu_trial_rec* fstar_rec,
                          int32_t n_req, cudaStream_t s);
cudaError_t launch_node_done(const uint32_t* st, int32_t n_trials, int32_t n_req, const int32_t* node,
                             int32_t* out_any_undone /*[n_nodes][n_trials]*/, int32_t n_nodes, cudaStream_t s);

// stage scoring (greedy): see k_reduce.cu
struct StageCand {
  int32_t n_entries;
  int32_t full_slot[16];       // record slot (in the full-sim cache) of each entry
  int32_t cut_slot[16];        // record slot of each entry's cut sim (after f* is known), -1 for f*
  int32_t node[16];
  int32_t gpus;                // #gpu of the candidate stage
  int32_t changed_node, changed_dp, changed_tp;
};
struct StageOut {
  int32_t fstar;               // entry index of f*
  int32_t pad;
  double TE, mean_tE;
};
cudaError_t launch_fstar(const samu_trial_rec* cache, int32_t T, const StageCand* sc, int32_t n, StageOut* out,
                         cudaStream_t s);
cudaError_t launch_stage_score(const samu_trial_rec* cache, int32_t T, const StageCand* sc, int32_t n,
                               StageOut* out, double TE_star, int32_t gpus_star, int32_t mode, int32_t* best,
                               double* max_dT, cudaStream_t s);
cudaError_t launch_fit(const int64_t* off, int32_t n_buckets, const double* x, const double* y, int32_t trim_permille,
                       uint8_t* gone, double* out_a, double* out_b, int32_t* out_n_used, int32_t* out_flags,
                       cudaStream_t s);
