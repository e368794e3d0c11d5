/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference of SamuLLM's sampling-then-simulation
 * estimator and greedy planner (arXiv 2503.16893; PAPER.md = "P:<line>").  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2503_16893_b200/) and neither
 * imports the other.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.
 *
 * Semantics: DESIGN.md §3 ("Readings"), which follows SURVEY.md §8(c).  Every function cites
 * the passage it follows.  fp64 throughout; compiled with -ffp-contract=off.
 */
#ifndef SAMU_ORACLE_H
#define SAMU_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_OK 0
#define OR_E_INVALID -1
#define OR_E_INFEASIBLE -2
#define OR_E_STATE -6

#define OR_N_TP_SLOTS 5   /* tp in {1,2,4,8,16} */
#define OR_MAX_DP 16
#define OR_MAX_SEQS 256

/* request status word (state arrays), bits 31..28 = status, 27..0 = rank / seq */
#define OR_ST_FRESH 0u
#define OR_ST_QUEUED 1u
#define OR_ST_PREEMPTED 2u
#define OR_ST_RUNNING 3u
#define OR_ST_DONE 4u

typedef struct or_model {
  uint32_t L, h;               /* layers, hidden dim */
  uint64_t c;                  /* sum of per-layer matmul weight elements */
  uint32_t l_max;              /* max sequence length */
  uint32_t tp_mask;            /* bit k => tp = 2^k allowed */
  uint64_t weight_bytes;
  uint64_t kv_bytes_per_token; /* all layers */
  int32_t n_buckets;
  const uint32_t* bucket_B;    /* [n_buckets] strictly increasing */
  const double* coeff;         /* [5 tp slots][3 phases][2 (a,b)][n_buckets] */
  const double* load;          /* [5 tp slots][16 dp] seconds */
  int32_t ecdf_k;
  const uint32_t* ecdf_values; /* [K] strictly increasing */
  const uint32_t* ecdf_cum;    /* [K] strictly increasing, n = cum[K-1] */
} or_model;

typedef struct or_engine {
  uint32_t max_num_seqs, block_size, min_batched_tokens, mem_util_permille;
  uint64_t mem_bytes_per_gpu, kv_cap_bytes_per_gpu;
  uint32_t n_gpus;             /* N planned GPUs (Alg. 1 input) */
} or_engine;

typedef struct or_app {
  or_engine engine;
  int32_t n_models;
  const or_model* models;
  int32_t n_nodes;
  const int32_t* node_model;
  int32_t n_req;
  const uint32_t* l_in_base;
  const uint32_t* cap_y;
  const int32_t* pred;
  const int32_t* node;
  const int32_t* chain;
} or_app;

typedef struct or_cand { int32_t node, dp, tp, resume; } or_cand;

typedef struct or_rec {
  double t_end;                /* max over dp replicas of the end clock (stage clock) */
  uint64_t flops_lo, flops_hi; /* exact sum of per-iteration FLOPs (u128) */
  uint64_t req_iters;          /* sum over iterations of B */
  uint32_t iters;              /* iterations over all replicas */
  uint32_t flags;              /* bit0 all requests of the node done; bit1 stopped by tau */
} or_rec;

typedef struct or_stage {
  int32_t n_entries;
  int32_t node[16], dp[16], tp[16];
  int32_t fstar;
  double mean_tE;
  double T_E;
} or_stage;

typedef struct or_plan {
  int32_t n_stages;
  or_stage stages[64];
  double total;                /* sum over stages of mean_k t_E^(k) */
  int64_t n_cand_evals;        /* candidate stages evaluated (complexity instrumentation) */
} or_plan;

typedef struct or_problem or_problem;

const char* or_last_error(void);
or_problem* or_problem_create(const or_app* app);
void or_problem_destroy(or_problem* p);

/* primitives (each cited in oracle.cpp) */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t or_ecdf_inverse(const or_problem* p, int32_t model, uint32_t u);
uint64_t or_flops_prefill(uint32_t L, uint64_t c, uint32_t h, uint32_t tp, uint64_t B, uint64_t s);
uint64_t or_flops_decode(uint32_t L, uint64_t c, uint32_t h, uint32_t tp, uint64_t B, uint64_t S);
int32_t or_dense_coeff(const or_problem* p, int32_t model, int32_t tp, double* a /*[3][max_seqs]*/,
                       double* b /*[3][max_seqs]*/);
int64_t or_plan_blocks(const or_problem* p, int32_t model, int32_t dp, int32_t tp); /* -1 invalid */
int32_t or_enumerate_plans(const or_problem* p, int32_t model, int32_t* dp, int32_t* tp, int32_t cap);
double or_iter_latency(const double* a3, const double* b3, uint64_t flops, uint64_t Bs, uint64_t S);

/* sampling: all app requests, trials [trial_begin, trial_begin + n_trials) */
int32_t or_sample_lengths(const or_problem* p, uint64_t seed, int32_t trial_begin, int32_t n_trials,
                          uint16_t* l_out /*[T][n]*/, uint16_t* l_in_eff /*[T][n]*/);

/* one candidate (model, plan) over n_trials.  state arrays may be NULL (fresh). */
int32_t or_simulate(const or_problem* p, const or_cand* cand, int32_t n_trials,
                    const uint16_t* l_out, const uint16_t* l_in_eff,
                    uint32_t* st, uint16_t* g, double* fin_t, double* overshoot /*[T][nodes][16]*/,
                    const double* tau /*[T] or NULL*/, const double* src_fin_t /*[T][n] or NULL*/,
                    int32_t commit, or_rec* out_rec /*[T]*/, uint32_t* out_fin_iter /*[T][n] or NULL*/,
                    double* out_fin_t /*[T][n] or NULL*/);

/* fresh-state full simulations of many candidates over trials on a thread pool (CPU baseline) */
int32_t or_simulate_many(const or_problem* p, int32_t n_cands, const or_cand* cands, int32_t n_trials,
                         const uint16_t* l_out, const uint16_t* l_in_eff, int32_t n_threads,
                         or_rec* out_rec /*[n_cands][T]*/);

/* per-candidate summaries over T trials (north star "segmented reduction to per-candidate mean
 * and percentile latency"; reading c17): mean = sequential fp64 sum in trial order / T,
 * percentiles nearest rank sorted[ceil(p T / 100) - 1], mean FLOPs = dbl(u128 sum) / T */
typedef struct or_summary {
  double mean_t, p50_t, p90_t, p99_t, mean_flops, mean_req_iters;
} or_summary;
int32_t or_summarise(int32_t n_cands, int32_t n_trials, const or_rec* recs /*[n_cands][T]*/, or_summary* out);

/* per-iteration descriptor of one replica-sim ("per-iteration trace dump":
 * t_start, kind, B, s, S, flops, latency), plus the KV state after the iteration */
typedef struct or_iter_desc {
  double t_start, lat;         /* clock at the iteration's start; its latency */
  uint64_t flops, s, S;        /* Eq. prefill / decode FLOPs; max and total length fed */
  int64_t free_blocks;         /* KV blocks free after the iteration (reading c5) */
  uint32_t kind;               /* 0 prefill, 1 decode */
  uint32_t B;                  /* batch size */
  uint32_t n_preempted;        /* victims of this (decode) iteration (c7) */
  uint32_t n_finished;
} or_iter_desc;
/* fresh-state full simulation of replica `replica` of one candidate in one trial (l_out, l_in
 * [n_req] of that trial); after every iteration the running set is listed as (request, g)
 * pairs, run_off[i]..run_off[i+1] for iteration i.  *n_desc / *n_run receive the needed sizes;
 * returns OR_E_INVALID (after filling them) when a capacity is too small. */
int32_t or_trace_replica(const or_problem* p, const or_cand* cand, const uint16_t* l_out, const uint16_t* l_in,
                         int32_t replica, int64_t cap_desc, or_iter_desc* out_desc, int64_t cap_run,
                         uint32_t* run_req, uint32_t* run_g, int64_t* run_off, int64_t* n_desc, int64_t* n_run);

/* Algorithm 1 greedy search with the estimator */
int32_t or_plan_greedy(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out);

/* the paper's competitors on the same estimator */
int32_t or_plan_max_heuristic(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out);
int32_t or_plan_min_heuristic(const or_problem* p, uint64_t seed, int32_t n_trials, or_plan* out);

/* known output lengths in place of the sampler: l_true [n_req] */
int32_t or_known_lengths(const or_problem* p, const uint32_t* l_true, uint16_t* l_out, uint16_t* l_in_eff);
/* algo 0 greedy / 1 max / 2 min; allow_preemption = 0 is the §5.5 no-preemption ablation;
 * known_l_out (NULL = sample) requires n_trials == 1 */
int32_t or_plan_run(const or_problem* p, uint64_t seed, int32_t n_trials, int32_t algo, int32_t allow_preemption,
                const uint32_t* known_l_out, or_plan* out);

/* runtime replay of a plan against true lengths with the dynamic scheduler */
typedef struct or_replay_stage {
  int32_t n_entries;
  int32_t node[16], dp[16], tp[16];
  uint32_t gpu_mask[16];       /* GPU ids of each pair (NVSwitch: any set) */
  int32_t resumed[16];         /* 1 = continued from the previous actual stage (no reload) */
  int32_t planned_stage;       /* index of the planned stage being executed */
  int32_t first_finisher;      /* node whose finish ended this actual stage */
  int32_t idle_gpus;
  double t_start, duration;
} or_replay_stage;

typedef struct or_replay {
  int32_t n_stages;
  or_replay_stage stages[64];
  double total;                /* simulated running time with the true lengths */
  double planned_total;        /* the plan's estimate */
  double idle_gpu_seconds;     /* sum over actual stages of unassigned GPUs x duration */
  int32_t n_kept_last, n_kept_room, n_stopped;
} or_replay;

/* true lengths: known_l_out [n_req], or NULL = trial 0 of the sampler with `seed` */
int32_t or_replay_plan(const or_problem* p, const or_plan* plan, uint64_t seed, const uint32_t* known_l_out,
                       or_replay* out);

/* least-squares coefficient fit per bucket with top-residual trimming; samples of
 * bucket k are [off[k], off[k+1]); flags bit0 = degenerate bucket (error), bit1 = a clamped */
int32_t or_fit_coeffs(int32_t n_buckets, const int64_t* off, const double* x, const double* y, int32_t trim_permille,
                      double* out_a, double* out_b, int32_t* out_n_used, int32_t* out_flags);

#ifdef __cplusplus
}
#endif
#endif
