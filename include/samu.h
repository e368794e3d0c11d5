/* samu.h — C ABI of libsamu: SamuLLM's sampling-then-simulation estimator and greedy planner
 * (arXiv 2503.16893) on B200 (sm_100a).
 *
 * Citations: P:<n> = PAPER.md line n; S:<n> = SPEC.md line n; readings cN = DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only.  "host" pointers are read before the call returns (copied);
 *     "device" pointers are caller-owned CUDA allocations on the context's device and are used in
 *     stream order on the context's stream.
 *   - Errors are status codes (samu_status, 0 = SAMU_OK).  No exception or abort crosses the ABI.
 *     samu_last_error() returns a context-owned message valid until the next call.
 *     Asynchronous CUDA / NCCL failures surface at the next synchronising call as SAMU_E_CUDA /
 *     SAMU_E_NCCL and poison the context (later calls return SAMU_E_STATE).
 *   - One context per process / GPU; a context is not thread-safe.
 *   - Determinism: results depend only on inputs, seed and trial ids — never on world size,
 *     launch configuration or scheduling.
 */
#ifndef SAMU_H
#define SAMU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t samu_status;
#define SAMU_OK 0
#define SAMU_E_INVALID -1     /* bad argument: l_in > l_max, unsorted eCDF, tp not dividing h,
                                 unregistered model, layout violation, ... */
#define SAMU_E_INFEASIBLE -2  /* capacity below one sequence / no plan fits an empty stage */
#define SAMU_E_NOMEM -3
#define SAMU_E_CUDA -4
#define SAMU_E_NCCL -5
#define SAMU_E_STATE -6       /* context poisoned, or inconsistent carried WorkloadState */

#define SAMU_N_TP_SLOTS 5     /* tp in {1, 2, 4, 8, 16}: slot = log2(tp) */
#define SAMU_MAX_DP 16
#define SAMU_MAX_SEQS 256     /* engine max_num_seqs limit of the simulation kernel */
#define SAMU_MAX_NODES 64

/* request status word (WorkloadState, c27): bits 31..28 status, bits 27..0 rank / seq */
#define SAMU_ST_FRESH 0u
#define SAMU_ST_QUEUED 1u
#define SAMU_ST_PREEMPTED 2u
#define SAMU_ST_RUNNING 3u
#define SAMU_ST_DONE 4u

typedef struct samu_ctx samu_ctx;

/* Model architecture + cost tables.  Symbols of Eq. prefill / decode FLOPs. */
typedef struct samu_model_spec {
  uint32_t n_layers;            /* L */
  uint32_t hidden;              /* h; every allowed tp must divide it (c12) */
  uint64_t c;                   /* sum of per-layer matmul weight elements */
  uint32_t l_max;               /* max sequence length, <= 65535 */
  uint32_t tp_mask;             /* bit k set => tp = 2^k is allowed, k < SAMU_N_TP_SLOTS */
  uint64_t weight_bytes;        /* model weights, for plan validity */
  uint64_t kv_bytes_per_token;  /* KV-cache bytes per token, all layers */
} samu_model_spec;

/* Engine + planned machine (readings c5, c6).  The planned machine (n_gpus GPUs of
 * mem_bytes_per_gpu) is the machine being planned for (Alg. 1 input "N GPUs"); it is
 * unrelated to the number of B200s running the estimator. */
typedef struct samu_engine_cfg {
  uint32_t max_num_seqs;        /* 1..256 */
  uint32_t block_size;          /* KV block tokens, 1..32 */
  uint32_t min_batched_tokens;  /* token budget per prefill = max(l_max, this) */
  uint32_t mem_util_permille;   /* usable fraction of GPU memory, 0..1000 */
  uint64_t mem_bytes_per_gpu;
  uint64_t kv_cap_bytes_per_gpu;
  uint32_t n_gpus;              /* N, 1..16 */
} samu_engine_cfg;

/* One application request.  Requests are passed as one array grouped by ascending node; a
 * request's pred (if any) has a smaller index.  l_in_eff = min(l_in_base + max(l_out(pred),1),
 * l_max) (c3); a same-node pred makes a chain (fused self-loop) whose links
 * share chain (the dp key, c13); a pred in another node is a cross-node input (evaluator,
 * P:476).  A node depends on at most one other node and does not mix the two kinds (c26). */
typedef struct samu_request {
  uint32_t l_in_base;           /* prompt tokens incl. template / update overhead, <= 65535 */
  uint32_t cap_y;               /* explicit output limit y */
  int32_t pred;                 /* -1 or index of the predecessor request */
  int32_t node;                 /* graph node (after self-loop fusion) */
  int32_t chain;                /* -1 or chain id within the node */
} samu_request;

/* Per-(candidate, trial) record (c16). 40 bytes. */
typedef struct samu_trial_rec {
  double t_end;                 /* stage-clock end time, max over dp replicas (incl. load) */
  uint64_t flops_lo, flops_hi;  /* exact u128 sum of per-iteration FLOPs */
  uint64_t req_iters;           /* sum over iterations of B (request-iterations) */
  uint32_t iters;               /* simulated iterations, all replicas */
  uint32_t flags;               /* bit0 all requests of the node done, bit1 cut by time limit */
} samu_trial_rec;

/* A candidate = one (node, plan) simulation over the context's local trials. */
typedef struct samu_candidate {
  int32_t node;
  int32_t dp, tp;               /* execution plan P = (dp, tp) */
  int32_t resume;               /* 1: keep plan — clock starts at the carried overshoot, state
                                   resumes exactly; 0: (re)load — clock starts at load(dp,tp) and
                                   partially decoded requests are recomputed (c18) */
  int32_t dep_src;              /* index of an earlier candidate in the same batch whose finish
                                   times give this node's cross-node ready times, or -1 (use the
                                   carried finish times) */
  int32_t commit;               /* 1: write the end state back into the WorkloadState */
} samu_candidate;

/* Per-candidate summary over all trials (c17). */
typedef struct samu_cand_summary {
  double mean_t, p50_t, p90_t, p99_t; /* mean: left-to-right sum / T; nearest-rank percentiles */
  double mean_flops;            /* dbl(sum of u128 FLOPs) / T */
  double mean_req_iters;
} samu_cand_summary;

typedef struct samu_plan_stage {
  int32_t n_entries;
  int32_t node[16], dp[16], tp[16];
  int32_t fstar;                /* node whose finish ends the stage (c16) */
  double mean_tE;               /* mean over trials of t_E^(k) */
  double T_E;                   /* stage throughput */
} samu_plan_stage;

typedef struct samu_plan {
  int32_t n_stages;
  samu_plan_stage stages[64];
  double total;                 /* sum over stages of mean t_E */
  int64_t n_cand_evals;         /* candidate stages scored (P:599 complexity) */
  int64_t n_sims;               /* candidate-trial simulations run by this rank */
  uint64_t req_iters;           /* simulated request-iterations by this rank */
} samu_plan;

/* ---- context ---------------------------------------------------------------------------- */

/* Create a context on CUDA device `cuda_device`, ordered on `cuda_stream` (a cudaStream_t; NULL
 * is the CUDA default stream, e.g. PyTorch's default current stream).  rank / world: this process's position among the processes
 * sharding the Monte-Carlo trials; world > 1 requires `nccl_unique_id` (128 bytes, host, from
 * samu_nccl_unique_id on rank 0 and broadcast by the caller).  *out owned by the caller until
 * samu_ctx_destroy. */
samu_status samu_ctx_create(samu_ctx** out, int32_t cuda_device, void* cuda_stream, int32_t rank,
                            int32_t world, const uint8_t* nccl_unique_id);
void samu_ctx_destroy(samu_ctx* ctx);

/* In-process rank group: `world` contexts created with samu_ctx_create_local in one process
 * (one thread per rank, any devices incl. the same one) run the multi-rank trial sharding with
 * device-to-device copies instead of NCCL (used to test the sharded path on one GPU).  The group
 * must outlive its contexts. */
typedef struct samu_local_group samu_local_group;
samu_status samu_local_group_create(samu_local_group** out, int32_t world);
void samu_local_group_destroy(samu_local_group* group);
samu_status samu_ctx_create_local(samu_ctx** out, int32_t cuda_device, void* cuda_stream, int32_t rank,
                                  samu_local_group* group);
const char* samu_last_error(const samu_ctx* ctx);
/* Number of CUDA kernels this context has launched so far (instrumentation). */
uint64_t samu_launch_count(const samu_ctx* ctx);
/* Schedule-sharing counters of this context since creation (instrumentation): out[0] shared-
 * schedule work items (a (node, dp) group's head replica-sim carrying up to 3 tp variants),
 * out[1] member items those carried, out[2] member items that fell out of sync (KV blocks bound
 * below the head's count, or a preemption) and were re-simulated on their own. */
void samu_share_stats(const samu_ctx* ctx, int64_t out[3]);
samu_status samu_nccl_unique_id(uint8_t out[128]);

/* Register model `model_id` (0..63): spec, per-B coefficient buckets and the loading table.
 *   bucket_B  host [n_buckets] strictly increasing batch sizes >= 1
 *   coeff     host [SAMU_N_TP_SLOTS][3 phases comp/prep/samp][2 (a,b)][n_buckets]
 *             (only slots allowed by tp_mask are read)
 *   load_s    host [SAMU_N_TP_SLOTS][SAMU_MAX_DP] seconds, load_s[slot][dp-1]
 * The dense per-B table (reading c11) is built on the device.
 * SAMU_E_INVALID: bad spec (l_max > 65535, tp_mask empty, ...), unsorted buckets, 2 L h >= 2^32
 * (a 32-bit FLOPs factor of K2), or a per-iteration FLOPs bound that could overflow u64. */
samu_status samu_model_register(samu_ctx* ctx, int32_t model_id, const samu_model_spec* spec,
                                int32_t n_buckets, const uint32_t* bucket_B, const double* coeff,
                                const double* load_s);

/* Load model `model_id`'s output-length eCDF F_out: host knots, K = n_points,
 * values strictly increasing, cum_counts strictly increasing with n = cum_counts[K-1] observed
 * lengths (10,000 in the paper).  Copied to the device.  SAMU_E_INVALID if unsorted. */
samu_status samu_ecdf_load(samu_ctx* ctx, int32_t model_id, const uint32_t* values,
                           const uint32_t* cum_counts, int32_t n_points);

/* Load the application: engine + planned machine, node -> model map (host [n_nodes]) and the
 * request array (host [n_req], layout rules above).  Validates (SAMU_E_INVALID) and uploads. */
samu_status samu_app_load(samu_ctx* ctx, const samu_engine_cfg* engine, int32_t n_nodes,
                          const int32_t* node_model, int32_t n_req, const samu_request* reqs);

/* Valid execution plans of `node`'s model on the planned machine: writes up
 * to `cap` (dp, tp) pairs in order of ascending dp*tp then tp into host dp[] / tp[] and returns
 * their total count (>= 0), or a negative samu_status. */
int32_t samu_enumerate_plans(samu_ctx* ctx, int32_t node, int32_t* dp, int32_t* tp, int32_t cap);

/* ---- sharding over ranks (north star: "candidates and Monte Carlo trials shard
 * naturally across the 8 GPUs") ---------------------------------------------------------------
 * Host-only: no context, no GPU.  These are the rules the sharded calls apply internally, so a
 * caller (bench.py, tests) can place its local trials / jobs the same way. */

/* A (jobs x trials) product over `world` ranks: world = trial_blocks x job_classes; rank r
 * simulates the contiguous trial block r % trial_blocks of n_trials (block sizes differ by at
 * most one, the lower blocks larger) for the jobs of class r / trial_blocks.  job_classes = 1
 * whenever n_trials >= world (pure trial sharding: trials are i.i.d., every rank holds every
 * candidate); with fewer trials than ranks, trial_blocks = the largest divisor of world not above
 * max(n_trials, 1).  forced_classes > 0 that divides world fixes job_classes (tests; the
 * SAMU_SHARD_CLASSES variable of the sharded calls).  Any output pointer may be NULL.
 * SAMU_E_INVALID: n_trials < 0, world < 1 or rank outside [0, world). */
samu_status samu_shard_plan(int32_t n_trials, int32_t world, int32_t rank, int32_t forced_classes,
                            int32_t* trial_blocks, int32_t* job_classes, int32_t* trial_begin,
                            int32_t* trial_count, int32_t* my_class);

/* Job classes of one batch: jobs (host work[n_jobs] >= 0, e.g. replica requests x expected
 * output) are placed longest-first (stable on ties) onto the least loaded class (lowest index
 * on ties); host out_class[n_jobs].  The greedy applies this to the jobs without a dependency
 * source (a dependent job runs in its source's class).  SAMU_E_INVALID: n_jobs < 0,
 * job_classes < 1, a negative or NaN work, or NULL arrays with n_jobs > 0. */
samu_status samu_shard_classes(int32_t n_jobs, const double* work, int32_t job_classes, int32_t* out_class);

/* ---- the hot path ---------------------------------------------------------------------- */

/* Output-length sampling (c1-c3) for every app request and trials
 * [trial_begin, trial_begin + n_trials): device out_l_out / out_l_in_eff [n_trials][n_req]
 * (u16, trial-major).  Counter-based: any trial range / world size gives identical values. */
samu_status samu_sample_lengths(samu_ctx* ctx, uint64_t seed, int32_t trial_begin, int32_t n_trials,
                                uint16_t* out_l_out, uint16_t* out_l_in_eff);

/* Output-length sampling of an arbitrary request set of one model (the §8(b) call shape,
 * P:431-433 "a set of requests per model"): no application needs to be loaded, only
 * the model's registration and eCDF.  reqs host [n_req]: l_in_base, cap_y, pred (-1, or the
 * index within this set of a chained predecessor, which must come earlier and have no other
 * successor; its generated tokens are added to the successor's prompt), node and chain
 * ignored.  Draw u of request i in trial k = word ((i + index_base) & 3) of
 * Philox4x32-10(ctr = ((i + index_base) >> 2, k, stream_id, 0), key = seed): with stream_id =
 * the node id and index_base = the node's first request index this is exactly what
 * samu_sample_lengths draws for that node.  Device out_l_out / out_l_in_eff [n_trials][n_req].
 * SAMU_E_INVALID: unregistered model / no eCDF, l_in_base > l_max, bad pred, stream_id >= 2^31. */
samu_status samu_sample_requests(samu_ctx* ctx, int32_t model_id, uint32_t stream_id, const samu_request* reqs,
                                 int32_t n_req, uint32_t index_base, uint64_t seed, int32_t trial_begin,
                                 int32_t n_trials, uint16_t* out_l_out, uint16_t* out_l_in_eff);

/* Known output lengths in place of the sampler (the §5.5 cost-model ablation):
 * host l_true [n_req] (copied before return) -> device out_l_out / out_l_in_eff [1][n_req] with
 * the sampler's clamps and chained-prompt arithmetic.  Synchronises the context stream. */
samu_status samu_known_lengths(samu_ctx* ctx, const uint32_t* l_true, uint16_t* out_l_out,
                               uint16_t* out_l_in_eff);

/* Simulate n_cands candidates over the n_trials local trials whose lengths are given
 * (device l_out / l_in_eff [n_trials][n_req], from samu_sample_lengths or known lengths).
 *   state       device WorkloadState or NULL (fresh, no commit):
 *                 st [n_trials][n_req] u32, g [n_trials][n_req] u16,
 *                 fin_t [n_trials][n_req] f64 (carried finish times, stage clock),
 *                 overshoot [n_trials][n_nodes][16] f64
 *   time_limit  device [n_cands][n_trials] f64 stage-clock limits tau, or NULL (+inf) (c15)
 *   out_recs    device [n_cands][n_trials] samu_trial_rec (required)
 *   out_summary host [n_cands] or NULL; if given, computed over ALL world trials (records are
 *               all-gathered over the context's ranks, trial order = rank order) and the call
 *               synchronises
 *   out_fin_iter device [n_cands][n_trials][n_req] u32 or NULL: iteration (within its replica)
 *               in which each request of the candidate's node finished, 0xFFFFFFFF otherwise
 *   out_fin_t   device [n_cands][n_trials][n_req] f64 or NULL: finish time (stage clock), +inf
 * Candidates with commit = 1 must be distinct nodes and need `state`.
 * SAMU_E_INVALID also when n_trials x n_req >= 2^32 (K2 indexes [trial][request] with 32 bits)
 * or the batch has >= 2^31 work items (trials x dp replicas).
 * Execution: one K2 launch per path present — LEAN (fresh state, independent requests, no
 * per-request outputs), FRESH (the same with chain successors), each with or without a time
 * limit, and the general one;
 * SAMU_K2_MODES=always|never in the environment overrides the batch-size rule that picks them.
 * The results do not depend on the path. */
samu_status samu_simulate_batch(samu_ctx* ctx, const samu_candidate* cands, int32_t n_cands,
                                const uint16_t* l_out, const uint16_t* l_in_eff, int32_t n_trials,
                                uint32_t* st, uint16_t* g, double* fin_t, double* overshoot,
                                const double* time_limit, samu_trial_rec* out_recs,
                                samu_cand_summary* out_summary, uint32_t* out_fin_iter,
                                double* out_fin_t);

/* Algorithm 1 greedy search with the estimator, readings c14-c18: samples the
 * lengths of this rank's share of n_trials (trials split in contiguous blocks by rank), keeps
 * the WorkloadState on the device, all-gathers per-trial records over NCCL when world > 1, and
 * scores candidate stages on the device.  Every rank returns the identical plan.  *out is
 * library-allocated; free with samu_plan_free. */
samu_status samu_plan_greedy(samu_ctx* ctx, uint64_t seed, int32_t n_trials, samu_plan** out);

/* The paper's competitors on the same estimator, stage commit and trial sharding:
 *   Max-heuristic: all GPUs to one model at a time (the lowest-id ready model) with the plan of
 *     highest stage throughput; each stage runs its model to completion.
 *   Min-heuristic: as many ready models as GPUs allow, GPUs split as evenly as possible, the
 *     split / plan combination of highest stage throughput (<= 10^4 evaluated); stages end at the
 *     first finish and every unfinished model is re-planned. */
samu_status samu_plan_max_heuristic(samu_ctx* ctx, uint64_t seed, int32_t n_trials, samu_plan** out);
samu_status samu_plan_min_heuristic(samu_ctx* ctx, uint64_t seed, int32_t n_trials, samu_plan** out);

/* General planner entry (all of the above plus the §5.5 ablations):
 *   algo              SAMU_ALGO_GREEDY / _MAX / _MIN
 *   allow_preemption  0 = no-preemption variant: a model keeps its plan and GPUs from the stage
 *                     it starts in until it finishes and is not re-planned (reading c29); the
 *                     Max-heuristic is the same either way
 *   known_l_out       host [n_req] true output lengths in place of the sampler, or NULL;
 *                     requires n_trials == 1 (reading c30) */
#define SAMU_ALGO_GREEDY 0
#define SAMU_ALGO_MAX 1
#define SAMU_ALGO_MIN 2
typedef struct samu_plan_opts {
  int32_t algo;
  int32_t allow_preemption;
  const uint32_t* known_l_out;
} samu_plan_opts;
samu_status samu_plan_run(samu_ctx* ctx, uint64_t seed, int32_t n_trials, const samu_plan_opts* opts, samu_plan** out);
void samu_plan_free(samu_plan* plan);

/* Per-iteration cost-model coefficients from profiled iterations (reading c34): for
 * each bucket k (one (model, tp, phase, B) combination), the samples [off[k], off[k+1]) of
 * (x, latency) -- x = FLOPs, B*s or S per phase -- are fitted by least squares, latency = a x + b
 * (a < 0 clamped to 0, b = mean latency).  trim_permille > 0 drops the floor(n * trim / 1000)
 * samples of largest |residual| (ties: lower index) and refits ("noise points", Fig. 5).
 * All arrays are device memory: off [n_buckets + 1] i64, x / y [off[n_buckets]] f64, out_a /
 * out_b [n_buckets] f64, out_n_used (samples kept) / out_flags (bit0 degenerate, bit1 a
 * clamped) [n_buckets] i32.  SAMU_E_INVALID if a bucket has fewer than two distinct x (its
 * outputs are 0).  Synchronises the context stream. */
samu_status samu_fit_coeffs(samu_ctx* ctx, int32_t n_buckets, const int64_t* off, const double* x, const double* y,
                            int32_t trim_permille, double* out_a, double* out_b, int32_t* out_n_used,
                            int32_t* out_flags);

/* Runtime replay with the dynamic scheduler (reading c33): executes `plan` against
 * true output lengths -- known_l_out host [n_req], or NULL = trial 0 of the sampler with `seed`
 * (a different seed than the plan's stands in for the real run) -- one trial on the device.
 * Each actual stage is the set of running (model, plan) pairs and ends at the first actual model
 * finish; then: an unfinished running pair keeps running if the current planned stage is its
 * model's last, or if it is in the next planned stage; next-stage pairs are placed first; other
 * running pairs keep running only if the whole next stage is placed and their GPUs are free,
 * else they are stopped (state carried).  GPU placement is trivial on NVSwitch (continuing pairs
 * keep their GPUs, new pairs take the lowest free ids).  `out` is caller-owned. */
typedef struct samu_replay_stage {
  int32_t n_entries;
  int32_t node[16], dp[16], tp[16];
  uint32_t gpu_mask[16];        /* GPU ids of each pair */
  int32_t resumed[16];          /* 1 = continued from the previous actual stage (no reload) */
  int32_t planned_stage;        /* planned stage being executed */
  int32_t first_finisher;       /* node whose finish ended this actual stage */
  int32_t idle_gpus;            /* GPUs with no pair during this actual stage */
  double t_start, duration;     /* seconds, replay clock */
} samu_replay_stage;

typedef struct samu_replay {
  int32_t n_stages;
  samu_replay_stage stages[64];
  double total;                 /* replayed running time */
  double planned_total;         /* the plan's estimate */
  double idle_gpu_seconds;      /* sum of idle_gpus x duration */
  int32_t n_kept_last, n_kept_room, n_stopped;
} samu_replay;

samu_status samu_replay_plan(samu_ctx* ctx, const samu_plan* plan, uint64_t seed, const uint32_t* known_l_out,
                             samu_replay* out);

#ifdef __cplusplus
}
#endif
#endif /* SAMU_H */
