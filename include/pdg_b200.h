/*
 * pdg_b200.h -- C ABI of the B200-native PDGraph scoring hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every pointer named
 * "dev" is device memory; "stream" is a cudaStream_t passed as void*.
 * Every entry point returns PDG_OK (0) or a PDG_E* status; no exception ever
 * crosses the ABI; pdg_last_error() returns a thread-local message.
 *
 * The reference (arXiv 2506.14851 "Hermes", /root/reference/pkg/src/pdgsim)
 * is pure Python with no FFI of its own; each entry point below names the
 * module-level Python function it replaces (file:line).  The Python shim
 * paper_2506_14851_b200/ binds these with ctypes and re-exposes the
 * reference's signatures.
 */
#ifndef PDG_B200_H
#define PDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PDG_OK = 0,
  PDG_EINVAL = 1,      /* bad argument (sizes, null pointers)             */
  PDG_ECUDA = 2,       /* CUDA runtime / launch failure                    */
  PDG_ENODEV = 3,      /* no sm_100 device                                 */
  PDG_EUNSUPPORTED = 4 /* shape outside the compiled kernel envelope       */
};

/* Row flags written by the scorers. */
#define PDG_FLAG_OVERRUN 0x1u   /* exhausted row: key = age * penalty (sched.py:295-300) */

const char* pdg_last_error(void);
int pdg_abi_version(void);
/* SM count, compute capability of the current device. */
int pdg_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------------------
 * K1a  Gittins rank over explicit float64 support rows.
 * Replaces pdgsim.sched.gittins_rank_batch (sched.py:102-129), same contract:
 *   values, probs : [n_rows, n_bins] row-major float64, rows ascending
 *   ages          : [n_rows] float64
 *   out_rank      : [n_rows] float64, NaN for exhausted rows
 * All pointers are device pointers.
 * ------------------------------------------------------------------------- */
int pdg_gittins_rank_f64(const double* values, const double* probs,
                         const double* ages, int64_t n_rows, int32_t n_bins,
                         double* out_rank, void* stream);
/* Same with HOST pointers (what the reference-facing drop-in passes): the
 * library stages them through a reused pinned buffer (batches up to 1 MiB in
 * mapped memory the kernel reads in place; larger ones copied up and back),
 * runs the kernel on `stream` and returns after the ranks are in out_rank. */
int pdg_gittins_rank_f64_host(const double* values, const double* probs,
                              const double* ages, int64_t n_rows, int32_t n_bins,
                              double* out_rank, void* stream);

/* Sample form: pdgsim.sched.gittins_rank (sched.py:51-85), bit-identical.
 * Row r's samples are samples[off[r] .. off[r] + len[r]) (len <= 16384); the
 * tail {s - age : s > age} is sorted and scanned exactly as the reference
 * scans it (sequential float64 prefix over groups of equal values).
 * out_rank NaN: no sample exceeds the age (the reference raises
 * ExhaustedDistributionError); len 0 rows give NaN too (EstimationError).
 * Device pointers; max_len >= every len[r]. */
#define PDG_SAMPLES_MAX 16384
int pdg_gittins_rank_samples(const double* samples, const int64_t* off, const int32_t* len,
                             const double* ages, int64_t n_rows, int32_t max_len,
                             double* out_rank, void* stream);
/* One distribution from HOST memory (the drop-in gittins_rank): staged in
 * mapped pinned memory, one launch, one sync. */
int pdg_gittins_rank_samples_host(const double* samples, int32_t n, double age,
                                  double* out_rank, void* stream);

/* ---------------------------------------------------------------------------
 * K1b  Gittins rank over the device-resident histogram queue (the
 * bucket_points view cached by ApplicationInstance.set_remaining,
 * sched.py:170-181 / distributions.py:79-133), fused with the overrun
 * penalty of refresh_priorities (sched.py:292-300) and the global sort key.
 *
 * Row i describes bucket_count equal-width buckets over [lo, lo + k*width]:
 *   value_j = ((lo + j*w) + (lo + (j+1)*w)) / 2 + est_age    (bit-exact f64)
 *   prob_j  = counts[j] / nsamp
 * nbins[i] == 1 with width 0 encodes the degenerate point-mass row.
 * ------------------------------------------------------------------------- */
typedef struct {
  const double* lo;        /* [N] lowest bucket edge (sample min)                 */
  const double* width;     /* [N] bucket width (hi-lo)/k; 0 for degenerate rows   */
  const double* est_age;   /* [N] attained service when the estimate was taken    */
  const int32_t* nbins;    /* [N] buckets in the row (k, or 1 when degenerate)     */
  const int32_t* nsamp;    /* [N] samples behind the histogram (n)                 */
  const uint16_t* counts;  /* [N, stride] bucket counts                            */
  int64_t stride;          /* counts row stride in elements, multiple of 8        */
} pdg_hist_rows;

/* age: [rows] attained service now.  penalty: overrun_penalty_factor.
 * out_key (optional): (float32 key bits << 32) | tiebreak[row]; tiebreak is
 * the position of (arrival_time, app_instance_id) in arrival order
 * (sched.py:168).  row_idx (optional): score only rows row_idx[0..n) (the
 * incremental re-score after refinement events); otherwise rows 0..n-1.
 * All per-row inputs and outputs are indexed by row. */
int pdg_gittins_score_hist(const pdg_hist_rows* rows, const double* age,
                           int64_t n, double penalty, float* out_key_f32,
                           uint8_t* out_flags, const uint32_t* tiebreak,
                           uint64_t* out_key, const int32_t* row_idx, void* stream);

/* ---------------------------------------------------------------------------
 * a4  ApplicationInstance.set_remaining's bucketing as a standalone call
 * (sched.py:170-181, distributions.py:79-105): rows of n float64 samples ->
 * (lo, width, nbins, u16 counts[stride]) in the pdg_hist_rows layout.  The
 * demand engine fuses the same epilogue.  n <= 65535.
 * ------------------------------------------------------------------------- */
int pdg_bucketize(const double* samples, int64_t rows, int32_t n, int32_t k, double* lo,
                  double* width, int32_t* nbins, uint16_t* counts, int64_t stride,
                  void* stream);

/* ---------------------------------------------------------------------------
 * K5  global order: stable radix sort of packed 64-bit keys ascending,
 * carrying a u32 payload (the queue slot).  Replaces the Python min()/sort
 * over _task_sort_key (simcore.py:339-344, 512-516).
 * begin_bit = 0 sorts the full (key, tiebreak) word; begin_bit = 32 sorts the
 * float key only and relies on stability -- valid when the input is already
 * in arrival (tiebreak) order, e.g. slots filled in arrival order or the
 * rank-major all-gather of arrival-ordered shards.
 * temp: device scratch of pdg_order_temp_bytes(n) bytes.
 * ------------------------------------------------------------------------- */
size_t pdg_order_temp_bytes(int64_t n);
int pdg_order(const uint64_t* keys_in, uint64_t* keys_out,
              const uint32_t* slots_in, uint32_t* slots_out, int64_t n,
              int32_t begin_bit, void* temp, size_t temp_bytes, void* stream);


/* K5 across ranks (distributed.global_order's exchange as one C call):
 * ncclAllGather of every rank's `width` packed keys (shards padded with
 * 0x7FFFFFFFFFFFFFFF, which sorts last) into gathered[world * width] on
 * `stream`, then a radix sort of the gathered keys into sorted_keys (the
 * positions are the low 32 bits).  begin_bit = 32 is exact when every shard
 * is in arrival order (the rank-major gather then is too).  nccl_comm: the
 * caller's ncclComm_t; NCCL is resolved at run time (libnccl.so.2), and
 * PDG_EUNSUPPORTED is returned if it cannot be found.  Replaces the Python
 * min()/sort over _task_sort_key for a sharded queue (simcore.py:339-344). */
size_t pdg_rank_allgather_sort_temp_bytes(int64_t width, int32_t world);
int pdg_rank_allgather_sort(void* nccl_comm, const uint64_t* local_keys, int64_t width,
                            int32_t world, uint64_t* gathered, uint64_t* sorted_keys,
                            int32_t begin_bit, void* temp, size_t temp_bytes, void* stream);

/* K5b  incremental order after re-scoring rows[0..m) (distinct): the previous
 * order (sorted_*_in, produced by pdg_order with begin_bit 0 or by this call)
 * minus those rows, merged with their new keys (keys[] holds every row's
 * packed key).  Same result as a full pdg_order (keys are unique).  mark: a
 * caller-owned zeroed uint8[n] (left zeroed).  temp:
 * pdg_order_update_temp_bytes(n, m) bytes. */
size_t pdg_order_update_temp_bytes(int64_t n, int64_t m);
int pdg_order_update(const uint64_t* keys, const uint64_t* sorted_keys_in,
                     const uint32_t* sorted_slots_in, int64_t n, const int32_t* rows, int64_t m,
                     uint8_t* mark, uint64_t* sorted_keys_out, uint32_t* sorted_slots_out,
                     void* temp, size_t temp_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * K2 + K3 + a4  demand engine.
 * Replaces pdgsim.estimator.monte_carlo_remaining_demand (estimator.py:305-362)
 * including _conditioning_for / conditional_filter (estimator.py:155-233,
 * 289-302), and ApplicationInstance.set_remaining's bucketing
 * (sched.py:170-181, distributions.py:79-105).  For the same graph, current
 * unit, relevant observation, n and seed the samples are bit-identical to the
 * reference (numpy PCG64 stream reproduced by position).
 *
 * The graph bank is compiled by paper_2506_14851_b200/graphs.py; its record
 * layouts (64-byte unit descriptor, K3 condition/pair records) are private to
 * that compiler and engine.cu.
 * ------------------------------------------------------------------------- */
typedef struct {
  const void* units;              /* unit descriptors, 64 B each            */
  const int32_t* graph_base;      /* [G] first unit of each graph           */
  const int32_t* graph_n;         /* [G] units per graph (<= 32)            */
  const int32_t* unit_capacity;   /* [U] FIFO capacity (kept-list cap, K3)  */
  const double* vals;             /* sample pools (float64)                 */
  const int32_t* pool_off;        /* own-input per-bucket output pools      */
  const int32_t* pool_len;
  const double* succ_cum;         /* cumulative successor probabilities     */
  const int32_t* succ_nxt;        /* next local unit, -1 = terminate        */
  const void* conds;              /* K3 (unit, upstream) descriptors        */
  const void* pairs;              /* K3 joined records                      */
  const uint64_t* jump;           /* PCG64 jump tables [3][1024][4]         */
  double prefill_rate, decode_rate; /* RateProfile (pdgraph.py:282-291)     */
  const uint64_t* succ_thr;       /* ceil(succ_cum * 2^53): integer cum <= u */
  int32_t max_units;              /* max over graph_n                        */
  const double* vals_div;         /* vals with LLM input pools / prefill_rate */
                                  /* and output pools / decode_rate (exact  */
                                  /* f64 divisions); durations as in vals   */
  int32_t features;               /* PDG_BANK_FEATURES_VALID | OR of the    */
                                  /* PDG_BANK_HAS_* kinds the bank holds;   */
                                  /* a speed hint only (0: assume all)      */
  const uint8_t* unit_class;      /* [U] optional scheduling hint: expected */
                                  /* remaining walk length class 0..15 of a */
                                  /* job starting at the unit; the engine   */
                                  /* hands out jobs longest-first when set  */
                                  /* and the scratch holds 8 * n_jobs bytes */
                                  /* (results do not depend on it)          */
} pdg_graph_bank;
enum {
  PDG_BANK_HAS_LLM = 1,           /* LLM units (input/output pools)         */
  PDG_BANK_HAS_OWN_INPUT = 2,     /* output_own_input pools                 */
  PDG_BANK_HAS_CONDITIONS = 4,    /* K3 masks (estimator.py:299)            */
  PDG_BANK_FEATURES_VALID = 0x40000000
};

typedef struct {
  const int32_t* graph;           /* [N] graph index in the bank                      */
  const int32_t* unit;            /* [N] current unit (index in sorted unit ids)      */
  const uint64_t* seed;           /* [N] np.random.default_rng seed (>= 0)           */
  const int32_t* obs_unit;        /* [N] relevant observed upstream unit, -1 = none   */
  const double* obs_val;          /* [N,3] (input_len, output_len, parallelism)      */
} pdg_mc_jobs;

typedef struct {
  double* samples;                /* [N, samples_stride] optional raw samples         */
  int64_t samples_stride;
  double* lo;                     /* histogram rows (pdg_hist_rows layout)            */
  double* width;
  int32_t* nbins;
  int32_t* nsamp;
  uint16_t* counts;
  int64_t stride;
  const int32_t* slot;            /* [N] row written for job i (NULL: row i)          */
  int32_t* capped;                /* [N] walks that hit the visit cap (optional)      */
  uint8_t* flags;                 /* [N] bit0 conditioned, bit1 override, bit2 serial,
                                     bit3 Lemire rejection redrawn in the fast kernel */
  double* mean;                   /* [rows] RemainingDemand.mean() (optional; Python  */
                                  /*   sum() semantics, see pdg_policy_keys)          */
  double* worst;                  /* [rows] max(samples) = worst_case (optional)      */
} pdg_mc_out;

/* Scratch for pdg_mc_remaining_demand: pdg_mc_scratch_bytes(n, max_pairs,
 * pdg_mc_grid_warps()) + 4 * n_jobs bytes (8 * n_jobs for the
 * longest-first job order, pdg_graph_bank.unit_class).  A numpy Lemire rejection (the
 * bounded draw redrawn, shifting every later half) is handled for n <= 512 by
 * a second, careful launch of the walk kernel over the handed-back
 * applications, which redraws the rejecting visit's bounded values with the
 * sequential generator (flags bit3); for n > 512 the application is replayed
 * by a sequential kernel in the same call (flags bit2). */
int pdg_mc_grid_warps(void);
size_t pdg_mc_scratch_bytes(int32_t n_samples, int32_t max_pairs, int32_t grid_warps);
int pdg_mc_remaining_demand(const pdg_graph_bank* bank, const pdg_mc_jobs* jobs,
                            int64_t n_jobs, int32_t n_samples, int32_t visit_cap,
                            int32_t bucket_count, int32_t max_unit_k, int32_t max_pairs,
                            const pdg_mc_out* out, void* scratch, size_t scratch_bytes,
                            void* stream);

/* ---------------------------------------------------------------------------
 * K1c  the other demand-aware priority keys over the device queue
 * (SURVEY.md 8(f) row 1), from the per-row outputs of the demand engine:
 *   PDG_POLICY_SRPT_MEAN  key = mean - (age - est_age)
 *                         compute_priority SRPT_MEAN (sched.py:216-218)
 *   PDG_POLICY_LSTF       key = deadline - now - ((worst + est_age) - age)
 *                         compute_priority LSTF -> lstf_slack (sched.py:219-224,
 *                         132-140); max(s + e) == max(s) + e bit-exactly
 * mean is RemainingDemand.mean() = sum(samples) / n (estimator.py:55-56) with
 * CPython >= 3.12 sum() semantics (Neumaier-compensated, in sample order),
 * written by the engine when pdg_mc_out.mean is set.  Keys are float64,
 * bit-identical to the reference; out_key (optional) is the order-preserving
 * uint64 image of the float64 key (sort with pdg_order, begin_bit = 0, on rows
 * in arrival order).  deadline may be NULL for SRPT_MEAN.  row_idx as in
 * pdg_gittins_score_hist.
 * ------------------------------------------------------------------------- */
enum { PDG_POLICY_SRPT_MEAN = 1, PDG_POLICY_LSTF = 2 };
int pdg_policy_keys(int32_t policy, const double* mean, const double* worst,
                    const double* est_age, const double* age, const double* deadline,
                    double now, int64_t n, const int32_t* row_idx, double* out_key_f64,
                    uint64_t* out_key, void* stream);

/* ---------------------------------------------------------------------------
 * K6  dispatch / preemption plan: the consumer of the
 * priority keys.  Replaces the min()/max() scans of Simulator._dispatch and
 * Simulator._preempt (simcore.py:512-516, 652-687) over _task_sort_key
 * (simcore.py:339-344) on one PriorityRefresh (simcore.py:636-644): first the
 * preemption swaps of every backend, then the dispatch fill of every backend.
 * Task t: backend[t] in [0, n_backends), active[t] (1 = holds a slot),
 * key[t] = the app's Priority.key (float64), app_rank[t] = position of the
 * app's (arrival_time, app_instance_id) in arrival order, stage[t] /
 * request[t] < 65536.  slots[b] <= 1024.  Events of backend b land in
 * ev_task/ev_kind[b * ev_cap ...]: ev_count[b] preemption events (pairs:
 * kind 1 = preempt, 2 = start), then ev_count[n_backends + b] dispatch starts
 * (kind 2).  ev_cap >= 3 * max(slots) always suffices.  After the call,
 * pdg_dispatch_status reports 0 = ok, 1 = a backend had more running tasks
 * than slots, 2 = a plan needed more than 2 * slots waiting candidates.
 * temp: pdg_dispatch_temp_bytes(n, n_backends) bytes of device scratch.
 * ------------------------------------------------------------------------- */
size_t pdg_dispatch_temp_bytes(int64_t n, int32_t n_backends);
int pdg_dispatch_plan(const int32_t* backend, const uint8_t* active, const double* key,
                      const uint32_t* app_rank, const int32_t* stage, const int32_t* request,
                      int64_t n, const int32_t* slots, int32_t n_backends, double hysteresis,
                      int32_t preempt, int32_t ev_cap, int32_t* ev_task, uint8_t* ev_kind,
                      int32_t* ev_count, void* temp, size_t temp_bytes, void* stream);
int pdg_dispatch_status(const void* temp, int64_t n, int32_t n_backends, int32_t* status_out,
                        void* stream);

/* a11b: Simulator._update_attained (simcore.py:306-313) for every application
 * of a queue: age_out[a] = completed[a] + max(progress[a], max over tasks t
 * with task_app[t] == a, task_active[t] != 0 and task_start[t] not NaN (the
 * backends' active tasks that have started) of min(task_service[t],
 * max(0, now - (task_start[t] + task_cold[t])))).  Bit-identical to the
 * reference loop (the max is order-free).  age_out may alias progress or
 * completed.  temp: 8 * n_apps bytes. */
int pdg_attained_service(const double* completed, const double* progress, int64_t n_apps,
                         const int32_t* task_app, const uint8_t* task_active,
                         const double* task_start, const double* task_cold,
                         const double* task_service, int64_t n_tasks, double now,
                         double* age_out, void* temp, size_t temp_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * K4a  batched plan_prewarm (prewarm.py:42-96), bit-exact: one job per
 * (application, successor).  Job j's completion samples (absolute times, the
 * caller's completion_dist.samples) are pool[off[j] .. off[j]+len[j]).
 * has_plan[j] = 0 when p_s < knob (the reference returns None); otherwise the
 * PrewarmPlan's (trigger_time, p_e).  Callers validate knob in [0,1], t_p >= 0.
 * ------------------------------------------------------------------------- */
int pdg_plan_prewarm(const double* pool, const int32_t* off, const int32_t* len,
                     const int32_t* bucket_count, const double* p_s, const double* t_p,
                     const double* knob, const double* now, int64_t n_jobs,
                     uint8_t* has_plan, double* trigger, double* p_e, void* stream);

/* ---------------------------------------------------------------------------
 * K4b  need probability per backend type and time window (BASELINE config 5).
 * need[a, t, k] = sum over successors v of a's current unit with type(v) = t
 * of p_s(v) * P(completion < now + W_k), completion = now + the current
 * unit's unconditioned service samples (simcore.py:480-487) conditioned on
 * "> now" as plan_prewarm does (prewarm.py:65-67).  agg[t, k] (optional) is
 * the sum over applications (expected number of applications needing a warm
 * type-t backend within W_k).  <= 32 windows, <= 64 types, <= 4 successors
 * per unit (further successors are ignored).
 * ------------------------------------------------------------------------- */
typedef struct {
  const double* svc_sorted;   /* service samples per unit, ascending          */
  const int32_t* svc_off;     /* [U]                                           */
  const int32_t* svc_len;     /* [U]                                           */
  const int32_t* graph_base;  /* [G]                                           */
  const int32_t* succ_off;    /* [U] into succ_nxt / succ_p                    */
  const int32_t* succ_len;    /* [U]                                           */
  const int32_t* succ_nxt;    /* local unit index of each successor            */
  const double* succ_p;       /* branch probability (pdgraph.py:182-194)       */
  const int32_t* unit_type;   /* [U] warm-content backend type, -1 = none      */
  const int32_t* win_idx;     /* optional [U, n_windows]: pdg_prewarm_window_index */
                              /* of the windows passed to pdg_prewarm_need       */
  const int32_t* unit_rec;    /* optional [U, 12], 16-B aligned: svc_off, svc_len, */
                              /* backend type of successors 0..3 (-1 = none),     */
                              /* float bits of (float)p_s of successors 0..3, 0, 0 */
} pdg_prewarm_tables;

/* lower_bound(svc_sorted[u], windows[k]) for every unit and window: lets
 * pdg_prewarm_need skip its per-application searches (a sample below W_k can
 * still complete at now + W_k after rounding; the kernel walks those back). */
int pdg_prewarm_window_index(const pdg_prewarm_tables* tables, int32_t n_units,
                             const double* windows, int32_t n_windows, int32_t* out,
                             void* stream);

int pdg_prewarm_need(const pdg_prewarm_tables* tables, const int32_t* graph,
                     const int32_t* unit, const double* now, int64_t n,
                     const double* windows, int32_t n_windows, int32_t n_types,
                     float* need, double* agg, void* stream);

/* Config 5's per-successor plans: plan_prewarm (prewarm.py:42-96) for every
 * (application, successor slot) of a queue, with the completion distribution
 * _plan_prewarms builds (simcore.py:450-478: now + the current unit's service
 * samples, bucket_count buckets), p_s the branch probability and t_p =
 * warmup_by_type[type of the successor].  Outputs [n, slots], successors in
 * sorted order as _plan_prewarms iterates them.  has_plan[a, s]:
 *   0  no plan: no successor in slot s, its successor has no warm content
 *      (type < 0), or plan_prewarm returned None;
 *   1  plan (trigger, p_e), bit-identical to plan_prewarm;
 *   PDG_PLAN_OVERFLOW  (every slot of the application) its unit has more
 *      than `slots` successors -- pass slots >= the bank's largest fan-out;
 *   PDG_PLAN_BAD_TYPE  the successor's type is >= n_types (no warmup entry).
 * temp: pdg_prewarm_triggers_temp_bytes(n, slots) bytes. */
#define PDG_PLAN_OVERFLOW 2
#define PDG_PLAN_BAD_TYPE 3
size_t pdg_prewarm_triggers_temp_bytes(int64_t n, int32_t slots);
int pdg_prewarm_triggers(const pdg_prewarm_tables* tables, const int32_t* graph,
                         const int32_t* unit, const double* now, int64_t n, int32_t slots,
                         const double* warmup_by_type, int32_t n_types, double knob,
                         int32_t bucket_count, uint8_t* has_plan, double* trigger, double* p_e,
                         void* temp, size_t temp_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Correlation masks: estimator.pearson (estimator.py:
 * 62-81) for a batch of (x, y) pairs laid out at x/y[off[j] .. off[j]+len[j]);
 * rho[j] = NaN where the reference raises (fewer than 2 points, constant
 * input), flag[j] = |rho| > threshold as _flag / build_masks set the mask
 * (estimator.py:97-142).  Sums follow CPython sum(); squares are d*d (the
 * reference's d**2 goes through libm pow, up to one ulp apart).
 * ------------------------------------------------------------------------- */
int pdg_pearson_flags(const double* x, const double* y, const int32_t* off, const int32_t* len,
                      int64_t n_jobs, double threshold, double* rho, uint8_t* flag,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PDG_B200_H */
