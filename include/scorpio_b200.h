/*
 * scorpio_b200 -- C ABI of the B200-native Scorpio scheduling hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every pointer passed to an
 * sl_* entry point that is documented as "device" must be CUDA device memory
 * on the current device; calls are asynchronous on `stream` and return 0 or a
 * negative SL_ERR_* code (no exceptions cross the ABI).  Per-simulation
 * engine failures are reported in sl_result.status (SL_SIM_*), which the
 * Python layer maps to slosim's EngineError (simengine.py:42-43).
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/slosim):
 *   sl_run_batch        <- simengine.run(trace, SimConfig)        simengine.py:168-303
 *                          (one call = many independent (trace, SimConfig) cells,
 *                           as report.sweep would issue them, report.py:180-221)
 *                          with ScorpioPolicy / plan_step          sched_scorpio.py:210-346
 *                          and the baselines                       sched_baselines.py:49-150
 *   sl_plan_step_batch  <- sched_scorpio.plan_step(state, ...)     sched_scorpio.py:210-316
 *                          over many independent SchedulerStates   schedtypes.py:60-64
 *   sl_ttft_sort_batch  <- the LDF sort inside ttft_guard          sched_scorpio.py:193
 *   sl_guard_admit_batch<- ttft_guard walk + admission scan        sched_scorpio.py:196-294
 *   sl_credit_select_batch <- select_batch                         sched_scorpio.py:161-180
 *   sl_predict_batch    <- LengthPredictor.predict                 predictor.py:115-126
 */
#ifndef SCORPIO_B200_H
#define SCORPIO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define SL_OK 0
#define SL_ERR_ARG (-1)
#define SL_ERR_CUDA (-2)
#define SL_ERR_NO_DEVICE (-3)

/* ---- per-sim status word (sl_result.status) ---------------------------- */
#define SL_SIM_OK 0
#define SL_SIM_NO_WORK_RUNNING 1 /* EngineError simengine.py:217 */
#define SL_SIM_NO_PROGRESS 2     /* EngineError simengine.py:220,224 */
#define SL_SIM_LOG_OVERFLOW 4    /* decision log capacity exceeded (run continues) */
#define SL_SIM_CAPACITY 8        /* fast kernel handoff: rerun by the general kernel (never final) */

/* ---- request status (core.Status, core.py:19-25) ----------------------- */
#define SL_COMPLETED 0
#define SL_REJECTED_TTFT 1
#define SL_REJECTED_ADMISSION 2
#define SL_INCOMPLETE 3

/* ---- policies (SimConfig.policy, simengine.py:64-77) ------------------- */
#define SL_POLICY_SCORPIO 0
#define SL_POLICY_GREEDY 1
#define SL_POLICY_SJF 2
#define SL_POLICY_EARLY_REJECT 3

/* ---- flags (ScorpioConfig sched_scorpio.py:43-60, BaselineConfig, horizon) */
#define SL_FLAG_TTFT_GUARD 1
#define SL_FLAG_TPOT_GUARD 2
#define SL_FLAG_R_ONLY 4
#define SL_FLAG_HAS_HORIZON 8
#define SL_FLAG_PREFILL_PRIORITY 16
#define SL_FLAG_GENERAL_ONLY 32 /* host: skip the register-resident fast kernel */

/* ---- sl_run_batch_ex modes --------------------------------------------- */
#define SL_MODE_AUTO 0    /* fast kernel, then the general kernel for handoffs */
#define SL_MODE_GENERAL 1 /* general kernel only (parity cross-check) */

typedef struct {
  double alpha, beta, gamma, delta, epsilon; /* ItlParams, costmodel.py:31-47 */
  double phi, theta, alpha_p, beta_p;        /* PrefillParams, costmodel.py:50-65 */
} sl_cost;

/* One simulation cell: a trace view under one SimConfig (simengine.py:46-61).
 * The rate axis divides arrivals by rate_factor (workload.rescale_arrivals,
 * workload.py:140-155); the SLO axis multiplies both thresholds by slo_scale.
 * Both are single IEEE operations applied on device, identical to building
 * the scaled Request objects on the host. */
typedef struct {
  int32_t trace;          /* index into sl_traces */
  int32_t policy;         /* SL_POLICY_* */
  int32_t flags;          /* SL_FLAG_* */
  int32_t max_batch_size; /* BaselineConfig.max_batch_size */
  double slo_scale;
  double rate_factor;
  double horizon; /* used iff SL_FLAG_HAS_HORIZON */
  int32_t credit_exp;  /* E of the fixed-point credits (sl_credit_params) */
  int32_t credit_wide; /* 1 -> 128-bit credits */
  int64_t ws_offset;   /* first request slot of this sim in the workspace */
  int64_t out_offset;  /* first row of this sim in sl_outcomes, -1 = none */
  int64_t log_slot;    /* row in sl_log, -1 = no log */
  sl_cost cost;
} sl_sim;

/* Trace table (device).  Request r of trace t lives at begin[t] + r. */
typedef struct {
  int32_t n_traces;
  int32_t _pad;
  const int64_t* begin; /* [n_traces + 1] */
  const double* arrival;
  const double* ttft_slo;
  const double* tpot_slo;
  const int32_t* prompt_len;
  const int32_t* true_out;
  const int32_t* predicted; /* LengthPredictor.predict output per request */
  const int64_t* id;
} sl_traces;

/* Per-sim result row: what summarize()/goodput()/adherence() reduce to
 * (report.py:71-134, core.py:168-179).  This is the row NCCL gathers. */
typedef struct {
  int32_t status;
  int32_t _pad;
  int64_t n_steps; /* work steps == len(EventLog.steps) */
  int64_t n_plans; /* plan_step calls */
  int64_t n_idle_skips;
  int64_t request_steps; /* sum over plans of |waiting| + |running| at entry */
  int64_t total;
  int64_t completed;
  int64_t compliant;
  int64_t rejected_ttft;
  int64_t rejected_admission;
  int64_t incomplete;
  int64_t ttft_violations;
  int64_t tpot_violations;
  double sim_end;
  double horizon;
  double goodput;
  double adherence;
  uint64_t digest; /* work-step decision digest */
} sl_result;

/* Optional per-request outcomes (RequestOutcome, core.py:59-77). */
typedef struct {
  int8_t* status;
  int8_t* compliant;
  int32_t* completion_step;
  double* first_token_time;
  double* completion_time;
  double* ttft;
  double* tpot;
} sl_outcomes;

/* Per-sim RunReport reductions (report.summarize, report.py:71-127) computed on
 * the device from the outcomes an sl_run_batch wrote (cells with outcomes):
 * nearest-rank p50/p90/p99 of TTFT (s) and TPOT (ms) over completed requests
 * (NaN when none; n_completed = -1 for cells without outcomes).
 * status_first[k]: index of the first request whose status code is k (total
 * when none) -- summarize() builds status_counts in first-occurrence order. */
typedef struct {
  double ttft_p[3];
  double tpot_ms_p[3];
  int64_t n_completed;
  int64_t status_first[4];
} sl_report_row;

/* Optional decision log (EventLog.steps, simengine.py:80-137), one row per
 * sim with log_slot >= 0: step_cap steps and id_cap ids per stream per row.
 * Ids of step k are the next n_admitted[k] / n_rejected[k] / n_batch[k]
 * entries of the three streams; rejected ids are encoded id*2+is_admission. */
typedef struct {
  int64_t step_cap, id_cap;
  double *now, *end, *prefill_s, *decode_s, *vbs, *min_slo; /* [rows*step_cap] */
  int32_t *n_admitted, *n_rejected, *n_batch;              /* [rows*step_cap] */
  int64_t *adm_ids, *rej_ids, *batch_ids;                  /* [rows*id_cap] */
  int64_t* n_steps; /* [rows] steps recorded */
  double* adm_rec;  /* [rows*id_cap*5] may be NULL: AdmissionRecord (vbs, l_avg, min_slo,
                       estimate, threshold) per admitted id of the scorpio TPOT guard */
  int64_t skip_cap;
  double* skip_now;     /* [rows*skip_cap] idle skips (EventLog.idle_skips) */
  double* skip_target;  /* [rows*skip_cap] */
  int32_t* skip_waiting; /* [rows*skip_cap] */
  int64_t* n_skips;     /* [rows] */
} sl_log;

/* Workspace bytes for `total_slots` request slots (sum over sims of trace length). */
int64_t sl_workspace_bytes(int64_t total_slots, int32_t n_sims);

/* Fixed-point credit parameters for one sim (host helper, no device work):
 * E = min over the sim's scaled TPOT SLOs of (frexp exponent - 53); wide = 1
 * when 2*max S >= 2^64. */
int sl_credit_params(int64_t n, const double* tpot_slo, double slo_scale, int32_t* credit_exp,
                     int32_t* credit_wide);

/* Run n_sims independent simulations to completion.  `traces`, `outcomes`
 * and `log` are host structs holding device pointers; `sims`, `order`,
 * `workspace` (sl_workspace_bytes(total_slots) bytes) and `results` are
 * device pointers.  order[] is the schedule (longest expected first); NULL =
 * 0..n_sims-1.  outcomes / log may be NULL. */
int sl_run_batch(const sl_traces* traces, const sl_sim* sims, const int32_t* order, int32_t n_sims,
                 void* workspace, int64_t total_slots, sl_result* results,
                 const sl_outcomes* outcomes, const sl_log* log, void* stream);

/* sl_run_batch with an explicit SL_MODE_*. */
int sl_run_batch_ex(const sl_traces* traces, const sl_sim* sims, const int32_t* order,
                    int32_t n_sims, void* workspace, int64_t total_slots, sl_result* results,
                    const sl_outcomes* outcomes, const sl_log* log, int32_t mode, void* stream);

/* RunReport reductions for n_sims cells (one launch): rows[n_sims]; per-category
 * totals / compliant counts cat_counts[n_sims][n_categories][2] for categories
 * 0..n_categories-1 (category[begin[t] + i] = category of request i of trace t,
 * may be NULL = all 0).  Replaces the per-run summarize() loop of report.sweep. */
int sl_report_batch(const sl_traces* traces, const sl_sim* sims, int32_t n_sims,
                    const sl_outcomes* outcomes, const int8_t* category, int32_t n_categories,
                    sl_report_row* rows, int64_t* cat_counts, void* stream);

/* Cumulative SLO-met series per sim (report.summarize's `cumulative`,
 * report.py:92): the completion times of the compliant requests, ascending,
 * written to out_times[out_offset .. out_offset + n_out[s]) (point i of the
 * series is (out_times[out_offset + i], i + 1)); n_out[s] = -1 for a sim
 * without outcomes.  scratch: device buffer of at least as many u64 as
 * out_times (the sort's second buffer).  One CTA per sim, stream-ordered. */
int sl_cumulative_batch(const sl_traces* traces, const sl_sim* sims, int32_t n_sims,
                        const sl_outcomes* outcomes, double* out_times, uint64_t* scratch,
                        int64_t* n_out, void* stream);

/* Number of kernels sl_run_batch launches per call (for the gpu_launches claim). */
int sl_run_batch_launches(void);

/* Self-test of the hot path's exact small-divisor division (device pointers):
 * out[i] = a[i] / b[i], a[i] an integer in [0, 2^53), 1 <= b[i]; must equal the
 * correctly rounded quotient (Python int / int), e.g. the L-average of
 * costmodel.itl (simengine.py:235-237) and _admission_math (sched_scorpio.py:104). */
int sl_selftest_div_small(const double* a, const int32_t* b, double* out, int64_t n, void* stream);

/* Self-test of the certified CPython sum used by the few-large-segments folds
 * (sum(1/slo), sched_scorpio.py:121; vbs, :312-315): for each s, the double-
 * double sum of the positive terms x[begin[s], begin[s+1]) (device pointers)
 * and its certificate.  out[3s] = the value CPython's sum() returns when the
 * certificate holds, else NaN; out[3s+1], out[3s+2] = the double-double. */
int sl_selftest_certified_sum(const double* x, const int64_t* begin, int32_t n_sums, double* out,
                              void* stream);

/* ---- batched plan_step over independent SchedulerStates ---------------
 * (sched_scorpio.plan_step, sched_scorpio.py:210-316; config 2).  A batch is S
 * "segments", each one SchedulerState (schedtypes.py:60-64): its waiting items
 * in current queue order and its running entries in admission order. */
#define SL_PLAN_WAITING 0
#define SL_PLAN_REJECTED_TTFT 1
#define SL_PLAN_REJECTED_ADMISSION 2
#define SL_PLAN_ADMITTED 3
#define SL_PLAN_GUARD_ONLY 64 /* flag: ttft_guard alone (no admission, sched_scorpio.py:183) */
#define SL_PLAN_FCFS_WALK 128 /* flag: TTFT walk over the unsorted FCFS queue
                                 (early_reject, sched_baselines.py:89-106) */
#define SL_PLAN_EXACT_WALK 256 /* flag: some prefill_s < 0 (legal when alpha_p < 0,
                                  costmodel.py:59-65): prefixes may shrink, so the
                                  walk runs without its monotone shortcuts */

typedef struct {
  int32_t n_segments;
  int32_t _pad;
  const int64_t* w_begin; /* [S+1] waiting-item ranges */
  const int64_t* r_begin; /* [S+1] running-entry ranges */
  /* waiting items (WaitingItem + its Request) */
  const double* w_arrival;
  const double* w_ttft;
  const double* w_tpot;
  const double* w_prefill; /* WaitingItem.prefill_s */
  const int32_t* w_prompt;
  const int32_t* w_pred; /* WaitingItem.predicted_len */
  const int64_t* w_id;
  /* running entries (RunningEntry) */
  const double* r_tpot;
  const int32_t* r_cur_len; /* prompt_len + tokens_generated */
  const int64_t* r_id;
  const uint64_t* r_credit; /* credit * tpot / 2^E (exact fixed point) */
  const uint8_t* r_exclude; /* may be NULL: 1 = excluded from the credit phase */
  /* per segment */
  const double* now;         /* [S] SchedulerState.now */
  const int32_t* credit_exp; /* [S] E (sl_credit_params over the segment's SLOs) */
} sl_plan_state;

typedef struct {
  int32_t flags; /* SL_FLAG_TTFT_GUARD | SL_FLAG_TPOT_GUARD | SL_FLAG_R_ONLY | SL_PLAN_GUARD_ONLY */
  int32_t _pad;
  sl_cost cost;
} sl_plan_config;

typedef struct {
  int32_t* perm;      /* [W] LDF order (global waiting indices), written by the sort */
  int32_t* scratch;   /* [W] sort / walk scratch */
  int32_t* adm_order; /* [W] admitted waiting indices in admission order (per segment) */
  int32_t* w_status;  /* [W] SL_PLAN_* */
  int32_t* w_pos;     /* [W] position in the new queue / in plan.rejected / admission order */
  double* w_rec;      /* [W*5] may be NULL: AdmissionRecord vbs, l_avg, min_slo, estimate, threshold */
  uint64_t* r_credit_out; /* [R] */
  uint8_t* r_batch;       /* [R] 1 = in decode_batch */
  int32_t* r_pos;         /* [R] position in decode_batch or -1 */
  int32_t* seg_counts;    /* [S*4] waiting kept, admitted, rejected, batch */
  uint64_t* seg_min_fixed; /* [S] min fixed-point slo over running + admitted (~0 if none) */
  double* seg_vbs;        /* [S] plan.vbs */
  double* seg_min_slo;    /* [S] plan.min_slo, NaN for None */
} sl_plan_out;

/* LDF sort of every segment's waiting queue by (deadline, arrival, id)
 * (sched_scorpio.py:193).  max_w: host bound on any segment's size (selects the
 * warp-bitonic, CTA-tile or tile+merge-path path). */
int sl_ttft_sort_batch(const sl_plan_state* st, int64_t max_w, sl_plan_out* out, void* stream);
/* TTFT walk + running aggregates + admission scan + vbs/min_slo per segment
 * (sched_scorpio.py:196-294, 312-315).  Reads out->perm when TTFT_GUARD. */
int sl_guard_admit_batch(const sl_plan_state* st, const sl_plan_config* cfg, sl_plan_out* out,
                         void* stream);
/* Credit phase select_batch (sched_scorpio.py:161-180), or decode-all when
 * TPOT_GUARD is off.  The per-segment minimum comes from out->seg_min_fixed
 * when use_seg_min (after sl_guard_admit_batch), else from the running entries. */
int sl_credit_select_batch(const sl_plan_state* st, const sl_plan_config* cfg, sl_plan_out* out,
                           int32_t use_seg_min, void* stream);
/* plan_step over every segment: sort (if TTFT_GUARD) + guard/admit + select. */
int sl_plan_step_batch(const sl_plan_state* st, const sl_plan_config* cfg, int64_t max_w,
                       sl_plan_out* out, void* stream);

/* vbs(running, min_slo) (sched_scorpio.py:70-74) for S segments of running
 * entries: Neumaier sum of min_slo[s] / tpot over each segment, in order. */
int sl_vbs_batch(int32_t n_segments, const int64_t* r_begin, const double* r_tpot,
                 const double* min_slo, double* out, void* stream);

/* ---- length predictor (LengthPredictor, predictor.py:93-126) ----------- */
#define SL_PREDICT_ORACLE 0
#define SL_PREDICT_NOISY_BUCKET 1

typedef struct {
  int32_t mode;         /* SL_PREDICT_* */
  int32_t num_buckets;  /* Bucketing.num_buckets */
  const double* boundaries; /* device, [num_buckets], strictly increasing */
  double error_prob;
  int32_t error_spread;
  int32_t _pad;
  uint64_t rng_seed;    /* default_rng([rng_seed, request.id]) */
} sl_predictor;

/* predicted_len for n requests (device arrays).  clamp_count (device, may be
 * NULL) accumulates lengths above the last boundary (the reference logs a
 * warning per clamp, predictor.py:75-81). */
int sl_predict_batch(const int64_t* id, const int32_t* true_out, int64_t n,
                     const sl_predictor* p, int32_t* out_pred, unsigned long long* clamp_count,
                     void* stream);

/* ABI self-description: writes sizeof(sl_sim), sizeof(sl_result),
 * sizeof(sl_traces), sizeof(sl_outcomes), sizeof(sl_log), sizeof(sl_cost),
 * sizeof(sl_predictor) into out[0..6] (n >= 7), and sizeof(sl_report_row) into
 * out[7] when n >= 8.  Lets bindings verify their struct mirrors. */
int sl_abi_layout(int64_t* out, int32_t n);

/* Device properties used for grid sizing. */
int sl_device_info(int32_t* sm_count, int32_t* l2_bytes);

#ifdef __cplusplus
}
#endif
#endif
