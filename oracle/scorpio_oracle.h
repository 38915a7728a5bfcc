/* TEST INFRASTRUCTURE ONLY: CPU restatement of the reference slosim hot path.
 * See scorpio_oracle.c for the reference file:line map. */
#ifndef SCORPIO_ORACLE_H
#define SCORPIO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_STATUS_COMPLETED = 0, /* core.Status, core.py:19-25 */
  ORC_STATUS_REJECTED_TTFT = 1,
  ORC_STATUS_REJECTED_ADMISSION = 2,
  ORC_STATUS_INCOMPLETE = 3,
};

enum {
  ORC_POLICY_SCORPIO = 0,
  ORC_POLICY_GREEDY = 1,
  ORC_POLICY_SJF = 2,
  ORC_POLICY_EARLY_REJECT = 3,
};

enum {
  ORC_FLAG_TTFT_GUARD = 1,
  ORC_FLAG_TPOT_GUARD = 2,
  ORC_FLAG_R_ONLY = 4,
  ORC_FLAG_HAS_HORIZON = 8,
  ORC_FLAG_PREFILL_PRIORITY = 16,
};

enum {
  ORC_OK = 0,
  ORC_ERR_UNSORTED = -1,
  ORC_ERR_RANGE = -2,
  ORC_ERR_NO_WORK_RUNNING = -3, /* EngineError, simengine.py:217 */
  ORC_ERR_NO_PROGRESS = -4,     /* EngineError, simengine.py:220,224 */
};

typedef struct {
  double alpha, beta, gamma, delta, epsilon; /* ItlParams */
  double phi, theta, alpha_p, beta_p;        /* PrefillParams */
} orc_cost;

typedef struct {
  int32_t policy;
  int32_t flags;
  int32_t max_batch_size;
  int32_t _pad;
  double horizon;
  orc_cost cost;
} orc_sim_params;

typedef struct {
  int64_t n;
  const double* arrival; /* already divided by the rate factor */
  const double* ttft_slo; /* already multiplied by the SLO scale */
  const double* tpot_slo;
  const int32_t* prompt_len;
  const int32_t* true_out;
  const int64_t* id;
  const int32_t* predicted;
} orc_trace;

typedef struct {
  int8_t* status;
  int8_t* compliant;
  int32_t* completion_step;
  double* first_token_time;
  double* completion_time;
  double* ttft;
  double* tpot;
} orc_outcomes;

typedef struct {
  int64_t status;
  int64_t n_steps;
  int64_t n_plans;
  int64_t n_idle_skips;
  int64_t request_steps;
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
  uint64_t digest;
} orc_summary;

typedef struct {
  int64_t step_cap, id_cap;
  double *now, *end, *prefill_s, *decode_s, *vbs, *min_slo;
  int32_t *n_admitted, *n_rejected, *n_batch;
  int64_t* ids; /* per step: admitted ids, rejected (id*2+is_admission), batch ids */
  int64_t n_steps, n_ids;
  int32_t overflow;
} orc_log;

int orc_run(const orc_trace* tr, const orc_sim_params* p, orc_outcomes* out, orc_summary* sum,
            orc_log* log);
uint64_t orc_digest_item(uint64_t step, uint32_t tag, uint32_t pos, uint64_t val);
int orc_credit_exponent(int64_t n, const double* tpot_slo, int* out_exp);

#ifdef __cplusplus
}
#endif
#endif
