/*
 * TEST INFRASTRUCTURE ONLY -- NOT PART OF THE PRODUCT PATH.
 *
 * CPU restatement (plain C, scalar, one simulation per call) of the reference
 * `slosim` hot path: the discrete-event engine `simengine.run`
 * (pkg/src/slosim/simengine.py:168-303) driving the scorpio policy
 * (`plan_step`, pkg/src/slosim/sched_scorpio.py:210-316) and the three
 * baselines (pkg/src/slosim/sched_baselines.py:49-150).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library, and only as the checker or the
 * CPU baseline.  The product path (paper_2505_23022_b200/) never calls it.
 *
 * Pinning: this restatement is checked against outputs of the real reference
 * (imported in the build container) committed as fixtures under tests/golden/
 * (generator: tests/golden/make_golden.py); see tests/test_oracle_golden.py.
 *
 * Exactness rules followed:
 *  - fp64 evaluated in Python's left-to-right order, no FMA contraction
 *    (build with -ffp-contract=off; SSE2 doubles on x86-64).
 *  - CPython 3.12 builtin sum() over floats is Neumaier-compensated
 *    (sched_scorpio.py:74,121; simengine.py:233) -> py_sum_*.
 *  - Credits are exact rationals in the reference (schedtypes.py:52,
 *    sched_scorpio.py:77-80,176).  Every increment of entry e has
 *    denominator slo_e, so credit_e * slo_e / 2^E is an integer N_e with
 *    E = min over the sim's TPOT SLOs of (frexp exponent - 53).  N_e is kept
 *    in unsigned __int128 here (always wide).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "scorpio_oracle.h"

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* CPython 3.12 sum() over a sequence of floats (Objects/bltinmodule.c):     */
/* int 0 start, first float leaves the int path as 0 + x, then Neumaier.     */
typedef struct {
  double f, c;
  int64_t n;
} py_sum;

static void py_sum_init(py_sum* s) { s->f = 0.0; s->c = 0.0; s->n = 0; }

static void py_sum_add(py_sum* s, double x) {
  if (s->n == 0) {
    s->f = 0.0 + x;
  } else {
    double t = s->f + x;
    if (fabs(s->f) >= fabs(x))
      s->c += (s->f - t) + x;
    else
      s->c += (x - t) + s->f;
    s->f = t;
  }
  s->n++;
}

/* empty sum returns the int 0; every use site adds it to a float, so 0.0 */
static double py_sum_result(const py_sum* s) {
  double f = s->f;
  if (s->n == 0) return 0.0;
  if (s->c != 0.0 && isfinite(s->c)) f += s->c;
  return f;
}

/* ------------------------------------------------------------------------ */
/* Cost models (costmodel.py:96-138).                                        */
static double prefill_time(const orc_cost* c, int32_t prompt_len) {
  /* costmodel.py:136: int <= float compares exactly; prompt_len < 2^53 */
  if ((double)prompt_len <= c->theta) return c->phi;
  return c->alpha_p * (double)prompt_len + c->beta_p;
}

static double itl(const orc_cost* c, int64_t batch_size, double avg_len) {
  /* costmodel.py:102-107, parsed ((((a*B)*L) + b*B) + g*L) + d */
  double B = (double)batch_size;
  return c->alpha * B * avg_len + c->beta * B + c->gamma * avg_len + c->delta;
}

/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t idx; /* position of the request in the trace */
  int32_t predicted_len;
  double prefill_s;
} witem; /* WaitingItem, schedtypes.py:18-36 */

typedef struct {
  int32_t idx;
  int32_t predicted_len;
  double prefill_s;
  int64_t tokens;
  u128 credit; /* credit * slo / 2^E, exact */
} rentry;      /* RunningEntry, schedtypes.py:39-57 */

typedef struct {
  /* trace (already rate/SLO scaled by the caller) */
  int64_t n;
  const double* arrival;
  const double* ttft_slo;
  const double* tpot_slo;
  const int32_t* prompt_len;
  const int32_t* true_out;
  const int64_t* id;
  const int32_t* predicted;
  const orc_sim_params* p;
  int credit_exp;
  /* state */
  witem* waiting;
  int64_t n_waiting;
  rentry* running;
  int64_t n_running;
  double now;
  /* per-request scratch */
  double* first_emit;
  int64_t* n_emits;
} sim_t;

static u128 slo_fixed(const sim_t* s, double slo) {
  /* exact: slo = m * 2^(e-53); E <= e-53, so slo * 2^-E is an integer */
  return (u128)ldexp(slo, -s->credit_exp);
}

static int wkey_less(const sim_t* s, const witem* a, const witem* b) {
  /* sort_key = (deadline, arrival_time, id), schedtypes.py:28-32 */
  double da = s->arrival[a->idx] + s->ttft_slo[a->idx];
  double db = s->arrival[b->idx] + s->ttft_slo[b->idx];
  if (da != db) return da < db;
  if (s->arrival[a->idx] != s->arrival[b->idx]) return s->arrival[a->idx] < s->arrival[b->idx];
  return s->id[a->idx] < s->id[b->idx];
}

/* stable insertion sort: list.sort is stable and the key is total anyway */
static void sort_waiting(sim_t* s) {
  for (int64_t i = 1; i < s->n_waiting; i++) {
    witem x = s->waiting[i];
    int64_t j = i - 1;
    while (j >= 0 && wkey_less(s, &x, &s->waiting[j])) {
      s->waiting[j + 1] = s->waiting[j];
      j--;
    }
    s->waiting[j + 1] = x;
  }
}

static int sjf_less(const sim_t* s, const witem* a, const witem* b) {
  /* sched_baselines.py:138-142 key (predicted_len, arrival_time, id) */
  if (a->predicted_len != b->predicted_len) return a->predicted_len < b->predicted_len;
  if (s->arrival[a->idx] != s->arrival[b->idx]) return s->arrival[a->idx] < s->arrival[b->idx];
  return s->id[a->idx] < s->id[b->idx];
}

/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t* admitted; /* indices into running (positions after append) */
  int64_t n_admitted;
  int32_t* batch; /* positions in running */
  int64_t n_batch;
  int32_t* rej_idx;
  int8_t* rej_reason; /* ORC_STATUS_REJECTED_TTFT / _ADMISSION */
  int64_t n_rej;
  double vbs;
  double min_slo; /* NAN when None */
} plan_t;

/* _admission_math, sched_scorpio.py:83-114 */
static int admission_math(int64_t n, double inv_slo_sum, double len_sum_f, int64_t len_sum_i,
                          int use_int_len, int has_min, double min_running_slo,
                          double candidate_slo, int32_t candidate_len, int32_t predicted_len,
                          const orc_cost* cost, int r_only) {
  double min_slo;
  if (!has_min || candidate_slo < min_running_slo)
    min_slo = candidate_slo;
  else
    min_slo = min_running_slo;
  double new_vbs = min_slo * (inv_slo_sum + 1.0 / candidate_slo);
  double l_avg;
  if (use_int_len) /* int / int true division: correctly rounded */
    l_avg = (double)(len_sum_i + candidate_len) / (double)(n + 1);
  else /* float + int, then / int */
    l_avg = (len_sum_f + (double)candidate_len) / (double)(n + 1);
  double estimate = cost->epsilon * ((cost->alpha * new_vbs + cost->gamma) *
                                         (l_avg + (double)predicted_len / 2.0) +
                                     cost->beta * new_vbs + cost->delta);
  double threshold = (r_only && has_min) ? min_running_slo : min_slo;
  return estimate <= threshold;
}

static void plan_scorpio(sim_t* s, plan_t* pl) {
  const orc_sim_params* p = s->p;
  int ttft_guard = (p->flags & ORC_FLAG_TTFT_GUARD) != 0;
  int tpot_guard = (p->flags & ORC_FLAG_TPOT_GUARD) != 0;
  int r_only = (p->flags & ORC_FLAG_R_ONLY) != 0;
  int64_t running_before = s->n_running;

  if (ttft_guard) { /* ttft_guard, sched_scorpio.py:183-207 */
    sort_waiting(s);
    int64_t k = 0;
    double prefix = 0.0;
    for (int64_t i = 0; i < s->n_waiting; i++) {
      witem it = s->waiting[i];
      double elapsed = s->now - s->arrival[it.idx];
      double estimate = elapsed + prefix + it.prefill_s;
      if (estimate > s->ttft_slo[it.idx]) {
        pl->rej_idx[pl->n_rej] = it.idx;
        pl->rej_reason[pl->n_rej] = ORC_STATUS_REJECTED_TTFT;
        pl->n_rej++;
      } else {
        prefix += it.prefill_s;
        s->waiting[k++] = it;
      }
    }
    s->n_waiting = k;
  }

  if (tpot_guard) { /* sched_scorpio.py:234-294 */
    /* _running_aggregates, :117-124 */
    int64_t n = s->n_running;
    py_sum ps;
    py_sum_init(&ps);
    int64_t lens = 0;
    int has_min = 0;
    double min_running = 0.0;
    for (int64_t j = 0; j < s->n_running; j++) {
      const rentry* e = &s->running[j];
      py_sum_add(&ps, 1.0 / s->tpot_slo[e->idx]);
      lens += (int64_t)s->prompt_len[e->idx] + e->tokens;
      double v = s->tpot_slo[e->idx];
      if (!has_min || v < min_running) { min_running = v; has_min = 1; }
    }
    double inv = py_sum_result(&ps);
    int64_t k = 0;
    for (int64_t i = 0; i < s->n_waiting; i++) {
      witem it = s->waiting[i];
      double cand = s->tpot_slo[it.idx];
      int ok = admission_math(n, inv, 0.0, lens, 1, has_min, min_running, cand,
                              s->prompt_len[it.idx], it.predicted_len, &p->cost, r_only);
      if (ok) {
        double min_slo = (!has_min || cand < min_running) ? cand : min_running;
        rentry* e = &s->running[s->n_running];
        e->idx = it.idx;
        e->predicted_len = it.predicted_len;
        e->prefill_s = it.prefill_s;
        e->tokens = 0;
        e->credit = 0;
        pl->admitted[pl->n_admitted++] = (int32_t)s->n_running;
        s->n_running++;
        n += 1;
        inv += 1.0 / cand; /* plain float add, :275 */
        lens += s->prompt_len[it.idx];
        min_running = min_slo;
        has_min = 1;
        continue;
      }
      /* solo test with (0, 0.0, 0.0, None), :279-289 */
      int solo_ok = admission_math(0, 0.0, 0.0, 0, 0, 0, 0.0, cand, s->prompt_len[it.idx],
                                   it.predicted_len, &p->cost, r_only);
      if (!solo_ok) {
        pl->rej_idx[pl->n_rej] = it.idx;
        pl->rej_reason[pl->n_rej] = ORC_STATUS_REJECTED_ADMISSION;
        pl->n_rej++;
      } else {
        s->waiting[k++] = it;
      }
    }
    s->n_waiting = k;
  } else { /* admit everything in queue order, :295-304 */
    for (int64_t i = 0; i < s->n_waiting; i++) {
      witem it = s->waiting[i];
      rentry* e = &s->running[s->n_running];
      e->idx = it.idx;
      e->predicted_len = it.predicted_len;
      e->prefill_s = it.prefill_s;
      e->tokens = 0;
      e->credit = 0;
      pl->admitted[pl->n_admitted++] = (int32_t)s->n_running;
      s->n_running++;
    }
    s->n_waiting = 0;
  }

  /* fresh entries are exactly the appended tail [running_before, n_running) */
  if (tpot_guard) { /* select_batch, :161-180 */
    if (s->n_running > 0) {
      double min_slo = s->tpot_slo[s->running[0].idx];
      for (int64_t j = 1; j < s->n_running; j++) {
        double v = s->tpot_slo[s->running[j].idx];
        if (v < min_slo) min_slo = v;
      }
      u128 MIN = slo_fixed(s, min_slo);
      for (int64_t j = 0; j < running_before; j++) {
        rentry* e = &s->running[j];
        u128 S = slo_fixed(s, s->tpot_slo[e->idx]);
        e->credit += MIN;
        if (e->credit >= S) {
          e->credit -= S;
          pl->batch[pl->n_batch++] = (int32_t)j;
        }
      }
    }
  } else {
    for (int64_t j = 0; j < running_before; j++) pl->batch[pl->n_batch++] = (int32_t)j;
  }

  if (s->n_running > 0) { /* :312-315 */
    double min_slo = s->tpot_slo[s->running[0].idx];
    for (int64_t j = 1; j < s->n_running; j++) {
      double v = s->tpot_slo[s->running[j].idx];
      if (v < min_slo) min_slo = v;
    }
    pl->min_slo = min_slo;
    py_sum vs;
    py_sum_init(&vs);
    for (int64_t j = 0; j < s->n_running; j++)
      py_sum_add(&vs, min_slo / s->tpot_slo[s->running[j].idx]); /* trp, :63-67 */
    pl->vbs = py_sum_result(&vs);
  }
}

/* baselines: sched_baselines.py:49-106 */
static void admit_fcfs(sim_t* s, plan_t* pl) {
  int64_t room = (int64_t)s->p->max_batch_size - s->n_running;
  int64_t take = room > 0 ? (room < s->n_waiting ? room : s->n_waiting) : 0;
  for (int64_t i = 0; i < take; i++) {
    witem it = s->waiting[i];
    rentry* e = &s->running[s->n_running];
    e->idx = it.idx;
    e->predicted_len = it.predicted_len;
    e->prefill_s = it.prefill_s;
    e->tokens = 0;
    e->credit = 0;
    pl->admitted[pl->n_admitted++] = (int32_t)s->n_running;
    s->n_running++;
  }
  memmove(s->waiting, s->waiting + take, (size_t)(s->n_waiting - take) * sizeof(witem));
  s->n_waiting -= take;
}

static void decode_all(sim_t* s, plan_t* pl, int64_t running_before) {
  if ((s->p->flags & ORC_FLAG_PREFILL_PRIORITY) && pl->n_admitted > 0) return;
  for (int64_t j = 0; j < running_before; j++) pl->batch[pl->n_batch++] = (int32_t)j;
}

static void plan_baseline(sim_t* s, plan_t* pl) {
  int64_t running_before = s->n_running;
  if (s->p->policy == ORC_POLICY_EARLY_REJECT) {
    int64_t k = 0;
    double prefix = 0.0;
    for (int64_t i = 0; i < s->n_waiting; i++) {
      witem it = s->waiting[i];
      double elapsed = s->now - s->arrival[it.idx];
      if (elapsed + prefix + it.prefill_s > s->ttft_slo[it.idx]) {
        pl->rej_idx[pl->n_rej] = it.idx;
        pl->rej_reason[pl->n_rej] = ORC_STATUS_REJECTED_TTFT;
        pl->n_rej++;
      } else {
        prefix += it.prefill_s;
        s->waiting[k++] = it;
      }
    }
    s->n_waiting = k;
  }
  admit_fcfs(s, pl);
  decode_all(s, pl, running_before);
}

/* ------------------------------------------------------------------------ */
/* digest item: mix(val ^ (step*K_STEP + tag*K_TAG + pos*K_POS)), mix(x) = y ^ (y >> 32)
 * with y = x*K_MIX (all mod 2^64); the digest sums the items of all work steps. */
uint64_t orc_digest_item(uint64_t step, uint32_t tag, uint32_t pos, uint64_t val) {
  uint64_t key = step * 0x9E3779B97F4A7C15ULL + (uint64_t)tag * 0xC2B2AE3D27D4EB4FULL +
                 (uint64_t)pos * 0x165667B19E3779F9ULL;
  uint64_t y = (val ^ key) * 0xD6E8FEB86659FD93ULL;
  return y ^ (y >> 32);
}

/* batch id hash: low 32 bits of mix(id); the batch of a work step is the one
 * item digest_item(step, 2, n_batch, sum of batch_hid mod 2^32). */
static uint32_t orc_batch_hid(uint64_t id) {
  uint64_t y = id * 0xD6E8FEB86659FD93ULL;
  return (uint32_t)(y ^ (y >> 32));
}

static uint64_t dbits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}

int orc_credit_exponent(int64_t n, const double* tpot_slo, int* out_exp) {
  int e_min = 0x7fffffff, e_max = -0x7fffffff;
  for (int64_t i = 0; i < n; i++) {
    int e;
    frexp(tpot_slo[i], &e);
    if (e < e_min) e_min = e;
    if (e > e_max) e_max = e;
  }
  if (n == 0) { *out_exp = 0; return 0; }
  *out_exp = e_min - 53;
  /* N < 2*S_max < 2^(54 + span); must fit u128 */
  return (54 + (e_max - e_min) + 1 <= 127) ? 0 : -1;
}

/* simengine.run, simengine.py:168-303 */
int orc_run(const orc_trace* tr, const orc_sim_params* p, orc_outcomes* out, orc_summary* sum,
            orc_log* log) {
  sim_t s;
  memset(&s, 0, sizeof(s));
  memset(sum, 0, sizeof(*sum));
  s.n = tr->n;
  s.arrival = tr->arrival;
  s.ttft_slo = tr->ttft_slo;
  s.tpot_slo = tr->tpot_slo;
  s.prompt_len = tr->prompt_len;
  s.true_out = tr->true_out;
  s.id = tr->id;
  s.predicted = tr->predicted;
  s.p = p;
  for (int64_t i = 1; i < tr->n; i++)
    if (tr->arrival[i] < tr->arrival[i - 1]) return ORC_ERR_UNSORTED;
  if (orc_credit_exponent(tr->n, tr->tpot_slo, &s.credit_exp) != 0) return ORC_ERR_RANGE;

  int64_t n = tr->n;
  size_t cap = (size_t)(n > 0 ? n : 1);
  s.waiting = (witem*)malloc(cap * sizeof(witem));
  s.running = (rentry*)malloc(cap * sizeof(rentry));
  s.first_emit = (double*)malloc(cap * sizeof(double));
  s.n_emits = (int64_t*)calloc(cap, sizeof(int64_t));
  plan_t pl;
  pl.admitted = (int32_t*)malloc(cap * sizeof(int32_t));
  pl.batch = (int32_t*)malloc(cap * sizeof(int32_t));
  pl.rej_idx = (int32_t*)malloc(cap * sizeof(int32_t));
  pl.rej_reason = (int8_t*)malloc(cap * sizeof(int8_t));
  int8_t* resolved = (int8_t*)calloc(cap, 1);
  int32_t* retire_buf = (int32_t*)malloc(cap * sizeof(int32_t));
  int rc = ORC_OK;

  for (int64_t i = 0; i < n; i++) {
    out->status[i] = ORC_STATUS_INCOMPLETE;
    out->compliant[i] = 0;
    out->completion_step[i] = -1;
    out->first_token_time[i] = NAN;
    out->completion_time[i] = NAN;
    out->ttft[i] = NAN;
    out->tpot[i] = NAN;
  }

  int64_t next_arrival = 0;
  int64_t step_idx = 0;
  uint64_t digest = 0;
  int64_t log_ids = 0;
  int is_scorpio = p->policy == ORC_POLICY_SCORPIO;

  for (;;) {
    while (next_arrival < n && s.arrival[next_arrival] <= s.now) { /* :186-188 */
      int64_t i = next_arrival;
      witem it;
      it.idx = (int32_t)i;
      it.predicted_len = s.predicted[i];
      it.prefill_s = prefill_time(&p->cost, s.prompt_len[i]);
      if (p->policy == ORC_POLICY_SJF) { /* bisect.insort (right) */
        int64_t lo = 0, hi = s.n_waiting;
        while (lo < hi) {
          int64_t mid = (lo + hi) / 2;
          if (sjf_less(&s, &it, &s.waiting[mid]))
            hi = mid;
          else
            lo = mid + 1;
        }
        memmove(s.waiting + lo + 1, s.waiting + lo, (size_t)(s.n_waiting - lo) * sizeof(witem));
        s.waiting[lo] = it;
        s.n_waiting++;
      } else {
        s.waiting[s.n_waiting++] = it;
      }
      next_arrival++;
    }

    if ((p->flags & ORC_FLAG_HAS_HORIZON) && s.now >= p->horizon) break; /* :190-191 */

    sum->n_plans++;
    sum->request_steps += s.n_waiting + s.n_running;
    pl.n_admitted = pl.n_batch = pl.n_rej = 0;
    pl.vbs = 0.0;
    pl.min_slo = NAN;
    int64_t running_before = s.n_running;
    if (is_scorpio)
      plan_scorpio(&s, &pl);
    else
      plan_baseline(&s, &pl);

    for (int64_t r = 0; r < pl.n_rej; r++) { /* :197-205 */
      int32_t i = pl.rej_idx[r];
      out->status[i] = pl.rej_reason[r];
      resolved[i] = 1;
      if (pl.rej_reason[r] == ORC_STATUS_REJECTED_TTFT)
        sum->rejected_ttft++;
      else
        sum->rejected_admission++;
    }

    if (pl.n_admitted == 0 && pl.n_batch == 0) { /* idle skip, :207-227 */
      int have = 0;
      double target = 0.0;
      for (int64_t w = 0; w < s.n_waiting; w++) {
        double d = s.arrival[s.waiting[w].idx] + s.ttft_slo[s.waiting[w].idx];
        if (d > s.now && (!have || d < target)) { target = d; have = 1; }
      }
      if (next_arrival < n) {
        double a = s.arrival[next_arrival];
        if (!have || a < target) target = a;
        have = 1;
      } else if (s.n_running > 0) {
        rc = ORC_ERR_NO_WORK_RUNNING;
        break;
      }
      if (!have) {
        if (s.n_waiting > 0) rc = ORC_ERR_NO_PROGRESS;
        break;
      }
      if (target <= s.now) { rc = ORC_ERR_NO_PROGRESS; break; }
      sum->n_idle_skips++;
      s.now = target;
      continue;
    }
    (void)running_before;

    /* step duration, :233-238 */
    py_sum pre;
    py_sum_init(&pre);
    for (int64_t a = 0; a < pl.n_admitted; a++) py_sum_add(&pre, s.running[pl.admitted[a]].prefill_s);
    double prefill_s = py_sum_result(&pre);
    double decode_s = 0.0;
    if (pl.n_batch > 0) {
      int64_t lsum = 0;
      for (int64_t b = 0; b < pl.n_batch; b++) {
        const rentry* e = &s.running[pl.batch[b]];
        lsum += (int64_t)s.prompt_len[e->idx] + e->tokens;
      }
      double l_avg = (double)lsum / (double)pl.n_batch;
      decode_s = itl(&p->cost, pl.n_batch, l_avg);
    }
    double end = s.now + prefill_s + decode_s;

    /* digest + log over work steps (EventLog.steps, :273-287) */
    for (int64_t a = 0; a < pl.n_admitted; a++)
      digest += orc_digest_item((uint64_t)step_idx, 0, (uint32_t)a,
                                (uint64_t)s.id[s.running[pl.admitted[a]].idx]);
    for (int64_t r = 0; r < pl.n_rej; r++)
      digest += orc_digest_item((uint64_t)step_idx, 1, (uint32_t)r,
                                (uint64_t)s.id[pl.rej_idx[r]] * 2u +
                                    (pl.rej_reason[r] == ORC_STATUS_REJECTED_ADMISSION));
    {
      uint32_t bh = 0; /* the batch: one item over the sum of batch_hid (mod 2^32) */
      for (int64_t b = 0; b < pl.n_batch; b++)
        bh += orc_batch_hid((uint64_t)s.id[s.running[pl.batch[b]].idx]);
      digest += orc_digest_item((uint64_t)step_idx, 2, (uint32_t)pl.n_batch, bh);
    }
    digest += orc_digest_item((uint64_t)step_idx, 3, 0, dbits(end));

    if (log && log->step_cap > 0) {
      if (step_idx < log->step_cap &&
          log_ids + pl.n_admitted + pl.n_rej + pl.n_batch <= log->id_cap) {
        log->now[step_idx] = s.now;
        log->end[step_idx] = end;
        log->prefill_s[step_idx] = prefill_s;
        log->decode_s[step_idx] = decode_s;
        log->vbs[step_idx] = pl.vbs;
        log->min_slo[step_idx] = pl.min_slo;
        log->n_admitted[step_idx] = (int32_t)pl.n_admitted;
        log->n_rejected[step_idx] = (int32_t)pl.n_rej;
        log->n_batch[step_idx] = (int32_t)pl.n_batch;
        for (int64_t a = 0; a < pl.n_admitted; a++)
          log->ids[log_ids++] = s.id[s.running[pl.admitted[a]].idx];
        for (int64_t r = 0; r < pl.n_rej; r++)
          log->ids[log_ids++] = s.id[pl.rej_idx[r]] * 2 +
                                (pl.rej_reason[r] == ORC_STATUS_REJECTED_ADMISSION);
        for (int64_t b = 0; b < pl.n_batch; b++)
          log->ids[log_ids++] = s.id[s.running[pl.batch[b]].idx];
        log->n_steps = step_idx + 1;
        log->n_ids = log_ids;
      } else {
        log->overflow = 1;
      }
    }

    /* token emits, :240-245 */
    for (int64_t a = 0; a < pl.n_admitted; a++) {
      rentry* e = &s.running[pl.admitted[a]];
      e->tokens = 1;
      s.first_emit[e->idx] = end;
      s.n_emits[e->idx] = 1;
    }
    for (int64_t b = 0; b < pl.n_batch; b++) {
      rentry* e = &s.running[pl.batch[b]];
      e->tokens += 1;
      s.n_emits[e->idx] += 1;
    }
    /* retire (stable), :247-271 */
    int64_t nret = 0, k = 0;
    for (int64_t j = 0; j < s.n_running; j++) {
      rentry e = s.running[j];
      if (e.tokens >= s.true_out[e.idx])
        retire_buf[nret++] = e.idx;
      else
        s.running[k++] = e;
    }
    s.n_running = k;
    for (int64_t r = 0; r < nret; r++) {
      int32_t i = retire_buf[r];
      double first = s.first_emit[i];
      int64_t ne = s.n_emits[i];
      double tpot = ne == 1 ? 0.0 : (end - first) / (double)(ne - 1); /* core.py:152-155 */
      double ttft = first - s.arrival[i];
      out->status[i] = ORC_STATUS_COMPLETED;
      out->first_token_time[i] = first;
      out->completion_time[i] = end;
      out->ttft[i] = ttft;
      out->tpot[i] = tpot;
      out->completion_step[i] = (int32_t)step_idx;
      int ok = ttft <= s.ttft_slo[i] && tpot <= s.tpot_slo[i]; /* core.py:158-165 */
      out->compliant[i] = (int8_t)ok;
      resolved[i] = 1;
      sum->completed++;
      sum->compliant += ok;
      sum->ttft_violations += ttft > s.ttft_slo[i];
      sum->tpot_violations += tpot > s.tpot_slo[i];
    }
    s.now = end;
    step_idx++;
  }

  sum->status = rc;
  sum->n_steps = step_idx;
  sum->sim_end = s.now;
  sum->digest = digest;
  sum->total = n;
  for (int64_t i = 0; i < n; i++)
    if (!resolved[i]) sum->incomplete++;
  double horizon = (p->flags & ORC_FLAG_HAS_HORIZON) ? p->horizon
                                                      : (s.now > 1e-12 ? s.now : 1e-12);
  sum->horizon = horizon;
  sum->goodput = (double)sum->compliant / horizon; /* core.py:168-172 */
  sum->adherence = n > 0 ? (double)sum->compliant / (double)n : 0.0;

  free(s.waiting);
  free(s.running);
  free(s.first_emit);
  free(s.n_emits);
  free(pl.admitted);
  free(pl.batch);
  free(pl.rej_idx);
  free(pl.rej_reason);
  free(resolved);
  free(retire_buf);
  return rc;
}
