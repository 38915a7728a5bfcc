// Persistent warp-per-simulation kernel: the whole slosim discrete-event loop
// (simengine.run, simengine.py:168-303) with the scorpio policy
// (sched_scorpio.plan_step, sched_scorpio.py:210-316) or a baseline
// (sched_baselines.py:49-150), for thousands of independent simulations.
//
// Mapping:
//  * one warp owns one simulation at a time and pulls the next one from a
//    device work counter over a host-ordered (longest-first) schedule;
//  * per-request arrival-time constants live in a 64-byte WRec, built for
//    every request of every sim by wrec_prepass_kernel ahead of the
//    simulation kernels; the waiting queue is an int32 index list kept in LDF
//    order by warp-parallel rank+shift insertion;
//  * the running set: in registers in the fast kernels (sim_fast.cuh: entry j
//    in lane j % 32, slot j / 32, up to 64 entries); in this general kernel a
//    positional SoA (32-byte RRec per entry, admission order), so credit
//    updates, emits and retire compaction are coalesced lane-parallel passes;
//    batch compaction = ballot + popc;
//  * the order-dependent fp64 chains (TTFT prefix walk, Neumaier aggregates,
//    greedy admission scan) run warp-uniformly over register-staged chunks
//    (one chunk load per 32 items, values broadcast with shuffles) so every
//    lane holds the same state and no lane diverges.
#include <cuda_runtime.h>

#include <atomic>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "scorpio_b200.h"
#include "sl_device.cuh"
#include "sim_common.cuh"
#include "sim_fast.cuh"
#include <stdlib.h>

using namespace sl;

namespace {

// TTFT prefix walk over wl[0, W) in list order (ttft_guard :196-205 /
// early_reject sched_baselines.py:95-103).  Rejected -> REJECTED_TTFT.
__device__ void ttft_walk(const Sim& s, const KArgs& a, bool has_out, int& W, int& nrej,
                          double now, int64_t step, Acc& acc, int lane, int64_t log_rej_base,
                          int64_t log_cap) {
  double prefix = 0.0;
  int kept = 0;
  for (int c0 = 0; c0 < W; c0 += 32) {
    int j = c0 + lane;
    bool valid = j < W;
    int idx = 0;
    double e = 0.0, pf = 0.0, tt = 0.0;
    if (valid) {
      idx = s.wl[j];
      const WRec& r = s.wr[idx];
      e = fsub_(now, r.arr);
      pf = r.prefill;
      tt = r.ttft;
    }
    int cnt = min(32, W - c0);
    unsigned rej = 0;
    for (int t = 0; t < cnt; ++t) {
      double et = bcast(e, t), pt = bcast(pf, t), tl = bcast(tt, t);
      double est = fadd_(fadd_(et, prefix), pt);
      if (est > tl)
        rej |= 1u << t;
      else
        prefix = fadd_(prefix, pt);
    }
    bool r_ = valid && ((rej >> lane) & 1u);
    bool keep = valid && !r_;
    unsigned km = __ballot_sync(SL_FULL, keep);
    __syncwarp();
    if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
    if (r_) {
      int pos = nrej + __popc(rej & lanemask_lt());
      int64_t rid = s.id[idx];
      acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u);
      acc.rej_ttft++;
      if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_TTFT;
      if (log_rej_base >= 0 && pos < log_cap) a.log.rej_ids[log_rej_base + pos] = rid * 2;
    }
    __syncwarp();
    kept += __popc(km);
    nrej += __popc(rej);
  }
  W = kept;
}

// Append waiting items wl[0, take) to the running list in order (admit-all /
// admit_fcfs) and drop them from the front of the waiting list by advancing
// its base (each request enters the list once, so base + W never passes the
// sim's n slots).  Returns the Neumaier prefill sum.
template <bool WIDE>
__device__ void admit_prefix(Sim& s, const KArgs& a, int& W, int& R, int take, int& nadm,
                             PySum& P, int64_t step, Acc& acc, int lane, int64_t log_adm_base,
                             int64_t log_cap) {
  for (int c0 = 0; c0 < take; c0 += 32) {
    int j = c0 + lane;
    bool valid = j < take;
    double pf = 0.0;
    if (valid) {
      int idx = s.wl[j];
      const WRec& w = s.wr[idx];
      pf = w.prefill;
      RRec r;
      r.N = 0;
      r.S = w.S;
      r.inv = w.inv;
      r.cur_len = w.prompt;
      r.rem = s.true_out[idx];
      s.rr[R + j] = r;
      s.rl[R + j] = idx;
      if constexpr (WIDE) {
        s.rNhi[R + j] = 0;
        s.rShi[R + j] = s.wShi[idx];
      }
      int64_t rid = s.id[idx];
      s.rh[R + j] = batch_hid((uint64_t)rid);
      acc.dig += digest_item((uint64_t)step, 0, (uint32_t)(nadm + j), (uint64_t)rid);
      if (log_adm_base >= 0 && nadm + j < log_cap) a.log.adm_ids[log_adm_base + nadm + j] = rid;
    }
    int cnt = min(32, take - c0);
    for (int t = 0; t < cnt; ++t) ps_add(P, bcast(pf, t));
  }
  __syncwarp();
  s.wl += take;
  R += take;
  nadm += take;
  W -= take;
}

template <bool WIDE>
__device__ __forceinline__ cred_t<WIDE> load_S(const Sim& s, int j) {
  if constexpr (WIDE)
    return ((unsigned __int128)s.rShi[j] << 64) | s.rr[j].S;
  else
    return s.rr[j].S;
}

// min over running S in [0, R) -> fixed value (warp-uniform)
template <bool WIDE>
__device__ cred_t<WIDE> running_min_S(const Sim& s, int R, int lane) {
  cred_t<WIDE> m = ~cred_t<WIDE>(0);
  for (int j = lane; j < R; j += 32) {
    cred_t<WIDE> v = load_S<WIDE>(s, j);
    m = v < m ? v : m;
  }
  return warp_min_cred<WIDE>(m);
}

template <bool WIDE>
__device__ void run_sim(Sim& s, const KArgs& a, bool has_out, int sim_index, int lane) {
  const int64_t n = s.n;
  const sl_cost& C = s.cost;
  const bool scorpio = s.policy == SL_POLICY_SCORPIO;
  const bool ttft_guard = (s.flags & SL_FLAG_TTFT_GUARD) != 0;
  const bool tpot_guard = (s.flags & SL_FLAG_TPOT_GUARD) != 0;
  const bool r_only = (s.flags & SL_FLAG_R_ONLY) != 0;
  const bool has_h = (s.flags & SL_FLAG_HAS_HORIZON) != 0;
  const bool sorted_ldf = scorpio && ttft_guard;
  const bool sjf = s.policy == SL_POLICY_SJF;

  if (has_out) {
    for (int64_t i = lane; i < n; i += 32) {
      int64_t o = s.out_off + i;
      a.out.status[o] = SL_INCOMPLETE;
      a.out.compliant[o] = 0;
      a.out.completion_step[o] = -1;
      a.out.first_token_time[o] = __longlong_as_double(0x7ff8000000000000LL);
      a.out.completion_time[o] = __longlong_as_double(0x7ff8000000000000LL);
      a.out.ttft[o] = __longlong_as_double(0x7ff8000000000000LL);
      a.out.tpot[o] = __longlong_as_double(0x7ff8000000000000LL);
    }
  }
  const bool logging = a.has_log && s.log_row >= 0;
  int64_t lg_step0 = logging ? s.log_row * a.log.step_cap : 0;
  int64_t lg_id0 = logging ? s.log_row * a.log.id_cap : 0;
  int64_t cur_adm = 0, cur_rej = 0, cur_batch = 0;  // log stream cursors
  bool log_over = false;

  Acc acc;
  memset(&acc, 0, sizeof(acc));
  double now = 0.0;
  int64_t next = 0;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  double next_t = n > 0 ? fdiv_(s.arrival[0], s.factor) : kInf;
  int W = 0, R = 0;
  int64_t step = 0, n_plans = 0, n_idle = 0, req_steps = 0;
  int status = SL_SIM_OK;

  for (;;) {
    // ---- arrivals become visible at step boundaries (simengine.py:186-188)
    while (next < n && next_t <= now) {
      int64_t i = next + lane;
      double ai = (i < n) ? fdiv_(s.arrival[i], s.factor) : kInf;
      bool c = ai <= now;
      unsigned m = __ballot_sync(SL_FULL, c);
      int k = __popc(m);  // arrivals are sorted: m is a lane prefix
      if (c) {
        WRec w;
        w.arr = ai;
        w.ttft = fmul_(s.ttft_b[i], s.scale);
        w.tpot = fmul_(s.tpot_b[i], s.scale);
        w.prompt = s.prompt[i];
        int32_t pred = s.predicted[i];
        w.prefill = prefill_time(C, w.prompt);
        w.inv = frcp_(w.tpot);
        w.deadline = fadd_(w.arr, w.ttft);
        cred_t<WIDE> S = slo_fixed<WIDE>(w.tpot, s.E);
        w.S = (uint64_t)S;
        if constexpr (WIDE) s.wShi[i] = (uint64_t)(S >> 64);
        bool solo = solo_ok(C, w.tpot, w.inv, w.prompt, pred);
        w.pred_solo = pred | (solo ? (int32_t)0x80000000 : 0);
        s.wr[i] = w;
      }
      __syncwarp();
      if (sorted_ldf || sjf) {
        for (int t = 0; t < k; ++t) insert_sorted(s, W, (int)(next + t), sjf, lane);
      } else {
        if (c) s.wl[W + lane] = (int32_t)i;
        __syncwarp();
        W += k;
      }
      next += k;
      next_t = next < n ? fdiv_(s.arrival[next], s.factor) : kInf;
    }

    if (has_h && now >= s.horizon) break;  // simengine.py:190-191

    // ---- quiet decode-all steps (baselines, admit-all ablation): nothing can be
    // admitted or rejected (no waiting request; or a full batch cap and no TTFT
    // walk) and every running entry decodes each step, so until the next
    // arrival, the horizon or the step before the first retirement only the
    // clock and the digest move; per-entry counters are settled once after.
    if (!(scorpio && tpot_guard) && !logging && R > 0 &&
        (W == 0 || (!scorpio && s.policy != SL_POLICY_EARLY_REJECT && R >= s.cap))) {
      int minrem = 1 << 30;
      int64_t bl = 0;
      uint32_t bh = 0;
      for (int j = lane; j < R; j += 32) {
        const RRec& r = s.rr[j];
        minrem = min(minrem, r.rem);
        bl += r.cur_len;
        bh += s.rh[j];
      }
      minrem = __reduce_min_sync(SL_FULL, minrem);
      bl = warp_sum_i64(bl);
      bh = __reduce_add_sync(SL_FULL, bh);
      int k = 0;
      while (k + 1 < minrem && next_t > now && !(has_h && now >= s.horizon)) {
        const double decode_s = itl(C, R, div_small((double)bl, R));
        const double end = fadd_(fadd_(now, 0.0), decode_s);  // prefill sum of no admission
        if (lane == 0)
          acc.dig += digest_item((uint64_t)step, 2, (uint32_t)R, bh) +
                     digest_item((uint64_t)step, 3, 0, (uint64_t)__double_as_longlong(end));
        n_plans++;
        req_steps += W + R;
        bl += R;
        now = end;
        step++;
        ++k;
      }
      if (k > 0) {
        for (int j = lane; j < R; j += 32) {
          RRec& r = s.rr[j];
          r.cur_len += k;
          r.rem -= k;
        }
        __syncwarp();
        continue;  // arrivals / horizon / the retiring step through the general step
      }
    }

    // ---- plan (policy.plan)
    n_plans++;
    req_steps += W + R;
    const int R0 = R;
    int nadm = 0, nrej = 0, nbatch = 0;
    PySum P;
    ps_init(P);
    int64_t blen = 0;  // per-lane partial of sum(current_len) over the batch
    uint32_t bhash = 0;  // per-lane partial of the batch id hash sum (digest tag 2)
    acc.dig_rej = 0;
    int64_t lg_adm = (logging && !log_over) ? lg_id0 + cur_adm : -1;
    int64_t lg_rej = (logging && !log_over) ? lg_id0 + cur_rej : -1;
    int64_t lg_bat = (logging && !log_over) ? lg_id0 + cur_batch : -1;
    // clamp stream bases so that positions beyond id_cap are dropped (overflow flagged below)
    int64_t cap_adm = logging ? a.log.id_cap - cur_adm : 0;
    int64_t cap_rej = logging ? a.log.id_cap - cur_rej : 0;
    int64_t cap_bat = logging ? a.log.id_cap - cur_batch : 0;

    if (scorpio) {
      if (ttft_guard && W > 0)
        ttft_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej);
      if (tpot_guard) {
        if (W > 0) {
          // _running_aggregates (sched_scorpio.py:117-124)
          int64_t n_run = R;
          int64_t lens = 0;
          for (int j = lane; j < R; j += 32) lens += s.rr[j].cur_len;
          lens = warp_sum_i64(lens);
          cred_t<WIDE> Smin = running_min_S<WIDE>(s, R, lane);
          bool has_min = R > 0;
          double min_d = has_min ? fixed_to_double<WIDE>(Smin, s.pow2E) : 0.0;
          PySum ps;
          ps_init(ps);
          for (int c0 = 0; c0 < R; c0 += 32) {
            int j = c0 + lane;
            double x = j < R ? s.rr[j].inv : 0.0;
            int cnt = min(32, R - c0);
            for (int t = 0; t < cnt; ++t) ps_add(ps, bcast(x, t));
          }
          double inv = ps_result(ps);
          // admission scan in queue order (sched_scorpio.py:237-294)
          int kept = 0;
          for (int c0 = 0; c0 < W; c0 += 32) {
            int j = c0 + lane;
            bool valid = j < W;
            int idx = 0;
            double tp = 0.0, ic = 0.0, pf = 0.0;
            int32_t ln = 0, ps_ = 0;
            cred_t<WIDE> Sc = 0;
            if (valid) {
              idx = s.wl[j];
              const WRec& w = s.wr[idx];
              tp = w.tpot;
              ic = w.inv;
              pf = w.prefill;
              ln = w.prompt;
              ps_ = w.pred_solo;
              if constexpr (WIDE)
                Sc = ((unsigned __int128)s.wShi[idx] << 64) | w.S;
              else
                Sc = w.S;
            }
            int cnt = min(32, W - c0);
            unsigned adm = 0;
            for (int t = 0; t < cnt; ++t) {
              double cand = bcast(tp, t);
              double icand = bcast(ic, t);
              int32_t clen = bcast(ln, t);
              int32_t cpred = bcast(ps_, t) & 0x7fffffff;
              bool lt = !has_min || cand < min_d;
              double minp = lt ? cand : min_d;
              double V = fmul_(minp, fadd_(inv, icand));
              double L = div_small((double)(lens + clen), (int)(n_run + 1));  // exact int / int
              double est = tpot_estimate(C, V, L, cpred);
              double thr = (r_only && has_min) ? min_d : minp;
              if (est <= thr) {
                if (lg_adm >= 0 && a.log.adm_rec && lane == 0) {  // AdmissionRecord inputs
                  const int q = nadm + __popc(adm);
                  if (q < cap_adm) {
                    double* rec = a.log.adm_rec + 5 * (lg_adm + q);
                    rec[0] = V;
                    rec[1] = L;
                    rec[2] = minp;
                    rec[3] = est;
                    rec[4] = thr;
                  }
                }
                adm |= 1u << t;
                n_run += 1;
                inv = fadd_(inv, icand);  // plain float add, :275
                lens += clen;
                if (lt) min_d = cand;
                has_min = true;
                ps_add(P, bcast(pf, t));
              }
            }
            bool is_adm = valid && ((adm >> lane) & 1u);
            bool solo = (ps_ & (int32_t)0x80000000) != 0;
            bool keep = valid && !is_adm && solo;
            bool rj = valid && !is_adm && !solo;
            unsigned km = __ballot_sync(SL_FULL, keep);
            unsigned rm = __ballot_sync(SL_FULL, rj);
            __syncwarp();
            if (is_adm) {
              int q = __popc(adm & lanemask_lt());
              RRec r;
              r.N = 0;
              r.S = (uint64_t)Sc;
              r.inv = ic;
              r.cur_len = ln;
              r.rem = s.true_out[idx];
              s.rr[R + q] = r;
              s.rl[R + q] = idx;
              if constexpr (WIDE) {
                s.rNhi[R + q] = 0;
                s.rShi[R + q] = (uint64_t)(Sc >> 64);
              }
              int64_t rid = s.id[idx];
              s.rh[R + q] = batch_hid((uint64_t)rid);
              acc.dig += digest_item((uint64_t)step, 0, (uint32_t)(nadm + q), (uint64_t)rid);
              if (lg_adm >= 0 && nadm + q < cap_adm) a.log.adm_ids[lg_adm + nadm + q] = rid;
            }
            if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
            if (rj) {
              int pos = nrej + __popc(rm & lanemask_lt());
              int64_t rid = s.id[idx];
              acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u + 1u);
              acc.rej_adm++;
              if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_ADMISSION;
              if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2 + 1;
            }
            __syncwarp();
            int na = __popc(adm);
            R += na;
            nadm += na;
            kept += __popc(km);
            nrej += __popc(rm);
          }
          W = kept;
        }
      } else {
        admit_prefix<WIDE>(s, a, W, R, W, nadm, P, step, acc, lane, lg_adm, cap_adm);
      }
    } else {
      if (s.policy == SL_POLICY_EARLY_REJECT && W > 0)
        ttft_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej);
      int room = s.cap - R;
      int take = room > 0 ? min(room, W) : 0;
      if (take > 0)
        admit_prefix<WIDE>(s, a, W, R, take, nadm, P, step, acc, lane, lg_adm, cap_adm);
    }

    // ---- decode batch
    cred_t<WIDE> MIN = 0;
    bool need_min = scorpio && (tpot_guard || logging);
    if (need_min && R > 0) MIN = running_min_S<WIDE>(s, R, lane);
    const bool credit = scorpio && tpot_guard;
    const bool decode_all = !credit && !(s.policy != SL_POLICY_SCORPIO &&
                                         (s.flags & SL_FLAG_PREFILL_PRIORITY) && nadm > 0);
    bool batch_ret = false;  // a batched entry emitted its last token
    if (credit || decode_all) {
      for (int c0 = 0; c0 < R0; c0 += 32) {
        int j = c0 + lane;
        bool b = false;
        if (j < R0) {
          if (credit) {  // select_batch, sched_scorpio.py:171-179
            RRec& r = s.rr[j];
            if constexpr (WIDE) {
              cred_t<WIDE> N = ((unsigned __int128)s.rNhi[j] << 64) | r.N;
              cred_t<WIDE> S = ((unsigned __int128)s.rShi[j] << 64) | r.S;
              N += MIN;
              if (N >= S) {
                N -= S;
                b = true;
              }
              r.N = (uint64_t)N;
              s.rNhi[j] = (uint64_t)(N >> 64);
            } else {
              uint64_t N = r.N + MIN;
              if (N >= r.S) {
                N -= r.S;
                b = true;
              }
              r.N = N;
            }
          } else {
            b = true;
          }
        }
        unsigned bm = __ballot_sync(SL_FULL, b);
        if (b) {
          RRec& r = s.rr[j];
          int pos = nbatch + __popc(bm & lanemask_lt());
          blen += r.cur_len;
          r.cur_len += 1;  // token emit (simengine.py:243-245); l_avg already taken
          r.rem -= 1;
          batch_ret |= r.rem <= 0;
          bhash += s.rh[j];  // batch_hid(id), kept per running position
          if (lg_bat >= 0 && pos < cap_bat) a.log.batch_ids[lg_bat + pos] = s.id[s.rl[j]];
        }
        nbatch += __popc(bm);
      }
    }

    // ---- no work: idle skip (simengine.py:207-227)
    if (nadm == 0 && nbatch == 0) {
      double dl = kInf;
      for (int j = lane; j < W; j += 32) {
        double d = s.wr[s.wl[j]].deadline;
        if (d > now && d < dl) dl = d;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) dl = fmin(dl, __shfl_xor_sync(SL_FULL, dl, o));
      bool have = dl != kInf;
      double target = dl;
      if (next < n) {
        if (!have || next_t < target) target = next_t;
        have = true;
      } else if (R > 0) {
        status = SL_SIM_NO_WORK_RUNNING;
        break;
      }
      if (!have) {
        if (W > 0) status = SL_SIM_NO_PROGRESS;
        break;
      }
      if (target <= now) {
        status = SL_SIM_NO_PROGRESS;
        break;
      }
      if (logging && a.log.skip_now && lane == 0 && n_idle < a.log.skip_cap) {
        const int64_t o = s.log_row * a.log.skip_cap + n_idle;
        a.log.skip_now[o] = now;
        a.log.skip_target[o] = target;
        a.log.skip_waiting[o] = W;
        a.log.n_skips[s.log_row] = n_idle + 1;
      }
      n_idle++;
      now = target;
      continue;
    }

    // ---- step duration (simengine.py:233-238)
    double prefill_s = ps_result(P);
    double decode_s = 0.0;
    int64_t bl = warp_sum_i64(blen);
    if (nbatch > 0) decode_s = itl(C, nbatch, div_small((double)bl, nbatch));  // exact int / int
    double end = fadd_(fadd_(now, prefill_s), decode_s);
    acc.dig += acc.dig_rej;
    bhash = __reduce_add_sync(SL_FULL, bhash);
    if (lane == 0)
      acc.dig += digest_item((uint64_t)step, 2, (uint32_t)nbatch, bhash) +
                 digest_item((uint64_t)step, 3, 0, (uint64_t)__double_as_longlong(end));

    // ---- decision log row
    if (logging) {
      bool fits = !log_over && step < a.log.step_cap && cur_adm + nadm <= a.log.id_cap &&
                  cur_rej + nrej <= a.log.id_cap && cur_batch + nbatch <= a.log.id_cap;
      if (fits) {
        double vbs = 0.0, mslo = __longlong_as_double(0x7ff8000000000000LL);
        if (scorpio && R > 0) {  // sched_scorpio.py:312-315 (before retirement); baselines keep defaults
          mslo = fixed_to_double<WIDE>(MIN, s.pow2E);
          PySum vs;
          ps_init(vs);
          for (int c0 = 0; c0 < R; c0 += 32) {
            int j = c0 + lane;
            double x = 0.0;
            if (j < R) x = fdiv_(mslo, fixed_to_double<WIDE>(load_S<WIDE>(s, j), s.pow2E));
            int cnt = min(32, R - c0);
            for (int t = 0; t < cnt; ++t) ps_add(vs, bcast(x, t));
          }
          vbs = ps_result(vs);
        }
        if (lane == 0) {
          int64_t o = lg_step0 + step;
          a.log.now[o] = now;
          a.log.end[o] = end;
          a.log.prefill_s[o] = prefill_s;
          a.log.decode_s[o] = decode_s;
          a.log.vbs[o] = vbs;
          a.log.min_slo[o] = mslo;
          a.log.n_admitted[o] = nadm;
          a.log.n_rejected[o] = nrej;
          a.log.n_batch[o] = nbatch;
          a.log.n_steps[s.log_row] = step + 1;
        }
        cur_adm += nadm;
        cur_rej += nrej;
        cur_batch += nbatch;
      } else {
        log_over = true;
      }
    }

    // ---- emits for fresh entries + retirement (simengine.py:240-271)
    // Only entries that emitted this step can finish: batched ones (batch_ret)
    // and the admitted (remaining 1).  Without any, just the first tokens.
    bool may_ret = batch_ret;
    for (int j = R0 + lane; j < R; j += 32) may_ret |= s.rr[j].rem <= 1;
    if (!__any_sync(SL_FULL, may_ret)) {
      for (int j = R0 + lane; j < R; j += 32) {
        RRec& r = s.rr[j];
        r.cur_len += 1;
        r.rem -= 1;
        s.first_emit[s.rl[j]] = end;
      }
      __syncwarp();
      now = end;
      step++;
      continue;
    }
    int keptR = 0;
    for (int c0 = 0; c0 < R; c0 += 32) {
      int j = c0 + lane;
      bool valid = j < R;
      RRec r;
      int idx = 0;
      uint32_t hid = 0;
      uint64_t nhi = 0, shi = 0;
      bool ret = false;
      if (valid) {
        r = s.rr[j];
        idx = s.rl[j];
        hid = s.rh[j];
        if constexpr (WIDE) {
          nhi = s.rNhi[j];
          shi = s.rShi[j];
        }
        if (j >= R0) {  // admitted this step: tokens = 1, first emit at `end`
          r.cur_len += 1;
          r.rem -= 1;
          s.first_emit[idx] = end;
        }
        ret = r.rem <= 0;
      }
      unsigned km = __ballot_sync(SL_FULL, valid && !ret);
      __syncwarp();
      if (valid && !ret) {
        int q = keptR + __popc(km & lanemask_lt());
        s.rr[q] = r;
        s.rl[q] = idx;
        s.rh[q] = hid;
        if constexpr (WIDE) {
          s.rNhi[q] = nhi;
          s.rShi[q] = shi;
        }
      }
      if (ret) {
        const WRec& w = s.wr[idx];
        double first = j >= R0 ? end : s.first_emit[idx];
        int32_t tout = s.true_out[idx];
        double tpot = tout == 1 ? 0.0 : fdiv_(fsub_(end, first), (double)(tout - 1));
        double ttft = fsub_(first, w.arr);
        bool ok = ttft <= w.ttft && tpot <= w.tpot;
        acc.completed++;
        acc.compliant += ok;
        acc.ttft_viol += ttft > w.ttft;
        acc.tpot_viol += tpot > w.tpot;
        if (has_out) {
          int64_t o = s.out_off + idx;
          a.out.status[o] = SL_COMPLETED;
          a.out.compliant[o] = ok;
          a.out.completion_step[o] = (int32_t)step;
          a.out.first_token_time[o] = first;
          a.out.completion_time[o] = end;
          a.out.ttft[o] = ttft;
          a.out.tpot[o] = tpot;
        }
      }
      __syncwarp();
      keptR += __popc(km);
    }
    R = keptR;
    now = end;
    step++;
  }

  write_result(a, sim_index, acc, status | (log_over ? SL_SIM_LOG_OVERFLOW : 0), n, step,
               n_plans, n_idle, req_steps, now, has_h, s.horizon, lane);
}

// General kernel: waiting and running lists in global memory (any size).
// handoff_only: run just the sims the fast kernel handed off (SL_SIM_CAPACITY).
__global__ void __launch_bounds__(128) sl_sim_kernel(const __grid_constant__ KArgs a,
                                                     int handoff_only) {
  const int lane = threadIdx.x & 31;
  Workspace ws = carve(a.ws_base, a.slots);
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(ws.counter + 1, 1);
    q = __shfl_sync(SL_FULL, q, 0);
    if (q >= a.n_sims) return;
    int si = a.order ? a.order[q] : q;
    if (handoff_only && !(a.results[si].status & SL_SIM_CAPACITY)) continue;
    Sim s = make_sim(a, ws, si);
    bool has_out = a.has_out && s.out_off >= 0;
    if (a.sims[si].credit_wide)
      run_sim<true>(s, a, has_out, si, lane);
    else
      run_sim<false>(s, a, has_out, si, lane);
  }
}

// Fast kernel: running set in registers (sim_fast.cuh); hands off sims that
// outgrow it or are flagged general-only.
constexpr int kFastWarps = 4;
#ifndef SL_SIM_IN_SMEM
#define SL_SIM_IN_SMEM 1
#endif
#ifndef SL_BASELINE_TO_GENERAL
#define SL_BASELINE_TO_GENERAL 1
#endif
#ifndef SL_HOT_MIN_BLOCKS
#define SL_HOT_MIN_BLOCKS 4  // 16 warps/SM for the hot kernel (<= 128 registers)
#endif
// WRec of every request of every sim handled by the fast kernels, built ahead
// of the simulation: one thread per (sim, request), streaming the shared trace
// and writing 64 B per request -- HBM-bound work taken off each simulation's
// serial step chain.  (The general kernel builds its own at arrival.)
__global__ void __launch_bounds__(256) wrec_prepass_kernel(const __grid_constant__ KArgs a) {
  const int si = blockIdx.y;
  const sl_sim& sp = a.sims[si];
  Workspace ws = carve(a.ws_base, a.slots);
  const int t = sp.trace;
  const int64_t n = a.tr.begin[t + 1] - a.tr.begin[t];
  Sim s = make_sim(a, ws, si);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t hi = 0;
    if (sp.credit_wide) {
      s.wr[i] = make_wrec<true>(s, i, &hi);
      s.wShi[i] = hi;
    } else {
      s.wr[i] = make_wrec<false>(s, i, &hi);
    }
  }
}

__device__ __forceinline__ bool hot_eligible(const sl_sim& sp) {
  const int f = SL_FLAG_TTFT_GUARD | SL_FLAG_TPOT_GUARD;
  return sp.policy == SL_POLICY_SCORPIO && (sp.flags & f) == f &&
         !(sp.flags & SL_FLAG_GENERAL_ONLY) && !sp.credit_wide;
}

// HOT = true: scorpio-with-both-guards sims only, no decision log (OUT: outcomes
// requested); HOT = false: every other sim (all sims when a log is requested).
template <bool HOT, bool OUT>
__global__ void __launch_bounds__(32 * kFastWarps, HOT ? SL_HOT_MIN_BLOCKS : 1) sl_sim_fast_kernel(
    const __grid_constant__ KArgs a) {
  __shared__ __align__(16) Slot<false> scratch[kFastWarps][kRunCap];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  Workspace ws = carve(a.ws_base, a.slots);
  for (;;) {
    int q = 0;
    if (lane == 0) q = atomicAdd(ws.counter + (HOT ? 0 : 2), 1);
    q = __shfl_sync(SL_FULL, q, 0);
    if (q >= a.n_sims) return;
    int si = a.order ? a.order[q] : q;
    const sl_sim& sp = a.sims[si];
    const bool hot = hot_eligible(sp);
    if (HOT ? !hot : (hot && !a.has_log)) continue;  // the other fast kernel's sim
    // 128-bit credits, or a baseline whose batch cap exceeds the register
    // slots (its running set soon outgrows them): the general kernel from the start
    if ((sp.flags & SL_FLAG_GENERAL_ONLY) || sp.credit_wide ||
        (!HOT && SL_BASELINE_TO_GENERAL && sp.policy != SL_POLICY_SCORPIO &&
         sp.max_batch_size > kRunCap)) {
      if (lane == 0) a.results[si].status = SL_SIM_CAPACITY;
      continue;
    }
    if (HOT) {
#if SL_SIM_IN_SMEM
      // per-sim constants live in shared memory: re-read where used instead of
      // pinning ~60 registers for the whole simulation
      __shared__ Sim sim_sm[kFastWarps];
      __syncwarp();
      if (lane == 0) sim_sm[warp] = make_sim(a, ws, si);
      __syncwarp();
      Sim& s = sim_sm[warp];  // read-only on the hot path (no append_prefix)
#else
      Sim s = make_sim(a, ws, si);
#endif
      run_fast<false, true>(s, a, OUT && s.out_off >= 0, si, lane, scratch[warp]);
    } else {
      Sim s = make_sim(a, ws, si);
      run_fast<false, false>(s, a, a.has_out && s.out_off >= 0, si, lane, scratch[warp]);
    }
  }
}

}  // namespace

extern "C" {

int64_t sl_workspace_bytes(int64_t total_slots, int32_t n_sims) {
  (void)n_sims;
  return workspace_bytes(total_slots);
}

int sl_credit_params(int64_t n, const double* tpot_slo, double slo_scale, int32_t* credit_exp,
                     int32_t* credit_wide) {
  if (!credit_exp || !credit_wide || (n > 0 && !tpot_slo)) return SL_ERR_ARG;
  int e_min = 1 << 30, e_max = -(1 << 30);
  for (int64_t i = 0; i < n; i++) {
    double v = tpot_slo[i] * slo_scale;
    if (!(v > 0.0) || !isfinite(v) || !isnormal(v)) return SL_ERR_ARG;
    int e;
    frexp(v, &e);
    if (e < e_min) e_min = e;
    if (e > e_max) e_max = e;
  }
  if (n == 0) {
    *credit_exp = 0;
    *credit_wide = 0;
    return SL_OK;
  }
  int E = e_min - 53;
  if (E < -1022) return SL_ERR_ARG;
  int span = e_max - e_min;  // S < 2^(53+span); need 2*S <= 2^64 (narrow) / 2^128 (wide)
  *credit_exp = E;
  *credit_wide = (53 + span + 1 > 64) ? 1 : 0;
  if (53 + span + 1 > 128) return SL_ERR_ARG;
  return SL_OK;
}

// Self-test hook for the exact small-divisor division used on the hot path
// (div_small, sl_device.cuh): out[i] = a[i] / b[i] correctly rounded.
__global__ void div_small_test_kernel(const double* a, const int32_t* b, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = div_small(a[i], b[i]);
}

int sl_selftest_div_small(const double* a, const int32_t* b, double* out, int64_t n,
                          void* stream) {
  if (n < 0 || (n > 0 && (!a || !b || !out))) return SL_ERR_ARG;
  if (n == 0) return SL_OK;
  div_small_test_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(a, b, out, n);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_run_batch_launches(void) { return 4; }  // WRec pre-pass + hot fast + generic fast + handoff

#if defined(SL_PHASE_PROF) || defined(SL_TIMELINE)
// Profiling builds only: per-sim phase cycles / counts of the fast kernel.
int sl_phase_prof_read(uint64_t* out, int32_t n_sims) {
  if (n_sims > kProfSims) n_sims = kProfSims;
  return cudaMemcpyFromSymbol(out, sl_prof_cycles, sizeof(unsigned long long) * kProfSlots * n_sims) ==
                 cudaSuccess ? n_sims : SL_ERR_CUDA;
}
#endif

int sl_abi_layout(int64_t* out, int32_t n) {
  if (!out || n < 7) return SL_ERR_ARG;
  if (n >= 8) out[7] = sizeof(sl_report_row);
  out[0] = sizeof(sl_sim);
  out[1] = sizeof(sl_result);
  out[2] = sizeof(sl_traces);
  out[3] = sizeof(sl_outcomes);
  out[4] = sizeof(sl_log);
  out[5] = sizeof(sl_cost);
  out[6] = sizeof(sl_predictor);
  return SL_OK;
}

int sl_device_info(int32_t* sm_count, int32_t* l2_bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SL_ERR_NO_DEVICE;
  int v = 0;
  if (sm_count) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    *sm_count = v;
  }
  if (l2_bytes) {
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
    *l2_bytes = v;
  }
  return SL_OK;
}

int sl_run_batch_ex(const sl_traces* traces, const sl_sim* sims, const int32_t* order,
                    int32_t n_sims, void* workspace, int64_t total_slots, sl_result* results,
                    const sl_outcomes* outcomes, const sl_log* log, int32_t mode, void* stream) {
  if (!traces || !sims || !workspace || !results || n_sims < 0 || total_slots < 0 ||
      (mode != SL_MODE_AUTO && mode != SL_MODE_GENERAL))
    return SL_ERR_ARG;
  if (n_sims == 0) return SL_OK;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.tr = *traces;
  a.sims = sims;
  a.order = order;
  a.n_sims = n_sims;
  a.slots = total_slots;
  a.ws_base = workspace;
  a.results = results;
  if (outcomes) {
    a.out = *outcomes;
    a.has_out = 1;
  }
  if (log) {
    a.log = *log;
    a.has_log = 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(workspace, 0, 256, st) != cudaSuccess) return SL_ERR_CUDA;
  if (mode == SL_MODE_AUTO) {  // WaitingItem fields of every request, ahead of the fast kernels
    dim3 grid(8, (unsigned)n_sims);  // 8 x 256 threads per sim, grid-stride over its requests
    wrec_prepass_kernel<<<grid, 256, 0, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return SL_ERR_CUDA;
  }
  // launch geometry per device, queried once (SM count, resident blocks per SM of
  // each kernel; the SL_* experiment knobs read once too) -- no per-call queries
  constexpr int kMaxDev = 64;
  static int geo_sms[kMaxDev], geo_per_sm[kMaxDev][4];
  static std::atomic<bool> geo_ok[kMaxDev];
  static const int env_cap = [] {
    const char* e = getenv("SL_BLOCKS_PER_SM");  // experiments: cap residency
    return e ? atoi(e) : 0;
  }();
  int dev = 0;
  cudaGetDevice(&dev);
  const void* fns[4] = {(const void*)sl_sim_fast_kernel<true, false>,
                        (const void*)sl_sim_fast_kernel<true, true>,
                        (const void*)sl_sim_fast_kernel<false, false>, (const void*)sl_sim_kernel};
  const int fthreads[4] = {32 * kFastWarps, 32 * kFastWarps, 32 * kFastWarps, 128};
  if (dev < 0 || dev >= kMaxDev) return SL_ERR_ARG;
  if (!geo_ok[dev].load(std::memory_order_acquire)) {  // (racing first calls compute the same)
    if (const char* e = getenv("SL_CARVEOUT")) {  // experiments: shared-memory carveout (percent)
      const int pct = atoi(e);
      cudaFuncSetAttribute(fns[0], cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaFuncSetAttribute(fns[1], cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    }
    cudaDeviceGetAttribute(&geo_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    for (int k = 0; k < 4; ++k) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[k], fthreads[k], 0);
      if (env_cap > 0 && env_cap < per_sm) per_sm = env_cap;
      geo_per_sm[dev][k] = per_sm < 1 ? 1 : per_sm;
    }
    geo_ok[dev].store(true, std::memory_order_release);
  }
  const int sms = geo_sms[dev];
  auto grid_for = [&](const void* fn, int threads) {
    int per_sm = 1;
    for (int k = 0; k < 4; ++k)
      if (fns[k] == fn) per_sm = geo_per_sm[dev][k];
    int64_t wpb = threads / 32;
    int64_t blocks = (n_sims + wpb - 1) / wpb;
    int64_t max_blocks = (int64_t)sms * per_sm;
    return (unsigned)(blocks < max_blocks ? blocks : max_blocks);
  };
  if (mode == SL_MODE_AUTO) {
    if (!a.has_log) {
      if (a.has_out)
        sl_sim_fast_kernel<true, true><<<grid_for((const void*)sl_sim_fast_kernel<true, true>,
                                                  32 * kFastWarps), 32 * kFastWarps, 0, st>>>(a);
      else
        sl_sim_fast_kernel<true, false><<<grid_for((const void*)sl_sim_fast_kernel<true, false>,
                                                   32 * kFastWarps), 32 * kFastWarps, 0, st>>>(a);
      if (cudaGetLastError() != cudaSuccess) return SL_ERR_CUDA;
    }
    sl_sim_fast_kernel<false, false><<<grid_for((const void*)sl_sim_fast_kernel<false, false>,
                                                32 * kFastWarps), 32 * kFastWarps, 0, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return SL_ERR_CUDA;
  }
  sl_sim_kernel<<<grid_for((const void*)sl_sim_kernel, 128), 128, 0, st>>>(
      a, mode == SL_MODE_AUTO ? 1 : 0);
  if (cudaGetLastError() != cudaSuccess) return SL_ERR_CUDA;
  return SL_OK;
}

int sl_run_batch(const sl_traces* traces, const sl_sim* sims, const int32_t* order, int32_t n_sims,
                 void* workspace, int64_t total_slots, sl_result* results,
                 const sl_outcomes* outcomes, const sl_log* log, void* stream) {
  return sl_run_batch_ex(traces, sims, order, n_sims, workspace, total_slots, results, outcomes,
                         log, SL_MODE_AUTO, stream);
}

}  // extern "C"
