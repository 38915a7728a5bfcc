// Fast simulation kernel (one warp per simulation, running set in registers).
//
// Same semantics as the general kernel (sim_kernel.cu), organised for the
// per-step latency that bounds a sweep: the lowest-rate simulations run
// ~4e5 steps with ~2 requests each, so a quiet step must not touch memory.
//  * running entry j lives in lane j%32, register slot j/32 (capacity 64);
//    a simulation that outgrows it is handed to the general kernel
//    (SL_SIM_CAPACITY) and rerun there from scratch, on the same stream;
//  * aggregates are cached and updated incrementally: min-SLO (fixed point
//    and double), sum of current lengths, and the Neumaier 1/slo sum (only
//    recomputed when membership changed and a candidate is waiting);
//  * TTFT walk and admission scan are speculative-parallel:
//    the order-dependent fp64 state is advanced serially only across
//    *decided* items, every candidate test runs lane-parallel, and ballots
//    find the first rejection / admission -- exact, because each decided item
//    sees exactly the sequential state.
#pragma once

#include "sim_common.cuh"

namespace sl {

constexpr int kSlots = 2;
constexpr int kRunCap = 32 * kSlots;

template <bool WIDE>
struct Slot {
  cred_t<WIDE> N, S;  // credit numerator, fixed-point slo
  double inv;         // 1 / tpot
  double first;       // first-token time
  int64_t id;         // request id
  int32_t idx;        // request index in the trace
  int32_t cur_len;    // prompt_len + tokens_generated
  int32_t rem;        // true_output_len - tokens_generated
};

// Conditional per-field moves (not `sl[pos >> 5] = e`, which would force the
// slot array into local memory through a dynamic index).
template <bool WIDE>
__device__ __forceinline__ void sel_slot(Slot<WIDE>& d, bool c, const Slot<WIDE>& e) {
  d.N = c ? e.N : d.N;
  d.S = c ? e.S : d.S;
  d.inv = c ? e.inv : d.inv;
  d.first = c ? e.first : d.first;
  d.id = c ? e.id : d.id;
  d.idx = c ? e.idx : d.idx;
  d.cur_len = c ? e.cur_len : d.cur_len;
  d.rem = c ? e.rem : d.rem;
}

template <bool WIDE>
__device__ __forceinline__ void put_slot(Slot<WIDE> (&sl)[kSlots], int pos, const Slot<WIDE>& e,
                                         int lane) {
  const bool mine = (pos & 31) == lane;
  const int k_at = pos >> 5;
#pragma unroll
  for (int k = 0; k < kSlots; ++k) sel_slot<WIDE>(sl[k], mine && k_at == k, e);
}

// Neumaier sum of 1/slo over the running set in order; the serial chain reads
// its operands from a per-warp smem broadcast buffer `bc` (32 doubles).
template <bool WIDE>
__device__ __forceinline__ double running_inv_sum(const Slot<WIDE> (&sl)[kSlots], int R, int lane,
                                                  double* bc) {
  PySum ps;
  ps_init(ps);
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int cnt = min(32, R - 32 * k);
    if (cnt <= 0) break;
    bc[lane] = sl[k].inv;
    __syncwarp();
    for (int t = 0; t < cnt; ++t) ps_add(ps, bc[t]);
    __syncwarp();
  }
  return ps_result(ps);
}

template <bool WIDE>
__device__ __forceinline__ cred_t<WIDE> running_min(const Slot<WIDE> (&sl)[kSlots], int R,
                                                    int lane) {
  cred_t<WIDE> m = ~cred_t<WIDE>(0);
#pragma unroll
  for (int k = 0; k < kSlots; ++k)
    if (32 * k + lane < R && sl[k].S < m) m = sl[k].S;
  return warp_min_cred<WIDE>(m);
}

// TTFT prefix walk over wl[0, W) in list order (ttft_guard sched_scorpio.py:196-205;
// early_reject sched_baselines.py:95-103).
//  1. Certified pass: an upper bound U_j of the sequential prefix (warp scan in
//     any order, inflated by (1 + 2^-30), which dominates the rounding error
//     of any summation order for W < 2^20) and monotonicity of IEEE addition
//     give est_j <= fl(fl(e_j + U_j) + pf_j); if that bound is <= ttft_j for
//     every item, no item is rejected and the queue is unchanged -- exactly.
//  2. Otherwise the exact walk, speculative-parallel: the sequential chain
//     assuming all undecided items are kept, lane-parallel tests, ballot for the
//     first rejection, restart after it.
__device__ __forceinline__ void spec_walk(const Sim& s, const KArgs& a, bool has_out, int& W,
                                          int& nrej, double now, int64_t step, Acc& acc, int lane,
                                          int64_t lg_rej, int64_t cap_rej, double* bc) {
  if (W < (1 << 20)) {
    const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
    double U = 0.0;
    bool all_ok = true;
    for (int c0 = 0; c0 < W && all_ok; c0 += 32) {
      const int j = c0 + lane;
      const bool valid = j < W;
      double e = 0.0, pf = 0.0, tt = 0.0;
      if (valid) {
        const WRec& r = s.wr[s.wl[j]];
        e = fsub_(now, r.arr);
        pf = r.prefill;
        tt = r.ttft;
      }
      double v = pf;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(SL_FULL, v, o);
        if (lane >= o) v = fadd_(v, y);
      }
      double excl = __shfl_up_sync(SL_FULL, v, 1);
      if (lane == 0) excl = 0.0;
      const double Uj = fmul_(fadd_(U, excl), inflate);
      all_ok = __all_sync(SL_FULL, !valid || fadd_(fadd_(e, Uj), pf) <= tt);
      U = fmul_(fadd_(U, __shfl_sync(SL_FULL, v, 31)), inflate);
    }
    if (all_ok) return;
  }
  double* pre = bc + 32;
  double prefix = 0.0;
  int kept = 0;
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int j = c0 + lane;
    const bool valid = j < W;
    const int cnt = min(32, W - c0);
    int idx = 0;
    double e = 0.0, pf = 0.0, tt = 0.0;
    if (valid) {
      idx = s.wl[j];
      const WRec& r = s.wr[idx];
      e = fsub_(now, r.arr);
      pf = r.prefill;
      tt = r.ttft;
    }
    bc[lane] = pf;
    __syncwarp();
    unsigned rejm = 0;
    int start = 0;
    while (start < cnt) {
      // assume every undecided item is kept: exact sequential prefix chain
      double run = prefix;
      for (int t = start; t < cnt; ++t) {
        if (lane == 0) pre[t] = run;
        run = fadd_(run, bc[t]);
      }
      __syncwarp();
      const double mine = pre[lane];
      const bool rj = lane >= start && lane < cnt && fadd_(fadd_(e, mine), pf) > tt;
      const unsigned m = __ballot_sync(SL_FULL, rj);
      if (m == 0) {
        prefix = run;
        break;
      }
      const int r = __ffs(m) - 1;  // first rejection; earlier items saw the true prefix
      rejm |= 1u << r;
      prefix = pre[r];  // a rejected item leaves the prefix unchanged
      start = r + 1;
      __syncwarp();
    }
    const bool r_ = valid && ((rejm >> lane) & 1u);
    const bool keep = valid && !r_;
    const unsigned km = __ballot_sync(SL_FULL, keep);
    __syncwarp();
    if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
    if (r_) {
      const int pos = nrej + __popc(rejm & lanemask_lt());
      const int64_t rid = s.id[idx];
      acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u);
      acc.rej_ttft++;
      if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_TTFT;
      if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2;
    }
    __syncwarp();
    kept += __popc(km);
    nrej += __popc(rejm);
  }
  W = kept;
}

// Cached running-set aggregates (sched_scorpio.py:117-124), warp-uniform.
template <bool WIDE>
struct Agg {
  cred_t<WIDE> Smin;  // min fixed-point slo over running (valid iff R > 0)
  double min_d;       // the same as a double
  int64_t lens;       // sum of current_len over running
  double inv;         // Neumaier sum of 1/slo over running, in order
  bool inv_valid;
};

// Greedy admission scan in queue order, speculative-parallel
// (sched_scorpio.py:234-294).  Returns false on register-capacity overflow.
template <bool WIDE>
__device__ __forceinline__ bool spec_admit(const Sim& s, const KArgs& a, bool has_out, int& W, int& R,
                           Slot<WIDE> (&sl)[kSlots], Agg<WIDE>& g, int& nadm, int& nrej,
                           PySum& P, bool r_only, int64_t step, Acc& acc, int lane,
                           int64_t lg_adm, int64_t cap_adm, int64_t lg_rej, int64_t cap_rej) {
  const sl_cost& C = s.cost;
  int64_t n_run = R;
  double inv = g.inv;
  int64_t lens = g.lens;
  bool has_min = R > 0;
  double mind = g.min_d;
  cred_t<WIDE> Smn = g.Smin;
  int kept = 0;
  bool ok_cap = true;
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int j = c0 + lane;
    const bool valid = j < W;
    int idx = 0;
    double tp = 0.0, ic = 0.0, pf = 0.0;
    int32_t ln = 0, ps_ = 0, tout = 0;
    int64_t rid = 0;
    cred_t<WIDE> Sc = 0;
    if (valid) {
      idx = s.wl[j];
      const WRec& w = s.wr[idx];
      tp = w.tpot;
      ic = w.inv;
      pf = w.prefill;
      ln = w.prompt;
      ps_ = w.pred_solo;
      tout = s.true_out[idx];
      rid = s.id[idx];
      if constexpr (WIDE)
        Sc = ((unsigned __int128)s.wShi[idx] << 64) | w.S;
      else
        Sc = w.S;
    }
    const int32_t pred = ps_ & 0x7fffffff;
    const bool solo = (ps_ & (int32_t)0x80000000) != 0;
    unsigned pend = __ballot_sync(SL_FULL, valid);
    while (pend) {
      // every pending candidate against the same state A (_admission_math :99-114)
      bool lt = !has_min || tp < mind;
      double minp = lt ? tp : mind;
      double V = fmul_(minp, fadd_(inv, ic));
      double L = fdiv_((double)(lens + ln), (double)(n_run + 1));
      double est = tpot_estimate(C, V, L, pred);
      double thr = (r_only && has_min) ? mind : minp;
      bool ok = ((pend >> lane) & 1u) && est <= thr;
      unsigned okm = __ballot_sync(SL_FULL, ok);
      int gl = okm ? __ffs(okm) - 1 : 32;
      unsigned fail = okm ? (pend & ((1u << gl) - 1u)) : pend;
      // failures before the first admit: outright reject unless feasible alone
      bool mf = (fail >> lane) & 1u;
      bool keep = mf && solo;
      bool rj = mf && !solo;
      unsigned km = __ballot_sync(SL_FULL, keep);
      unsigned rm = __ballot_sync(SL_FULL, rj);
      if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
      if (rj) {
        int pos = nrej + __popc(rm & lanemask_lt());
        acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u + 1u);
        acc.rej_adm++;
        if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_ADMISSION;
        if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2 + 1;
      }
      kept += __popc(km);
      nrej += __popc(rm);
      pend &= ~fail;
      if (!okm) break;
      // admit candidate gl (warp-uniform state update, :250-278)
      if (R >= kRunCap) {
        ok_cap = false;
        break;
      }
      Slot<WIDE> e;
      e.N = 0;
      e.S = shfl_cred<WIDE>(Sc, gl);
      e.inv = bcast(ic, gl);
      e.first = 0.0;
      e.id = bcast(rid, gl);
      e.idx = bcast(idx, gl);
      e.cur_len = bcast(ln, gl);
      e.rem = bcast(tout, gl);
      const double tp_g = bcast(tp, gl);
      const double pf_g = bcast(pf, gl);
      const bool lt_g = bcast((int)lt, gl) != 0;
      put_slot<WIDE>(sl, R, e, lane);
      if (lg_adm >= 0 && a.log.adm_rec) {  // AdmissionRecord inputs (sched_scorpio.py:254-271)
        const double r0 = bcast(V, gl), r1 = bcast(L, gl), r2 = bcast(minp, gl);
        const double r3 = bcast(est, gl), r4 = bcast(thr, gl);
        if (lane == 0 && nadm < cap_adm) {
          double* rec = a.log.adm_rec + 5 * (lg_adm + nadm);
          rec[0] = r0;
          rec[1] = r1;
          rec[2] = r2;
          rec[3] = r3;
          rec[4] = r4;
        }
      }
      if (lane == 0) {
        acc.dig += digest_item((uint64_t)step, 0, (uint32_t)nadm, (uint64_t)e.id);
        if (lg_adm >= 0 && nadm < cap_adm) a.log.adm_ids[lg_adm + nadm] = e.id;
      }
      n_run += 1;
      inv = fadd_(inv, e.inv);  // plain float add, :275
      lens += e.cur_len;
      if (lt_g) {
        mind = tp_g;
        Smn = e.S;
      }
      has_min = true;
      ps_add(P, pf_g);
      ++nadm;
      ++R;
      pend &= ~(1u << gl);
    }
    __syncwarp();
    if (!ok_cap) break;
  }
  W = kept;
  g.lens = lens;
  if (nadm) {
    g.min_d = mind;
    g.Smin = Smn;
    g.inv_valid = false;  // the scan's plain adds are not the Neumaier sum
  }
  return ok_cap;
}

// Append waiting items wl[0, take) to the running set in order (admit-all,
// sched_scorpio.py:295-304, and admit_fcfs, sched_baselines.py:49-60).
template <bool WIDE>
__device__ __forceinline__ bool append_prefix(const Sim& s, const KArgs& a, int& W, int& R,
                              Slot<WIDE> (&sl)[kSlots], Agg<WIDE>& g, int take, int& nadm,
                              PySum& P, int64_t step, Acc& acc, int lane, int64_t lg_adm,
                              int64_t cap_adm) {
  if (R + take > kRunCap) return false;
  for (int c0 = 0; c0 < take; c0 += 32) {
    const int j = c0 + lane;
    const bool valid = j < take;
    Slot<WIDE> e;
    double pf = 0.0, tp = 0.0;
    if (valid) {
      int idx = s.wl[j];
      const WRec& w = s.wr[idx];
      pf = w.prefill;
      tp = w.tpot;
      e.N = 0;
      if constexpr (WIDE)
        e.S = ((unsigned __int128)s.wShi[idx] << 64) | w.S;
      else
        e.S = w.S;
      e.inv = w.inv;
      e.first = 0.0;
      e.id = s.id[idx];
      e.idx = idx;
      e.cur_len = w.prompt;
      e.rem = s.true_out[idx];
      acc.dig += digest_item((uint64_t)step, 0, (uint32_t)(nadm + j), (uint64_t)e.id);
      if (lg_adm >= 0 && nadm + j < cap_adm) a.log.adm_ids[lg_adm + nadm + j] = e.id;
    }
    const int cnt = min(32, take - c0);
    for (int t = 0; t < cnt; ++t) {
      Slot<WIDE> x;
      x.N = 0;
      x.S = shfl_cred<WIDE>(e.S, t);
      x.inv = bcast(e.inv, t);
      x.first = 0.0;
      x.id = bcast(e.id, t);
      x.idx = bcast(e.idx, t);
      x.cur_len = bcast(e.cur_len, t);
      x.rem = bcast(e.rem, t);
      double tpt = bcast(tp, t);
      put_slot<WIDE>(sl, R, x, lane);
      ps_add(P, bcast(pf, t));
      g.lens += x.cur_len;
      if (R == 0 || x.S < g.Smin) {
        g.Smin = x.S;
        g.min_d = tpt;
      }
      ++R;
    }
  }
  __syncwarp();
  int rest = W - take;
  for (int c0 = 0; c0 < rest; c0 += 32) {
    int j = c0 + lane;
    int v = 0;
    if (j < rest) v = s.wl[take + j];
    __syncwarp();
    if (j < rest) s.wl[j] = v;
    __syncwarp();
  }
  nadm += take;
  W = rest;
  if (take) g.inv_valid = false;
  return true;
}

// Retire entries whose last token was emitted at `end` (simengine.py:247-271):
// outcomes, then stable compaction of the register slots through smem.
template <bool WIDE>
__device__ __forceinline__ void retire(const Sim& s, const KArgs& a, bool has_out,
                                       Slot<WIDE> (&sl)[kSlots], int& R, Agg<WIDE>& g,
                                       double end, int64_t step, Acc& acc, int lane,
                                       Slot<WIDE>* scr) {
  int q0 = 0;
  unsigned retired_len = 0;
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int j = 32 * k + lane;
    const bool ret = j < R && sl[k].rem <= 0;
    const bool kp = j < R && !ret;
    unsigned km = __ballot_sync(SL_FULL, kp);
    if (kp) scr[q0 + __popc(km & lanemask_lt())] = sl[k];
    q0 += __popc(km);
    retired_len += __reduce_add_sync(SL_FULL, ret ? (unsigned)sl[k].cur_len : 0u);
    if (ret) {
      const int idx = sl[k].idx;
      const WRec& w = s.wr[idx];
      const double first = sl[k].first;
      const int32_t tout = s.true_out[idx];
      const double tpot = tout == 1 ? 0.0 : fdiv_(fsub_(end, first), (double)(tout - 1));
      const double ttft = fsub_(first, w.arr);
      const bool okc = ttft <= w.ttft && tpot <= w.tpot;
      acc.completed++;
      acc.compliant += okc;
      acc.ttft_viol += ttft > w.ttft;
      acc.tpot_viol += tpot > w.tpot;
      if (has_out) {
        const int64_t o = s.out_off + idx;
        a.out.status[o] = SL_COMPLETED;
        a.out.compliant[o] = okc;
        a.out.completion_step[o] = (int32_t)step;
        a.out.first_token_time[o] = first;
        a.out.completion_time[o] = end;
        a.out.ttft[o] = ttft;
        a.out.tpot[o] = tpot;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kSlots; ++k)
    if (32 * k + lane < q0) sl[k] = scr[32 * k + lane];
  __syncwarp();
  R = q0;
  g.lens -= retired_len;
  g.inv_valid = false;
  if (R > 0) {
    g.Smin = running_min<WIDE>(sl, R, lane);
    g.min_d = fixed_to_double<WIDE>(g.Smin, s.pow2E);
  }
}

// Quiet steps: nothing waiting, no arrival due, <= 32 running, credit
// batching, no decision log.  Exactly the general step restricted to that
// case (no admission, so prefill_s is the empty sum 0 and now + 0 == now,
// and the strictest entry always batches, so the step has work); kept as a
// tight loop because these steps are the critical path of a sweep.
template <bool WIDE>
__device__ __forceinline__ void quiet_steps(const Sim& s, const KArgs& a, bool has_out,
                                            Slot<WIDE> (&sl)[kSlots], int& R, Agg<WIDE>& g,
                                            double& now, int64_t& step, int64_t& n_plans,
                                            int64_t& req_steps, double next_t, bool has_h,
                                            Acc& acc, int lane, Slot<WIDE>* scr) {
  const sl_cost& C = s.cost;
  const double horizon = has_h ? s.horizon : __longlong_as_double(0x7ff0000000000000LL);
  // Digest items of the step end times are deferred: lane (step % 32) keeps the
  // end of its step and the 32 items are hashed together (one SIMT pass per 32
  // steps instead of one lane-0 pass per step).
  int64_t base = step;      // first step of the current 32-step window
  uint64_t end_bits = 0;    // this lane's pending end time (step base + lane)
  bool have_end = false;
  uint64_t key2 = digest_key((uint64_t)step, 2);
  while (R > 0 && R <= 32 && next_t > now && now < horizon) {
    ++n_plans;
    req_steps += R;
    // select_batch (sched_scorpio.py:171-179), fixed point
    const bool live = lane < R;
    const cred_t<WIDE> N = sl[0].N + g.Smin;
    const bool b = live && N >= sl[0].S;
    if (live) sl[0].N = b ? N - sl[0].S : N;
    const unsigned bm = __ballot_sync(SL_FULL, b);
    const int nb = __popc(bm);
    const unsigned blen = __reduce_add_sync(SL_FULL, b ? (unsigned)sl[0].cur_len : 0u);
    if (b) {
      acc.dig += digest_item_k(key2, __popc(bm & lanemask_lt()), (uint64_t)sl[0].id);
      sl[0].cur_len += 1;
      sl[0].rem -= 1;
    }
    g.lens += nb;
    double L;
    if ((nb & (nb - 1)) == 0)
      L = fmul_((double)blen, __longlong_as_double((long long)(1023 - (__ffs(nb) - 1)) << 52));
    else
      L = fdiv_((double)blen, (double)nb);
    const double end = fadd_(now, itl(C, nb, L));
    if (lane == (int)(step - base)) {
      end_bits = (uint64_t)__double_as_longlong(end);
      have_end = true;
    }
    if (__any_sync(SL_FULL, live && sl[0].rem <= 0))
      retire<WIDE>(s, a, has_out, sl, R, g, end, step, acc, lane, scr);
    now = end;
    ++step;
    key2 += kDigStep;
    if (step - base == 32) {
      if (have_end) acc.dig += digest_item((uint64_t)(base + lane), 3, 0, end_bits);
      have_end = false;
      base = step;
    }
  }
  if (have_end) acc.dig += digest_item((uint64_t)(base + lane), 3, 0, end_bits);
}

template <bool WIDE>
__device__ __forceinline__ void run_fast(const Sim& s, const KArgs& a, bool has_out, int si, int lane,
                         Slot<WIDE>* scr) {
  const int64_t n = s.n;
  const sl_cost& C = s.cost;
  const bool scorpio = s.policy == SL_POLICY_SCORPIO;
  const bool ttft_guard = (s.flags & SL_FLAG_TTFT_GUARD) != 0;
  const bool tpot_guard = (s.flags & SL_FLAG_TPOT_GUARD) != 0;
  const bool r_only = (s.flags & SL_FLAG_R_ONLY) != 0;
  const bool has_h = (s.flags & SL_FLAG_HAS_HORIZON) != 0;
  const bool sorted_ldf = scorpio && ttft_guard;
  const bool sjf = s.policy == SL_POLICY_SJF;
  const bool credit = scorpio && tpot_guard;
  const bool prio = !scorpio && (s.flags & SL_FLAG_PREFILL_PRIORITY);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);

  if (has_out) init_outcomes(s, a, lane);
  const bool logging = a.has_log && s.log_row >= 0;
  const int64_t lg_step0 = logging ? s.log_row * a.log.step_cap : 0;
  const int64_t lg_id0 = logging ? s.log_row * a.log.id_cap : 0;
  int64_t cur_adm = 0, cur_rej = 0, cur_bat = 0;
  bool log_over = false;

  Acc acc = {0, 0, 0, 0, 0, 0, 0, 0};
  Slot<WIDE> sl[kSlots];
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    sl[k].N = 0;
    sl[k].S = 0;
    sl[k].inv = 0.0;
    sl[k].first = 0.0;
    sl[k].id = 0;
    sl[k].idx = 0;
    sl[k].cur_len = 0;
    sl[k].rem = 0;
  }
  Agg<WIDE> g;
  g.Smin = 0;
  g.min_d = 0.0;
  g.lens = 0;
  g.inv = 0.0;
  g.inv_valid = true;

  double now = 0.0;
  int64_t next = 0;
  double next_t = n > 0 ? fdiv_(s.arrival[0], s.factor) : kInf;
  int W = 0, R = 0;
  int64_t step = 0, n_plans = 0, n_idle = 0, req_steps = 0;
  int status = SL_SIM_OK;

  for (;;) {
    if (next < n && next_t <= now)
      process_arrivals<WIDE>(s, W, next, next_t, now, sorted_ldf, sjf, lane);
    if (has_h && now >= s.horizon) break;  // simengine.py:190-191
    if (W == 0 && credit && !logging && R > 0 && R <= 32) {
      quiet_steps<WIDE>(s, a, has_out, sl, R, g, now, step, n_plans, req_steps, next_t, has_h, acc,
                        lane, scr);
      continue;
    }

    ++n_plans;
    req_steps += W + R;
    const int R0 = R;
    int nadm = 0, nrej = 0;
    PySum P;
    ps_init(P);
    acc.dig_rej = 0;
    const bool lg = logging && !log_over;
    const int64_t lg_adm = lg ? lg_id0 + cur_adm : -1;
    const int64_t lg_rej = lg ? lg_id0 + cur_rej : -1;
    const int64_t lg_bat = lg ? lg_id0 + cur_bat : -1;
    const int64_t cap_adm = logging ? a.log.id_cap - cur_adm : 0;
    const int64_t cap_rej = logging ? a.log.id_cap - cur_rej : 0;
    const int64_t cap_bat = logging ? a.log.id_cap - cur_bat : 0;

    bool fits = true;
    if (W > 0) {
      if (scorpio) {
        if (ttft_guard)
          spec_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej,
                    reinterpret_cast<double*>(scr));
        if (tpot_guard) {
          if (W > 0) {
            if (!g.inv_valid) {
              g.inv = running_inv_sum<WIDE>(sl, R, lane, reinterpret_cast<double*>(scr));
              g.inv_valid = true;
            }
            fits = spec_admit<WIDE>(s, a, has_out, W, R, sl, g, nadm, nrej, P, r_only, step, acc,
                                    lane, lg_adm, cap_adm, lg_rej, cap_rej);
          }
        } else {
          fits = append_prefix<WIDE>(s, a, W, R, sl, g, W, nadm, P, step, acc, lane, lg_adm,
                                     cap_adm);
        }
      } else {
        if (s.policy == SL_POLICY_EARLY_REJECT)
          spec_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej,
                    reinterpret_cast<double*>(scr));
        int room = s.cap - R;
        int take = room > 0 ? min(room, W) : 0;
        if (take > 0)
          fits = append_prefix<WIDE>(s, a, W, R, sl, g, take, nadm, P, step, acc, lane, lg_adm,
                                     cap_adm);
      }
    }
    if (!fits) {
      status = SL_SIM_CAPACITY;
      break;
    }

    // ---- decode batch: credit phase (select_batch :161-180) or decode-all
    unsigned bm[kSlots];
    unsigned blen = 0;
    int nb = 0;
    const bool decode = credit || !(prio && nadm > 0);
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      const int j = 32 * k + lane;
      bool b = false;
      if (decode && j < R0) {
        if (credit) {
          cred_t<WIDE> N = sl[k].N + g.Smin;
          b = N >= sl[k].S;
          sl[k].N = b ? N - sl[k].S : N;
        } else {
          b = true;
        }
      }
      bm[k] = __ballot_sync(SL_FULL, b);
      blen += __reduce_add_sync(SL_FULL, b ? (unsigned)sl[k].cur_len : 0u);
      if (b) {
        int pos = nb + __popc(bm[k] & lanemask_lt());
        acc.dig += digest_item((uint64_t)step, 2, (uint32_t)pos, (uint64_t)sl[k].id);
        if (lg_bat >= 0 && pos < cap_bat) a.log.batch_ids[lg_bat + pos] = sl[k].id;
        sl[k].cur_len += 1;  // token emit (simengine.py:243-245), after l_avg's input
        sl[k].rem -= 1;
      }
      nb += __popc(bm[k]);
    }
    g.lens += nb;

    // ---- no work: idle skip (simengine.py:207-227)
    if (nadm == 0 && nb == 0) {
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
      if (logging && a.log.skip_now && lane == 0) {  // EventLog.idle_skips (simengine.py:225)
        if (n_idle < a.log.skip_cap) {
          const int64_t o = s.log_row * a.log.skip_cap + n_idle;
          a.log.skip_now[o] = now;
          a.log.skip_target[o] = target;
          a.log.skip_waiting[o] = W;
          a.log.n_skips[s.log_row] = n_idle + 1;
        }
      }
      ++n_idle;
      now = target;
      continue;
    }

    // ---- step duration (simengine.py:233-238)
    const double prefill_s = ps_result(P);
    double decode_s = 0.0;
    if (nb > 0) {
      double L;
      if ((nb & (nb - 1)) == 0)  // exact: division by a power of two is a scaling
        L = fmul_((double)blen, __longlong_as_double((long long)(1023 - (__ffs(nb) - 1)) << 52));
      else
        L = fdiv_((double)blen, (double)nb);
      decode_s = itl(C, nb, L);
    }
    const double end = fadd_(fadd_(now, prefill_s), decode_s);
    acc.dig += acc.dig_rej;
    if (lane == 0) acc.dig += digest_item((uint64_t)step, 3, 0, (uint64_t)__double_as_longlong(end));

    // ---- decision log row (EventLog.steps)
    if (logging) {
      bool ok = !log_over && step < a.log.step_cap && cur_adm + nadm <= a.log.id_cap &&
                cur_rej + nrej <= a.log.id_cap && cur_bat + nb <= a.log.id_cap;
      if (ok) {
        double vbs = 0.0, mslo = __longlong_as_double(0x7ff8000000000000LL);
        if (scorpio && R > 0) {  // sched_scorpio.py:312-315, before retirement
          mslo = g.min_d;
          PySum vs;
          ps_init(vs);
#pragma unroll
          for (int k = 0; k < kSlots; ++k) {
            int cnt = min(32, R - 32 * k);
            double x = 32 * k + lane < R
                           ? fdiv_(mslo, fixed_to_double<WIDE>(sl[k].S, s.pow2E))
                           : 0.0;
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
          a.log.n_batch[o] = nb;
          a.log.n_steps[s.log_row] = step + 1;
        }
        cur_adm += nadm;
        cur_rej += nrej;
        cur_bat += nb;
      } else {
        log_over = true;
      }
    }

    // ---- fresh entries emit their first token; retirement (simengine.py:240-271)
    if (nadm > 0) {
#pragma unroll
      for (int k = 0; k < kSlots; ++k) {
        const int j = 32 * k + lane;
        if (j >= R0 && j < R) {
          sl[k].cur_len += 1;
          sl[k].rem -= 1;
          sl[k].first = end;
        }
      }
      g.lens += nadm;
    }
    bool any_ret = false;
#pragma unroll
    for (int k = 0; k < kSlots; ++k)
      any_ret |= __any_sync(SL_FULL, 32 * k + lane < R && sl[k].rem <= 0);
    if (any_ret) retire<WIDE>(s, a, has_out, sl, R, g, end, step, acc, lane, scr);
    now = end;
    ++step;
  }

  write_result(a, si, acc, status | (log_over ? SL_SIM_LOG_OVERFLOW : 0), n, step, n_plans,
               n_idle, req_steps, now, has_h, s.horizon, lane);
}

}  // namespace sl
