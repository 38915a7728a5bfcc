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
#ifndef SL_INV_UNROLL
#define SL_INV_UNROLL 0  // unrolled branch-free 1/slo fold (measured: 112 -> 118 ms, registers)
#endif
#ifndef SL_QUIET_SMEM
#define SL_QUIET_SMEM 1  // quiet loop: per-step digest inputs in a shared-memory ring
#endif
#ifndef SL_ARR2
#define SL_ARR2 0  // keep the arrival time after next in a register (single-arrival fast path)
#endif
#ifndef SL_QUIET_NOLIVE
#define SL_QUIET_NOLIVE 0  // quiet loop: dead lanes neutralised once instead of tested per step
#endif
#ifndef SL_ACC_SMEM
#define SL_ACC_SMEM 0  // per-lane outcome counters in shared memory instead of registers
#endif
#if SL_ACC_SMEM
constexpr int kAccWarps = 4;  // == kFastWarps (sim_kernel.cu)
enum { kAccCompleted, kAccCompliant, kAccRejTtft, kAccRejAdm, kAccTtftViol, kAccTpotViol };
__shared__ int32_t sl_acc_sm[kAccWarps][6][32];
#define SL_ACC_ADD(acc, field, K, v) (sl_acc_sm[threadIdx.x >> 5][K][threadIdx.x & 31] += (v))
#else
#define SL_ACC_ADD(acc, field, K, v) ((acc).field += (v))
#endif
#ifndef SL_QUIET_PIPE
#define SL_QUIET_PIPE 0  // quiet loop: step k+1's batch formed during step k's clock update
#endif
#ifndef SL_INV_FOLD
#define SL_INV_FOLD 0  // branch-free ps_add_nz loop for the 1/slo fold rebuild
#endif
#ifndef SL_WALK_SKIP
#define SL_WALK_SKIP 1  // general steps skip the walk while now < walk_until
#endif

// Optional per-phase cycle accounting (profiling builds only: -DSL_PHASE_PROF,
// read back with sl_phase_prof_read).  Slots 0-7: cycles per phase, 8-13: counts,
// 14-15: %globaltimer (ns) at the sim's start and end, 16-19: walks, exact walks,
// sum of W over walks, sum of W over admission scans.
#ifdef SL_PHASE_PROF
constexpr int kProfSims = 1 << 16;
constexpr int kProfSlots = 26;
__device__ __forceinline__ unsigned long long prof_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long sl_prof_cycles[kProfSims][kProfSlots];
#define SL_PROF_DECL              \
  unsigned long long prof_acc[kProfSlots] = {0}; \
  prof_acc[14] = prof_gtime();                   \
  long long prof_t = clock64();
#define SL_PROF_MARK(k)                 \
  {                                     \
    const long long t_ = clock64();     \
    prof_acc[k] += (unsigned long long)(t_ - prof_t); \
    prof_t = t_;                        \
  }
#define SL_PROF_COUNT(k, v) prof_acc[k] += (v);
#define SL_PROF_WRITE(si)                                                  \
  prof_acc[15] = prof_gtime();                                             \
  if (lane == 0 && (si) < kProfSims)                                       \
    for (int k_ = 0; k_ < kProfSlots; ++k_) sl_prof_cycles[si][k_] = prof_acc[k_];
#elif defined(SL_TIMELINE)
// Timeline-only build (-DSL_TIMELINE): %globaltimer at each sim's start and end,
// stored straight to global memory (no live registers), read with
// sl_phase_prof_read into slots 14-15.
constexpr int kProfSims = 1 << 16;
constexpr int kProfSlots = 26;
__device__ unsigned long long sl_prof_cycles[kProfSims][kProfSlots];
__device__ __forceinline__ unsigned long long prof_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SL_PROF_DECL \
  if (lane == 0 && si < kProfSims) sl_prof_cycles[si][14] = prof_gtime();
#define SL_PROF_MARK(k)
#define SL_PROF_COUNT(k, v)
#define SL_PROF_WRITE(si) \
  if (lane == 0 && (si) < kProfSims) sl_prof_cycles[si][15] = prof_gtime();
#else
#define SL_PROF_DECL
#define SL_PROF_MARK(k)
#define SL_PROF_COUNT(k, v)
#define SL_PROF_WRITE(si)
#endif

// A running entry held in registers.  1/slo is recomputed from S when the
// Neumaier fold has to be rebuilt, the first-token time lives in the
// workspace (first_emit[idx]); the id is only read by the decision log.
template <bool WIDE>
struct Slot {
  cred_t<WIDE> N, S;  // credit numerator, fixed-point slo
  int64_t id;         // request id
  int32_t idx;        // request index in the trace
  int32_t cur_len;    // prompt_len + tokens_generated
  int32_t rem;        // true_output_len - tokens_generated
  uint32_t hid;       // batch_hid(id), the digest's per-entry hash
};

// Conditional per-field moves (not `sl[pos >> 5] = e`, which would force the
// slot array into local memory through a dynamic index).
template <bool WIDE>
__device__ __forceinline__ void sel_slot(Slot<WIDE>& d, bool c, const Slot<WIDE>& e) {
  d.N = c ? e.N : d.N;
  d.S = c ? e.S : d.S;
  d.id = c ? e.id : d.id;
  d.hid = c ? e.hid : d.hid;
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
__device__ __forceinline__ PySum running_inv_sum(const Sim& s, const Slot<WIDE> (&sl)[kSlots],
                                                 int R, int lane, double* bc) {
  PySum ps;
  ps_init(ps);
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int cnt = min(32, R - 32 * k);
    if (cnt <= 0) break;
    // 1.0 / tpot: S * 2^E is tpot exactly, so this is the WRec's inv bit for bit
    if (32 * k + lane < R) bc[lane] = frcp_(fixed_to_double<WIDE>(sl[k].S, s.pow2E));
    __syncwarp();
    if (SL_INV_UNROLL && cnt == 32 && ps.n > 0) {
      double v[32];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const double2 p = reinterpret_cast<const double2*>(bc)[t];
        v[2 * t] = p.x;
        v[2 * t + 1] = p.y;
      }
#pragma unroll
      for (int t = 0; t < 32; ++t) ps_add_nz(ps, v[t]);
    } else if (SL_INV_FOLD) {
      ps_fold_buf(ps, bc, cnt);
    } else {
      for (int t = 0; t < cnt; ++t) ps_add(ps, bc[t]);
    }
    __syncwarp();
  }
  return ps;
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

// Time up to which the walk provably rejects nothing: item j passed at `now`
// with prefix bound U (est0 = fl(fl(fl(now - arr) + U) + pf) <= ttft).  Until
// the next insertion its prefix can only shrink, so at a later now1 its est stays
// <= ttft while now1 - now < sigma - m, sigma = fl(ttft - est0),
// m = 2^-39 (now + U + pf + sigma) >> the <= 8u relative rounding error of the
// three-op chain at now and now1 (+ that of sigma and of this sum).  Clamped
// to >= 0 so that the bit patterns order like the values (warp_min_nonneg).
__device__ __forceinline__ double walk_pass_until(double now, double U, double pf, double tt,
                                                  double est0) {
  const double sig = fsub_(tt, est0);
  const double m = fmul_(1.8189894035458565e-12, fadd_(fadd_(fadd_(now, U), pf), sig));
  const double t = fsub_(fadd_(now, sig), m);
  return t >= 0.0 ? t : 0.0;  // also maps NaN to 0 (no skipping)
}

// Warp minimum of non-negative doubles (their bit patterns order like the values).
__device__ __forceinline__ double warp_min_nonneg(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const unsigned hi = __reduce_min_sync(SL_FULL, (unsigned)(b >> 32));
  const unsigned lo = __reduce_min_sync(SL_FULL, (unsigned)(b >> 32) == hi ? (unsigned)b : ~0u);
  return __longlong_as_double((long long)(((uint64_t)hi << 32) | lo));
}

// Certified pass over chunks [c_from, W) of the queue given an upper bound U of
// the prefix before c_from (see spec_walk): true iff no item can be rejected;
// tmin / U accumulate the walk bound and the inflated running prefix bound.
__device__ __forceinline__ bool cert_scan(const Sim& s, double now, int W, int c_from, int lane,
                                          double& U, double& tmin) {
  const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
  bool all_ok = true;
  for (int c0 = c_from; c0 < W && all_ok; c0 += 32) {
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
    const double est0 = fadd_(fadd_(e, Uj), pf);
    all_ok = __all_sync(SL_FULL, !valid || est0 <= tt);
    if (valid) tmin = fmin(tmin, walk_pass_until(now, Uj, pf, tt, est0));
    U = fmul_(fadd_(U, __shfl_sync(SL_FULL, v, 31)), inflate);
  }
  return all_ok;
}

#ifndef SL_BLOCK_ARR
#define SL_BLOCK_ARR 1  // a blocked queue stays blocked across a failing arrival
#endif
#ifndef SL_BOUND_WALK
#define SL_BOUND_WALK 1  // two-sided certified walk (see spec_walk_bounds)
#endif
#ifndef SL_WALK_MARGIN
// relative margin of the walk's prefix bounds (2^-30); any larger value is as
// exact (wider bounds, more chunks on the serial form): the parity tests run a
// 2^-8 build to exercise that form (tests/test_gpu_variant_builds.py)
#define SL_WALK_MARGIN 9.313225746154785e-10
#endif

// Rejection side effects of one walk chunk and the stable compaction of its
// kept items to wl[kept, ...) (shared by both walk forms).
__device__ __forceinline__ void walk_commit(const Sim& s, const KArgs& a, bool has_out, int& kept,
                                            int& nrej, bool valid, int idx, unsigned rejm,
                                            int64_t step, Acc& acc, int lane, int64_t lg_rej,
                                            int64_t cap_rej) {
  const bool r_ = valid && ((rejm >> lane) & 1u);
  const bool keep = valid && !r_;
  const unsigned km = __ballot_sync(SL_FULL, keep);
  __syncwarp();
  if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
  if (r_) {
    const int pos = nrej + __popc(rejm & lanemask_lt());
    const int64_t rid = s.id[idx];
    acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u);
    SL_ACC_ADD(acc, rej_ttft, kAccRejTtft, 1);
    if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_TTFT;
    if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2;
  }
  __syncwarp();
  kept += __popc(km);
  nrej += __popc(rejm);
}

// TTFT prefix walk, two-sided certified form (ttft_guard sched_scorpio.py:196-205;
// early_reject sched_baselines.py:95-103).  The exact walk keeps a sequential
// fl-sum `prefix` of the kept prefills and rejects item j iff
// fl(fl(e_j + prefix_j) + pf_j) > ttft_j, e_j = fl(now - arr_j).  That test is
// monotone in prefix_j, so bounds Lj <= prefix_j <= Uj decide it exactly
// whenever both agree.  Per chunk, one warp scan (any order) of the prefills of
// the items not yet rejected gives excl_j; with Pl <= (exact real sum of the
// kept prefills before the chunk) <= ... and Pu an upper bound of the
// sequential prefix,
//   Uj = fl(fl(Pu + excl_j) (1 + 2^-30)),  Lj = fl(fl(Pl + excl_j) (1 - 2^-30))
// bound prefix_j: any-order fl-sums of n < 2^20 non-negative terms are within
// (n-1) u < 2^-33 relative of the real sum, which the 2^-30 factors dominate
// (with the rounding of the two ops).  The first item that is not certain to
// pass is either certain to fail (rejected; the chunk is re-scanned without it,
// since later prefixes shrink) or undecided (|est - ttft| within ~2^-29 of the
// prefix): then the chunk runs the serial exact walk from the exact prefix (the
// sequential sum of the kept prefills so far, recomputed when not known).
// Items failing at Pl fail at any prefix: rejected outright.  Returns true when
// anything was rejected or a chunk ran serially; `until` / `p_up` as spec_walk.
__device__ __forceinline__ bool spec_walk_bounds(const Sim& s, const KArgs& a, bool has_out,
                                                 int& W, int& nrej, double now, int64_t step,
                                                 Acc& acc, int lane, int64_t lg_rej,
                                                 int64_t cap_rej, double* bc, double& until,
                                                 double& p_up) {
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const double up = 1.0 + SL_WALK_MARGIN, dn = 1.0 - SL_WALK_MARGIN;
  const bool certifiable = W < (1 << 20);
  double Pl = 0.0, Pu = 0.0;  // bounds of the incoming prefix (equal and exact while pex)
  bool pex = true;
  double tmin = kInf;
  int kept = 0;
  bool any = false;
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int j = c0 + lane;
    const bool valid = j < W;
    int idx = 0;
    double e = 0.0, pf = 0.0, tt = 0.0;
    if (valid) {
      idx = s.wl[j];
      const WRec& r = s.wr[idx];
      e = fsub_(now, r.arr);
      pf = r.prefill;
      tt = r.ttft;
    }
    unsigned rejm = __ballot_sync(SL_FULL, valid && fadd_(fadd_(e, Pl), pf) > tt);
    bool serial = !certifiable;
    double Uj = 0.0, estU = 0.0, tot = 0.0;
    while (!serial) {
      const bool live = valid && !((rejm >> lane) & 1u);
      double v = live ? pf : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(SL_FULL, v, o);
        if (lane >= o) v = fadd_(v, y);
      }
      double excl = __shfl_up_sync(SL_FULL, v, 1);
      if (lane == 0) excl = 0.0;
      tot = __shfl_sync(SL_FULL, v, 31);
      Uj = fmul_(fadd_(Pu, excl), up);
      estU = fadd_(fadd_(e, Uj), pf);
      const unsigned m = __ballot_sync(SL_FULL, live && !(estU <= tt));
      if (!m) break;
      const int f = __ffs(m) - 1;
      const double Lj = fmul_(fadd_(Pl, excl), dn);
      const bool fails = fadd_(fadd_(e, Lj), pf) > tt;
      if (__shfl_sync(SL_FULL, (int)fails, f)) {
        rejm |= 1u << f;
      } else {
        serial = true;
      }
    }
    if (!serial) {
      if (valid && !((rejm >> lane) & 1u))
        tmin = fmin(tmin, walk_pass_until(now, Uj, pf, tt, estU));
      Pl = fmul_(fadd_(Pl, tot), dn);
      Pu = fmul_(fadd_(Pu, tot), up);
      pex = false;
    } else {
      // exact incoming prefix, then the reference's loop over the chunk
      double p = Pl;
      if (!pex) {
        p = 0.0;
        for (int t = 0; t < kept; ++t) p = fadd_(p, s.wr[s.wl[t]].prefill);
      }
      double* bcE = bc + 32;
      double* bcT = bc + 64;
      bc[lane] = pf;
      bcE[lane] = e;
      bcT[lane] = tt;
      __syncwarp();
      rejm = 0u;
      double mine = 0.0;
      const int cnt = min(32, W - c0);
      for (int t = 0; t < cnt; ++t) {
        const double pt = bc[t];
        if (lane == t) mine = p;
        if (fadd_(fadd_(bcE[t], p), pt) > bcT[t])
          rejm |= 1u << t;
        else
          p = fadd_(p, pt);
      }
      __syncwarp();
      if (valid && !((rejm >> lane) & 1u))
        tmin = fmin(tmin, walk_pass_until(now, mine, pf, tt, fadd_(fadd_(e, mine), pf)));
      Pl = Pu = p;
      pex = true;
      any = true;
    }
    if (rejm) any = true;
    if (rejm || kept != c0)
      walk_commit(s, a, has_out, kept, nrej, valid, idx, rejm, step, acc, lane, lg_rej, cap_rej);
    else
      kept += min(32, W - c0);
  }
  W = kept;
  until = warp_min_nonneg(tmin);
  p_up = pex ? fmul_(Pu, up) : Pu;
  return any;
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
//     first rejection; from there one serial pass with the test inline.
// `until` receives the time before which the walk over the remaining queue
// provably rejects nothing (walk_pass_until), valid until the next insertion.
__device__ __forceinline__ bool spec_walk(const Sim& s, const KArgs& a, bool has_out, int& W,
                                          int& nrej, double now, int64_t step, Acc& acc, int lane,
                                          int64_t lg_rej, int64_t cap_rej, double* bc,
                                          double& until, double& p_up) {
#if SL_BOUND_WALK
  return spec_walk_bounds(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej, bc,
                          until, p_up);
#endif
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const bool certifiable = W < (1 << 20);
  if (certifiable) {
    double U = 0.0;
    double tmin = kInf;
    if (cert_scan(s, now, W, 0, lane, U, tmin)) {
      until = warp_min_nonneg(tmin);
      p_up = U;  // inflated total: bounds every prefix of the queue
      return false;
    }
  }
  double* bcE = bc + 32;
  double* bcT = bc + 64;
  double prefix = 0.0;
  double tmin = kInf;
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
    // items failing at the chunk's incoming prefix fail at any later one
    // (prefixes only grow, est is monotone in them): rejected outright
    unsigned rejm = __ballot_sync(SL_FULL, valid && fadd_(fadd_(e, prefix), pf) > tt);
    bc[lane] = ((rejm >> lane) & 1u) ? 0.0 : pf;  // x + 0.0 == x: rejected items add nothing
    __syncwarp();
    // speculative pass: the exact sequential prefix chain assuming every
    // undecided item is kept, tested lane-parallel
    double run = prefix, mine = 0.0;
    for (int t = 0; t < cnt; ++t) {
      if (lane == t) mine = run;
      run = fadd_(run, bc[t]);
    }
    const unsigned m = __ballot_sync(SL_FULL, valid && !((rejm >> lane) & 1u) &&
                                                  fadd_(fadd_(e, mine), pf) > tt);
    if (m) {
      // first rejection r: earlier items saw the true prefix; from r on the
      // chain runs serially with the test inline (one pass however many reject)
      const int r = __ffs(m) - 1;
      rejm |= 1u << r;
      double p = __shfl_sync(SL_FULL, mine, r);  // a rejected item leaves the prefix unchanged
      bcE[lane] = e;
      bcT[lane] = tt;
      __syncwarp();
      for (int t = r + 1; t < cnt; ++t) {
        if ((rejm >> t) & 1u) continue;
        const double pt = bc[t];
        const double est = fadd_(fadd_(bcE[t], p), pt);
        if (lane == t) mine = p;
        if (est > bcT[t])
          rejm |= 1u << t;
        else
          p = fadd_(p, pt);
      }
      run = p;
    }
    prefix = run;
    const bool r_ = valid && ((rejm >> lane) & 1u);
    const bool keep = valid && !r_;
    if (keep) tmin = fmin(tmin, walk_pass_until(now, mine, pf, tt, fadd_(fadd_(e, mine), pf)));
    const unsigned km = __ballot_sync(SL_FULL, keep);
    __syncwarp();
    if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
    if (r_) {
      const int pos = nrej + __popc(rejm & lanemask_lt());
      const int64_t rid = s.id[idx];
      acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u);
      SL_ACC_ADD(acc, rej_ttft, kAccRejTtft, 1);
      if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_TTFT;
      if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2;
    }
    __syncwarp();
    kept += __popc(km);
    nrej += __popc(rejm);
    if (rejm && certifiable && c0 + 32 < W) {
      // rejections come first in deadline order: if the rest of the queue is
      // certified from the exact prefix here, it only moves down the list
      double U = prefix, tc = tmin;
      if (cert_scan(s, now, W, c0 + 32, lane, U, tc)) {
        for (int c1 = c0 + 32; c1 < W; c1 += 32) {
          const bool v1 = c1 + lane < W;
          const int i1 = v1 ? s.wl[c1 + lane] : 0;
          __syncwarp();
          if (v1) s.wl[kept + lane] = i1;
          __syncwarp();
          kept += min(32, W - c1);
        }
        W = kept;
        until = warp_min_nonneg(tc);
        p_up = U;
        return true;
      }
    }
  }
  W = kept;
  until = warp_min_nonneg(tmin);
  p_up = fmul_(prefix, 1.0 + 9.313225746154785e-10);  // kept total, inflated by 2^-30
  return true;  // the exact walk ran
}

// Cached running-set aggregates (sched_scorpio.py:117-124), warp-uniform.
template <bool WIDE>
struct Agg {
  cred_t<WIDE> Smin;  // min fixed-point slo over running (valid iff R > 0)
  double min_d;       // the same as a double
  int64_t lens;       // sum of current_len over running
  PySum pinv;         // Neumaier fold of 1/slo over running, in order (CPython sum state);
  bool inv_valid;      // appends extend the fold exactly, removals invalidate it
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
  double inv = ps_result(g.pinv);  // plain adds below (:275); the fold is extended separately
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
    double tp = 0.0, ic = 0.0;
    int32_t ln = 0, ps_ = 0;
    if (valid) {  // the test's inputs; prefill / fixed slo are read for the admitted only
      idx = s.wl[j];
      const WRec& w = s.wr[idx];
      tp = w.tpot;
      ic = w.inv;
      ln = w.prompt;
      ps_ = w.pred_solo;
    }
    const int32_t pred = ps_ & 0x7fffffff;
    const bool solo = (ps_ & (int32_t)0x80000000) != 0;
    const unsigned vmask = __ballot_sync(SL_FULL, valid);
    unsigned pend = vmask, admm = 0;
    // one round per admission: every pending candidate against the same state A
    // (_admission_math :99-114); lanes before the first admit fail against A and
    // are decided; the chunk's failures are settled once after the rounds
    while (pend) {
      bool lt = !has_min || tp < mind;
      double minp = lt ? tp : mind;
      double V = fmul_(minp, fadd_(inv, ic));
      double L = div_small((double)(lens + ln), (int)(n_run + 1));
      double est = tpot_estimate(C, V, L, pred);
      double thr = (r_only && has_min) ? mind : minp;
      const unsigned okm = __ballot_sync(SL_FULL, ((pend >> lane) & 1u) && est <= thr);
      if (!okm) break;
      const int gl = __ffs(okm) - 1;
      // admit candidate gl (warp-uniform state update, :250-278)
      if (R >= kRunCap) {
        ok_cap = false;
        break;
      }
      Slot<WIDE> e;
      e.N = 0;
      e.idx = bcast(idx, gl);
      const WRec& wg = s.wr[e.idx];
      if constexpr (WIDE)
        e.S = ((unsigned __int128)s.wShi[e.idx] << 64) | wg.S;
      else
        e.S = wg.S;
      e.id = s.id[e.idx];
      e.hid = batch_hid((uint64_t)e.id);
      const double e_inv = bcast(ic, gl);
      e.cur_len = bcast(ln, gl);
      e.rem = s.true_out[e.idx];
      const double tp_g = bcast(tp, gl);
      const double pf_g = wg.prefill;
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
      inv = fadd_(inv, e_inv);  // plain float add, :275
      ps_add(g.pinv, e_inv);    // next step's sum() over the running list
      lens += e.cur_len;
      if (lt_g) {
        mind = tp_g;
        Smn = e.S;
      }
      has_min = true;
      ps_add(P, pf_g);
      ++nadm;
      ++R;
      admm |= 1u << gl;
      pend &= ~((2u << gl) - 1u);
    }
    if (!ok_cap) break;
    // failures: outright reject unless feasible alone (:279-291), in queue order
    const unsigned fail = vmask & ~admm;
    const bool mf = (fail >> lane) & 1u;
    const bool keep = mf && solo;
    const bool rj = mf && !solo;
    const unsigned km = __ballot_sync(SL_FULL, keep);
    const unsigned rm = fail & ~km;
    __syncwarp();
    if (keep) s.wl[kept + __popc(km & lanemask_lt())] = idx;
    if (rj) {
      const int64_t rid = s.id[idx];  // ids only for decided requests
      int pos = nrej + __popc(rm & lanemask_lt());
      acc.dig_rej += digest_item((uint64_t)step, 1, (uint32_t)pos, (uint64_t)rid * 2u + 1u);
      SL_ACC_ADD(acc, rej_adm, kAccRejAdm, 1);
      if (has_out) a.out.status[s.out_off + idx] = SL_REJECTED_ADMISSION;
      if (lg_rej >= 0 && pos < cap_rej) a.log.rej_ids[lg_rej + pos] = rid * 2 + 1;
    }
    kept += __popc(km);
    nrej += __popc(rm);
    __syncwarp();
  }
  W = kept;
  g.lens = lens;
  if (nadm) {
    g.min_d = mind;
    g.Smin = Smn;
    // the fold g.pinv was extended entry by entry (the scan's plain adds are not it)
  }
  return ok_cap;
}

// Append waiting items wl[0, take) to the running set in order (admit-all,
// sched_scorpio.py:295-304, and admit_fcfs, sched_baselines.py:49-60), then
// drop them from the front of the waiting list by advancing its base (each
// request enters the list once, so base + W stays within the sim's n slots).
// `s` is this thread's own copy of the Sim (never called by the hot kernel,
// whose Sim is shared in shared memory).
template <bool WIDE>
__device__ __forceinline__ bool append_prefix(Sim& s, const KArgs& a, int& W, int& R,
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
      e.id = s.id[idx];
      e.hid = batch_hid((uint64_t)e.id);
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
      x.id = bcast(e.id, t);
      x.hid = bcast(e.hid, t);
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
  s.wl += take;
  nadm += take;
  W -= take;
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
      const double first = s.first_emit[idx];
      const int32_t tout = s.true_out[idx];
      const double tpot = tout == 1 ? 0.0 : fdiv_(fsub_(end, first), (double)(tout - 1));
      const double ttft = fsub_(first, w.arr);
      const bool okc = ttft <= w.ttft && tpot <= w.tpot;
      SL_ACC_ADD(acc, completed, kAccCompleted, 1);
      SL_ACC_ADD(acc, compliant, kAccCompliant, okc);
      SL_ACC_ADD(acc, ttft_viol, kAccTtftViol, ttft > w.ttft);
      SL_ACC_ADD(acc, tpot_viol, kAccTpotViol, tpot > w.tpot);
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

// Quiet steps (<= 32 running, credit batching, no log, and either nothing
// waiting or a waiting queue that provably stays untouched: `blocked` -- the
// admission scan fails for every request, see run_fast -- and the walk passes
// every request while now < walk_until): the general step restricted to that
// case, where a step's only decisions are the credit batch and the clock.
// One step per iteration; the digest items are deferred and hashed
// lane-parallel, 32 steps per pass (lane j keeps step base+j).  (A 32-step
// lookahead form -- per-lane credit recurrences, parallel itl(), serial clock --
// cut the critical-path sim by 15-25% but its code cost the sweep 10-25% in
// instruction-cache stalls.)
// Returns true when entries retire at the end of the last step (at `now`, step
// index `step - 1`): the caller runs retire() -- its one call site, which keeps
// the hot instruction footprint small.
template <bool WIDE>
__device__ __forceinline__ bool quiet_steps(const Sim& s, const KArgs& a, bool has_out,
                                            Slot<WIDE> (&sl)[kSlots], int& R, const int W,
                                            Agg<WIDE>& g, double& now, int64_t& step,
                                            int64_t& n_plans, int64_t& req_steps, double next_t,
                                            double walk_until, bool has_h, Acc& acc, int lane,
                                            Slot<WIDE>* scr, bool all = false) {
  const sl_cost& C = s.cost;
  const double horizon = has_h ? s.horizon : __longlong_as_double(0x7ff0000000000000LL);
  // a step runs while now < lim (next arrival, horizon, walk bound: all strict)
  const double lim = fmin(fmin(next_t, horizon), walk_until);
  const bool live = lane < R;
  const uint32_t hh = sl[0].hid;
  // per-call bookkeeping: the running set and the queue are fixed within the
  // loop, so plan / request-step / length counters are settled at exit
  const int64_t step0 = step;
  const unsigned cl0 = live ? (unsigned)sl[0].cur_len : 0u;
  int k = 0;  // steps done in this call; digest window = steps [k & ~31, k)
  uint64_t end_bits = 0;
  uint32_t d_nb = 0, d_bh = 0;
  bool have = false;
  bool ret = false;
#if SL_QUIET_PIPE
#if SL_QUIET_SMEM
  uint4* ring = reinterpret_cast<uint4*>(scr);
  int flushed = 0;  // steps [0, flushed) of this call are hashed
#endif
  // One-step software pipeline: the credit recurrence does not depend on the
  // clock, so step k+1's batch (credits, ballot, length / hash sums) is formed
  // while step k's itl() chain is in flight, and committed only when step k+1
  // runs (a retirement at step k, or the loop bound, discards it).
  if (R > 0 && R <= 32 && now < lim) {
    cred_t<WIDE> N1 = sl[0].N + g.Smin;
    bool b1 = live && (all || N1 >= sl[0].S);
    unsigned nb1 = __popc(__ballot_sync(SL_FULL, b1));
    unsigned blen1 = __reduce_add_sync(SL_FULL, b1 ? (unsigned)sl[0].cur_len : 0u);
    unsigned bh1 = __reduce_add_sync(SL_FULL, b1 ? hh : 0u);
    for (;;) {
      if (live && !all) sl[0].N = b1 ? N1 - sl[0].S : N1;
      if (b1) {
        sl[0].cur_len += 1;
        sl[0].rem -= 1;
      }
      const int nb = (int)nb1;
      const unsigned blen = blen1, bh = bh1;
      ret = __any_sync(SL_FULL, live && sl[0].rem <= 0);
      N1 = sl[0].N + g.Smin;  // step k+1, speculative
      b1 = live && (all || N1 >= sl[0].S);
      nb1 = __popc(__ballot_sync(SL_FULL, b1));
      blen1 = __reduce_add_sync(SL_FULL, b1 ? (unsigned)sl[0].cur_len : 0u);
      bh1 = __reduce_add_sync(SL_FULL, b1 ? hh : 0u);
      const double end = fadd_(now, itl(C, nb, div_small((double)blen, nb)));
#if SL_QUIET_SMEM
      if (lane == (k & 31)) {
        const uint64_t eb = (uint64_t)__double_as_longlong(end);
        ring[k & 31] = make_uint4((unsigned)nb, bh, (unsigned)eb, (unsigned)(eb >> 32));
      }
#else
      if (lane == (k & 31)) {
        end_bits = (uint64_t)__double_as_longlong(end);
        d_nb = nb;
        d_bh = bh;
        have = true;
      }
#endif
      now = end;
      ++k;
      if (ret || !(now < lim)) break;
      if ((k & 31) == 0) {
#if SL_QUIET_SMEM
        __syncwarp();
        const uint4 q = ring[lane];
        const uint64_t st = (uint64_t)(step0 + k - 32 + lane);
        acc.dig += digest_item(st, 2, q.x, q.y) +
                   digest_item(st, 3, 0, ((uint64_t)q.w << 32) | q.z);
        flushed = k;
        __syncwarp();
#else
        if (have)
          acc.dig += digest_item((uint64_t)(step0 + k - 32 + lane), 2, d_nb, d_bh) +
                     digest_item((uint64_t)(step0 + k - 32 + lane), 3, 0, end_bits);
        have = false;
#endif
      }
    }
  }
#if SL_QUIET_SMEM
  __syncwarp();
  if (flushed + lane < k) {
    const uint4 q = ring[lane];
    const uint64_t st = (uint64_t)(step0 + flushed + lane);
    acc.dig += digest_item(st, 2, q.x, q.y) + digest_item(st, 3, 0, ((uint64_t)q.w << 32) | q.z);
  }
  __syncwarp();
#endif
#elif SL_QUIET_SMEM
  // the step's digest inputs (batch size, batch hash, end time) go to a 32-entry
  // ring in the (here unused) scratch: one lane's store per step, hashed 32 steps
  // at a time lane-parallel
  uint4* ring = reinterpret_cast<uint4*>(scr);
  int flushed = 0;  // steps [0, flushed) of this call are hashed
#if SL_QUIET_NOLIVE
  // lanes past R hold no entry: zero credit, earn 0, S = 1 -> never batched, and
  // rem = 1 -> never retire, so the step needs no liveness tests (their slot
  // fields are dead and are overwritten by put_slot when an entry arrives)
  const cred_t<WIDE> earn = live ? g.Smin : cred_t<WIDE>(0);
  if (!live) {
    sl[0].N = 0;
    sl[0].S = 1;
    sl[0].rem = 1;
  }
#endif
  while (R > 0 && R <= 32 && now < lim) {
#if SL_QUIET_NOLIVE
    const cred_t<WIDE> N = sl[0].N + earn;
    const bool b = all ? live : N >= sl[0].S;  // all: decode-all policies, no credits
    if (!all) sl[0].N = b ? N - sl[0].S : N;
#else
    const cred_t<WIDE> N = sl[0].N + g.Smin;
    const bool b = live && (all || N >= sl[0].S);  // all: decode-all policies, no credits
    if (live && !all) sl[0].N = b ? N - sl[0].S : N;
#endif
    const int nb = __popc(__ballot_sync(SL_FULL, b));
    const unsigned blen = __reduce_add_sync(SL_FULL, b ? (unsigned)sl[0].cur_len : 0u);
    const unsigned bh = __reduce_add_sync(SL_FULL, b ? hh : 0u);
    if (b) {
      sl[0].cur_len += 1;
      sl[0].rem -= 1;
    }
    const double end = fadd_(now, itl(C, nb, div_small((double)blen, nb)));
    if (lane == (k & 31)) {
      const uint64_t eb = (uint64_t)__double_as_longlong(end);
      ring[k & 31] = make_uint4((unsigned)nb, bh, (unsigned)eb, (unsigned)(eb >> 32));
    }
#if SL_QUIET_NOLIVE
    ret = __any_sync(SL_FULL, sl[0].rem <= 0);
#else
    ret = __any_sync(SL_FULL, live && sl[0].rem <= 0);
#endif
    now = end;
    ++k;
    if (ret) break;
    if ((k & 31) == 0) {
      __syncwarp();
      const uint4 q = ring[lane];
      const uint64_t st = (uint64_t)(step0 + k - 32 + lane);
      acc.dig += digest_item(st, 2, q.x, q.y) +
                 digest_item(st, 3, 0, ((uint64_t)q.w << 32) | q.z);
      flushed = k;
      __syncwarp();
    }
  }
  __syncwarp();
  if (flushed + lane < k) {
    const uint4 q = ring[lane];
    const uint64_t st = (uint64_t)(step0 + flushed + lane);
    acc.dig += digest_item(st, 2, q.x, q.y) + digest_item(st, 3, 0, ((uint64_t)q.w << 32) | q.z);
  }
  __syncwarp();
#else
  while (R > 0 && R <= 32 && now < lim) {
    const cred_t<WIDE> N = sl[0].N + g.Smin;
    const bool b = live && (all || N >= sl[0].S);  // all: decode-all policies, no credits
    if (live && !all) sl[0].N = b ? N - sl[0].S : N;
    const int nb = __popc(__ballot_sync(SL_FULL, b));
    const unsigned blen = __reduce_add_sync(SL_FULL, b ? (unsigned)sl[0].cur_len : 0u);
    const unsigned bh = __reduce_add_sync(SL_FULL, b ? hh : 0u);
    if (b) {
      sl[0].cur_len += 1;
      sl[0].rem -= 1;
    }
    const double end = fadd_(now, itl(C, nb, div_small((double)blen, nb)));
    if (lane == (k & 31)) {
      end_bits = (uint64_t)__double_as_longlong(end);
      d_nb = nb;
      d_bh = bh;
      have = true;
    }
    ret = __any_sync(SL_FULL, live && sl[0].rem <= 0);
    now = end;
    ++k;
    if (ret) break;
    if ((k & 31) == 0) {
      if (have)
        acc.dig += digest_item((uint64_t)(step0 + k - 32 + lane), 2, d_nb, d_bh) +
                   digest_item((uint64_t)(step0 + k - 32 + lane), 3, 0, end_bits);
      have = false;
    }
  }
#endif
  if (have)
    acc.dig += digest_item((uint64_t)(step0 + ((k - 1) & ~31) + lane), 2, d_nb, d_bh) +
               digest_item((uint64_t)(step0 + ((k - 1) & ~31) + lane), 3, 0, end_bits);
  step = step0 + k;
  n_plans += k;
  req_steps += (int64_t)k * (R + W);
  g.lens += __reduce_add_sync(SL_FULL, (live ? (unsigned)sl[0].cur_len : 0u) - cl0);
  return ret;
}

// New arrivals (requests [n0, n0 + kn), their WRec already built) inserted into
// a waiting queue with a walk bound `walk_until`: an insertion grows the
// prefixes of later requests by at most D = (sum of new prefills) (1 + 2^-30)
// + 2^-30 p_up (a fresh fl-sum of n < 2^20 positive terms stays within 2^-30 of
// any other order), which lowers every old bound by at most D (est has slope 1
// in the prefix; the rounding margin m of walk_pass_until is unchanged since
// sigma + U is); each new request gets its own bound with prefix <= p_up + D.
// `blocked` is cleared: the next step runs the admission scan.  (Keeping it
// when every new request provably fails too was measured slower.)
__device__ __forceinline__ void arrivals_keep_bounds(const Sim& s, int64_t n0, int kn, double now,
                                                     bool ttft_guard, bool& blocked,
                                                     double& walk_until, double& p_up, int lane) {
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const bool keep_w = ttft_guard && walk_until > now && kn <= 32;
  const double wu_old = walk_until;
  blocked = false;
  if (ttft_guard) walk_until = -kInf;
  if (!keep_w) return;
  const bool v = lane < kn;
  double pf = 0.0, arr = 0.0, tt = 0.0;
  if (v) {
    const WRec& w = s.wr[n0 + lane];
    pf = w.prefill;
    arr = w.arr;
    tt = w.ttft;
  }
  const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
  double sp = pf;  // sum of the new prefills (any order; inflated below)
  if (kn > 1) {
#pragma unroll
    for (int o = 16; o; o >>= 1) sp = fadd_(sp, __shfl_xor_sync(SL_FULL, sp, o));
  } else {
    sp = __shfl_sync(SL_FULL, pf, 0);  // one arrival (the common case)
  }
  const double D = fadd_(fmul_(sp, inflate), fmul_(p_up, 9.313225746154785e-10));
  const double Dup = fmul_(D, 1.0 + 1.1368683772161603e-13);  // + 2^-43: rounding of D
  const double old_w = fsub_(fsub_(wu_old, Dup), fmul_(wu_old, 9.094947017729282e-13));
  const double Ux = fmul_(fadd_(p_up, Dup), inflate);  // bound on a new request's prefix
  double tx = kInf;
  if (v) {
    const double est0 = fadd_(fadd_(fsub_(now, arr), Ux), pf);
    tx = est0 <= tt ? walk_pass_until(now, Ux, pf, tt, est0) : 0.0;
  }
  walk_until = fmin(old_w, warp_min_nonneg(tx));
  p_up = Ux;
}

// HOT: compile-time specialisation for the sweep's common case -- scorpio with
// both guards, no decision log -- so the hot kernel carries no baseline,
// ablation or logging code (smaller instruction footprint, fewer registers).
template <bool WIDE, bool HOT = false>
__device__ __forceinline__ void run_fast(Sim& s, const KArgs& a, bool has_out, int si, int lane,
                         Slot<WIDE>* scr) {
  const int64_t n = s.n;
  const sl_cost& C = s.cost;
  const bool scorpio = HOT || s.policy == SL_POLICY_SCORPIO;
  const bool ttft_guard = HOT || (s.flags & SL_FLAG_TTFT_GUARD) != 0;
  const bool tpot_guard = HOT || (s.flags & SL_FLAG_TPOT_GUARD) != 0;
  const bool r_only = (s.flags & SL_FLAG_R_ONLY) != 0;
  const bool has_h = (s.flags & SL_FLAG_HAS_HORIZON) != 0;
  const bool sorted_ldf = scorpio && ttft_guard;
  const bool sjf = !HOT && s.policy == SL_POLICY_SJF;
  const bool credit = scorpio && tpot_guard;
  const bool prio = !HOT && !scorpio && (s.flags & SL_FLAG_PREFILL_PRIORITY);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);

  if (has_out) init_outcomes(s, a, lane);
  const bool logging = !HOT && a.has_log && s.log_row >= 0;
  const int64_t lg_step0 = logging ? s.log_row * a.log.step_cap : 0;
  const int64_t lg_id0 = logging ? s.log_row * a.log.id_cap : 0;
  int64_t cur_adm = 0, cur_rej = 0, cur_bat = 0;
  bool log_over = false;

  Acc acc = {0, 0, 0, 0, 0, 0, 0, 0};
#if SL_ACC_SMEM
#pragma unroll
  for (int k = 0; k < 6; ++k) sl_acc_sm[threadIdx.x >> 5][k][lane] = 0;
#endif
  Slot<WIDE> sl[kSlots];
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    sl[k].N = 0;
    sl[k].S = 0;
    sl[k].id = 0;
    sl[k].hid = 0;
    sl[k].idx = 0;
    sl[k].cur_len = 0;
    sl[k].rem = 0;
  }
  Agg<WIDE> g;
  g.Smin = 0;
  g.min_d = 0.0;
  g.lens = 0;
  ps_init(g.pinv);
  g.inv_valid = true;

  double now = 0.0;
  int64_t next = 0;
  double next_t = n > 0 ? s.wr[0].arr : kInf;  // WRec built by wrec_prepass_kernel
#if SL_ARR2
  // the arrival after next, so that the common single arrival needs no load on
  // the step's path (the next one is then already known)
  double next_t2 = n > 1 ? s.wr[1].arr : kInf;
#endif
  int W = 0, R = 0;
  int64_t step = 0, n_plans = 0, n_idle = 0, req_steps = 0;
  int status = SL_SIM_OK;
  bool blocked = false;
  // the walk provably rejects nothing while now < walk_until (until an insertion)
  double walk_until = ttft_guard ? -kInf : kInf;
  double p_up = 0.0;  // upper bound on the prefill sum of the whole waiting queue
  const bool mono = C.alpha >= 0.0 && C.gamma >= 0.0 && C.epsilon >= 0.0;  // est monotone in L
  SL_PROF_DECL

  for (;;) {
    if (next < n && next_t <= now) {
      const int64_t n0 = next;
#if SL_ARR2
      if (next_t2 > now && (sorted_ldf || sjf)) {  // exactly one request arrives
        insert_sorted(s, W, (int)next, sjf, lane);
        ++next;
        next_t = next_t2;
        next_t2 = next + 1 < n ? (s.factor == 1.0 ? s.arrival[next + 1] : s.wr[next + 1].arr)
                               : kInf;
#if SL_PREFETCH
        if (lane == 0 && next < n) asm volatile("prefetch.global.L1 [%0];" ::"l"(s.wr + next));
#endif
      } else {
        process_arrivals<WIDE>(s, W, next, next_t, now, sorted_ldf, sjf, lane);
        next_t2 = next + 1 < n ? (s.factor == 1.0 ? s.arrival[next + 1] : s.wr[next + 1].arr)
                               : kInf;
      }
#else
      process_arrivals<WIDE>(s, W, next, next_t, now, sorted_ldf, sjf, lane);
#endif
      const bool was_blocked = blocked;
      arrivals_keep_bounds(s, n0, (int)(next - n0), now, ttft_guard, blocked, walk_until, p_up,
                           lane);
#if SL_BLOCK_ARR
      // A blocked queue (every waiting request fails against the unchanged
      // running state and is feasible alone) stays blocked when the one new
      // request fails against that state too and is feasible alone: this
      // step's scan would admit and reject nothing.
      if (HOT && was_blocked && mono && next - n0 == 1) {
        const WRec& w = s.wr[n0];
        const double tp = w.tpot, ic = w.inv;
        const int32_t ps_ = w.pred_solo;
        const bool has_min = R > 0;
        const bool lt = !has_min || tp < g.min_d;
        const double minp = lt ? tp : g.min_d;
        const double V = fmul_(minp, fadd_(ps_result(g.pinv), ic));
        const double L = div_small((double)(g.lens + w.prompt), R + 1);
        const double est = tpot_estimate(C, V, L, ps_ & 0x7fffffff);
        const double thr = (r_only && has_min) ? g.min_d : minp;
        blocked = !(est <= thr) && (ps_ & (int32_t)0x80000000) != 0;
      }
#endif
    }
    SL_PROF_MARK(0)
    if (has_h && now >= s.horizon) break;  // simengine.py:190-191
    bool ret;  // entries retire at the end of step `step - 1` (at `now`)
    // quiet / blocked steps: nothing can be admitted or rejected (W == 0, or
    // the admission scan provably fails and the walk provably passes)
    if (!logging && R > 0 && R <= 32 &&
        (credit ? (W == 0 || (blocked && now < walk_until)) : W == 0)) {
      SL_PROF_COUNT(9, 1)
      SL_PROF_COUNT(10, -step)
      ret = quiet_steps<WIDE>(s, a, has_out, sl, R, W, g, now, step, n_plans, req_steps, next_t,
                              W > 0 ? walk_until : kInf, has_h, acc, lane, scr, !credit);
      SL_PROF_COUNT(10, step)
      SL_PROF_MARK(1)
    } else {
    SL_PROF_COUNT(8, 1)
    // general-step kinds: quiet-eligible but for R > 32 (nothing waiting / blocked
    // with the walk bound ahead), and R > 32 at all
    SL_PROF_COUNT(22, R > 32 && W == 0)
    SL_PROF_COUNT(23, R > 32 && W > 0 && blocked && now < walk_until)
    SL_PROF_COUNT(24, R > 32)
    SL_PROF_COUNT(25, W > 0 && !blocked)
#ifdef SL_PHASE_PROF
    prof_acc[12] = prof_acc[12] > (unsigned long long)W ? prof_acc[12] : (unsigned long long)W;
    prof_acc[13] = prof_acc[13] > (unsigned long long)R ? prof_acc[13] : (unsigned long long)R;
#endif

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
        // the walk provably rejects nothing before walk_until (no insertion
        // since it was computed, or insertions accounted for at arrival)
        if (ttft_guard && !(SL_WALK_SKIP && now < walk_until)) {
          SL_PROF_COUNT(16, 1)
          SL_PROF_COUNT(18, W)
          const bool exact = spec_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej,
                                       cap_rej, reinterpret_cast<double*>(scr), walk_until, p_up);
          SL_PROF_COUNT(17, exact)
#ifdef SL_PHASE_PROF
          {
            const long long t_ = clock64();
            prof_acc[exact ? 20 : 21] += (unsigned long long)(t_ - prof_t);
          }
#endif
          (void)exact;
        }
        SL_PROF_MARK(2)
        if (tpot_guard) {
          // `blocked`: every waiting request failed the admission test at a
          // previous step and is feasible alone, and since then only `lens`
          // has grown (no arrival, admission or retirement); the estimate is
          // monotone in L, so the whole scan would admit and reject nothing.
          if (W > 0 && !blocked) {
            if (!g.inv_valid) {
              g.pinv = running_inv_sum<WIDE>(s, sl, R, lane, reinterpret_cast<double*>(scr));
              g.inv_valid = true;
            }
            SL_PROF_MARK(3)
            SL_PROF_COUNT(19, W)
            fits = spec_admit<WIDE>(s, a, has_out, W, R, sl, g, nadm, nrej, P, r_only, step, acc,
                                    lane, lg_adm, cap_adm, lg_rej, cap_rej);
            blocked = mono && nadm == 0;
          }
        } else {
          fits = append_prefix<WIDE>(s, a, W, R, sl, g, W, nadm, P, step, acc, lane, lg_adm,
                                     cap_adm);
        }
      } else {
        if (s.policy == SL_POLICY_EARLY_REJECT && !(SL_WALK_SKIP && now < walk_until))
          spec_walk(s, a, has_out, W, nrej, now, step, acc, lane, lg_rej, cap_rej,
                    reinterpret_cast<double*>(scr), walk_until, p_up);
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
    SL_PROF_MARK(4)

    // ---- decode batch: credit phase (select_batch :161-180) or decode-all
    unsigned bm[kSlots];
    unsigned blen = 0, bhash = 0;
    int nb = 0;
    const bool decode = credit || !(prio && nadm > 0);
#pragma unroll
    for (int k = 0; k < kSlots; ++k) {
      bm[k] = 0u;
      if (k > 0 && R0 <= 32 * k) break;
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
      bhash += __reduce_add_sync(SL_FULL, b ? sl[k].hid : 0u);
      if (b) {
        int pos = nb + __popc(bm[k] & lanemask_lt());
        if (lg_bat >= 0 && pos < cap_bat) a.log.batch_ids[lg_bat + pos] = sl[k].id;
        sl[k].cur_len += 1;  // token emit (simengine.py:243-245), after l_avg's input
        sl[k].rem -= 1;
      }
      nb += __popc(bm[k]);
    }
    g.lens += nb;
    SL_PROF_MARK(5)

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
      decode_s = itl(C, nb, div_small((double)blen, nb));
    }
    const double end = fadd_(fadd_(now, prefill_s), decode_s);
    acc.dig += acc.dig_rej;
    if (lane == 0)
      acc.dig += digest_item((uint64_t)step, 2, (uint32_t)nb, bhash) +
                 digest_item((uint64_t)step, 3, 0, (uint64_t)__double_as_longlong(end));

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
          s.first_emit[sl[k].idx] = end;
        }
      }
      g.lens += nadm;
    }
    bool any_ret = false;
#pragma unroll
    for (int k = 0; k < kSlots; ++k)
      any_ret |= __any_sync(SL_FULL, 32 * k + lane < R && sl[k].rem <= 0);
    SL_PROF_MARK(6)
    SL_PROF_COUNT(11, W > 0 && nadm == 0 && nrej == 0)
    now = end;
    ++step;
    ret = any_ret;
    }  // general step
    if (ret) {  // the one retire() call site
      retire<WIDE>(s, a, has_out, sl, R, g, now, step - 1, acc, lane, scr);
      blocked = false;
    }
    SL_PROF_MARK(7)
  }
  SL_PROF_WRITE(si)

#if SL_ACC_SMEM
  acc.completed = sl_acc_sm[threadIdx.x >> 5][kAccCompleted][lane];
  acc.compliant = sl_acc_sm[threadIdx.x >> 5][kAccCompliant][lane];
  acc.rej_ttft = sl_acc_sm[threadIdx.x >> 5][kAccRejTtft][lane];
  acc.rej_adm = sl_acc_sm[threadIdx.x >> 5][kAccRejAdm][lane];
  acc.ttft_viol = sl_acc_sm[threadIdx.x >> 5][kAccTtftViol][lane];
  acc.tpot_viol = sl_acc_sm[threadIdx.x >> 5][kAccTpotViol][lane];
#endif
  write_result(a, si, acc, status | (log_over ? SL_SIM_LOG_OVERFLOW : 0), n, step, n_plans,
               n_idle, req_steps, now, has_h, s.horizon, lane);
}

}  // namespace sl
