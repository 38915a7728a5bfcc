// Shared device-side state layout of the simulation kernels (general and fast).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "scorpio_b200.h"
#include "sl_device.cuh"

#ifndef SL_PREFETCH
#define SL_PREFETCH 1  // prefetch the next arriving request's WRec into L1 (measured -1%;
                        // 2: also its id / output length, measured +3%)
#endif

namespace sl {


struct __align__(16) WRec {  // per request, written at arrival (WaitingItem + Request fields)
  double arr;       // arrival_time / rate_factor
  double ttft;      // ttft_slo * slo_scale
  double prefill;   // prefill_time(prompt_len), costmodel.py:132-138
  double tpot;      // tpot_slo * slo_scale
  double inv;       // 1.0 / tpot
  double deadline;  // arr + ttft, core.py:50-53
  uint64_t S;       // fixed-point tpot (low 64 bits)
  int32_t prompt;
  int32_t pred_solo;  // predicted_len | solo_ok << 31
};
static_assert(sizeof(WRec) == 64, "WRec layout");

struct __align__(16) RRec {  // per running entry, positional (RunningEntry)
  uint64_t N;   // credit * slo / 2^E (low 64 bits)
  uint64_t S;   // slo / 2^E (low 64 bits)
  double inv;   // 1.0 / tpot
  int32_t cur_len;  // prompt_len + tokens_generated
  int32_t rem;      // true_output_len - tokens_generated
};
static_assert(sizeof(RRec) == 32, "RRec layout");

struct Workspace {  // SoA regions over all request slots
  int* counter;
  int32_t* wl;       // waiting list (request index), per sim [n]
  int32_t* rl;       // running list (request index), per sim [n]
  WRec* wr;          // per request
  RRec* rr;          // per running position
  uint64_t* wShi;    // wide credits: S high word per request
  uint64_t* rNhi;    // wide credits: per running position
  uint64_t* rShi;
  double* first_emit;  // per request
  uint32_t* rh;        // batch_hid(id) per running position (general kernel)
};

__host__ __device__ inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

__host__ __device__ inline Workspace carve(void* base, int64_t slots) {
  Workspace w;
  char* p = (char*)base;
  int64_t off = 0;
  w.counter = (int*)(p + off);
  off += 256;
  w.wl = (int32_t*)(p + off);
  off = align256(off + slots * 4);
  w.rl = (int32_t*)(p + off);
  off = align256(off + slots * 4);
  w.wr = (WRec*)(p + off);
  off = align256(off + slots * 64);
  w.rr = (RRec*)(p + off);
  off = align256(off + slots * 32);
  w.wShi = (uint64_t*)(p + off);
  off = align256(off + slots * 8);
  w.rNhi = (uint64_t*)(p + off);
  off = align256(off + slots * 8);
  w.rShi = (uint64_t*)(p + off);
  off = align256(off + slots * 8);
  w.first_emit = (double*)(p + off);
  off = align256(off + slots * 8);
  w.rh = (uint32_t*)(p + off);
  return w;
}

__host__ __device__ inline int64_t workspace_bytes(int64_t slots) {
  return 256 + 8 * 256 + align256(slots * 4) * 3 + align256(slots * 64) + align256(slots * 32) +
         align256(slots * 8) * 4;
}

struct KArgs {
  sl_traces tr;
  const sl_sim* sims;
  const int32_t* order;
  int32_t n_sims;
  int64_t slots;
  void* ws_base;
  sl_result* results;
  sl_outcomes out;
  int has_out;
  sl_log log;
  int has_log;
};

// Pointer known to address global memory.  The hot kernel keeps its per-sim
// view in shared memory, so nvcc cannot infer the address space of pointers it
// reloads from there and would emit generic LD/ST; the assumption restores
// LDG/STG on every access.
template <class T>
struct gptr {
  T* p;
  __device__ __forceinline__ T* get() const {
    T* q = p;
    __builtin_assume(__isGlobal(q));
    return q;
  }
  __device__ __forceinline__ gptr& operator=(T* q) {
    p = q;
    return *this;
  }
  __device__ __forceinline__ gptr& operator+=(int64_t k) {
    p += k;
    return *this;
  }
  __device__ __forceinline__ T& operator[](int64_t i) const { return get()[i]; }
  __device__ __forceinline__ T* operator+(int64_t i) const { return get() + i; }
  __device__ __forceinline__ operator T*() const { return get(); }
};

// Per-sim view, warp-uniform.
struct Sim {
  // trace
  gptr<const double> arrival;
  gptr<const double> ttft_b;
  gptr<const double> tpot_b;
  gptr<const int32_t> prompt;
  gptr<const int32_t> true_out;
  gptr<const int32_t> predicted;
  gptr<const int64_t> id;
  int64_t n;
  // params
  sl_cost cost;
  double scale, factor, horizon, pow2E;
  int policy, flags, cap, E;
  // workspace slices
  gptr<int32_t> wl;
  gptr<int32_t> rl;
  gptr<uint32_t> rh;
  gptr<WRec> wr;
  gptr<RRec> rr;
  gptr<uint64_t> wShi;
  gptr<uint64_t> rNhi;
  gptr<uint64_t> rShi;
  gptr<double> first_emit;
  // outputs
  int64_t out_off;
  int64_t log_row;
};

__device__ __forceinline__ bool key_less_ldf(const Sim& s, double da, double aa, int ia, double db,
                                             double ab, int ib) {
  // sort_key = (deadline, arrival_time, id), schedtypes.py:28-32
  if (da != db) return da < db;
  if (aa != ab) return aa < ab;
  return s.id[ia] < s.id[ib];
}

__device__ __forceinline__ bool key_less_sjf(const Sim& s, int32_t pa, double aa, int ia,
                                             int32_t pb, double ab, int ib) {
  // sched_baselines.py:138-142 key (predicted_len, arrival_time, id)
  if (pa != pb) return pa < pb;
  if (aa != ab) return aa < ab;
  return s.id[ia] < s.id[ib];
}

// Insert request `idx` into the sorted waiting list at its rank (keys are
// unique, so rank == bisect position).  Warp-cooperative: O(W/32) compares
// and a top-down chunked shift.
__device__ __forceinline__ void insert_sorted(const Sim& s, int& W, int idx, bool sjf, int lane) {
  const WRec& me = s.wr[idx];
  double dk = me.deadline, ak = me.arr;
  int32_t pk = me.pred_solo & 0x7fffffff;
  int pos = 0;
  if (sjf && W > 64) {
    // SJF arrivals land anywhere: 32-ary search (32 probes per round) over the
    // sorted list, then one chunk.  Invariant: keys below lo are smaller,
    // keys from hi on larger than the new one.
    auto less_new = [&](int j) {
      const int o = s.wl[j];
      const int32_t pr = s.wr[o].pred_solo & 0x7fffffff;
      return pr != pk ? pr < pk : key_less_sjf(s, pr, s.wr[o].arr, o, pk, ak, idx);
    };
    int lo = 0, hi = W;
    while (hi - lo > 32) {
      const int stride = (hi - lo + 31) / 32;
      const int q = lo + lane * stride;
      const int cnt = __popc(__ballot_sync(SL_FULL, q < hi && less_new(q)));
      const int nhi = lo + cnt * stride;
      lo = cnt ? lo + (cnt - 1) * stride + 1 : lo;
      hi = nhi < hi ? nhi : hi;
    }
    pos = lo + __popc(__ballot_sync(SL_FULL, lo + lane < hi && less_new(lo + lane)));
  } else {
  // keys below the new one form a prefix of the list: scan chunks from the end
  // and stop at the first chunk holding one (new arrivals mostly land late)
  for (int c0 = (W - 1) & ~31; c0 >= 0; c0 -= 32) {
    int j = c0 + lane;
    bool lt = false;
    if (j < W) {  // primary key first; arrival / id read only on a tie
      const int o = s.wl[j];
      const WRec& r = s.wr[o];
      if (sjf) {
        const int32_t pr = r.pred_solo & 0x7fffffff;
        lt = pr != pk ? pr < pk : key_less_sjf(s, pr, r.arr, o, pk, ak, idx);
      } else {
        const double dr = r.deadline;
        lt = dr != dk ? dr < dk : key_less_ldf(s, dr, r.arr, o, dk, ak, idx);
      }
    }
    const unsigned m = __ballot_sync(SL_FULL, lt);
    if (m) {
      pos = c0 + __popc(m);
      break;
    }
  }
  }
  // shift [pos, W) up by one, highest chunk first
  int tail = W - pos;
  for (int c = (tail - 1) / 32; c >= 0 && tail > 0; --c) {
    int j = pos + c * 32 + lane;
    int v = 0;
    bool ok = j < W;
    if (ok) v = s.wl[j];
    __syncwarp();
    if (ok) s.wl[j + 1] = v;
    __syncwarp();
  }
  if (lane == 0) s.wl[pos] = idx;
  __syncwarp();
  W += 1;
}


// Make the warp-uniform per-sim view of cell `si` (traces, params, workspace slices).
__device__ __forceinline__ Sim make_sim(const KArgs& a, const Workspace& ws, int si) {
  const sl_sim& sp = a.sims[si];
  Sim s;
  int t = sp.trace;
  int64_t b = a.tr.begin[t];
  s.n = a.tr.begin[t + 1] - b;
  s.arrival = a.tr.arrival + b;
  s.ttft_b = a.tr.ttft_slo + b;
  s.tpot_b = a.tr.tpot_slo + b;
  s.prompt = a.tr.prompt_len + b;
  s.true_out = a.tr.true_out + b;
  s.predicted = a.tr.predicted + b;
  s.id = a.tr.id + b;
  s.cost = sp.cost;
  s.scale = sp.slo_scale;
  s.factor = sp.rate_factor;
  s.horizon = sp.horizon;
  s.policy = sp.policy;
  s.flags = sp.flags;
  s.cap = sp.max_batch_size;
  s.E = sp.credit_exp;
  s.pow2E = __longlong_as_double((long long)(sp.credit_exp + 1023) << 52);
  int64_t o = sp.ws_offset;
  s.wl = ws.wl + o;
  s.rl = ws.rl + o;
  s.rh = ws.rh + o;
  s.wr = ws.wr + o;
  s.rr = ws.rr + o;
  s.wShi = ws.wShi + o;
  s.rNhi = ws.rNhi + o;
  s.rShi = ws.rShi + o;
  s.first_emit = ws.first_emit + o;
  s.out_off = sp.out_offset;
  s.log_row = sp.log_slot;
  return s;
}

__device__ __forceinline__ void init_outcomes(const Sim& s, const KArgs& a, int lane) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t i = lane; i < s.n; i += 32) {
    int64_t o = s.out_off + i;
    a.out.status[o] = SL_INCOMPLETE;
    a.out.compliant[o] = 0;
    a.out.completion_step[o] = -1;
    a.out.first_token_time[o] = qnan;
    a.out.completion_time[o] = qnan;
    a.out.ttft[o] = qnan;
    a.out.tpot[o] = qnan;
  }
}

// The WaitingItem fields of request i of a sim (arrival / rate factor, scaled
// SLOs, prefill_time, 1/slo, deadline, fixed-point slo, solo feasibility): one
// IEEE op each, exactly as the reference builds them (core.py:50-53,
// costmodel.py:132-138, sched_scorpio.py:279-289).
template <bool WIDE>
__device__ __forceinline__ WRec make_wrec(const Sim& s, int64_t i, uint64_t* S_hi) {
  const sl_cost& C = s.cost;
  WRec w;
  w.arr = s.factor == 1.0 ? s.arrival[i] : fdiv_(s.arrival[i], s.factor);
  w.ttft = fmul_(s.ttft_b[i], s.scale);
  w.tpot = fmul_(s.tpot_b[i], s.scale);
  w.prompt = s.prompt[i];
  const int32_t pred = s.predicted[i];
  w.prefill = prefill_time(C, w.prompt);
  w.inv = frcp_(w.tpot);
  w.deadline = fadd_(w.arr, w.ttft);
  const cred_t<WIDE> S = slo_fixed<WIDE>(w.tpot, s.E);
  w.S = (uint64_t)S;
  if constexpr (WIDE) *S_hi = (uint64_t)(S >> 64);
  const bool solo = solo_ok(C, w.tpot, w.inv, w.prompt, pred);
  w.pred_solo = pred | (solo ? (int32_t)0x80000000 : 0);
  return w;
}

// Requests with arrival <= now become visible (simengine.py:186-188) and join
// the waiting list in queue order (LDF / SJF insertion or FCFS append).  Their
// WRec were built in advance by wrec_prepass_kernel (a bandwidth-bound pass
// over all requests of all sims), so only the queue update stays on the
// simulation's serial path.
template <bool WIDE>
__device__ __forceinline__ void process_arrivals(const Sim& s, int& W, int64_t& next, double& next_t, double now,
                                 bool sorted_ldf, bool sjf, int lane) {
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  while (next < s.n && next_t <= now) {
    const int64_t i = next + lane;
    // arrival / rate factor: the trace value itself when the factor is 1 (x / 1.0 == x)
    const bool c = i < s.n && (s.factor == 1.0 ? s.arrival[i] : s.wr[i].arr) <= now;
    const int k = __popc(__ballot_sync(SL_FULL, c));  // arrivals are sorted: a lane prefix
    if (sorted_ldf || sjf) {
      for (int t = 0; t < k; ++t) insert_sorted(s, W, (int)(next + t), sjf, lane);
    } else {
      if (c) s.wl[W + lane] = (int32_t)i;
      __syncwarp();
      W += k;
    }
    next += k;
    next_t = next < s.n ? (s.factor == 1.0 ? s.arrival[next] : s.wr[next].arr) : kInf;
  }
#if SL_PREFETCH
  // the next request's WRec (first touched at its arrival): start the L1 fill now
  if (lane == 0 && next < s.n) asm volatile("prefetch.global.L1 [%0];" ::"l"(s.wr + next));
#if SL_PREFETCH >= 2
  // and its id / output length (read when it is admitted)
  if (lane == 1 && next < s.n) asm volatile("prefetch.global.L1 [%0];" ::"l"(s.id + next));
  if (lane == 2 && next < s.n) asm volatile("prefetch.global.L1 [%0];" ::"l"(s.true_out + next));
#endif
#endif
}

// Per-lane accumulators folded into the result row at the end.
struct Acc {
  uint64_t dig;      // committed digest partial
  uint64_t dig_rej;  // pending: rejections of the current plan (committed iff it has work)
  int32_t completed, compliant, rej_ttft, rej_adm, ttft_viol, tpot_viol;  // per-lane partials
};

__device__ __forceinline__ void write_result(const KArgs& a, int si, const Acc& acc, int status,
                                             int64_t n, int64_t step, int64_t n_plans,
                                             int64_t n_idle, int64_t req_steps, double now,
                                             bool has_h, double horizon, int lane) {
  uint64_t dig = warp_sum_u64(acc.dig);
  // per-lane partial counts are < 2^31 and their sums <= n < 2^32
  int64_t completed = __reduce_add_sync(SL_FULL, (unsigned)acc.completed);
  int64_t compliant = __reduce_add_sync(SL_FULL, (unsigned)acc.compliant);
  int64_t rj_t = __reduce_add_sync(SL_FULL, (unsigned)acc.rej_ttft);
  int64_t rj_a = __reduce_add_sync(SL_FULL, (unsigned)acc.rej_adm);
  int64_t tv = __reduce_add_sync(SL_FULL, (unsigned)acc.ttft_viol);
  int64_t pv = __reduce_add_sync(SL_FULL, (unsigned)acc.tpot_viol);
  if (lane == 0) {
    sl_result res;
    res.status = status;
    res._pad = 0;
    res.n_steps = step;
    res.n_plans = n_plans;
    res.n_idle_skips = n_idle;
    res.request_steps = req_steps;
    res.total = n;
    res.completed = completed;
    res.compliant = compliant;
    res.rejected_ttft = rj_t;
    res.rejected_admission = rj_a;
    res.incomplete = n - completed - rj_t - rj_a;
    res.ttft_violations = tv;
    res.tpot_violations = pv;
    res.sim_end = now;
    double h = has_h ? horizon : (now > 1e-12 ? now : 1e-12);  // report.py:130-134
    res.horizon = h;
    res.goodput = fdiv_((double)compliant, h);                   // core.py:168-172
    res.adherence = n > 0 ? fdiv_((double)compliant, (double)n) : 0.0;
    res.digest = dig;
    a.results[si] = res;
  }
}

}  // namespace sl
