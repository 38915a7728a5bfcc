// Batched plan_step over independent SchedulerStates (config 2 and the drop-in
// sched_scorpio API): three separately launchable kernels.
//
//  sort   -- LDF order of each segment's waiting queue by (deadline, arrival,
//            id) (sched_scorpio.py:193): warp bitonic network in registers for
//            segments <= 32 items, CTA bitonic over shared memory for tiles of
//            <= 2048, then merge-path passes between tiles for larger segments.
//  guard  -- one warp per segment: speculative-parallel TTFT prefix walk,
//            running aggregates (Neumaier 1/slo in running order), speculative
//            greedy admission scan, then min_slo and vbs over running+admitted
//            (sched_scorpio.py:196-294, 312-315).
//  select -- one warp per segment: fixed-point credit earn/debit with ballot
//            batch compaction (sched_scorpio.py:161-180), or decode-all.
// All fp64 on the decision path uses the unfused *_rn intrinsics (sl_device.cuh).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "scorpio_b200.h"
#include "sl_device.cuh"

using namespace sl;

#ifndef SL_SORT32
#define SL_SORT32 1  // warp LDF networks on 32-bit range-relative keys (near-ties: full keys)
#endif

namespace {

constexpr int kTile = 2048;  // CTA sort tile
constexpr int kSortThreads = 256;
constexpr int kMergeItems = 4;  // outputs per thread in a merge pass

struct Key {
  double d, a;
  int64_t id;
  int32_t idx;
};

__device__ __forceinline__ bool key_lt(const Key& x, const Key& y) {
  if (x.d != y.d) return x.d < y.d;
  if (x.a != y.a) return x.a < y.a;
  return x.id < y.id;
}

__device__ __forceinline__ Key load_key(const sl_plan_state& st, int32_t i) {
  Key k;
  k.a = st.w_arrival[i];
  k.d = fadd_(k.a, st.w_ttft[i]);  // Request.deadline, core.py:50-53
  k.id = st.w_id[i];
  k.idx = i;
  return k;
}

__device__ __forceinline__ Key inf_key() {
  Key k;
  k.d = __longlong_as_double(0x7ff0000000000000LL);
  k.a = k.d;
  k.id = INT64_MAX;
  k.idx = -1;
  return k;
}

// LDF order of <= 32 items held one per lane (deadline d >= 0, valid lanes <
// n) by a bitonic network over 32-bit keys: the deadline's bit pattern minus the
// warp minimum (monotone for non-negative doubles), shifted right so that the
// range fits 27 bits, with the lane (input position) in the low 5 bits.
// Returns the input lane at this lane's sorted position, or -1 when two
// adjacent sorted keys share their top 27 bits (equal or near-equal deadlines:
// the caller falls back to a full-key network).
__device__ __forceinline__ int warp_ldf_src32(double d, bool valid, int n, int lane) {
  const uint64_t b = valid ? (uint64_t)__double_as_longlong(d) : 0ull;
  const unsigned hmin = __reduce_min_sync(SL_FULL, valid ? (unsigned)(b >> 32) : ~0u);
  const unsigned lmin = __reduce_min_sync(SL_FULL, valid && (unsigned)(b >> 32) == hmin
                                                       ? (unsigned)b : ~0u);
  const uint64_t bmin = ((uint64_t)hmin << 32) | lmin;
  const uint64_t off = valid ? b - bmin : 0ull;
  const unsigned ohi = __reduce_max_sync(SL_FULL, (unsigned)(off >> 32));
  const unsigned olo = __reduce_max_sync(SL_FULL, (unsigned)(off >> 32) == ohi ? (unsigned)off : 0u);
  const uint64_t omax = ((uint64_t)ohi << 32) | olo;
  const int bits = omax ? 64 - __clzll((long long)omax) : 0;  // significant bits of the range
  const int sh = bits > 27 ? bits - 27 : 0;
  unsigned key = valid ? ((unsigned)(off >> sh) << 5) | (unsigned)lane : ~0u;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      const unsigned ok = __shfl_xor_sync(SL_FULL, key, j);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & j) == 0;
      key = ((lower == up) == (ok < key)) ? ok : key;
    }
  }
  const unsigned next = __shfl_down_sync(SL_FULL, key, 1);
  if (__any_sync(SL_FULL, lane + 1 < n && (next >> 5) == (key >> 5))) return -1;
  return (int)(key & 31);
}

// ---- sort: one warp per segment (<= 32 items), bitonic network over shuffles
// (d_pre: this lane's deadline when the caller has loaded it already -- the
// grid-stride kernel pipelines the next segment's loads -- else loaded here)
__device__ __forceinline__ void seg_sort_warp(const sl_plan_state& st, int32_t* perm, int seg,
                                              int lane, const double* d_pre = nullptr) {
  const int64_t b = st.w_begin[seg];
  const int n = (int)(st.w_begin[seg + 1] - b);
  // Fast path: non-negative deadlines order like their bit patterns.  The
  // network sorts one 32-bit key per lane (warp_ldf_src32: range-relative
  // deadline bits, lane in the low 5 bits; SL_SORT32=0: the 64-bit form, the
  // deadline bits with the low 5 bits replaced by the lane).  Distinct keys
  // above the lane bits make that the LDF order; otherwise (ties or near-ties,
  // rare) the full (deadline, arrival, id) network below decides.
  double d = 0.0;
  if (d_pre)
    d = *d_pre;
  else if (lane < n)
    d = fadd_(st.w_arrival[b + lane], st.w_ttft[b + lane]);  // core.py:50-53
  if (SL_SORT32 && __all_sync(SL_FULL, lane >= n || d >= 0.0)) {
    const int src = warp_ldf_src32(d, lane < n, n, lane);
    if (src >= 0) {
      if (lane < n) perm[b + lane] = (int32_t)(b + src);
      return;
    }
  }
  if (!SL_SORT32 && __all_sync(SL_FULL, lane >= n || d >= 0.0)) {
    uint64_t key = lane < n ? (((uint64_t)__double_as_longlong(d) & ~31ull) | (uint64_t)lane)
                            : ~0ull;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int j = size >> 1; j > 0; j >>= 1) {
        const uint64_t ok = __shfl_xor_sync(SL_FULL, key, j);
        const bool up = (lane & size) == 0;
        const bool lower = (lane & j) == 0;
        key = ((lower == up) == (ok < key)) ? ok : key;
      }
    }
    const uint64_t next = __shfl_down_sync(SL_FULL, key, 1);
    if (!__any_sync(SL_FULL, lane + 1 < n && (next >> 5) == (key >> 5))) {
      if (lane < n) perm[b + lane] = (int32_t)(b + (int)(key & 31));
      return;
    }
  }
  Key k = lane < n ? load_key(st, (int32_t)(b + lane)) : inf_key();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      Key o;
      o.d = __shfl_xor_sync(SL_FULL, k.d, j);
      o.a = __shfl_xor_sync(SL_FULL, k.a, j);
      o.id = __shfl_xor_sync(SL_FULL, k.id, j);
      o.idx = __shfl_xor_sync(SL_FULL, k.idx, j);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & j) == 0;
      const bool take = (lower == up) ? key_lt(o, k) : key_lt(k, o);
      if (take) k = o;
    }
  }
  if (lane < n) perm[b + lane] = k.idx;
}

// grid-stride over segments: a bounded grid (resident warps) instead of one
// 4-warp block per 4 segments, so block launches do not pace large batches
__global__ void sort_warp_kernel(const sl_plan_state st, int32_t* perm) {
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // the next segment's deadline inputs are in flight while this one is sorted
  auto fetch = [&](int sg, double& a, double& t) {
    a = t = 0.0;
    if (sg < st.n_segments) {
      const int64_t b = st.w_begin[sg];
      if (lane < st.w_begin[sg + 1] - b) {
        a = st.w_arrival[b + lane];
        t = st.w_ttft[b + lane];
      }
    }
  };
  double a_n, t_n;
  fetch(seg, a_n, t_n);
  for (; seg < st.n_segments; seg += nw) {
    const double d = fadd_(a_n, t_n);  // core.py:50-53 (unused past the segment's end)
    fetch(seg + nw, a_n, t_n);
    seg_sort_warp(st, perm, seg, lane, &d);
  }
}

// ---- sort: one CTA per (segment, tile of <= kTile items), bitonic over smem
__global__ void __launch_bounds__(kSortThreads) sort_tile_kernel(const sl_plan_state st,
                                                                 int tiles_per_seg, int32_t* out) {
  extern __shared__ unsigned char smem_raw[];
  double* sd = reinterpret_cast<double*>(smem_raw);
  double* sa = sd + kTile;
  int64_t* sid = reinterpret_cast<int64_t*>(sa + kTile);
  int32_t* sidx = reinterpret_cast<int32_t*>(sid + kTile);
  const int seg = blockIdx.x / tiles_per_seg;
  const int tile = blockIdx.x % tiles_per_seg;
  const int64_t sb = st.w_begin[seg], se = st.w_begin[seg + 1];
  const int64_t b = sb + (int64_t)tile * kTile;
  if (b >= se) return;
  const int n = (int)min((int64_t)kTile, se - b);
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    Key k = i < n ? load_key(st, (int32_t)(b + i)) : inf_key();
    sd[i] = k.d;
    sa[i] = k.a;
    sid[i] = k.id;
    sidx[i] = k.idx;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * j * (t / j) + (t % j);
        const int hi = lo + j;
        const bool up = (lo & size) == 0;
        Key x{sd[lo], sa[lo], sid[lo], sidx[lo]};
        Key y{sd[hi], sa[hi], sid[hi], sidx[hi]};
        const bool swap = up ? key_lt(y, x) : key_lt(x, y);
        if (swap) {
          sd[lo] = y.d; sa[lo] = y.a; sid[lo] = y.id; sidx[lo] = y.idx;
          sd[hi] = x.d; sa[hi] = x.a; sid[hi] = x.id; sidx[hi] = x.idx;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[b + i] = sidx[i];
}

// ---- sort: merge-path pass over runs of width w inside each segment
__global__ void merge_pass_kernel(const sl_plan_state st, int64_t w, int blocks_per_seg,
                                  const int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  const int seg = blockIdx.x / blocks_per_seg;
  const int64_t sb = st.w_begin[seg], se = st.w_begin[seg + 1];
  const int64_t p0 = ((int64_t)(blockIdx.x % blocks_per_seg) * blockDim.x + threadIdx.x) *
                     kMergeItems;  // output offset inside the segment
  const int64_t n = se - sb;
  if (p0 >= n) return;
  const int64_t pair = p0 / (2 * w);
  const int64_t base = sb + pair * 2 * w;
  const int64_t la = min(w, se - base);
  const int64_t lb = max((int64_t)0, min(w, se - base - w));
  const int32_t* A = src + base;
  const int32_t* B = src + base + w;
  const int64_t q = p0 - pair * 2 * w;  // diagonal inside the pair
  // merge path: first i with A[i] > B[q-i-1] (A wins ties; keys are unique)
  int64_t lo = max((int64_t)0, q - lb), hi = min(q, la);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key_lt(load_key(st, B[q - mid - 1]), load_key(st, A[mid])))
      hi = mid;
    else
      lo = mid + 1;
  }
  int64_t i = lo, j = q - lo;
  for (int t = 0; t < kMergeItems && q + t < la + lb; ++t) {
    bool takeA;
    if (i >= la)
      takeA = false;
    else if (j >= lb)
      takeA = true;
    else
      takeA = !key_lt(load_key(st, B[j]), load_key(st, A[i]));
    dst[base + q + t] = takeA ? A[i++] : B[j++];
  }
}

__global__ void copy_kernel(const sl_plan_state st, const int32_t* __restrict__ src,
                            int32_t* __restrict__ dst) {
  const int64_t n = st.w_begin[st.n_segments] - st.w_begin[0];
  src += st.w_begin[0];
  dst += st.w_begin[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// A segment's waiting-item fields staged in shared memory by cp.async while the
// warp works on the previous segment (guard_admit_group_kernel, <= 32 waiting).
struct GStage {
  double arr[32], pf[32], tt[32], tp[32];
  int32_t idx[32], ln[32], pd[32], klane[32];
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// ---- guard + admission: one warp per segment
// GROUP: the Neumaier folds are done lane-per-segment by the caller
// (guard_admit_group_kernel): `inv_pre` is this segment's sum(1/slo) fold, and
// the caller folds vbs from the returned min_d / has_min / nadm.
template <bool GROUP = false>
__device__ __forceinline__ void seg_guard_admit(const sl_plan_state& st, const sl_plan_config& cfg,
                                                const sl_plan_out& out, int seg, int lane,
                                                double inv_pre = 0.0, double* min_out = nullptr,
                                                bool* has_min_out = nullptr,
                                                int* nadm_out = nullptr,
                                                int32_t* klist32 = nullptr,
                                                long long lens_pre = 0, double min_pre = 0.0,
                                                GStage* stg = nullptr) {
  const sl_cost& C = cfg.cost;
  const bool ttft_guard = cfg.flags & SL_FLAG_TTFT_GUARD;
  const bool tpot_guard = cfg.flags & SL_FLAG_TPOT_GUARD;
  const bool r_only = cfg.flags & SL_FLAG_R_ONLY;
  const bool guard_only = cfg.flags & SL_PLAN_GUARD_ONLY;
  const bool walk = ttft_guard || (cfg.flags & SL_PLAN_FCFS_WALK);
  // negative prefills: no certified pass, no outright rejection (both assume
  // the prefix only grows); the speculative chain + serial pass stays exact
  const bool exact = cfg.flags & SL_PLAN_EXACT_WALK;
  const int64_t wb = st.w_begin[seg], rb = st.r_begin[seg];
  const int W = (int)(st.w_begin[seg + 1] - wb);
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const double now = st.now[seg];
  const int E = st.credit_exp[seg];
  const double pow2E = __longlong_as_double((long long)(E + 1023) << 52);
  // the walk's kept list: the warp's 32-entry shared buffer for segments of <= 32
  // waiting (no global round trip), else the segment's slice of out.scratch
  int32_t* kept_list = (klist32 && W <= 32) ? klist32 : out.scratch + wb;
  int nrej = 0, kept = 0;
  // fields staged in shared memory by the caller (one chunk: lane == position)
  const bool staged = stg != nullptr && W <= 32;

  // 1. TTFT walk over the LDF order (speculative-parallel, exact), or the FCFS queue.
  // Certified pass first (as spec_walk in sim_fast.cuh): an inflated any-order
  // prefix bound U_j >= the sequential prefix and monotone IEEE addition give
  // est_j <= fl(fl(e_j + U_j) + pf_j); if that passes for every item nothing is
  // rejected and the exact chain is not needed.
  bool certified = !walk;
  if (walk && !exact && W < (1 << 20)) {
    const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
    double U = 0.0;
    bool all_ok = true;
    for (int c0 = 0; c0 < W && all_ok; c0 += 32) {
      const int p = c0 + lane;
      const bool valid = p < W;
      double e = 0.0, pf = 0.0, tt = 0.0;
      if (valid && staged) {
        e = fsub_(now, stg->arr[lane]);
        pf = stg->pf[lane];
        tt = stg->tt[lane];
      } else if (valid) {
        const int32_t idx = ttft_guard ? out.perm[wb + p] : (int32_t)(wb + p);
        e = fsub_(now, st.w_arrival[idx]);
        pf = st.w_prefill[idx];
        tt = st.w_ttft[idx];
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
    certified = all_ok;
  }
  {
    double prefix = 0.0;
    // software pipelined over chunks (large segments are DRAM-latency bound):
    // queue slots of chunk c+2 and the fields of chunk c+1 are requested before
    // chunk c is walked
    auto slot = [&](int c0) -> int32_t {
      const int p = c0 + lane;
      return p < W ? (ttft_guard ? out.perm[wb + p] : (int32_t)(wb + p)) : -1;
    };
    int32_t idx_n = staged ? (lane < W ? stg->idx[lane] : -1) : slot(0);
    int32_t idx_nn = staged ? -1 : slot(32);
    double ar_n = 0.0, pf_n = 0.0, tt_n = 0.0;
    if (staged) {
      if (idx_n >= 0) {
        ar_n = stg->arr[lane];
        pf_n = stg->pf[lane];
        tt_n = stg->tt[lane];
      }
    } else if (idx_n >= 0) {
      ar_n = st.w_arrival[idx_n];
      pf_n = st.w_prefill[idx_n];
      tt_n = st.w_ttft[idx_n];
    }
    for (int c0 = 0; c0 < W; c0 += 32) {
      const int p = c0 + lane;
      const bool valid = p < W;
      const int cnt = min(32, W - c0);
      const int32_t idx = valid ? idx_n : 0;
      const double e = fsub_(now, ar_n), pf = pf_n, tt = tt_n;
      idx_n = idx_nn;
      idx_nn = slot(c0 + 64);
      if (idx_n >= 0) {
        ar_n = st.w_arrival[idx_n];
        pf_n = st.w_prefill[idx_n];
        tt_n = st.w_ttft[idx_n];
      }
      unsigned rejm = 0;
      if (!certified) {
        // items failing at the chunk's incoming prefix fail at any later one
        // (prefixes only grow, est is monotone in them): rejected outright,
        // and the speculative chain runs over the remaining items only
        rejm = exact ? 0u : __ballot_sync(SL_FULL, valid && fadd_(fadd_(e, prefix), pf) > tt);
        const unsigned live = (cnt == 32 ? ~0u : (1u << cnt) - 1u) & ~rejm;
        if (live) {
          // speculative chain over the undecided items (assumed kept), tested
          // lane-parallel; from the first rejection on, one serial pass with the
          // test inline (as spec_walk in sim_fast.cuh)
          const double pfk = ((live >> lane) & 1u) ? pf : 0.0;  // x + 0.0 == x
          double run = prefix, mine = 0.0;
          for (int t = __ffs(live) - 1; t < cnt; ++t) {
            const double x = bcast(pfk, t);
            if (lane == t) mine = run;
            run = fadd_(run, x);
          }
          const unsigned m = __ballot_sync(SL_FULL, ((live >> lane) & 1u) &&
                                                        fadd_(fadd_(e, mine), pf) > tt);
          if (m) {
            const int r = __ffs(m) - 1;
            rejm |= 1u << r;
            double q = bcast(mine, r);  // a rejected item leaves the prefix unchanged
            for (int t = r + 1; t < cnt; ++t) {
              if ((rejm >> t) & 1u) continue;
              const double x = bcast(pf, t), et = bcast(e, t), tt_t = bcast(tt, t);
              if (fadd_(fadd_(et, q), x) > tt_t)
                rejm |= 1u << t;
              else
                q = fadd_(q, x);
            }
            run = q;
          }
          prefix = run;
        }
      }
      const bool rj = valid && ((rejm >> lane) & 1u);
      const bool keep = valid && !rj;
      const unsigned km = __ballot_sync(SL_FULL, keep);
      if (keep) {
        const int q = kept + __popc(km & lanemask_lt());
        kept_list[q] = idx;
        if (staged) stg->klane[q] = lane;
      }
      if (rj) {
        out.w_status[idx] = SL_PLAN_REJECTED_TTFT;
        out.w_pos[idx] = nrej + __popc(rejm & lanemask_lt());
      }
      kept += __popc(km);
      nrej += __popc(rejm);
    }
    __syncwarp();
  }
  if (guard_only) {
    for (int p = lane; p < kept; p += 32) {
      out.w_status[kept_list[p]] = SL_PLAN_WAITING;
      out.w_pos[kept_list[p]] = p;
    }
    if (lane == 0) {
      out.seg_counts[4 * seg + 0] = kept;
      out.seg_counts[4 * seg + 1] = 0;
      out.seg_counts[4 * seg + 2] = nrej;
    }
    return;
  }

  // 2. running aggregates (sched_scorpio.py:117-124); GROUP: reduced lane-per-
  // segment by the caller with its sum(1/slo) fold
  int64_t lens = lens_pre;
  double min_d = min_pre;
  if (!GROUP) {
    lens = 0;
    min_d = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll 4
    for (int j = lane; j < R; j += 32) {
      lens += st.r_cur_len[rb + j];
      min_d = fmin(min_d, st.r_tpot[rb + j]);
    }
    lens = warp_sum_i64(lens);
#pragma unroll
    for (int o = 16; o; o >>= 1) min_d = fmin(min_d, __shfl_xor_sync(SL_FULL, min_d, o));
  }
  bool has_min = R > 0;
  int nadm = 0, nwait = 0;
  int32_t* adm = out.adm_order + wb;

  if (tpot_guard) {
    double inv = inv_pre;
    if (!GROUP && kept > 0) {
      PySum ps;
      ps_init(ps);
      double t_n = lane < R ? st.r_tpot[rb + lane] : 1.0;  // next chunk's operand, in flight
      for (int c0 = 0; c0 < R; c0 += 32) {
        const double x = frcp_(t_n);
        const int jn = c0 + 32 + lane;
        t_n = jn < R ? st.r_tpot[rb + jn] : 1.0;
        ps_add_warp(ps, x, min(32, R - c0));
      }
      inv = ps_result(ps);
    }
    int64_t n_run = R;
    // 3. admission scan, speculative-parallel (sched_scorpio.py:237-294)
    for (int c0 = 0; c0 < kept; c0 += 32) {
      const int p = c0 + lane;
      const bool valid = p < kept;
      int32_t idx = 0, ln = 0, pred = 0;
      double tp = 1.0, ic = 0.0;
      if (valid) {
        idx = kept_list[p];
        if (staged) {
          const int q = stg->klane[p];
          tp = stg->tp[q];
          ln = stg->ln[q];
          pred = stg->pd[q];
        } else {
          tp = st.w_tpot[idx];
          ln = st.w_prompt[idx];
          pred = st.w_pred[idx];
        }
        ic = frcp_(tp);
      }
      // feasible alone? (solo test, :279-289)
      const bool solo = solo_ok(C, tp, ic, ln, pred);
      unsigned pend = __ballot_sync(SL_FULL, valid);
      while (pend) {
        const bool lt = !has_min || tp < min_d;
        const double minp = lt ? tp : min_d;
        const double V = fmul_(minp, fadd_(inv, ic));
        // Python's int / int: exact small-divisor form up to 128 (div_small)
        const double L = n_run < 128 ? div_small((double)(lens + ln), (int)(n_run + 1))
                                     : fdiv_((double)(lens + ln), (double)(n_run + 1));
        const double est = tpot_estimate(C, V, L, pred);
        const double thr = (r_only && has_min) ? min_d : minp;
        const bool ok = ((pend >> lane) & 1u) && est <= thr;
        const unsigned okm = __ballot_sync(SL_FULL, ok);
        const int g = okm ? __ffs(okm) - 1 : 32;
        const unsigned fail = okm ? (pend & ((1u << g) - 1u)) : pend;
        const bool mf = (fail >> lane) & 1u;
        const bool keep = mf && solo;
        const bool rj = mf && !solo;
        const unsigned km = __ballot_sync(SL_FULL, keep);
        const unsigned rm = __ballot_sync(SL_FULL, rj);
        if (keep) {
          out.w_status[idx] = SL_PLAN_WAITING;
          out.w_pos[idx] = nwait + __popc(km & lanemask_lt());
        }
        if (rj) {
          out.w_status[idx] = SL_PLAN_REJECTED_ADMISSION;
          out.w_pos[idx] = nrej + __popc(rm & lanemask_lt());
        }
        nwait += __popc(km);
        nrej += __popc(rm);
        pend &= ~fail;
        if (!okm) break;
        if (lane == g) {
          out.w_status[idx] = SL_PLAN_ADMITTED;
          out.w_pos[idx] = nadm;
          adm[nadm] = idx;
          if (out.w_rec) {
            double* r5 = out.w_rec + 5 * (int64_t)idx;
            r5[0] = V;
            r5[1] = L;
            r5[2] = minp;
            r5[3] = est;
            r5[4] = thr;
          }
        }
        // state update (:272-277)
        const double tp_g = bcast(tp, g);
        n_run += 1;
        inv = fadd_(inv, bcast(ic, g));
        lens += bcast(ln, g);
        if (!has_min || tp_g < min_d) min_d = tp_g;
        has_min = true;
        ++nadm;
        pend &= ~(1u << g);
      }
    }
  } else {  // admit everything in queue order (:295-304)
    for (int p = lane; p < kept; p += 32) {
      const int32_t idx = kept_list[p];
      out.w_status[idx] = SL_PLAN_ADMITTED;
      out.w_pos[idx] = p;
      adm[p] = idx;
    }
    for (int c0 = 0; c0 < kept; c0 += 32) {
      const int p = c0 + lane;
      double v = p < kept ? st.w_tpot[kept_list[p]] : min_d;
#pragma unroll
      for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(SL_FULL, v, o));
      min_d = fmin(min_d, v);
    }
    has_min = has_min || kept > 0;
    nadm = kept;
  }
  __syncwarp();

  if (GROUP) {
    *min_out = min_d;
    *has_min_out = has_min;
    *nadm_out = nadm;
    if (lane == 0) {
      out.seg_counts[4 * seg + 0] = nwait;
      out.seg_counts[4 * seg + 1] = nadm;
      out.seg_counts[4 * seg + 2] = nrej;
    }
    return;
  }
  // 4. plan.min_slo / plan.vbs over running + admitted, in order (:312-315)
  double vbs = 0.0;
  if (has_min) {
    PySum vs;
    ps_init(vs);
    const int tot = R + nadm;
    auto slo = [&](int j) { return j < tot ? (j < R ? st.r_tpot[rb + j] : st.w_tpot[adm[j - R]]) : 1.0; };
    double t_n = slo(lane);  // next chunk's operand, in flight
    for (int c0 = 0; c0 < tot; c0 += 32) {
      const double x = fdiv_(min_d, t_n);
      t_n = slo(c0 + 32 + lane);
      ps_add_warp(vs, x, min(32, tot - c0));
    }
    vbs = ps_result(vs);
  }
  if (lane == 0) {
    out.seg_counts[4 * seg + 0] = nwait;
    out.seg_counts[4 * seg + 1] = nadm;
    out.seg_counts[4 * seg + 2] = nrej;
    out.seg_vbs[seg] = vbs;
    out.seg_min_slo[seg] = has_min ? min_d : __longlong_as_double(0x7ff8000000000000LL);
    out.seg_min_fixed[seg] = has_min ? slo_fixed<false>(min_d, E) : ~0ull;
  }
  (void)pow2E;
}

__global__ void guard_admit_kernel(const sl_plan_state st, const sl_plan_config cfg,
                                   sl_plan_out out) {
  __shared__ int32_t klist[32][32];  // per warp (blockDim <= 1024)
  const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= st.n_segments) return;
  seg_guard_admit(st, cfg, out, seg, threadIdx.x & 31, 0.0, nullptr, nullptr, nullptr,
                  klist[threadIdx.x >> 5]);
}

// Large batches: one warp per kPlanGroup segments.  The order-dependent Neumaier folds
// (sum(1/slo) over running, sched_scorpio.py:121; vbs over running + admitted,
// :312-315) run lane-per-segment -- one warp instruction advances 32 folds
// instead of 32 lanes repeating one -- and the walk / admission scan run
// warp-per-segment in between (seg_guard_admit<true>).
#ifndef SL_PLAN_GROUP
#define SL_PLAN_GROUP 16  // segments per warp (measured: 16 with 7 blocks/SM beats 32, 8 and 4)
#endif
#ifndef SL_PLAN_STAGE
#define SL_PLAN_STAGE 1  // cp.async staging of the next segment's fields (group kernel)
#endif
#ifndef SL_SELECT_PF
#define SL_SELECT_PF 1  // credit select: next segment's lines prefetched into L1
#endif
#ifndef SL_PLAN_GROUP_BLOCKS
#define SL_PLAN_GROUP_BLOCKS 7  // <= 72 registers: 28 warps/SM
#endif
constexpr int kPlanGroup = SL_PLAN_GROUP;
__global__ void __launch_bounds__(128, SL_PLAN_GROUP_BLOCKS) guard_admit_group_kernel(
    const sl_plan_state st, const sl_plan_config cfg, sl_plan_out out) {
  __shared__ int32_t klist[4][32];  // per warp (128 threads)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int seg0 = warp * kPlanGroup;
  if (seg0 >= st.n_segments) return;
  const int nseg = min(kPlanGroup, st.n_segments - seg0);
  const int my = seg0 + lane;
  const bool mine = lane < nseg;
  const bool tpot_guard = cfg.flags & SL_FLAG_TPOT_GUARD;
  // fold 1: sum(1.0 / slo) over this lane's segment's running entries, in order,
  // with the segment's min slo and sum of current lengths
  double inv = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL);
  long long lsum = 0;
  if (mine) {
    const int64_t rb = st.r_begin[my], re = st.r_begin[my + 1];
    PySum ps;
    ps_init(ps);
    for (int64_t j = rb; j < re; ++j) {
      const double t = st.r_tpot[j];
      if (tpot_guard) ps_add(ps, frcp_(t));
      mn = fmin(mn, t);
      lsum += st.r_cur_len[j];
    }
    inv = ps_result(ps);
  }
  double min_d = 0.0;
  bool has_min = false;
  int nadm = 0;
#if SL_PLAN_STAGE
  // segment k+1's waiting fields are copied into shared memory (cp.async)
  // while the warp walks and admits segment k; segment k+2's queue slots are
  // loaded into a register meanwhile (two dependent global round trips per
  // segment off the warp's path)
  __shared__ GStage stage[4][2];
  GStage* sg = stage[threadIdx.x >> 5];
  const bool ttft_guard = cfg.flags & SL_FLAG_TTFT_GUARD;
  auto seg_slot = [&](int seg) -> int32_t {
    const int64_t wb = st.w_begin[seg];
    const int W = (int)(st.w_begin[seg + 1] - wb);
    return (W <= 32 && lane < W) ? (ttft_guard ? out.perm[wb + lane] : (int32_t)(wb + lane)) : -1;
  };
  auto issue = [&](GStage& b, int32_t idx) {
    b.idx[lane] = idx;
    if (idx >= 0) {
      cp_async8(&b.arr[lane], st.w_arrival + idx);
      cp_async8(&b.pf[lane], st.w_prefill + idx);
      cp_async8(&b.tt[lane], st.w_ttft + idx);
      cp_async8(&b.tp[lane], st.w_tpot + idx);
      cp_async4(&b.ln[lane], st.w_prompt + idx);
      cp_async4(&b.pd[lane], st.w_pred + idx);
    }
    cp_async_commit();
  };
  issue(sg[0], seg_slot(seg0));
  int32_t i_next = nseg > 1 ? seg_slot(seg0 + 1) : -1;
#endif
  for (int k = 0; k < nseg; ++k) {
    double m_k = 0.0;
    bool h_k = false;
    int a_k = 0;
#if SL_PLAN_STAGE
    issue(sg[(k + 1) & 1], i_next);  // (an empty group past the last segment)
    i_next = k + 2 < nseg ? seg_slot(seg0 + k + 2) : -1;
    cp_async_wait1();  // segment k's group has landed
    __syncwarp();
    GStage* cur = &sg[k & 1];
#else
    GStage* cur = nullptr;
#endif
    seg_guard_admit<true>(st, cfg, out, seg0 + k, lane, __shfl_sync(SL_FULL, inv, k), &m_k, &h_k,
                          &a_k, klist[threadIdx.x >> 5], __shfl_sync(SL_FULL, lsum, k),
                          __shfl_sync(SL_FULL, mn, k), cur);
    __syncwarp();  // the next segment reuses the warp's kept-list and stage buffers
    if (lane == k) {
      min_d = m_k;
      has_min = h_k;
      nadm = a_k;
    }
  }
  __syncwarp();
  if (!mine || (cfg.flags & SL_PLAN_GUARD_ONLY)) return;
  // fold 2: vbs = sum(min_slo / slo) over running then admitted, in order
  double vbs = 0.0;
  if (has_min) {
    const int64_t rb = st.r_begin[my], re = st.r_begin[my + 1];
    const int32_t* adm = out.adm_order + st.w_begin[my];
    PySum vs;
    ps_init(vs);
    for (int64_t j = rb; j < re; ++j) ps_add(vs, fdiv_(min_d, st.r_tpot[j]));
    for (int q = 0; q < nadm; ++q) ps_add(vs, fdiv_(min_d, st.w_tpot[adm[q]]));
    vbs = ps_result(vs);
  }
  const int E = st.credit_exp[my];
  out.seg_vbs[my] = vbs;
  out.seg_min_slo[my] = has_min ? min_d : __longlong_as_double(0x7ff8000000000000LL);
  out.seg_min_fixed[my] = has_min ? slo_fixed<false>(min_d, E) : ~0ull;
}

// Self-test of the certified CPython sum (DD, dd_certify in sl_device.cuh): one
// warp per sum of x[begin[s], begin[s+1]); out[3 s] = the certified result (NaN
// when the certificate fails), out[3 s + 1], out[3 s + 2] = the double-double.
__global__ void certified_sum_test_kernel(const double* __restrict__ x,
                                          const int64_t* __restrict__ begin, int n_sums,
                                          double* __restrict__ out) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (s >= n_sums) return;
  DD a = {0.0, 0.0};
  for (int64_t j = begin[s] + lane; j < begin[s + 1]; j += 32) dd_add(a, x[j]);
  a = dd_warp(a);
  double r = __longlong_as_double(0x7ff8000000000000LL);
  if (!dd_certify(a, begin[s + 1] - begin[s], &r)) r = __longlong_as_double(0x7ff8000000000000LL);
  if (lane == 0) {
    out[3 * s] = r;
    out[3 * s + 1] = a.s;
    out[3 * s + 2] = a.c;
  }
}

// ---- credit select / decode-all: one warp per segment
__device__ __forceinline__ void seg_credit_select(const sl_plan_state& st,
                                                  const sl_plan_config& cfg,
                                                  const sl_plan_out& out, int use_seg_min,
                                                  int seg, int lane) {
  const bool credit = cfg.flags & SL_FLAG_TPOT_GUARD;
  const int64_t rb = st.r_begin[seg];
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const int E = st.credit_exp[seg];
  uint64_t MIN = ~0ull;
  if (credit) {
    if (use_seg_min) {
      MIN = out.seg_min_fixed[seg];
    } else {
      for (int j = lane; j < R; j += 32) {
        const uint64_t S = slo_fixed<false>(st.r_tpot[rb + j], E);
        MIN = S < MIN ? S : MIN;
      }
      MIN = warp_min_cred<false>(MIN);
    }
  }
  int nb = 0;
  for (int c0 = 0; c0 < R; c0 += 32) {
    const int j = c0 + lane;
    bool b = false;
    if (j < R) {
      const int64_t r = rb + j;
      const bool ex = st.r_exclude && st.r_exclude[r];
      uint64_t N = st.r_credit[r];
      if (!ex) {
        if (credit) {
          const uint64_t S = slo_fixed<false>(st.r_tpot[r], E);
          N += MIN;
          b = N >= S;
          if (b) N -= S;
        } else {
          b = true;
        }
      }
      out.r_credit_out[r] = N;
    }
    const unsigned bm = __ballot_sync(SL_FULL, b);
    if (j < R) {
      out.r_batch[rb + j] = b;
      out.r_pos[rb + j] = b ? nb + __popc(bm & lanemask_lt()) : -1;
    }
    nb += __popc(bm);
  }
  if (lane == 0) out.seg_counts[4 * seg + 3] = nb;
}

__global__ void credit_select_kernel(const sl_plan_state st, const sl_plan_config cfg,
                                     sl_plan_out out, int use_seg_min) {
  const int nw = (gridDim.x * blockDim.x) >> 5;  // grid-stride, as sort_warp_kernel
  const int lane = threadIdx.x & 31, S = st.n_segments;
  int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#if SL_SELECT_PF
  // the next segment's running lines are prefetched into L1 while this one is
  // selected (its start loaded one segment earlier, so no prefetch waits on it)
  int64_t bn = seg + nw < S ? st.r_begin[seg + nw] : 0;
#endif
  for (; seg < S; seg += nw) {
#if SL_SELECT_PF
    const int nx = seg + nw;
    if (nx < S && lane < 5) {
      const char* q = lane < 2 ? reinterpret_cast<const char*>(st.r_credit + bn) + 128 * lane
                      : lane < 4 ? reinterpret_cast<const char*>(st.r_tpot + bn) + 128 * (lane - 2)
                                 : reinterpret_cast<const char*>(st.r_exclude ? st.r_exclude + bn
                                                                              : nullptr);
      if (q) asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
    }
    const int64_t bnn = nx + nw < S ? st.r_begin[nx + nw] : 0;
#endif
    seg_credit_select(st, cfg, out, use_seg_min, seg, lane);
#if SL_SELECT_PF
    bn = bnn;
#endif
  }
}

// Few, large segments (the config-2 stress shape): one 1024-thread CTA per
// segment instead of one warp.  Entries go in super-tiles of 32 x 1024: pass 1
// earns / debits every entry (coalesced) and keeps its batch bit in a register,
// one count per (tile, warp) in shared memory; one CTA-wide scan of the 1,024
// counts; pass 2 writes the batch positions.  Same per-entry arithmetic as
// seg_credit_select.
constexpr int kSelCta = 1024;
__global__ void __launch_bounds__(kSelCta) credit_select_cta_kernel(const sl_plan_state st,
                                                                    const sl_plan_config cfg,
                                                                    sl_plan_out out,
                                                                    int use_seg_min) {
  __shared__ int cnt[kSelCta];
  __shared__ int wtot[32];
  __shared__ unsigned long long smin;
  __shared__ int sbase;
  const int seg = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool credit = cfg.flags & SL_FLAG_TPOT_GUARD;
  const int64_t rb = st.r_begin[seg];
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const int E = st.credit_exp[seg];
  if (tid == 0) {
    smin = ~0ull;
    sbase = 0;
  }
  __syncthreads();
  if (credit) {
    if (use_seg_min) {
      if (tid == 0) smin = out.seg_min_fixed[seg];
    } else {
      uint64_t m = ~0ull;
      for (int j = tid; j < R; j += kSelCta) {
        const uint64_t S = slo_fixed<false>(st.r_tpot[rb + j], E);
        m = S < m ? S : m;
      }
      m = warp_min_cred<false>(m);
      if (lane == 0) atomicMin(&smin, (unsigned long long)m);
    }
  }
  __syncthreads();
  const uint64_t MIN = smin;
  constexpr int kSuper = 32 * kSelCta;
  for (int s0 = 0; s0 < R; s0 += kSuper) {
    unsigned bits = 0;
#pragma unroll 4
    for (int it = 0; it < 32; ++it) {
      const int j = s0 + it * kSelCta + tid;
      bool b = false;
      if (j < R) {
        const int64_t r = rb + j;
        const bool ex = st.r_exclude && st.r_exclude[r];
        uint64_t N = st.r_credit[r];
        if (!ex) {
          if (credit) {
            const uint64_t S = slo_fixed<false>(st.r_tpot[r], E);
            N += MIN;
            b = N >= S;
            if (b) N -= S;
          } else {
            b = true;
          }
        }
        out.r_credit_out[r] = N;
        out.r_batch[r] = b;
      }
      bits |= (unsigned)b << it;
      const unsigned bm = __ballot_sync(SL_FULL, b);
      if (lane == 0) cnt[it * 32 + w] = __popc(bm);
    }
    __syncthreads();
    // exclusive scan of cnt[0..1023] (tile-major, warp-minor = entry order)
    const int v = cnt[tid];
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(SL_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = wtot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(SL_FULL, t, o);
        if (lane >= o) t += y;
      }
      wtot[lane] = t;  // inclusive
    }
    __syncthreads();
    const int base = sbase;
    cnt[tid] = base + (w ? wtot[w - 1] : 0) + x - v;
    __syncthreads();
#pragma unroll 4
    for (int it = 0; it < 32; ++it) {
      const int j = s0 + it * kSelCta + tid;
      const bool b = (bits >> it) & 1u;
      const unsigned bm = __ballot_sync(SL_FULL, b);
      if (j < R) out.r_pos[rb + j] = b ? cnt[it * 32 + w] + __popc(bm & lanemask_lt()) : -1;
    }
    __syncthreads();
    if (tid == 0) sbase = base + wtot[31];
    __syncthreads();
  }
  if (tid == 0) out.seg_counts[4 * seg + 3] = sbase;
}

// Segment count below which credit select runs one CTA per segment.
constexpr int kSelCtaMaxSegments = 64;

// Credit select for few, large segments over a cluster of kSelCluster CTAs per
// segment: CTA q takes the q-th contiguous slice of the running list.  Pass 1:
// every entry's credit update and batch flag (written out), the slice's batch
// count; the counts (and, without a given minimum, the slices' minima first)
// are pushed into every CTA's shared memory with one cluster barrier each; pass
// 2: batch positions from the count of the slices before this one plus a
// blocked ballot scan over the slice (the flags re-read from r_batch).
#ifndef SL_SEL_CLUSTER
#define SL_SEL_CLUSTER 16  // CTAs per segment (measured at the stress shape: 4 22 us, 8 15.8 us, 16 11.5 us)
#endif
constexpr int kSelCluster = SL_SEL_CLUSTER;
__device__ __forceinline__ int cta_excl_scan_i(int v, int* wtot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(SL_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = wtot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(SL_FULL, t, o);
      if (lane >= o) t += y;
    }
    wtot[lane] = t;  // inclusive
  }
  __syncthreads();
  const int r = (w ? wtot[w - 1] : 0) + x - v;
  return r;
}

__global__ void __launch_bounds__(kSelCta) credit_select_cluster_kernel(const sl_plan_state st,
                                                                        const sl_plan_config cfg,
                                                                        sl_plan_out out,
                                                                        int use_seg_min) {
  namespace cg = cooperative_groups;
  __shared__ int wtot[32];
  __shared__ unsigned long long cmin[kSelCluster];  // pushed by every CTA
  __shared__ int ctot[kSelCluster];
  __shared__ unsigned long long smin;
  __shared__ int lcount;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int seg = blockIdx.x / kSelCluster;
  const int tid = threadIdx.x;
  const bool credit = cfg.flags & SL_FLAG_TPOT_GUARD;
  const int64_t rb = st.r_begin[seg];
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const int E = st.credit_exp[seg];
  const int chunk = (R + kSelCluster - 1) / kSelCluster;
  const int lo = min(R, q * chunk), hi = min(R, lo + chunk);
  if (tid == 0) {
    smin = ~0ull;
    lcount = 0;
  }
  cl.sync();  // every CTA started (DSMEM stores below), locals initialised
  uint64_t MIN = ~0ull;
  if (credit) {
    if (use_seg_min) {
      MIN = out.seg_min_fixed[seg];
    } else {  // min fixed-point slo over the whole running list
      uint64_t m = ~0ull;
      for (int j = lo + tid; j < hi; j += kSelCta) {
        const uint64_t S = slo_fixed<false>(st.r_tpot[rb + j], E);
        m = S < m ? S : m;
      }
      m = warp_min_cred<false>(m);
      if ((tid & 31) == 0) atomicMin(&smin, (unsigned long long)m);
      __syncthreads();
      if (tid < kSelCluster) cl.map_shared_rank(cmin, tid)[q] = smin;
      cl.sync();
      for (int k = 0; k < kSelCluster; ++k) MIN = min(MIN, (uint64_t)cmin[k]);
    }
  }
  // pass 1: credits and batch flags of this slice
  int cnt = 0;
  for (int j = lo + tid; j < hi; j += kSelCta) {
    const int64_t r = rb + j;
    const bool ex = st.r_exclude && st.r_exclude[r];
    uint64_t N = st.r_credit[r];
    bool b = false;
    if (!ex) {
      if (credit) {
        const uint64_t S = slo_fixed<false>(st.r_tpot[r], E);
        N += MIN;
        b = N >= S;
        if (b) N -= S;
      } else {
        b = true;
      }
    }
    out.r_credit_out[r] = N;
    out.r_batch[r] = b;
    cnt += b;
  }
  cnt = __reduce_add_sync(SL_FULL, (unsigned)cnt);
  if ((tid & 31) == 0) atomicAdd(&lcount, cnt);
  __syncthreads();
  if (tid < kSelCluster) cl.map_shared_rank(ctot, tid)[q] = lcount;
  cl.sync();  // every slice's count everywhere; r_batch written (block-scope visibility below)
  int base = 0, total = 0;
  for (int k = 0; k < kSelCluster; ++k) {
    base += k < q ? ctot[k] : 0;
    total += ctot[k];
  }
  // pass 2: positions, 1024 entries per round in slice order
  for (int j0 = lo; j0 < hi; j0 += kSelCta) {
    const int j = j0 + tid;
    const bool b = j < hi && out.r_batch[rb + j];
    const int e = cta_excl_scan_i(b ? 1 : 0, wtot);
    if (j < hi) out.r_pos[rb + j] = b ? base + e : -1;
    base += wtot[31];
    __syncthreads();  // wtot reused by the next round
  }
  if (q == 0 && tid == 0) out.seg_counts[4 * seg + 3] = total;
}



// ---- plan_step of one segment with <= 32 waiting and <= 32 running, all in
// registers (the config-2 primary shape).  Every input of the segment is loaded
// up front -- one memory latency instead of one per stage -- and the stages
// exchange values by shuffles: LDF sort (packed-key network, full-key network on
// near-ties), TTFT walk (certified any-order bound, else rounds of "first item
// that passes at the current prefix"), sum(1/slo), admission rounds, vbs, and
// the credit phase.  Same decisions and fp64 values as seg_sort_warp +
// seg_guard_admit + seg_credit_select (sched_scorpio.py:117-207, 210-316).
#ifdef SL_LARGE_PROF
__device__ unsigned long long sl_fused_prof[16];
#define SL_FSTAMP()                                                 \
  do {                                                              \
    if (seg == 0 && lane == 0) {                                    \
      const unsigned long long k_ = sl_fused_prof[0] + 1;           \
      if (k_ < 16) sl_fused_prof[k_] = clock64();                   \
      sl_fused_prof[0] = k_;                                        \
    }                                                               \
  } while (0)
#else
#define SL_FSTAMP() do {} while (0)
#endif
// Warp pairs of the fused step (plan_fused_pair_kernel): the fold warp loads the
// running set, computes its aggregates, sum(1/slo) and -- speculatively with the
// pre-admission minimum -- the running part of vbs, hands them over through
// shared memory (named barrier 1 + pair), then waits for the plan warp's final
// minimum (barrier 5 + pair) and runs the credit phase on the entries it holds.
struct PairShared {
  long long lens;
  double min_pre, inv, vf, vc;
  int vn;
  int has_min;
  unsigned long long MIN;
};
__device__ __forceinline__ void pair_bar_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void pair_bar_arrive(int id) {
  asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

// The fold warp of a pair (see PairShared): running-set work of seg_plan_small.
__device__ __forceinline__ void seg_plan_fold(const sl_plan_state& st, const sl_plan_config& cfg,
                                              const sl_plan_out& out, int seg, int lane,
                                              double* buf, PairShared& ps_sh, int pair) {
  const bool tpot_guard = cfg.flags & SL_FLAG_TPOT_GUARD;
  if (cfg.flags & SL_PLAN_GUARD_ONLY) return;  // the plan warp stops after the walk
  const int64_t rb = st.r_begin[seg];
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const int E = st.credit_exp[seg];
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const bool rv = lane < R;
  double rt = 1.0;
  int32_t rlen = 0;
  uint64_t rcred = 0;
  bool rex = false;
  if (rv) {
    rt = st.r_tpot[rb + lane];
    rlen = st.r_cur_len[rb + lane];
    rcred = st.r_credit[rb + lane];
    rex = st.r_exclude && st.r_exclude[rb + lane];
  }
  // running aggregates (:117-124), sum(1/slo) (:121), vbs running part (:312-315)
  const int64_t lens = warp_sum_i64(rv ? (int64_t)rlen : 0);
  double min_pre = rv ? rt : kInf;
#pragma unroll
  for (int o = 16; o; o >>= 1) min_pre = fmin(min_pre, __shfl_xor_sync(SL_FULL, min_pre, o));
  double inv = 0.0;
  if (tpot_guard && R > 0) {
    PySum ps;
    ps_init(ps);
    ps_add_warp_smem(ps, frcp_(rt), R, buf);
    inv = ps_result(ps);
  }
  PySum vs;
  ps_init(vs);
  if (R > 0) ps_add_warp_smem(vs, fdiv_(min_pre, rt), R, buf);
  if (lane == 0) {
    ps_sh.lens = lens;
    ps_sh.min_pre = min_pre;
    ps_sh.inv = inv;
    ps_sh.vf = vs.f;
    ps_sh.vc = vs.c;
    ps_sh.vn = vs.n;
  }
  __syncwarp();
  pair_bar_arrive(1 + pair);
  pair_bar_sync(5 + pair);  // the plan warp's final minimum
  const uint64_t MIN = ps_sh.MIN;
  // ---- credit phase (:161-180) or decode-all
  bool b = false;
  uint64_t N = rcred;
  if (rv && !rex) {
    if (tpot_guard) {
      const uint64_t S = slo_fixed<false>(rt, E);
      N += MIN;
      b = N >= S;
      if (b) N -= S;
    } else {
      b = true;
    }
  }
  const unsigned bm = __ballot_sync(SL_FULL, b);
  if (rv) {
    out.r_credit_out[rb + lane] = N;
    out.r_batch[rb + lane] = b;
    out.r_pos[rb + lane] = b ? __popc(bm & lanemask_lt()) : -1;
  }
  if (lane == 0) out.seg_counts[4 * seg + 3] = __popc(bm);
}

template <bool PAIR = false>
__device__ __forceinline__ void seg_plan_small(const sl_plan_state& st, const sl_plan_config& cfg,
                                               const sl_plan_out& out, int seg, int lane,
                                               double* buf, PairShared* ps_sh = nullptr,
                                               int pair = 0) {
  const sl_cost& C = cfg.cost;
  const bool ttft_guard = cfg.flags & SL_FLAG_TTFT_GUARD;
  const bool tpot_guard = cfg.flags & SL_FLAG_TPOT_GUARD;
  const bool r_only = cfg.flags & SL_FLAG_R_ONLY;
  const bool guard_only = cfg.flags & SL_PLAN_GUARD_ONLY;
  const bool walk = ttft_guard || (cfg.flags & SL_PLAN_FCFS_WALK);
  const bool exact = cfg.flags & SL_PLAN_EXACT_WALK;
  const int64_t wb = st.w_begin[seg], rb = st.r_begin[seg];
  const int W = (int)(st.w_begin[seg + 1] - wb);
  const int R = (int)(st.r_begin[seg + 1] - rb);
  const double now = st.now[seg];
  const int E = st.credit_exp[seg];
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  SL_FSTAMP();
  // ---- every input at once
  const bool wv = lane < W, rv = lane < R;
  double arr = 0.0, tt0 = 0.0, pf0 = 0.0, tp0 = 1.0;
  int32_t pr0 = 0, pd0 = 0;
  int64_t id0 = 0;
  if (wv) {
    arr = st.w_arrival[wb + lane];
    tt0 = st.w_ttft[wb + lane];
    pf0 = st.w_prefill[wb + lane];
    tp0 = st.w_tpot[wb + lane];
    pr0 = st.w_prompt[wb + lane];
    pd0 = st.w_pred[wb + lane];
    id0 = st.w_id[wb + lane];
  }
  double rt = 1.0;
  int32_t rlen = 0;
  uint64_t rcred = 0;
  bool rex = false;
  if (!PAIR && rv) {
    rt = st.r_tpot[rb + lane];
    rlen = st.r_cur_len[rb + lane];
    rcred = st.r_credit[rb + lane];
    rex = st.r_exclude && st.r_exclude[rb + lane];
  }
  SL_FSTAMP();
  // ---- LDF order (sched_scorpio.py:193): src = input position at walk position lane
  int src = lane;
  if (ttft_guard) {
    const double d = wv ? fadd_(arr, tt0) : 0.0;  // core.py:50-53
    bool done = false;
    if (SL_SORT32 && __all_sync(SL_FULL, !wv || d >= 0.0)) {
      const int sr = warp_ldf_src32(d, wv, W, lane);
      if (sr >= 0) {
        src = sr;
        done = true;
      }
    }
    if (!SL_SORT32 && __all_sync(SL_FULL, !wv || d >= 0.0)) {
      uint64_t key = wv ? (((uint64_t)__double_as_longlong(d) & ~31ull) | (uint64_t)lane) : ~0ull;
#pragma unroll
      for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
          const uint64_t ok = __shfl_xor_sync(SL_FULL, key, j);
          const bool up = (lane & size) == 0;
          const bool lower = (lane & j) == 0;
          key = ((lower == up) == (ok < key)) ? ok : key;
        }
      }
      const uint64_t next = __shfl_down_sync(SL_FULL, key, 1);
      if (!__any_sync(SL_FULL, lane + 1 < W && (next >> 5) == (key >> 5))) {
        src = (int)(key & 31);
        done = true;
      }
    }
    if (!done) {  // ties / near-ties: the full (deadline, arrival, id) network
      Key k;
      if (wv) {
        k.d = d;
        k.a = arr;
        k.id = id0;
        k.idx = lane;
      } else {
        k = inf_key();
      }
#pragma unroll
      for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
          Key o;
          o.d = __shfl_xor_sync(SL_FULL, k.d, j);
          o.a = __shfl_xor_sync(SL_FULL, k.a, j);
          o.id = __shfl_xor_sync(SL_FULL, k.id, j);
          o.idx = __shfl_xor_sync(SL_FULL, k.idx, j);
          const bool up = (lane & size) == 0;
          const bool lower = (lane & j) == 0;
          const bool take = (lower == up) ? key_lt(o, k) : key_lt(k, o);
          if (take) k = o;
        }
      }
      src = k.idx < 0 ? lane : k.idx;
    }
    if (wv) out.perm[wb + lane] = (int32_t)(wb + src);
  }
  SL_FSTAMP();
  // fields in walk order
  const double e = __shfl_sync(SL_FULL, fsub_(now, arr), src);
  const double pf = __shfl_sync(SL_FULL, pf0, src);
  const double tt = __shfl_sync(SL_FULL, tt0, src);
  const double tp = __shfl_sync(SL_FULL, tp0, src);
  const int32_t ln = __shfl_sync(SL_FULL, pr0, src);
  const int32_t pred = __shfl_sync(SL_FULL, pd0, src);
  const int32_t idx = (int32_t)(wb + src);
  const unsigned vmask = __ballot_sync(SL_FULL, wv);

  // ---- TTFT walk (:196-205)
  unsigned kept = vmask;
  if (walk) {
    bool certified = false;
    if (!exact) {  // any-order inflated prefix bound (see seg_guard_admit)
      const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
      double v = wv ? pf : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(SL_FULL, v, o);
        if (lane >= o) v = fadd_(v, y);
      }
      double excl = __shfl_up_sync(SL_FULL, v, 1);
      if (lane == 0) excl = 0.0;
      const double Uj = fmul_(fadd_(0.0, excl), inflate);
      certified = __all_sync(SL_FULL, !wv || fadd_(fadd_(e, Uj), pf) <= tt);
    }
    if (!certified) {  // exact: rounds of the first item passing at the current prefix
      unsigned alive = vmask;
      kept = 0;
      double prefix = 0.0;
      for (;;) {
        const unsigned okm =
            __ballot_sync(SL_FULL, ((alive >> lane) & 1u) && !(fadd_(fadd_(e, prefix), pf) > tt));
        if (!okm) break;
        const int g = __ffs(okm) - 1;
        kept |= 1u << g;
        alive &= ~((2u << g) - 1u);
        prefix = fadd_(prefix, bcast(pf, g));
      }
    }
  }
  SL_FSTAMP();
  const unsigned rejw = vmask & ~kept;
  if ((rejw >> lane) & 1u) {
    out.w_status[idx] = SL_PLAN_REJECTED_TTFT;
    out.w_pos[idx] = __popc(rejw & lanemask_lt());
  }
  int nrej = __popc(rejw);
  if (guard_only) {
    if ((kept >> lane) & 1u) {
      out.w_status[idx] = SL_PLAN_WAITING;
      out.w_pos[idx] = __popc(kept & lanemask_lt());
    }
    if (lane == 0) {
      out.seg_counts[4 * seg + 0] = __popc(kept);
      out.seg_counts[4 * seg + 1] = 0;
      out.seg_counts[4 * seg + 2] = nrej;
    }
    return;
  }

  // ---- running aggregates (:117-124)
  int64_t lens;
  double min_d;
  double inv_pair = 0.0;
  if (PAIR) {  // from the fold warp
    pair_bar_sync(1 + pair);
    lens = ps_sh->lens;
    min_d = ps_sh->min_pre;
    inv_pair = ps_sh->inv;
  } else {
    lens = warp_sum_i64(rv ? (int64_t)rlen : 0);
    min_d = rv ? rt : kInf;
#pragma unroll
    for (int o = 16; o; o >>= 1) min_d = fmin(min_d, __shfl_xor_sync(SL_FULL, min_d, o));
  }
  const double min_pre = min_d;
  bool has_min = R > 0;
  unsigned admm = 0, keepm = 0, rejm = 0;
  if (tpot_guard) {
    double inv = 0.0;
    if (PAIR) {
      inv = inv_pair;
    } else if (kept && R > 0) {
      PySum ps;
      ps_init(ps);
      ps_add_warp_smem(ps, frcp_(rt), R, buf);
      inv = ps_result(ps);
    }
  SL_FSTAMP();
    // ---- admission rounds (:237-294): every pending candidate against one state
    const double ic = frcp_(tp);
    const bool solo = solo_ok(C, tp, ic, ln, pred);
    int64_t n_run = R;
    unsigned pend = kept;
    while (pend) {
      const bool lt = !has_min || tp < min_d;
      const double minp = lt ? tp : min_d;
      const double V = fmul_(minp, fadd_(inv, ic));
      const double L = div_small((double)(lens + ln), (int)(n_run + 1));  // n_run + 1 <= 65
      const double est = tpot_estimate(C, V, L, pred);
      const double thr = (r_only && has_min) ? min_d : minp;
      const unsigned okm = __ballot_sync(SL_FULL, ((pend >> lane) & 1u) && est <= thr);
      if (!okm) break;
      const int g = __ffs(okm) - 1;
      if (lane == g && out.w_rec) {
        double* r5 = out.w_rec + 5 * (int64_t)idx;
        r5[0] = V;
        r5[1] = L;
        r5[2] = minp;
        r5[3] = est;
        r5[4] = thr;
      }
      admm |= 1u << g;
      pend &= ~((2u << g) - 1u);
      const double tp_g = bcast(tp, g);
      n_run += 1;
      inv = fadd_(inv, bcast(ic, g));  // :275
      lens += bcast(ln, g);
      if (!has_min || tp_g < min_d) min_d = tp_g;
      has_min = true;
    }
    const unsigned fail = kept & ~admm;
    keepm = __ballot_sync(SL_FULL, ((fail >> lane) & 1u) && solo);
    rejm = fail & ~keepm;
  } else {  // admit everything in queue order (:295-304)
    admm = kept;
    double v = (kept >> lane) & 1u ? tp : kInf;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(SL_FULL, v, o));
    min_d = fmin(min_d, v);
    has_min = has_min || kept != 0;
  }
  SL_FSTAMP();
  const int nadm = __popc(admm);
  if ((admm >> lane) & 1u) {
    const int q = __popc(admm & lanemask_lt());
    out.w_status[idx] = SL_PLAN_ADMITTED;
    out.w_pos[idx] = q;
    out.adm_order[wb + q] = idx;
  } else if ((keepm >> lane) & 1u) {
    out.w_status[idx] = SL_PLAN_WAITING;
    out.w_pos[idx] = __popc(keepm & lanemask_lt());
  } else if ((rejm >> lane) & 1u) {
    out.w_status[idx] = SL_PLAN_REJECTED_ADMISSION;
    out.w_pos[idx] = nrej + __popc(rejm & lanemask_lt());
  }
  nrej += __popc(rejm);

  // ---- plan.min_slo / plan.vbs over running + admitted, in order (:312-315)
  double vbs = 0.0;
  if (has_min) {
    PySum vs;
    ps_init(vs);
    if (PAIR && R > 0 && min_d == min_pre) {
      vs.f = ps_sh->vf;  // the fold warp's running part, folded with this minimum
      vs.c = ps_sh->vc;
      vs.n = ps_sh->vn;
    } else if (R > 0) {
      if (PAIR && rv) rt = st.r_tpot[rb + lane];  // admission lowered the minimum (rare)
      ps_add_warp_smem(vs, fdiv_(min_d, rt), R, buf);
    }
    if (nadm) {
      const bool a = (admm >> lane) & 1u;
      const double x = a ? fdiv_(min_d, tp) : 0.0;
      __syncwarp();
      if (a) buf[__popc(admm & lanemask_lt())] = x;
      __syncwarp();
      ps_fold_buf(vs, buf, nadm);
    }
    vbs = ps_result(vs);
  }
  SL_FSTAMP();
  const uint64_t MIN = has_min ? slo_fixed<false>(min_d, E) : ~0ull;
  if (PAIR) {
    if (lane == 0) ps_sh->MIN = MIN;
    __syncwarp();
    pair_bar_arrive(5 + pair);  // the fold warp runs the credit phase
  }
  if (lane == 0) {
    out.seg_counts[4 * seg + 0] = __popc(keepm);
    out.seg_counts[4 * seg + 1] = nadm;
    out.seg_counts[4 * seg + 2] = nrej;
    out.seg_vbs[seg] = vbs;
    out.seg_min_slo[seg] = has_min ? min_d : __longlong_as_double(0x7ff8000000000000LL);
    out.seg_min_fixed[seg] = MIN;
  }
  if (PAIR) return;
  // ---- credit phase (:161-180) or decode-all
  bool b = false;
  uint64_t N = rcred;
  if (rv && !rex) {
    if (tpot_guard) {
      const uint64_t S = slo_fixed<false>(rt, E);
      N += MIN;
      b = N >= S;
      if (b) N -= S;
    } else {
      b = true;
    }
  }
  const unsigned bm = __ballot_sync(SL_FULL, b);
  if (rv) {
    out.r_credit_out[rb + lane] = N;
    out.r_batch[rb + lane] = b;
    out.r_pos[rb + lane] = b ? __popc(bm & lanemask_lt()) : -1;
  }
  if (lane == 0) out.seg_counts[4 * seg + 3] = __popc(bm);
  SL_FSTAMP();
}

// ---- the fused plan step with a warp pair per segment (PairShared): 4 segments
// per 256-thread CTA; the plan warp sorts, walks and admits while the fold warp
// reduces the running set; segments with more than 32 running run unpaired.
__global__ void __launch_bounds__(256) plan_fused_pair_kernel(const sl_plan_state st,
                                                              const sl_plan_config cfg,
                                                              sl_plan_out out) {
  __shared__ __align__(16) double bufs[8][32];
  __shared__ PairShared psh[4];
  const int w = threadIdx.x >> 5, pair = w >> 1;
  const int seg = blockIdx.x * 4 + pair;
  if (seg >= st.n_segments) return;
  const int lane = threadIdx.x & 31;
  const bool small = st.r_begin[seg + 1] - st.r_begin[seg] <= 32;  // (w <= 32 here)
  if (small) {
    if (w & 1)
      seg_plan_fold(st, cfg, out, seg, lane, bufs[w], psh[pair], pair);
    else
      seg_plan_small<true>(st, cfg, out, seg, lane, bufs[w], &psh[pair], pair);
    return;
  }
  if (w & 1) return;
  if (cfg.flags & SL_FLAG_TTFT_GUARD) {
    seg_sort_warp(st, out.perm, seg, lane);
    __syncwarp();
  }
  seg_guard_admit(st, cfg, out, seg, lane);
  if (cfg.flags & SL_PLAN_GUARD_ONLY) return;
  __syncwarp();
  seg_credit_select(st, cfg, out, 1, seg, lane);
}

// ---- the whole plan_step in one launch (segments of <= 32 waiting items):
// sort, guard + admission, credit select back to back in one warp; the stages
// hand over through the segment's own global slices (L1-resident), so inputs
// cross HBM once and there is one launch instead of three.
__global__ void __launch_bounds__(256) plan_fused_kernel(const sl_plan_state st,
                                                         const sl_plan_config cfg,
                                                         sl_plan_out out) {
  __shared__ __align__(16) double bufs[8][32];
  const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (seg >= st.n_segments) return;
  const int lane = threadIdx.x & 31;
  if (st.r_begin[seg + 1] - st.r_begin[seg] <= 32) {  // (w <= 32 for every segment here)
    seg_plan_small(st, cfg, out, seg, lane, bufs[threadIdx.x >> 5]);
    return;
  }
  if (cfg.flags & SL_FLAG_TTFT_GUARD) {
    seg_sort_warp(st, out.perm, seg, lane);
    __syncwarp();
  }
  seg_guard_admit(st, cfg, out, seg, lane);
  if (cfg.flags & SL_PLAN_GUARD_ONLY) return;
  __syncwarp();
  seg_credit_select(st, cfg, out, 1, seg, lane);
}

__global__ void vbs_kernel(int S, const int64_t* r_begin, const double* r_tpot,
                           const double* min_slo, double* out) {
  const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (seg >= S) return;
  const int64_t rb = r_begin[seg];
  const int R = (int)(r_begin[seg + 1] - rb);
  const double m = min_slo[seg];
  PySum vs;
  ps_init(vs);
  for (int c0 = 0; c0 < R; c0 += 32) {
    const int j = c0 + lane;
    const double x = j < R ? fdiv_(m, r_tpot[rb + j]) : 0.0;  // trp, :63-67
    const int cnt = min(32, R - c0);
    for (int t = 0; t < cnt; ++t) ps_add(vs, bcast(x, t));
  }
  if (lane == 0) out[seg] = ps_result(vs);  // empty -> 0.0 (:72-73)
}

int warps_grid(int n_warps, int threads) { return (n_warps * 32 + threads - 1) / threads; }

// Grid for the grid-stride warp-per-segment kernels: at most `per_sm` blocks
// per SM (SL_STRIDE_BLOCKS overrides for experiments).
int stride_grid(int n_warps, int threads, int per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (const char* e = getenv("SL_STRIDE_BLOCKS")) per_sm = atoi(e);
  const int need = warps_grid(n_warps, threads);
  const int cap = sms * per_sm;
  return need < cap ? need : cap;
}

// Segment count from which guard_admit uses the 32-segments-per-warp kernel
// (enough groups to fill the GPU); SL_PLAN_GROUP_MIN overrides it (tests force
// either path).  The fused single-launch plan step is used below it.
int plan_group_min() {
  if (const char* e = getenv("SL_PLAN_GROUP_MIN")) return atoi(e);
  return 8192;
}

// The fused single-launch plan step for segments of <= 32 waiting, below
// plan_group_min segments (above it the separate kernels are faster: measured
// 704 vs 492 us at 262,144 segments); SL_PLAN_FUSED=0 disables it (tests).
bool plan_fused_on() {
  const char* e = getenv("SL_PLAN_FUSED");
  return !(e && e[0] == '0');
}

// Segment count up to which guard + admission runs one CTA per segment
// (guard_admit_cta_kernel, plan_large.cuh); SL_PLAN_CTA_MAX overrides it.
int plan_cta_max() {
  if (const char* e = getenv("SL_PLAN_CTA_MAX")) return atoi(e);
  return kSelCtaMaxSegments;
}

}  // namespace

#include "plan_large.cuh"

#ifdef SL_LARGE_PROF
extern "C" int sl_fused_prof_read(unsigned long long* out) {  // and reset
  static const unsigned long long z[16] = {0};
  if (cudaMemcpyFromSymbol(out, sl_fused_prof, sizeof(z)) != cudaSuccess) return SL_ERR_CUDA;
  return cudaMemcpyToSymbol(sl_fused_prof, z, sizeof(z)) == cudaSuccess ? 0 : SL_ERR_CUDA;
}
#endif

extern "C" {

int sl_ttft_sort_batch(const sl_plan_state* st, int64_t max_w, sl_plan_out* out, void* stream) {
  if (!st || !out || !out->perm || max_w < 0) return SL_ERR_ARG;
  const int S = st->n_segments;
  if (S == 0 || max_w == 0) return SL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (max_w <= 32) {
    sort_warp_kernel<<<stride_grid(S, 128, 32), 128, 0, s>>>(*st, out->perm);
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  if (S <= plan_cta_max() && max_w <= kSortMaxCluster * kSortLoc) {  // few large segments
    const int cs = (int)((max_w + kSortLoc - 1) / kSortLoc);  // one cluster per segment
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(sort_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(sort_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(RadixSmem));
      attr_set = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(S * cs);
    lc.blockDim = dim3(kSortCtaThreads);
    lc.dynamicSmemBytes = sizeof(RadixSmem);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, sort_cluster_kernel, *st, out->perm) != cudaSuccess)
      return SL_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  if (!out->scratch) return SL_ERR_ARG;
  const int tiles = (int)((max_w + kTile - 1) / kTile);
  const size_t smem = (size_t)kTile * (8 + 8 + 8 + 4);
  cudaFuncSetAttribute(sort_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sort_tile_kernel<<<S * tiles, kSortThreads, smem, s>>>(*st, tiles, out->perm);
  int32_t* src = out->perm;
  int32_t* dst = out->scratch;
  for (int64_t w = kTile; w < max_w; w *= 2) {
    const int per_block = 256 * kMergeItems;
    const int bps = (int)((max_w + per_block - 1) / per_block);
    merge_pass_kernel<<<S * bps, 256, 0, s>>>(*st, w, bps, src, dst);
    int32_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != out->perm) {
    copy_kernel<<<592, 256, 0, s>>>(*st, src, out->perm);
  }
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_guard_admit_batch(const sl_plan_state* st, const sl_plan_config* cfg, sl_plan_out* out,
                         void* stream) {
  if (!st || !cfg || !out || !out->scratch || !out->w_status || !out->w_pos || !out->seg_counts)
    return SL_ERR_ARG;
  if (!(cfg->flags & SL_PLAN_GUARD_ONLY) &&
      (!out->adm_order || !out->seg_vbs || !out->seg_min_slo || !out->seg_min_fixed))
    return SL_ERR_ARG;
  if ((cfg->flags & SL_FLAG_TTFT_GUARD) && !out->perm) return SL_ERR_ARG;
  if (st->n_segments == 0) return SL_OK;
  if (st->n_segments <= plan_cta_max()) {
    const int smem = (int)sizeof(LargeSmem);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(guard_admit_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem);
    // a 2-CTA cluster per segment: the CPython folds on their own SM (SL_PLAN_SPLIT=0: one CTA)
    const char* e = getenv("SL_PLAN_SPLIT");
    const int cs = (e && e[0] == '0') ? 1 : 2;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(st->n_segments * cs);
    lc.blockDim = dim3(kLThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, guard_admit_cta_kernel, *st, *cfg, *out) != cudaSuccess)
      return SL_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  if (st->n_segments >= plan_group_min()) {
    guard_admit_group_kernel<<<warps_grid((st->n_segments + kPlanGroup - 1) / kPlanGroup, 128), 128, 0,
                               (cudaStream_t)stream>>>(*st, *cfg, *out);
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  guard_admit_kernel<<<warps_grid(st->n_segments, 128), 128, 0, (cudaStream_t)stream>>>(*st, *cfg,
                                                                                        *out);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_credit_select_batch(const sl_plan_state* st, const sl_plan_config* cfg, sl_plan_out* out,
                           int32_t use_seg_min, void* stream) {
  if (!st || !cfg || !out || !out->r_credit_out || !out->r_batch || !out->r_pos ||
      !out->seg_counts || (use_seg_min && !out->seg_min_fixed))
    return SL_ERR_ARG;
  if (st->n_segments == 0) return SL_OK;
  const char* ce = getenv("SL_SELECT_CLUSTER");
  if (st->n_segments <= kSelCtaMaxSegments && !(ce && ce[0] == '0')) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(st->n_segments * kSelCluster);
    lc.blockDim = dim3(kSelCta);
    lc.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kSelCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (kSelCluster > 8)
      cudaFuncSetAttribute(credit_select_cluster_kernel,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (cudaLaunchKernelEx(&lc, credit_select_cluster_kernel, *st, *cfg, *out, use_seg_min) !=
        cudaSuccess)
      return SL_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  if (st->n_segments <= kSelCtaMaxSegments)
    credit_select_cta_kernel<<<st->n_segments, kSelCta, 0, (cudaStream_t)stream>>>(
        *st, *cfg, *out, use_seg_min);
  else
    credit_select_kernel<<<stride_grid(st->n_segments, 128, 32), 128, 0, (cudaStream_t)stream>>>(
        *st, *cfg, *out, use_seg_min);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_vbs_batch(int32_t n_segments, const int64_t* r_begin, const double* r_tpot,
                 const double* min_slo, double* out, void* stream) {
  if (n_segments < 0 || (n_segments > 0 && (!r_begin || !min_slo || !out))) return SL_ERR_ARG;
  if (n_segments == 0) return SL_OK;
  vbs_kernel<<<warps_grid(n_segments, 128), 128, 0, (cudaStream_t)stream>>>(n_segments, r_begin,
                                                                           r_tpot, min_slo, out);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_plan_step_batch(const sl_plan_state* st, const sl_plan_config* cfg, int64_t max_w,
                       sl_plan_out* out, void* stream) {
  if (!st || !cfg || !out) return SL_ERR_ARG;
  if (max_w <= 32 && st->n_segments < plan_group_min() && plan_fused_on()) {  // one launch
    if (!out->scratch || !out->w_status || !out->w_pos || !out->seg_counts ||
        ((cfg->flags & SL_FLAG_TTFT_GUARD) && !out->perm))
      return SL_ERR_ARG;
    if (!(cfg->flags & SL_PLAN_GUARD_ONLY) &&
        (!out->adm_order || !out->seg_vbs || !out->seg_min_slo || !out->seg_min_fixed ||
         !out->r_credit_out || !out->r_batch || !out->r_pos))
      return SL_ERR_ARG;
    if (st->n_segments == 0) return SL_OK;
    // warp pairs while the GPU has room for them (measured: faster up to ~1,500
    // segments, one warp per segment from 2,048); SL_PLAN_PAIR=0 / =1 forces
    const char* pe = getenv("SL_PLAN_PAIR");
    const bool pair = pe ? pe[0] != '0' : st->n_segments <= 1536;
    if (pair) {
      plan_fused_pair_kernel<<<(st->n_segments + 3) / 4, 256, 0, (cudaStream_t)stream>>>(*st, *cfg,
                                                                                       *out);
      return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
    }
    plan_fused_kernel<<<warps_grid(st->n_segments, 256), 256, 0, (cudaStream_t)stream>>>(*st, *cfg,
                                                                                        *out);
    return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
  }
  int rc;
  if (cfg->flags & SL_FLAG_TTFT_GUARD) {
    rc = sl_ttft_sort_batch(st, max_w, out, stream);
    if (rc) return rc;
  }
  rc = sl_guard_admit_batch(st, cfg, out, stream);
  if (rc) return rc;
  if (cfg->flags & SL_PLAN_GUARD_ONLY) return SL_OK;
  return sl_credit_select_batch(st, cfg, out, 1, stream);
}

int sl_selftest_certified_sum(const double* x, const int64_t* begin, int32_t n_sums, double* out,
                              void* stream) {
  if (n_sums < 0 || (n_sums > 0 && (!x || !begin || !out))) return SL_ERR_ARG;
  if (n_sums == 0) return SL_OK;
  certified_sum_test_kernel<<<(n_sums + 7) / 8, 256, 0, (cudaStream_t)stream>>>(x, begin, n_sums,
                                                                               out);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

}  // extern "C"
