// Device-side building blocks shared by the sweep (persistent per-sim) kernel
// and the batched plan-step kernels.  sm_100a only.
//
// fp64 rules: every floating-point operation on the
// decision path goes through the *_rn intrinsics below, which nvcc never
// contracts into FMA, so results equal CPython's left-to-right unfused
// evaluation bit for bit.  The library is additionally built with
// --fmad=false as a second line of defence.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "scorpio_b200.h"

#define SL_FULL 0xffffffffu

namespace sl {

__device__ __forceinline__ double fadd_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fdiv_(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T bcast(T v, int src) {
  return __shfl_sync(SL_FULL, v, src);
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(SL_FULL, v, o);
  return v;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(SL_FULL, v, o);
  return v;
}

// ---- CPython 3.12 builtin sum() over floats (Neumaier), SURVEY Appendix B.
struct PySum {
  double f, c;
  int n;
};
__device__ __forceinline__ void ps_init(PySum& s) {
  s.f = 0.0;
  s.c = 0.0;
  s.n = 0;
}
__device__ __forceinline__ void ps_add(PySum& s, double x) {
  if (s.n == 0) {
    s.f = fadd_(0.0, x);  // int 0 + float leaves the int fast path
    s.n = 1;
  } else {
    double t = fadd_(s.f, x);
    double a = (fabs(s.f) >= fabs(x)) ? fadd_(fsub_(s.f, t), x) : fadd_(fsub_(x, t), s.f);
    s.c = fadd_(s.c, a);
    s.f = t;
  }
}
__device__ __forceinline__ double ps_result(const PySum& s) {
  if (s.n == 0) return 0.0;  // int 0; every use adds it to a float
  double f = s.f;
  if (s.c != 0.0 && isfinite(s.c)) f = fadd_(f, s.c);
  return f;
}

// ---- cost models (costmodel.py:96-138)
__device__ __forceinline__ double prefill_time(const sl_cost& c, int32_t prompt) {
  double p = (double)prompt;  // exact (|prompt| < 2^53); int<=float compare is exact
  if (p <= c.theta) return c.phi;
  return fadd_(fmul_(c.alpha_p, p), c.beta_p);
}

// ((((alpha*B)*L) + beta*B) + gamma*L) + delta, costmodel.py:102-107
__device__ __forceinline__ double itl(const sl_cost& c, int64_t batch, double l_avg) {
  double B = (double)batch;
  return fadd_(fadd_(fadd_(fmul_(fmul_(c.alpha, B), l_avg), fmul_(c.beta, B)), fmul_(c.gamma, l_avg)),
              c.delta);
}

// estimate of _admission_math (sched_scorpio.py:105-109):
// eps * ((((alpha*V) + gamma) * (L + P/2.0) + beta*V) + delta)
__device__ __forceinline__ double tpot_estimate(const sl_cost& c, double V, double L, int32_t pred) {
  double half = fmul_((double)pred, 0.5);  // == pred / 2.0 exactly
  return fmul_(c.epsilon,
              fadd_(fadd_(fmul_(fadd_(fmul_(c.alpha, V), c.gamma), fadd_(L, half)), fmul_(c.beta, V)),
                   c.delta));
}

// solo test: _admission_math(0, 0.0, 0.0, None, cand, len, pred), sched_scorpio.py:279-289
__device__ __forceinline__ bool solo_ok(const sl_cost& c, double cand, double inv_cand,
                                        int32_t len, int32_t pred) {
  double V = fmul_(cand, fadd_(0.0, inv_cand));
  double L = (double)len;  // (0 + len) / 1 exactly
  return tpot_estimate(c, V, L, pred) <= cand;
}

// ---- fixed-point credits.  S = tpot / 2^E, exact.
template <bool WIDE>
using cred_t = typename std::conditional<WIDE, unsigned __int128, uint64_t>::type;

template <bool WIDE>
__device__ __forceinline__ cred_t<WIDE> slo_fixed(double tpot, int E) {
  uint64_t b = (uint64_t)__double_as_longlong(tpot);
  int ex = (int)((b >> 52) & 0x7ff);
  uint64_t m = (b & 0xFFFFFFFFFFFFFull) | (1ull << 52);
  int sh = (ex - 1075) - E;  // >= 0 by construction of E
  if constexpr (WIDE) {
    return (unsigned __int128)m << sh;
  } else {
    return m << sh;
  }
}

template <bool WIDE>
__device__ __forceinline__ double fixed_to_double(cred_t<WIDE> S, double pow2E) {
  if constexpr (WIDE) {
    uint64_t lo = (uint64_t)S, hi = (uint64_t)(S >> 64);
    // both parts and their sum are exact: S has <= 53 significant bits
    double d = fadd_(fmul_(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
    return fmul_(d, pow2E);
  } else {
    return fmul_(__ull2double_rn(S), pow2E);
  }
}

template <bool WIDE>
__device__ __forceinline__ cred_t<WIDE> shfl_cred(cred_t<WIDE> v, int src) {
  if constexpr (WIDE) {
    uint64_t lo = __shfl_sync(SL_FULL, (uint64_t)v, src);
    uint64_t hi = __shfl_sync(SL_FULL, (uint64_t)(v >> 64), src);
    return ((unsigned __int128)hi << 64) | lo;
  } else {
    return __shfl_sync(SL_FULL, v, src);
  }
}

template <bool WIDE>
__device__ __forceinline__ cred_t<WIDE> warp_min_cred(cred_t<WIDE> v) {
  if constexpr (!WIDE) {  // two 32-bit warp reductions: high word, then low word among ties
    const unsigned hi = __reduce_min_sync(SL_FULL, (unsigned)(v >> 32));
    const unsigned lo = __reduce_min_sync(SL_FULL, (unsigned)(v >> 32) == hi ? (unsigned)v : ~0u);
    return ((uint64_t)hi << 32) | lo;
  } else {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      uint64_t lo = __shfl_xor_sync(SL_FULL, (uint64_t)v, o);
      uint64_t hi = __shfl_xor_sync(SL_FULL, (uint64_t)(v >> 64), o);
      cred_t<WIDE> w = ((unsigned __int128)hi << 64) | lo;
      v = w < v ? w : v;
    }
    return v;
  }
}

// ---- work-step decision digest (oracle orc_digest_item).
// item = mix(val ^ (step*K_STEP + tag*K_TAG + pos*K_POS)), mix(x) = (x*K_MIX) ^ ((x*K_MIX) >> 32);
// the digest is the sum mod 2^64 of the items of all work steps: per admitted
// id (tag 0), per rejection (tag 1), one per step for the batch (tag 2, see
// batch_hid) and one per step for the end time (tag 3).
constexpr uint64_t kDigStep = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kDigTag = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t kDigPos = 0x165667B19E3779F9ULL;
constexpr uint64_t kDigMix = 0xD6E8FEB86659FD93ULL;
__device__ __forceinline__ uint64_t digest_key(uint64_t step, uint32_t tag) {
  return step * kDigStep + (uint64_t)tag * kDigTag;
}
__device__ __forceinline__ uint64_t digest_item_k(uint64_t key, uint32_t pos, uint64_t val) {
  uint64_t x = (val ^ (key + (uint64_t)pos * kDigPos)) * kDigMix;
  return x ^ (x >> 32);
}
__device__ __forceinline__ uint64_t digest_item(uint64_t step, uint32_t tag, uint32_t pos,
                                                uint64_t val) {
  return digest_item_k(digest_key(step, tag), pos, val);
}
// Batch id hash: the low 32 bits of mix(id).  The batch of a work step enters
// the digest as ONE item, digest_item(step, 2, n_batch, sum of batch_hid mod
// 2^32) -- a warp reduction per step instead of a hash per (step, entry).
__device__ __forceinline__ uint32_t batch_hid(uint64_t id) {
  const uint64_t y = id * kDigMix;
  return (uint32_t)(y ^ (y >> 32));
}

}  // namespace sl
