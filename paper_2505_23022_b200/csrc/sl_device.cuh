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

#ifndef SL_PSADD_SEL
#define SL_PSADD_SEL 0  // CPython sum() step: select the operands, then one error expression
#endif

namespace sl {

__device__ __forceinline__ double fadd_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fdiv_(double a, double b) { return __ddiv_rn(a, b); }
// 1.0 / x, correctly rounded (== fdiv_(1.0, x)): the reciprocal intrinsic has no
// general-division slow path.
__device__ __forceinline__ double frcp_(double x) { return __drcp_rn(x); }

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
#if SL_PSADD_SEL
    // operands selected first, one error expression (2 DADDs, not 4 + a select)
    const bool big = fabs(s.f) >= fabs(x);
    const double hi = big ? s.f : x, lo = big ? x : s.f;
    double a = fadd_(fsub_(hi, t), lo);
#else
    double a = (fabs(s.f) >= fabs(x)) ? fadd_(fsub_(s.f, t), x) : fadd_(fsub_(x, t), s.f);
#endif
    s.c = fadd_(s.c, a);
    s.f = t;
  }
}
// Fold the first `cnt` lanes' values of x (lane order) into s.  The operands are
// gathered by unrolled shuffles that do not depend on the (serial) sum chain.
__device__ __forceinline__ void ps_add_warp(PySum& s, double x, int cnt) {
  if (cnt == 32) {
    double v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = __shfl_sync(0xffffffffu, x, t);
#pragma unroll
    for (int t = 0; t < 32; ++t) ps_add(s, v[t]);
  } else {
    for (int t = 0; t < cnt; ++t) ps_add(s, __shfl_sync(0xffffffffu, x, t));
  }
}

// ps_add for a sum that already holds a float (s.n > 0): branch-free, so an
// unrolled run of these keeps only the t = f + x dependency on the chain.
__device__ __forceinline__ void ps_add_nz(PySum& s, double x) {
  const double t = fadd_(s.f, x);
  const bool big = fabs(s.f) >= fabs(x);
  const double hi = big ? s.f : x, lo = big ? x : s.f;
  s.c = fadd_(s.c, fadd_(fsub_(hi, t), lo));
  s.f = t;
}

// Fold the first `cnt` lanes' values of x into s (as ps_add_warp), the full-chunk
// case unrolled over ps_add_nz: long folds (thousands of entries) run at about
// one DADD latency per entry.
__device__ __forceinline__ void ps_add_warp_long(PySum& s, double x, int cnt) {
  if (cnt == 32 && s.n > 0) {
    double v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = __shfl_sync(0xffffffffu, x, t);
#pragma unroll
    for (int t = 0; t < 32; ++t) ps_add_nz(s, v[t]);
  } else {
    for (int t = 0; t < cnt; ++t) ps_add(s, __shfl_sync(0xffffffffu, x, t));
  }
}

// Fold buf[0, cnt) into s in order: the first term of an empty sum takes the
// int-0 path, every later one the branch-free ps_add_nz (same result as ps_add).
__device__ __forceinline__ void ps_fold_buf(PySum& s, const double* buf, int cnt) {
  int t = 0;
  if (s.n == 0 && cnt > 0) {
    s.f = fadd_(0.0, buf[0]);
    s.n = 1;
    t = 1;
  }
  for (; t < cnt; ++t) ps_add_nz(s, buf[t]);
}

// As ps_add_warp_long with the operands gathered through a per-warp shared
// buffer `buf` (32 doubles, 16-byte aligned) as 16 x LDS.128 broadcasts instead
// of 64 shuffles: the fold is then bound by its own fp64 issue (~19 cycles per
// entry measured, tools/ubench_fold.cu) instead of shuffle throughput (~27).
__device__ __forceinline__ void ps_add_warp_smem(PySum& s, double x, int cnt, double* buf) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  buf[lane] = x;
  __syncwarp();
  if (cnt == 32) {
    double v[32];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const double2 p = reinterpret_cast<const double2*>(buf)[t];
      v[2 * t] = p.x;
      v[2 * t + 1] = p.y;
    }
    if (s.n == 0) {  // first term of an empty sum: the int-0 path
      s.f = fadd_(0.0, v[0]);
      s.n = 1;
#pragma unroll
      for (int t = 1; t < 32; ++t) ps_add_nz(s, v[t]);
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) ps_add_nz(s, v[t]);
    }
  } else {
    ps_fold_buf(s, buf, cnt);
  }
}

__device__ __forceinline__ double ps_result(const PySum& s) {
  if (s.n == 0) return 0.0;  // int 0; every use adds it to a float
  double f = s.f;
  if (s.c != 0.0 && isfinite(s.c)) f = fadd_(f, s.c);
  return f;
}

// ---- exact small-divisor division.  kRecip[b] = RN(1/b).  For an integer
// 0 <= a < 2^53 and 1 <= b <= 128: q0 = RN(a*y) is within 2 ulp of a/b, so the
// remainder r = a - b*q0 is a multiple of ulp(q0) below 2^8 ulp(q0) and the FMA
// computes it exactly; q1 = RN(q0 + r*y) = RN(a/b + (a/b - q0)*eps), |eps| <=
// 2^-53, and a/b is either dyadic (exact) or at least ulp/(2b) away from every
// rounding midpoint, which that perturbation cannot cross: q1 == a / b correctly
// rounded, i.e. Python's int / int.  Three fp64 ops instead of __ddiv_rn.
__constant__ double kRecip[129] = {0.0, 1.0, 0.5, 0.3333333333333333, 0.25, 0.2, 0.16666666666666666, 0.14285714285714285, 0.125, 0.1111111111111111, 0.1, 0.09090909090909091, 0.08333333333333333, 0.07692307692307693, 0.07142857142857142, 0.06666666666666667, 0.0625, 0.058823529411764705, 0.05555555555555555, 0.05263157894736842, 0.05, 0.047619047619047616, 0.045454545454545456, 0.043478260869565216, 0.041666666666666664, 0.04, 0.038461538461538464, 0.037037037037037035, 0.03571428571428571, 0.034482758620689655, 0.03333333333333333, 0.03225806451612903, 0.03125, 0.030303030303030304, 0.029411764705882353, 0.02857142857142857, 0.027777777777777776, 0.02702702702702703, 0.02631578947368421, 0.02564102564102564, 0.025, 0.024390243902439025, 0.023809523809523808, 0.023255813953488372, 0.022727272727272728, 0.022222222222222223, 0.021739130434782608, 0.02127659574468085, 0.020833333333333332, 0.02040816326530612, 0.02, 0.0196078431372549, 0.019230769230769232, 0.018867924528301886, 0.018518518518518517, 0.01818181818181818, 0.017857142857142856, 0.017543859649122806, 0.017241379310344827, 0.01694915254237288, 0.016666666666666666, 0.01639344262295082, 0.016129032258064516, 0.015873015873015872, 0.015625, 0.015384615384615385, 0.015151515151515152, 0.014925373134328358, 0.014705882352941176, 0.014492753623188406, 0.014285714285714285, 0.014084507042253521, 0.013888888888888888, 0.0136986301369863, 0.013513513513513514, 0.013333333333333334, 0.013157894736842105, 0.012987012987012988, 0.01282051282051282, 0.012658227848101266, 0.0125, 0.012345679012345678, 0.012195121951219513, 0.012048192771084338, 0.011904761904761904, 0.011764705882352941, 0.011627906976744186, 0.011494252873563218, 0.011363636363636364, 0.011235955056179775, 0.011111111111111112, 0.01098901098901099, 0.010869565217391304, 0.010752688172043012, 0.010638297872340425, 0.010526315789473684, 0.010416666666666666, 0.010309278350515464, 0.01020408163265306, 0.010101010101010102, 0.01, 0.009900990099009901, 0.00980392156862745, 0.009708737864077669, 0.009615384615384616, 0.009523809523809525, 0.009433962264150943, 0.009345794392523364, 0.009259259259259259, 0.009174311926605505, 0.00909090909090909, 0.009009009009009009, 0.008928571428571428, 0.008849557522123894, 0.008771929824561403, 0.008695652173913044, 0.008620689655172414, 0.008547008547008548, 0.00847457627118644, 0.008403361344537815, 0.008333333333333333, 0.008264462809917356, 0.00819672131147541, 0.008130081300813009, 0.008064516129032258, 0.008, 0.007936507936507936, 0.007874015748031496, 0.0078125};

__device__ __forceinline__ double div_small(double a, int b) {
  if (b > 128) return fdiv_(a, (double)b);
  const double y = kRecip[b];
  const double q0 = fmul_(a, y);
  const double r = __fma_rn(-q0, (double)b, a);
  return __fma_rn(r, y, q0);
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

// ---- certified CPython sums of positive terms.
// CPython's sum() over floats (Neumaier: f_i = fl(f_{i-1} + x_i), the exact
// error e_i of each add -- FastTwoSum -- chained into c by rounded adds, result
// fl(f_n + c_n)) satisfies f_n + sum(e_i) = S exactly, and for positive terms
// |e_i| <= u S, so |c_n - sum(e_i)| <= gamma_{n-1} n u S: f_n + c_n lies within
// n^2 u^2 S (1 + 2nu) of the exact sum S and the result is RN(S) unless a
// rounding midpoint of the double grid lies within that distance of S.  A
// double-double sum (s, c) of the same terms in any order -- TwoSum per term,
// the errors added rounded -- is within n^2 u^2 S of S as well, so with
// T = 4 n^2 u^2 hi: if |lo| + T < half the gap from hi = RN(s + c) toward lo,
// the sequential fold's result is hi, bit for bit.  Otherwise (probability
// ~2^-20 n^2 u / ...: never seen) the caller runs the sequential fold.
#ifndef SL_CERT_FOLD
#define SL_CERT_FOLD 1  // 0: always the sequential folds (the tests build this too)
#endif
struct DD {
  double s, c;
};
__device__ __forceinline__ void dd_add(DD& a, double x) {
  const double t = fadd_(a.s, x);
  const double bv = fsub_(t, a.s);
  const double e = fadd_(fsub_(a.s, fsub_(t, bv)), fsub_(x, bv));  // exact: a.s + x - t
  a.s = t;
  a.c = fadd_(a.c, e);
}
__device__ __forceinline__ DD dd_merge(DD a, const DD& b) {
  dd_add(a, b.s);
  a.c = fadd_(a.c, b.c);
  return a;
}
// lane 0's tree of the warp's partials, broadcast (every lane the same value)
__device__ __forceinline__ DD dd_warp(DD a) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    DD b;
    b.s = __shfl_down_sync(SL_FULL, a.s, o);
    b.c = __shfl_down_sync(SL_FULL, a.c, o);
    a = dd_merge(a, b);
  }
  a.s = __shfl_sync(SL_FULL, a.s, 0);
  a.c = __shfl_sync(SL_FULL, a.c, 0);
  return a;
}
__device__ __forceinline__ bool dd_certify(const DD& a, int64_t n, double* res) {
  const double hi = fadd_(a.s, a.c);
  const double bv = fsub_(hi, a.s);
  const double lo = fadd_(fsub_(a.s, fsub_(hi, bv)), fsub_(a.c, bv));  // exact: a.s + a.c - hi
  if (!(hi > 1e-290) || !(hi < 1e300)) return false;  // normal, gap formula valid
  const double nn = (double)n;
  const double T = fmul_(fmul_(fmul_(nn, nn), 4.930380657631324e-32), hi);  // 4 n^2 2^-106 hi
  // the gap to the next double above hi, or below (half at a power of two)
  const uint64_t b = (uint64_t)__double_as_longlong(hi);
  const double up = __longlong_as_double((long long)(((b >> 52) - 52) << 52));
  const double gap = (lo >= 0.0 || (b & 0xFFFFFFFFFFFFFull) != 0) ? up : fmul_(up, 0.5);
  if (!(fadd_(fabs(lo), T) < fmul_(gap, 0.4999))) return false;
  *res = hi;
  return true;
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
