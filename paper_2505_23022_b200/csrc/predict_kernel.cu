// LengthPredictor.predict on device (predictor.py:115-126), one thread per request.
//
//   oracle       -> true_output_len
//   noisy_bucket -> true bucket (bisect_left over the boundaries, overflow to the
//                   last bucket), then with probability error_prob a shift of
//                   +-U[1, spread] buckets, clamped, and the bucket representative
//                   max(1, ceil((lo + hi) / 2.0))            (predictor.py:71-90)
//
// The noise stream is numpy's: default_rng([rng_seed, id]) = SeedSequence
// (pool 4, uint32 hashmix/mix) -> PCG64 (128-bit LCG, XSL-RR output) with the
// draws random() [53-bit double], integers(1, spread+1) [Lemire on the low
// 32 bits, retries from the buffered high half], random() for the sign.
// Pinned by tests/golden/predictor_kat.npz (numpy 2.3.5 outputs).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "scorpio_b200.h"

namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

__device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t buf32;
};

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
}
__device__ __forceinline__ void pcg_step(Pcg64& g) { g.state = g.state * pcg_mult() + g.inc; }
__device__ __forceinline__ uint64_t pcg_next64(Pcg64& g) {
  pcg_step(g);
  uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
  unsigned rot = (unsigned)(g.state >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ uint32_t pcg_next32(Pcg64& g) {
  if (g.has32) {
    g.has32 = false;
    return g.buf32;
  }
  uint64_t v = pcg_next64(g);
  g.has32 = true;
  g.buf32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}
__device__ __forceinline__ double next_double(Pcg64& g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Split a non-negative integer into little-endian uint32 words (0 -> [0]).
__device__ __forceinline__ int words_of(uint64_t v, uint32_t* w) {
  if (v == 0) {
    w[0] = 0;
    return 1;
  }
  int k = 0;
  while (v) {
    w[k++] = (uint32_t)v;
    v >>= 32;
  }
  return k;
}

// default_rng([seed, id]) -> seeded PCG64
__device__ Pcg64 seeded_pcg(uint64_t seed, uint64_t id) {
  uint32_t ent[4];
  int ne = words_of(seed, ent);
  ne += words_of(id, ent + ne);
  uint32_t pool[4];
  uint32_t h = kInitA;
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, h);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
  // ne <= 4 == pool size: no remaining entropy words
  uint32_t st[8];
  uint32_t hb = kInitB;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t w0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  uint64_t w1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  uint64_t w2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  uint64_t w3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
  Pcg64 g;
  u128 initstate = ((u128)w0 << 64) | w1;
  u128 initseq = ((u128)w2 << 64) | w3;
  g.state = 0;
  g.inc = (initseq << 1) | 1;
  pcg_step(g);
  g.state += initstate;
  pcg_step(g);
  g.has32 = false;
  g.buf32 = 0;
  return g;
}

// integers(1, spread + 1): Lemire over [0, spread) on 32-bit draws
__device__ __forceinline__ int64_t bounded_1_to(Pcg64& g, int32_t spread) {
  uint32_t rng = (uint32_t)(spread - 1);
  if (rng == 0) return 1;  // no draw
  uint32_t excl = rng + 1;
  uint64_t m = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return 1 + (int64_t)(m >> 32);
}

__device__ __forceinline__ int bucket_of(const double* b, int nb, int32_t len, int* clamped) {
  double x = (double)len;
  if (x > b[nb - 1]) {
    *clamped = 1;
    return nb - 1;
  }
  int lo = 0, hi = nb;  // bisect_left
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (b[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int32_t representative(const double* b, int k) {
  double lo = k > 0 ? b[k - 1] : 0.0;
  double hi = b[k];
  double c = ceil(__ddiv_rn(__dadd_rn(lo, hi), 2.0));
  return c < 1.0 ? 1 : (int32_t)c;
}

__global__ void sl_predict_kernel(const int64_t* __restrict__ id,
                                  const int32_t* __restrict__ true_out, int64_t n,
                                  sl_predictor p, int32_t* __restrict__ out,
                                  unsigned long long* __restrict__ clamps) {
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t t = true_out[i];
    if (p.mode == SL_PREDICT_ORACLE) {
      out[i] = t;
      continue;
    }
    int clamped = 0;
    int tb = bucket_of(p.boundaries, p.num_buckets, t, &clamped);
    local += clamped;
    Pcg64 g = seeded_pcg(p.rng_seed, (uint64_t)id[i]);
    int b = tb;
    if (next_double(g) < p.error_prob) {
      int64_t shift = bounded_1_to(g, p.error_spread);
      if (next_double(g) < 0.5) shift = -shift;
      int64_t nbk = tb + shift;
      nbk = nbk < 0 ? 0 : nbk;
      nbk = nbk > p.num_buckets - 1 ? p.num_buckets - 1 : nbk;
      b = (int)nbk;
    }
    out[i] = representative(p.boundaries, b);
  }
  if (clamps && local) atomicAdd(clamps, (unsigned long long)local);
}

}  // namespace

extern "C" int sl_predict_batch(const int64_t* id, const int32_t* true_out, int64_t n,
                                const sl_predictor* p, int32_t* out_pred,
                                unsigned long long* clamp_count, void* stream) {
  if (!p || n < 0 || (n > 0 && (!id || !true_out || !out_pred))) return SL_ERR_ARG;
  if (p->mode != SL_PREDICT_ORACLE && p->mode != SL_PREDICT_NOISY_BUCKET) return SL_ERR_ARG;
  if (p->mode == SL_PREDICT_NOISY_BUCKET &&
      (!p->boundaries || p->num_buckets < 1 || p->error_spread < 1 || !(p->error_prob >= 0.0) ||
       p->error_prob > 1.0))
    return SL_ERR_ARG;
  if (n == 0) return SL_OK;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  sl_predict_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(id, true_out, n, *p,
                                                                        out_pred, clamp_count);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}
