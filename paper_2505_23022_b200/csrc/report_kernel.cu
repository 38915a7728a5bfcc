// Per-simulation RunReport reductions on the device (report.summarize,
// report.py:71-127), over the per-request outcomes an sl_run_batch wrote:
// nearest-rank percentiles of TTFT and TPOT over completed requests and the
// per-category totals / compliant counts.  One CTA per simulation.
//
// Nearest rank (report.py:_nearest_rank): the ceil(p / 100.0 * n)-th smallest
// (1-based; p / 100.0 * n evaluated in fp64 as Python does).  The order
// statistic is found by an exact radix select on the value's bit pattern:
// TTFT and TPOT of completed requests are non-negative doubles, whose bit
// patterns order like the values; 8 passes of 8 bits, the three ranks of a
// metric selected together.  TPOT is reported in ms: x -> fl(1000 x) is
// monotone, so the k-th smallest of the scaled list is fl(1000 * k-th smallest).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "scorpio_b200.h"
#include "sl_device.cuh"

using namespace sl;

namespace {

constexpr int kThreads = 256;
constexpr int kRanks = 3;  // p50, p90, p99
__constant__ double kPct[kRanks] = {50.0, 90.0, 99.0};

// k-th smallest (0-based ranks rk[q]) of the values v(i) of the completed
// requests [0, n) of one sim; all threads of the CTA call it.
template <class F>
__device__ void radix_select3(F value, const int8_t* status, int64_t n, const int64_t* rk,
                              uint64_t* out, unsigned* hist) {
  __shared__ uint64_t prefix[kRanks];
  __shared__ int64_t rem[kRanks];
  if (threadIdx.x < kRanks) {
    prefix[threadIdx.x] = 0;
    rem[threadIdx.x] = rk[threadIdx.x];
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < kRanks * 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint64_t hi_mask = shift == 56 ? 0ull : ~0ull << (shift + 8);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      if (status[i] != SL_COMPLETED) continue;
      const uint64_t bits = (uint64_t)__double_as_longlong(value(i));
      const unsigned digit = (unsigned)(bits >> shift) & 255u;
#pragma unroll
      for (int q = 0; q < kRanks; ++q)
        if (rem[q] >= 0 && (bits & hi_mask) == prefix[q]) atomicAdd(&hist[q * 256 + digit], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kRanks) {  // bin holding rank rem[q] among the candidates
      const int q = threadIdx.x;
      if (rem[q] >= 0) {
        int64_t r = rem[q];
        unsigned d = 0;
        for (; d < 256; ++d) {
          if (r < (int64_t)hist[q * 256 + d]) break;
          r -= hist[q * 256 + d];
        }
        prefix[q] |= (uint64_t)d << shift;
        rem[q] = r;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < kRanks) out[threadIdx.x] = prefix[threadIdx.x];
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) report_kernel(const sl_traces tr, const sl_sim* sims,
                                                          sl_outcomes oc, const int8_t* category,
                                                          int32_t n_cat, sl_report_row* rows,
                                                          int64_t* cat_counts) {
  __shared__ unsigned hist[kRanks * 256];
  __shared__ unsigned long long ncomp;
  __shared__ uint64_t sel[kRanks];
  __shared__ unsigned long long sfirst[4];
  extern __shared__ unsigned long long cat_sm[];  // [n_cat][2]
  const int si = blockIdx.x;
  const sl_sim& sp = sims[si];
  const int t = sp.trace;
  const int64_t b = tr.begin[t];
  const int64_t n = tr.begin[t + 1] - b;
  sl_report_row* row = rows + si;
  if (sp.out_offset < 0) {  // no outcomes for this cell
    if (threadIdx.x == 0) row->n_completed = -1;
    return;
  }
  const int8_t* status = oc.status + sp.out_offset;
  const int8_t* compliant = oc.compliant + sp.out_offset;
  const double* ttft = oc.ttft + sp.out_offset;
  const double* tpot = oc.tpot + sp.out_offset;
  if (threadIdx.x == 0) ncomp = 0;
  if (threadIdx.x < 4) sfirst[threadIdx.x] = (unsigned long long)n;
  for (int c = threadIdx.x; c < 2 * n_cat; c += blockDim.x) cat_sm[c] = 0;
  __syncthreads();
  unsigned long long mine = 0;
  unsigned long long first[4] = {(unsigned long long)n, (unsigned long long)n,
                                 (unsigned long long)n, (unsigned long long)n};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int sc = status[i];
    mine += sc == SL_COMPLETED;
    if (sc >= 0 && sc < 4 && first[sc] == (unsigned long long)n) first[sc] = (unsigned long long)i;
    const int c = category ? category[b + i] : 0;
    if (c >= 0 && c < n_cat) {
      atomicAdd(&cat_sm[2 * c], 1ull);
      if (compliant[i]) atomicAdd(&cat_sm[2 * c + 1], 1ull);
    }
  }
  atomicAdd(&ncomp, mine);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (first[k] < (unsigned long long)n) atomicMin(&sfirst[k], first[k]);
  __syncthreads();
  const int64_t nc = (int64_t)ncomp;
  int64_t rk[kRanks];
#pragma unroll
  for (int q = 0; q < kRanks; ++q) {  // max(1, ceil(p / 100.0 * n)) - 1 (report.py:_nearest_rank)
    const double pos = fmul_(fdiv_(kPct[q], 100.0), (double)nc);
    const int64_t r = (int64_t)ceil(pos);
    rk[q] = nc > 0 ? (r < 1 ? 1 : r) - 1 : -1;
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  radix_select3([&](int64_t i) { return ttft[i]; }, status, n, rk, sel, hist);
  if (threadIdx.x < kRanks)
    row->ttft_p[threadIdx.x] = nc > 0 ? __longlong_as_double((long long)sel[threadIdx.x]) : qnan;
  __syncthreads();
  radix_select3([&](int64_t i) { return tpot[i]; }, status, n, rk, sel, hist);
  if (threadIdx.x < kRanks)
    row->tpot_ms_p[threadIdx.x] =
        nc > 0 ? fmul_(__longlong_as_double((long long)sel[threadIdx.x]), 1000.0) : qnan;
  if (threadIdx.x == 0) row->n_completed = nc;
  if (threadIdx.x < 4) row->status_first[threadIdx.x] = (int64_t)sfirst[threadIdx.x];
  for (int c = threadIdx.x; c < 2 * n_cat; c += blockDim.x)
    cat_counts[(int64_t)si * 2 * n_cat + c] = (int64_t)cat_sm[c];
}

// Cumulative SLO-met series (report.py:92: sorted completion times of the
// compliant requests; point i is (t_i, i + 1)).  One CTA per simulation:
// stream-compact the compliant requests' completion times (index order) into
// `out`, then a stable LSD radix sort of their bit patterns (non-negative
// doubles order like their bits) between `out` and `scratch`, 8-bit digits,
// passes whose digit is constant over the keys skipped.  Rank within a
// 256-key tile: warp peers by __match_any_sync, warps in order through a
// per-warp digit count table.
constexpr int kWarps = kThreads / 32;

__device__ int64_t block_compact(const int8_t* flag, const double* val, int64_t n, uint64_t* out,
                                 unsigned* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t base = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kThreads) {
    const int64_t i = t0 + threadIdx.x;
    const bool f = i < n && flag[i] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    unsigned before = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      before += q < w ? wsum[q] : 0;
      tot += wsum[q];
    }
    if (f)
      out[base + before + __popc(bal & ((1u << lane) - 1u))] =
          (uint64_t)__double_as_longlong(val[i]);
    base += tot;
    __syncthreads();
  }
  return base;
}

__global__ void __launch_bounds__(kThreads) cumulative_kernel(const sl_traces tr,
                                                              const sl_sim* sims, sl_outcomes oc,
                                                              double* out_times, uint64_t* scratch,
                                                              int64_t* n_out) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long bucket[256];
  __shared__ unsigned wc[kWarps][256];
  __shared__ unsigned wsum[kWarps];
  __shared__ int skip;
  const sl_sim& sp = sims[blockIdx.x];
  if (sp.out_offset < 0) {
    if (threadIdx.x == 0) n_out[blockIdx.x] = -1;
    return;
  }
  const int64_t n = tr.begin[sp.trace + 1] - tr.begin[sp.trace];
  uint64_t* a = reinterpret_cast<uint64_t*>(out_times) + sp.out_offset;
  uint64_t* b = scratch + sp.out_offset;
  const int64_t c = block_compact(oc.compliant + sp.out_offset, oc.completion_time + sp.out_offset,
                                  n, a, wsum);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int shift = 0; shift < 64; shift += 8) {
    hist[threadIdx.x] = 0;
    for (int q = 0; q < kWarps; ++q) wc[q][threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < c; i += kThreads) atomicAdd(&hist[(a[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan; a pass with one occupied digit is the identity
      unsigned long long run = 0;
      skip = 0;
      for (int d = 0; d < 256; ++d) {
        bucket[d] = run;
        run += hist[d];
        skip |= (int64_t)hist[d] == c;
      }
    }
    __syncthreads();
    if (skip) continue;
    for (int64_t t0 = 0; t0 < c; t0 += kThreads) {
      const int64_t i = t0 + threadIdx.x;
      const bool v = i < c;
      const uint64_t key = v ? a[i] : 0;
      const unsigned d = (unsigned)(key >> shift) & 255u;
      const unsigned peers = __match_any_sync(0xffffffffu, v ? d : 256u + lane);
      if (v && lane == __ffs(peers) - 1) wc[w][d] = __popc(peers);
      __syncthreads();
      if (v) {
        unsigned long long pos = bucket[d] + __popc(peers & ((1u << lane) - 1u));
        for (int q = 0; q < w; ++q) pos += wc[q][d];
        b[pos] = key;
      }
      __syncthreads();
      unsigned add = 0;
#pragma unroll
      for (int q = 0; q < kWarps; ++q) {
        add += wc[q][threadIdx.x];
        wc[q][threadIdx.x] = 0;
      }
      bucket[threadIdx.x] += add;
      __syncthreads();
    }
    uint64_t* t = a;
    a = b;
    b = t;
  }
  uint64_t* dst = reinterpret_cast<uint64_t*>(out_times) + sp.out_offset;
  if (a != dst)
    for (int64_t i = threadIdx.x; i < c; i += kThreads) dst[i] = a[i];
  if (threadIdx.x == 0) n_out[blockIdx.x] = c;
}

}  // namespace

extern "C" {

int sl_report_batch(const sl_traces* traces, const sl_sim* sims, int32_t n_sims,
                    const sl_outcomes* outcomes, const int8_t* category, int32_t n_categories,
                    sl_report_row* rows, int64_t* cat_counts, void* stream) {
  if (!traces || !sims || !outcomes || !rows || n_sims < 0 || n_categories < 0 ||
      (n_categories > 0 && !cat_counts) || n_categories > 4096)
    return SL_ERR_ARG;
  if (n_sims == 0) return SL_OK;
  const size_t smem = sizeof(unsigned long long) * 2 * (size_t)n_categories;
  report_kernel<<<n_sims, kThreads, smem, (cudaStream_t)stream>>>(
      *traces, sims, *outcomes, category, n_categories, rows, cat_counts);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

int sl_cumulative_batch(const sl_traces* traces, const sl_sim* sims, int32_t n_sims,
                        const sl_outcomes* outcomes, double* out_times, uint64_t* scratch,
                        int64_t* n_out, void* stream) {
  if (!traces || !sims || !outcomes || !out_times || !scratch || !n_out || n_sims < 0)
    return SL_ERR_ARG;
  if (n_sims == 0) return SL_OK;
  cumulative_kernel<<<n_sims, kThreads, 0, (cudaStream_t)stream>>>(*traces, sims, *outcomes,
                                                                   out_times, scratch, n_out);
  return cudaGetLastError() == cudaSuccess ? SL_OK : SL_ERR_CUDA;
}

}  // extern "C"
