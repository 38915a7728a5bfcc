// Batched plan_step for FEW, LARGE segments (the config-2 stress shape: one
// SchedulerState with 32,768 waiting + 32,768 running): one CTA per segment.
// Included by plan_kernels.cu (same translation unit and helpers).
//
// A segment's plan_step is three order-dependent chains -- the TTFT prefix walk
// over the LDF queue, CPython's compensated sum(1/slo) over the running list
// (sched_scorpio.py:121), the greedy admission scan (:237-294) -- plus the
// sum(min_slo/slo) of plan.vbs (:312-315).  One warp walking all of it
// serially took 2.3 ms at the stress shape.  Here the CTA splits the roles
// so that the chains overlap and only the unavoidable serial parts stay serial:
//   walk warps (kLW): tiles of kLTile queue items in walk order; every item that
//       fails at the tile's incoming prefix is rejected outright in parallel
//       (prefixes only grow and the estimate is monotone in them), the
//       survivors are compacted in order to shared memory and warp 0 runs the
//       exact speculative chain over them alone; statuses / positions by
//       CTA-wide ballot scans.  A whole-queue certified pass (inflated
//       any-order prefix bound) first: if nothing can be rejected the queue is
//       kept as is.
//   fold warp F0: sum(1/slo) over running, in order (one DADD latency/entry).
//   aggregate warps F1..F3: min slo and sum of lengths over running; then F1
//       folds vbs over running with that minimum, speculatively: admission
//       rarely lowers the minimum, and when it does warp 0 refolds.
//   warp 0 then runs the admission scan (speculative-parallel rounds, one per
//       admission per chunk; bookkeeping once per chunk) and finishes vbs over
//       the admitted entries from F1's fold state.
// Exactness: every decision and fp64 value comes from the same sequential
// operations as seg_guard_admit (the reference's order); only independent work
// moved to other warps.

namespace {

constexpr int kLW = 12;                    // walk warps
constexpr int kLF = 4;                     // fold / aggregate warps
constexpr int kLThreads = (kLW + kLF) * 32;
constexpr int kLWalkThreads = kLW * 32;
#ifndef SL_LK
#define SL_LK 2
#endif
constexpr int kLK = SL_LK;                   // queue items per walk thread per tile
constexpr int kLTile = kLWalkThreads * kLK;
constexpr int kLChunks = kLK * kLW;        // warp chunks per tile

// named barriers (0 is __syncthreads)
constexpr int kBarWalk = 1;   // walk warps
constexpr int kBarAgg = 2;    // F0 (inv), F1..F3 (min, lens) -> warp 0
constexpr int kBarRed = 3;    // F1..F3 reduction
constexpr int kBarVbs = 4;    // vbs pair (fold over running) -> warp 0
constexpr int kBarInvRing = 5;   // 5..8: inv fold handover (full x2, empty x2)
constexpr int kBarVbsRing = 9;   // 9..12: vbs fold handover
constexpr int kBarInvPair = 13;  // split launch: the inv f / c warps
constexpr int kBarPipe = 14;     // pipelined walk: warp 0 (chains) + the helper warps
constexpr int kBarHelp = 15;     // pipelined walk: the helper warps
#ifndef SL_PIPE_SOLO
#define SL_PIPE_SOLO 1  // pipelined walk: warps 4 and 8 (warp 0's SMSP) idle (measured: 239 -> 233 us)
#endif
constexpr int kAdmChunks = 1024;  // kept lists of up to 32,768 items
#ifndef SL_ADM_PAR
#define SL_ADM_PAR 1  // first admission round over every chunk in parallel (all walk warps)
#endif
#ifndef SL_WALK_PIPE
#define SL_WALK_PIPE 1  // walk tiles staged / settled by warps 1.. under warp 0's chains
#endif

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Profiling builds only (-DSL_LARGE_PROF): %globaltimer stamps per phase of
// segment 0, read with sl_large_prof_read: 0 start, 1 walk done, 2 inv fold done,
// 3 min/lens done, 4 vbs(running) done, 5 admission done, 6 end.
#ifdef SL_LARGE_PROF
__device__ unsigned long long sl_large_prof[16];
#define SL_LCLK(v) (v = clock64())
#define SL_LSTAMP(k)                                                      \
  do {                                                                    \
    if (seg == 0 && lane == 0) {                                          \
      unsigned long long t_;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      sl_large_prof[k] = t_;                                              \
    }                                                                     \
  } while (0)
__device__ unsigned long long sl_sort_prof[32];  // sort_cluster_kernel: [0] count, clock64 stamps
__device__ unsigned long long sl_sort_cta[16][4];  // per CTA: globaltimer after scatter / local sort, big, my_n
#define SL_CTASTAMP(k, v)                                                        \
  do {                                                                           \
    if (threadIdx.x == 0 && blockIdx.x < 16) sl_sort_cta[blockIdx.x][k] = (v);   \
  } while (0)
__device__ __forceinline__ unsigned long long sl_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SL_SSTAMP()                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                   \
      const unsigned long long k_ = sl_sort_prof[0] + 1;                         \
      if (k_ < 32) sl_sort_prof[k_] = clock64();                                 \
      sl_sort_prof[0] = k_;                                                      \
    }                                                                            \
  } while (0)
#else
#define SL_CTASTAMP(k, v) do {} while (0)
#define SL_SSTAMP() do {} while (0)
#define SL_LSTAMP(k) do {} while (0)
#define SL_LCLK(v) do {} while (0)
#endif

// A long CPython sum() split over two warps (split_fold_f / split_fold_c):
// slot s of the handover ring holds 32 operands and the running float sum
// before each of them.
struct SplitRing {
  double x[2][32];
  double fb[2][32];
};

struct LargeSmem {
  SplitRing sf[2];     // inv, vbs (16-byte aligned: first)
  double ebuf[2][32];  // c-chain operand broadcast buffers
  double fbuf[32];     // warp 0's fold operand buffer
  // survivors of a tile, in order, and the chain's decisions (1 = rejected); two
  // buffers: the pipelined walk stages tile i+1 while warp 0 chains tile i
  double sv_e[2][kLTile], sv_pf[2][kLTile], sv_tt[2][kLTile];
  uint8_t dec[2][kLTile];
  int32_t m_idx[2][kLTile];   // pipelined walk: each helper item's queue slot and
  int16_t m_code[2][kLTile];  // -2 invalid, -1 rejected outright, else survivor slot
  int n_svb[2];
  double Pb[2];  // the prefix after each chained tile (pipelined walk)
  // parallel first admission round: per 32-item chunk of the kept list, the
  // first item passing against the pre-admission state, the failing items before
  // it (kept waiting / rejected, as lane masks) and their output offsets
  int a_first[kAdmChunks];
  unsigned a_keepm[kAdmChunks], a_rejm[kAdmChunks];
  int a_kofs[kAdmChunks], a_rofs[kAdmChunks];
  double adm_inv;
  int a_cstar, a_nwait, a_nrej;
  int cnt[2][kLChunks];
  int off[2][kLChunks];
  double P;        // walk prefix (exact, sequential)
  double U;        // certified pass: inflated prefix bound
  int all_ok;
  int n_sv, kept, nrej, kbase, rbase;
  // aggregates
  double inv_f, inv_c;  // sum(1/slo) over running: the float sum and its compensation
  double vbs_f, vbs_c;  // vbs over running with min_pre
  // certified folds (dd_certify): the pair's double-double partials, the vbs
  // running part as a double-double for warp 0 and whether it was certified
  double dd_part[2][2][2];  // [inv, vbs][warp of the pair][s, c]
  double vbs_s, vbs_cc;
  int vbs_cert;
  double min_pre;  // min slo over running (+inf if none)
  long long lens;  // sum of current lengths over running
  double red_min[2];
  long long red_len[2];
  // split launch: one-shot mbarriers (expected count 1) in CTA 0, arrived on by
  // the fold CTA after it has stored its results there, waited on by warp 0
  unsigned long long agg_ready, inv_ready, vbs_ready;
};

// Split launch (a cluster of 2 CTAs per segment): the fold warps run in CTA 1 on
// their own SM and publish their results into CTA 0's shared memory, then
// arrive (release, cluster scope) on an mbarrier there; warp 0 of CTA 0 waits
// on it (acquire) where it would otherwise wait on the named barrier.
__device__ __forceinline__ void mbar_init1(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void flag_release(unsigned long long* local_bar_in_cta0) {
  // the mbarrier at the same offset in CTA 0's shared memory
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;"
               : "=r"(remote)
               : "r"((unsigned)__cvta_generic_to_shared(local_bar_in_cta0)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void flag_acquire(unsigned long long* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a)
        : "memory");
  }
}

// exclusive scan of the nch (<= kLChunks) counts of row r (one warp), totals to *tot
__device__ __forceinline__ void chunk_scan(LargeSmem& sm, int r, int lane, int* tot,
                                           int nch = kLChunks) {
  static_assert(kLChunks <= 64, "two chunks per lane");
  const int a = lane < nch ? sm.cnt[r][lane] : 0;
  const int b = lane + 32 < nch ? sm.cnt[r][lane + 32] : 0;
  // chunks 0..31 in lanes, then 32..63
  int x = a;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(SL_FULL, x, o);
    if (lane >= o) x += y;
  }
  const int tot_a = __shfl_sync(SL_FULL, x, 31);
  int z = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(SL_FULL, z, o);
    if (lane >= o) z += y;
  }
  const int tot_b = __shfl_sync(SL_FULL, z, 31);
  if (lane < nch) sm.off[r][lane] = x - a;
  if (lane + 32 < nch) sm.off[r][lane + 32] = tot_a + z - b;
  if (lane == 0) *tot = tot_a + tot_b;
}

// The sequential walk over the survivors [0, n) in shared memory (warp 0):
// dec[i] = 1 for rejected; returns the prefix after them.  Rounds of "first
// item that passes at the current prefix": every item before it fails at this
// prefix -- rejected, the prefix unchanged -- and it is kept, adding its
// prefill.  One round per kept item plus one per 64 rejected items, each a
// lane-parallel test of a 64-item window; exact for any prefill sign.
__device__ __forceinline__ double survivor_chain(LargeSmem& sm, int n, double prefix, int lane,
                                                 int b = 0) {
  // items in reversed lane order (item t of a half in lane 31 - t): the first
  // passing item is the highest set ballot bit (one FLO, no bit reversal)
  const int rl = 31 - lane;
  for (int base = 0; base < n; base += 64) {
    const int j0 = base + rl, j1 = base + 32 + rl;
    const bool v0 = j0 < n, v1 = j1 < n;
    double e0 = 0.0, p0 = 0.0, t0 = 0.0, e1 = 0.0, p1 = 0.0, t1 = 0.0;
    if (v0) {
      e0 = sm.sv_e[b][j0];
      p0 = sm.sv_pf[b][j0];
      t0 = sm.sv_tt[b][j0];
    }
    if (v1) {
      e1 = sm.sv_e[b][j1];
      p1 = sm.sv_pf[b][j1];
      t1 = sm.sv_tt[b][j1];
    }
    // the window stays in registers; each round retires the lanes up to the
    // first one that passes at the current prefix
    bool a0 = v0, a1 = v1, k0 = false, k1 = false;
    for (;;) {
      // every lane also forms the prefix it would leave if kept (prefix + its
      // prefill, the same IEEE add) alongside the tests, so that the next
      // prefix is one shuffle away from the first passing lane
      const double n0 = fadd_(prefix, p0), n1 = fadd_(prefix, p1);
      const unsigned ok0 = __ballot_sync(SL_FULL, a0 && !(fadd_(fadd_(e0, prefix), p0) > t0));
      const unsigned ok1 = __ballot_sync(SL_FULL, a1 && !(fadd_(fadd_(e1, prefix), p1) > t1));
      if (!(ok0 | ok1)) break;  // every remaining item fails at this prefix
      // the first passing item: lane gl of the lower half, else of the upper;
      // the half is chosen before the shuffle (one 64-bit shuffle on the path)
      const bool hi = ok0 == 0;
      const int gl = 31 - __clz(hi ? ok1 : ok0);
      prefix = __shfl_sync(SL_FULL, hi ? n1 : n0, gl);
      k0 |= !hi && lane == gl;
      k1 |= hi && lane == gl;
      a0 &= !hi && lane < gl;  // later items of the lower half: lower lanes
      a1 &= !hi || lane < gl;
    }
    if (v0) sm.dec[b][j0] = !k0;
    if (v1) sm.dec[b][j1] = !k1;
  }
  return prefix;
}

// CPython's sum() over n operands (f += x with Neumaier's
// compensation c), split over two warps so that each serial chain is one DADD
// per operand.  split_fold_f (warp A) computes the operands lane-parallel and
// the float chain f, handing each 32-operand chunk to split_fold_c (warp B)
// with the value of f before every operand; B forms the exact rounding errors
// lane-parallel (the same FastTwoSum as ps_add) and chains c over them in order.
// The pair equals ps_add over the operands bit for bit: the first operand's
// error is exactly 0 (0.0 + x), so c = 0.0 + 0.0 as ps_add leaves it.
// Handover: a 2-slot ring, named barriers full[s] (A arrives, B syncs) and
// empty[s] (B arrives, A syncs): barrier ids bar .. bar + 3.
// The operand of element j is op(src[j]); loads run two chunks ahead and the
// operand one chunk ahead of the chain (global-load and division latency off it).
template <class OP>
__device__ __forceinline__ double split_fold_f(int n, const double* src, OP op, SplitRing& ring,
                                               int bar, int lane) {
  double f = 0.0;
  int k = 0;
  double x = lane < n ? op(src[lane]) : 0.0;
  double raw = 32 + lane < n ? src[32 + lane] : 1.0;
  for (int c0 = 0; c0 < n; c0 += 32, ++k) {
    const int s = k & 1;
    const int cnt = min(32, n - c0);
    const double xn = op(raw);  // next chunk's operand (1.0 past the end: never folded)
    const int jnn = c0 + 64 + lane;
    raw = jnn < n ? src[jnn] : 1.0;
    if (k >= 2) bar_sync(bar + 2 + s, 64);  // B has read chunk k - 2 from slot s
    ring.x[s][lane] = x;
    __syncwarp();
    if (cnt == 32) {
      double v[32];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const double2 p = reinterpret_cast<const double2*>(ring.x[s])[t];
        v[2 * t] = p.x;
        v[2 * t + 1] = p.y;
      }
      // one predicated store per element keeps the chain at ~12 cycles per
      // element (a register array stored after the chain measured ~19)
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if (lane == 0) ring.fb[s][t] = f;
        f = fadd_(f, v[t]);
      }
    } else {
      double mine = 0.0;
      for (int t = 0; t < cnt; ++t) {
        if (lane == t) mine = f;
        f = fadd_(f, ring.x[s][t]);
      }
      ring.fb[s][lane] = mine;
    }
    __syncwarp();
    bar_arrive(bar + s, 64);
    x = xn;
  }
  // balance the empty barriers of the last two chunks
  for (int q = max(0, k - 2); q < k; ++q) bar_sync(bar + 2 + (q & 1), 64);
  return f;
}

__device__ __forceinline__ double split_fold_c(int n, SplitRing& ring, int bar, double* ebuf,
                                               int lane) {
  double c = 0.0;
  int k = 0;
  for (int c0 = 0; c0 < n; c0 += 32, ++k) {
    const int s = k & 1;
    const int cnt = min(32, n - c0);
    bar_sync(bar + s, 64);
    double err = 0.0;
    if (lane < cnt) {
      const double f = ring.fb[s][lane], x = ring.x[s][lane];
      const double t = fadd_(f, x);
      const bool big = fabs(f) >= fabs(x);
      const double hi = big ? f : x, lo = big ? x : f;
      err = fadd_(fsub_(hi, t), lo);  // exact: f + x - t
    }
    __syncwarp();  // (err depends on both loads: the slot is read)
    bar_arrive(bar + 2 + s, 64);
    ebuf[lane] = err;
    __syncwarp();
    if (cnt == 32) {
      double e[32];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const double2 p = reinterpret_cast<const double2*>(ebuf)[t];
        e[2 * t] = p.x;
        e[2 * t + 1] = p.y;
      }
#pragma unroll
      for (int t = 0; t < 32; ++t) c = fadd_(c, e[t]);
    } else {
      for (int t = 0; t < cnt; ++t) c = fadd_(c, ebuf[t]);
    }
    __syncwarp();
  }
  return c;
}

__device__ __forceinline__ double div_int(int64_t a, int64_t b) {
  return b <= 128 ? div_small((double)a, (int)b) : fdiv_((double)a, (double)b);
}

// certified CPython sums (DD, dd_certify): sl_device.cuh

__global__ void __launch_bounds__(kLThreads, 1) guard_admit_cta_kernel(const sl_plan_state st,
                                                                       const sl_plan_config cfg,
                                                                       sl_plan_out out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LargeSmem& sm = *reinterpret_cast<LargeSmem*>(smem_raw);
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  // split: a 2-CTA cluster per segment -- CTA 0 walks and admits, CTA 1 folds
  const bool split = cl.num_blocks() == 2;
  const int crank = split ? (int)cl.block_rank() : 0;
  const int seg = split ? blockIdx.x >> 1 : blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0 && crank == 0) SL_LSTAMP(7);  // kernel entry
  if (split) {
    if (tid == 0) {
      mbar_init1(&sm.agg_ready);
      mbar_init1(&sm.inv_ready);
      mbar_init1(&sm.vbs_ready);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();  // both CTAs started, mbarriers initialised, before any DSMEM access
  }
  LargeSmem* res = split ? cl.map_shared_rank(&sm, 0) : &sm;  // where fold results go
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
  int32_t* kept_list = out.scratch + wb;
  const bool need_inv = !guard_only && tpot_guard && R > 0 && W > 0;
  const bool need_vbs = !guard_only && R > 0;
  if (tid == 0 && crank == 0) SL_LSTAMP(0);

  if (split && crank == 1 && warp < kLW) {
    // CTA 1's spare warps: pull the segment's inputs into L2 (128-byte lines)
    // so that neither the walk's gathers nor the folds' streams wait on HBM
    const int nt = kLW * 32;
    auto pf = [&](const void* base, int64_t bytes) {
      const char* b = static_cast<const char*>(base);
      for (int64_t o = (int64_t)tid * 128; o < bytes; o += (int64_t)nt * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b + o));
    };
    pf(st.r_tpot + rb, 8 * (int64_t)R);
    pf(st.r_cur_len + rb, 4 * (int64_t)R);
    pf(st.w_arrival + wb, 8 * (int64_t)W);
    pf(st.w_prefill + wb, 8 * (int64_t)W);
    pf(st.w_ttft + wb, 8 * (int64_t)W);
    if (ttft_guard) pf(out.perm + wb, 4 * (int64_t)W);
    pf(st.w_tpot + wb, 8 * (int64_t)W);
    pf(st.w_prompt + wb, 4 * (int64_t)W);
    pf(st.w_pred + wb, 4 * (int64_t)W);
    return;
  }
  if (split && (crank == 0) == (warp >= kLW)) return;  // the other CTA's role
  // named-barrier counts: warp 0 takes part in the aggregate / vbs barriers
  // unless it polls CTA 0's flags instead (split)
  const int agg_cnt = 5 * 32, vbs_cnt = split ? 2 * 32 : 3 * 32;
  if (warp >= kLW) {
    // ------------------------------------------------------------ fold warps
    if (guard_only) return;  // warp 0 waits on none of their barriers
    // roles by SMSP (warp % 4); warp 0 (the serial walk) is on SMSP 0:
    //   kLW+0 (SMSP 0) vbs c-chain, kLW+1 inv f-chain, kLW+2 inv c-chain,
    //   kLW+3 vbs f-chain; the vbs pair first reduces min slo / lengths
    static_assert(kLW % 4 == 0 && kLF == 4, "fold warps kLW..kLW+3");
    const int f = warp - kLW;
    const double* tp = st.r_tpot + rb;
    if (f == 1 || f == 2) {  // sum(1.0 / slo) over running, in order (:121)
      bool cert = false;
      if (need_inv && SL_CERT_FOLD) {
        // the certified sum over both warps of the pair first (dd_certify)
        DD a = {0.0, 0.0};
        bool pos = true;
        for (int j = (f - 1) * 32 + lane; j < R; j += 64) {
          const double x = frcp_(tp[j]);
          pos = pos && x > 0.0 && x < 1e300;
          dd_add(a, x);
        }
        pos = __all_sync(SL_FULL, pos);
        a = dd_warp(a);
        if (lane == 0) {
          sm.dd_part[0][f - 1][0] = pos ? a.s : -1.0;
          sm.dd_part[0][f - 1][1] = a.c;
        }
        bar_sync(kBarInvPair, 64);
        const DD a0 = {sm.dd_part[0][0][0], sm.dd_part[0][0][1]};
        const DD a1 = {sm.dd_part[0][1][0], sm.dd_part[0][1][1]};
        double r = 0.0;
        cert = a0.s >= 0.0 && a1.s >= 0.0 && dd_certify(dd_merge(a0, a1), R, &r);
        if (cert && f == 1 && lane == 0) {
          res->inv_f = r;
          res->inv_c = 0.0;
        }
      }
      if (need_inv && !cert) {
        if (f == 1) {
          const double fs = split_fold_f(R, tp, [](double t) { return frcp_(t); }, sm.sf[0],
                                         kBarInvRing, lane);
          if (lane == 0) res->inv_f = fs;
        } else {
          const double cs = split_fold_c(R, sm.sf[0], kBarInvRing, sm.ebuf[0], lane);
          if (lane == 0) res->inv_c = cs;
        }
      }
      if (f == 1) SL_LSTAMP(2);
      if (split) {  // the inv pair alone: the min / lengths warps do not wait for it
        bar_sync(kBarInvPair, 64);
        if (f == 1 && lane == 0) flag_release(&sm.inv_ready);
      } else {
        bar_arrive(kBarAgg, agg_cnt);
      }
      return;
    }
    // vbs pair: min slo and sum of lengths over running
    const int ft = (f == 0 ? 0 : 32) + lane;  // 0..63
    long long lens = 0;
    double mn = kInf;
    for (int j = ft; j < R; j += 64) {
      lens += st.r_cur_len[rb + j];
      mn = fmin(mn, tp[j]);
    }
    lens = warp_sum_i64(lens);
#pragma unroll
    for (int o = 16; o; o >>= 1) mn = fmin(mn, __shfl_xor_sync(SL_FULL, mn, o));
    if (lane == 0) {
      sm.red_min[f == 0] = mn;
      sm.red_len[f == 0] = lens;
    }
    bar_sync(kBarRed, 64);
    const double min_pre = fmin(sm.red_min[0], sm.red_min[1]);
    if (f == 3 && lane == 0) {
      res->min_pre = min_pre;
      res->lens = sm.red_len[0] + sm.red_len[1];
    }
    if (f == 3) SL_LSTAMP(3);
    if (split) {
      if (f == 3 && lane == 0) flag_release(&sm.agg_ready);  // min / lengths
    } else {
      bar_arrive(kBarAgg, agg_cnt);
    }
    bool vcert = false;
    if (need_vbs && SL_CERT_FOLD) {
      // certified sum of min_pre / slo over running (the pair's 64 lanes); warp 0
      // extends the double-double with the admitted entries and certifies the total
      DD a = {0.0, 0.0};
      bool pos = true;
      for (int j = ft; j < R; j += 64) {
        const double x = fdiv_(min_pre, tp[j]);
        pos = pos && x > 0.0 && x < 1e300;
        dd_add(a, x);
      }
      pos = __all_sync(SL_FULL, pos);
      a = dd_warp(a);
      if (lane == 0) {
        sm.dd_part[1][f == 0][0] = pos ? a.s : -1.0;
        sm.dd_part[1][f == 0][1] = a.c;
      }
      bar_sync(kBarRed, 64);
      const DD a0 = {sm.dd_part[1][0][0], sm.dd_part[1][0][1]};
      const DD a1 = {sm.dd_part[1][1][0], sm.dd_part[1][1][1]};
      const DD t = dd_merge(a0, a1);
      double r = 0.0;
      vcert = a0.s >= 0.0 && a1.s >= 0.0 && dd_certify(t, R, &r);
      if (f == 3 && lane == 0) {
        res->vbs_s = t.s;
        res->vbs_cc = t.c;
        res->vbs_cert = vcert;
      }
    } else if (f == 3 && lane == 0) {
      res->vbs_cert = 0;
    }
    if (need_vbs) {  // vbs over running with the pre-admission minimum (:312-315)
      if (vcert) {
        // certified above
      } else if (f == 3) {
        const double fs = split_fold_f(R, tp, [&](double t) { return fdiv_(min_pre, t); },
                                       sm.sf[1], kBarVbsRing, lane);
        if (lane == 0) res->vbs_f = fs;
      } else {
        const double cs = split_fold_c(R, sm.sf[1], kBarVbsRing, sm.ebuf[1], lane);
        if (lane == 0) res->vbs_c = cs;
      }
      if (f == 3) SL_LSTAMP(4);
      if (split) {
        bar_sync(kBarVbs, vbs_cnt);
        if (f == 3 && lane == 0) flag_release(&sm.vbs_ready);
      } else {
        bar_arrive(kBarVbs, vbs_cnt);  // warp 0 waits on it iff R > 0
      }
    }
    return;
  }

  // -------------------------------------------------------------- walk warps
  if (tid == 0) {
    sm.P = 0.0;
    sm.U = 0.0;
    sm.all_ok = 1;
    sm.kept = 0;
    sm.nrej = 0;
  }
  bar_sync(kBarWalk, kLWalkThreads);
  auto qidx = [&](int p) -> int32_t {
    return ttft_guard ? out.perm[wb + p] : (int32_t)(wb + p);
  };
  // certified pass over the whole queue (see seg_guard_admit): an inflated
  // any-order prefix bound U_j >= the sequential prefix; if every item passes
  // against it, the walk keeps everything in order.
  bool certified = !walk;
  if (walk && !exact && W < (1 << 20)) {
    const double inflate = 1.0 + 9.313225746154785e-10;  // 1 + 2^-30
    for (int t0 = 0; t0 < W; t0 += kLTile) {
      const double U = sm.U;
      double e[kLK], pf[kLK], tt[kLK], v[kLK];
      bool ok = true;
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        const int p = t0 + k * kLWalkThreads + tid;
        e[k] = pf[k] = tt[k] = 0.0;
        if (p < W) {
          const int32_t idx = qidx(p);
          e[k] = fsub_(now, st.w_arrival[idx]);
          pf[k] = st.w_prefill[idx];
          tt[k] = st.w_ttft[idx];
        }
        v[k] = pf[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(SL_FULL, v[k], o);
          if (lane >= o) v[k] = fadd_(v[k], y);
        }
      }
      // chunk totals -> chunk offsets (any order, inflated below); reuse off[] as doubles
      double* ctot = reinterpret_cast<double*>(sm.sv_e[0]);
#pragma unroll
      for (int k = 0; k < kLK; ++k)
        if (lane == 31) ctot[k * kLW + warp] = v[k];
      bar_sync(kBarWalk, kLWalkThreads);
      if (warp == 0) {
        double c = 0.0;
        for (int q = 0; q < kLChunks; ++q) {  // serial, tiny
          const double x = ctot[q];
          if (lane == 0) ctot[kLChunks + q] = c;
          c = fadd_(c, x);
        }
        if (lane == 0) ctot[2 * kLChunks] = c;
      }
      bar_sync(kBarWalk, kLWalkThreads);
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        const int p = t0 + k * kLWalkThreads + tid;
        double excl = __shfl_up_sync(SL_FULL, v[k], 1);
        if (lane == 0) excl = 0.0;
        const double Uj = fmul_(fadd_(fmul_(fadd_(U, ctot[kLChunks + k * kLW + warp]), inflate),
                                      excl), inflate);
        if (p < W && fadd_(fadd_(e[k], Uj), pf[k]) > tt[k]) ok = false;
      }
      const double tile_tot = ctot[2 * kLChunks];
      if (!__all_sync(SL_FULL, ok)) sm.all_ok = 0;  // benign race: every writer stores 0
      bar_sync(kBarWalk, kLWalkThreads);
      if (!sm.all_ok) break;
      if (tid == 0) sm.U = fmul_(fmul_(fadd_(U, tile_tot), inflate), inflate);
      bar_sync(kBarWalk, kLWalkThreads);
    }
    certified = sm.all_ok != 0;
  }
#ifdef SL_LARGE_PROF
  long long pc[6] = {0, 0, 0, 0, 0, 0}, pt0 = 0, pt1 = 0;
  long long n_sv_tot = 0;
#endif
  if (certified) {
    for (int p = tid; p < W; p += kLWalkThreads) kept_list[p] = qidx(p);
    if (tid == 0) sm.kept = W;
  } else if (SL_WALK_PIPE) {
    // Pipelined walk: warp 0 runs the exact chains tile after tile; warps 1..11
    // ("helpers") stage tile i+1 (loads, the outright filter at a lower bound of
    // its incoming prefix -- the prefix after tile i-1 --, survivor compaction)
    // and settle tile i-1 (kept list, rejections) while warp 0 chains tile i.
    // The outright filter only shortens the chain: an item failing at a lower
    // bound of its prefix fails at the prefix, and the chain rejects the same
    // items either way, so the decisions and their order do not depend on the
    // bound used.
#if SL_PIPE_SOLO
    // warp 0's SMSP (warps 0, 4, 8) runs the chain alone: warps 4 and 8 sit out
    constexpr int kPH = kLW - kLW / 4;
#else
    constexpr int kPH = kLW - 1;
#endif
    constexpr int kPHT = kPH * 32, kPTile = kPHT * kLK, kPCh = kLK * kPH;
    static_assert(kPTile <= kLTile && kPCh <= kLChunks, "pipelined tile fits the buffers");
    const int ntiles = (W + kPTile - 1) / kPTile;
    if (SL_PIPE_SOLO && warp != 0 && (warp & 3) == 0) {
      // idle: the walk's closing barrier below
    } else if (warp == 0) {
      double P = 0.0;
      for (int i = 0; i < ntiles; ++i) {
        bar_sync(kBarPipe, 32 + kPHT);  // tile i staged; tile i-1's chain published
        const int b = i & 1;
        P = survivor_chain(sm, sm.n_svb[b], P, lane, b);
        if (lane == 0) sm.Pb[b] = P;
        __syncwarp();
      }
      bar_sync(kBarPipe, 32 + kPHT);  // the last chain's decisions are in
      if (lane == 0) sm.P = P;
    } else {
      const int hw = SL_PIPE_SOLO ? warp - 1 - (warp >> 2) : warp - 1, h = hw * 32 + lane;
      auto slot_of = [&](int p) -> int32_t { return p < W ? qidx(p) : -1; };
      int32_t idx_n[kLK], idx_nn[kLK];
      double ar_n[kLK], pf_n[kLK], tt_n[kLK];
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        idx_n[k] = slot_of(k * kPHT + h);
        idx_nn[k] = slot_of(kPTile + k * kPHT + h);
        ar_n[k] = pf_n[k] = tt_n[k] = 0.0;
        if (idx_n[k] >= 0) {
          ar_n[k] = st.w_arrival[idx_n[k]];
          pf_n[k] = st.w_prefill[idx_n[k]];
          tt_n[k] = st.w_ttft[idx_n[k]];
        }
      }
      // stage tile t into buffer t & 1 with outright-filter prefix P0
      auto stage = [&](int t, double P0) {
        const int b = t & 1, t0 = t * kPTile;
        double e[kLK], pf[kLK], tt[kLK];
        int32_t idx[kLK];
        bool valid[kLK], sv[kLK];
        int slot[kLK];
#pragma unroll
        for (int k = 0; k < kLK; ++k) {
          const int p = t0 + k * kPHT + h;
          valid[k] = p < W;
          e[k] = valid[k] ? fsub_(now, ar_n[k]) : 0.0;
          pf[k] = valid[k] ? pf_n[k] : 0.0;
          tt[k] = valid[k] ? tt_n[k] : 0.0;
          idx[k] = valid[k] ? idx_n[k] : 0;
          idx_n[k] = idx_nn[k];
          idx_nn[k] = slot_of(t0 + 2 * kPTile + k * kPHT + h);
          if (idx_n[k] >= 0) {
            ar_n[k] = st.w_arrival[idx_n[k]];
            pf_n[k] = st.w_prefill[idx_n[k]];
            tt_n[k] = st.w_ttft[idx_n[k]];
          }
          const bool rej0 = valid[k] && !exact && fadd_(fadd_(e[k], P0), pf[k]) > tt[k];
          sv[k] = valid[k] && !rej0;
          const unsigned m = __ballot_sync(SL_FULL, sv[k]);
          slot[k] = __popc(m & lanemask_lt());
          if (lane == 0) sm.cnt[0][k * kPH + hw] = __popc(m);
          sm.m_idx[b][k * kPHT + h] = idx[k];
          sm.m_code[b][k * kPHT + h] = (int16_t)(valid[k] ? (rej0 ? -1 : 0) : -2);
        }
        bar_sync(kBarHelp, kPHT);
        if (hw == 0) chunk_scan(sm, 0, lane, &sm.n_svb[b], kPCh);
        bar_sync(kBarHelp, kPHT);
#pragma unroll
        for (int k = 0; k < kLK; ++k) {
          if (sv[k]) {
            const int q = slot[k] + sm.off[0][k * kPH + hw];
            sm.sv_e[b][q] = e[k];
            sm.sv_pf[b][q] = pf[k];
            sm.sv_tt[b][q] = tt[k];
            sm.m_code[b][k * kPHT + h] = (int16_t)q;
          }
        }
      };
      // settle tile t (its chain's decisions are in buffer t & 1)
      auto settle = [&](int t) {
        const int b = t & 1;
        bool keep[kLK], rj[kLK];
        int kr[kLK], rr[kLK];
        int32_t idx[kLK];
#pragma unroll
        for (int k = 0; k < kLK; ++k) {
          const int c = sm.m_code[b][k * kPHT + h];
          idx[k] = sm.m_idx[b][k * kPHT + h];
          rj[k] = c == -1 || (c >= 0 && sm.dec[b][c]);
          keep[k] = c != -2 && !rj[k];
          const unsigned mk = __ballot_sync(SL_FULL, keep[k]);
          const unsigned mr = __ballot_sync(SL_FULL, rj[k]);
          kr[k] = __popc(mk & lanemask_lt());
          rr[k] = __popc(mr & lanemask_lt());
          if (lane == 0) {
            sm.cnt[0][k * kPH + hw] = __popc(mk);
            sm.cnt[1][k * kPH + hw] = __popc(mr);
          }
        }
        bar_sync(kBarHelp, kPHT);
        if (hw == 0) {
          int tk, tr;
          chunk_scan(sm, 0, lane, &tk, kPCh);
          chunk_scan(sm, 1, lane, &tr, kPCh);
          if (lane == 0) {
            sm.kbase = sm.kept;
            sm.rbase = sm.nrej;
            sm.kept += tk;
            sm.nrej += tr;
          }
        }
        bar_sync(kBarHelp, kPHT);
        const int kbase = sm.kbase, rbase = sm.rbase;
#pragma unroll
        for (int k = 0; k < kLK; ++k) {
          if (keep[k]) kept_list[kbase + sm.off[0][k * kPH + hw] + kr[k]] = idx[k];
          if (rj[k]) {
            out.w_status[idx[k]] = SL_PLAN_REJECTED_TTFT;
            out.w_pos[idx[k]] = rbase + sm.off[1][k * kPH + hw] + rr[k];
          }
        }
        bar_sync(kBarHelp, kPHT);  // off / kbase are reused by the next stage / settle
      };
      if (ntiles > 0) stage(0, 0.0);
      for (int i = 0; i < ntiles; ++i) {
        bar_sync(kBarPipe, 32 + kPHT);  // tile i staged; tile i-1's chain published
        if (i >= 1) settle(i - 1);
        // tile i+1's outright filter at the prefix after tile i-1 (<= its own)
        if (i + 1 < ntiles) stage(i + 1, i >= 1 ? sm.Pb[(i - 1) & 1] : 0.0);
      }
      bar_sync(kBarPipe, 32 + kPHT);  // the last chain's decisions are in
      if (ntiles > 0) settle(ntiles - 1);
    }
  } else {
    // software pipelined over tiles: the next tile's fields and the queue slots
    // of the tile after it are requested before this tile's chain (each tile's
    // gathers are two dependent round trips)
    auto slot_of = [&](int p) -> int32_t { return p < W ? qidx(p) : -1; };
    int32_t idx_n[kLK], idx_nn[kLK];
    double ar_n[kLK], pf_n[kLK], tt_n[kLK];
#pragma unroll
    for (int k = 0; k < kLK; ++k) {
      idx_n[k] = slot_of(k * kLWalkThreads + tid);
      idx_nn[k] = slot_of(kLTile + k * kLWalkThreads + tid);
      ar_n[k] = pf_n[k] = tt_n[k] = 0.0;
      if (idx_n[k] >= 0) {
        ar_n[k] = st.w_arrival[idx_n[k]];
        pf_n[k] = st.w_prefill[idx_n[k]];
        tt_n[k] = st.w_ttft[idx_n[k]];
      }
    }
    for (int t0 = 0; t0 < W; t0 += kLTile) {
      SL_LCLK(pt0);
      const double P0 = sm.P;
      double e[kLK], pf[kLK], tt[kLK];
      int32_t idx[kLK];
      bool valid[kLK], rej0[kLK], sv[kLK];
      int slot[kLK];
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        const int p = t0 + k * kLWalkThreads + tid;
        valid[k] = p < W;
        e[k] = valid[k] ? fsub_(now, ar_n[k]) : 0.0;
        pf[k] = valid[k] ? pf_n[k] : 0.0;
        tt[k] = valid[k] ? tt_n[k] : 0.0;
        idx[k] = valid[k] ? idx_n[k] : 0;
        idx_n[k] = idx_nn[k];
        idx_nn[k] = slot_of(t0 + 2 * kLTile + k * kLWalkThreads + tid);
        if (idx_n[k] >= 0) {
          ar_n[k] = st.w_arrival[idx_n[k]];
          pf_n[k] = st.w_prefill[idx_n[k]];
          tt_n[k] = st.w_ttft[idx_n[k]];
        }
        // fails at the tile's incoming prefix -> fails at every later one
        rej0[k] = valid[k] && !exact && fadd_(fadd_(e[k], P0), pf[k]) > tt[k];
        sv[k] = valid[k] && !rej0[k];
        const unsigned m = __ballot_sync(SL_FULL, sv[k]);
        slot[k] = __popc(m & lanemask_lt());
        if (lane == 0) sm.cnt[0][k * kLW + warp] = __popc(m);
      }
      bar_sync(kBarWalk, kLWalkThreads);
#ifdef SL_LARGE_PROF
      SL_LCLK(pt1); pc[0] += pt1 - pt0; pt0 = pt1;
#endif
      if (warp == 0) chunk_scan(sm, 0, lane, &sm.n_sv);
      bar_sync(kBarWalk, kLWalkThreads);
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        if (sv[k]) {
          slot[k] += sm.off[0][k * kLW + warp];
          sm.sv_e[0][slot[k]] = e[k];
          sm.sv_pf[0][slot[k]] = pf[k];
          sm.sv_tt[0][slot[k]] = tt[k];
        }
      }
      bar_sync(kBarWalk, kLWalkThreads);
#ifdef SL_LARGE_PROF
      SL_LCLK(pt1); pc[1] += pt1 - pt0; pt0 = pt1; n_sv_tot += sm.n_sv;
#endif
      if (warp == 0) {
        const double P1 = survivor_chain(sm, sm.n_sv, P0, lane);
        if (lane == 0) sm.P = P1;
      } else {
        // while warp 0 runs the chain: pull the next tile's inputs into L2 (the
        // walk order gathers them through perm, two dependent round trips cold)
        for (int p = t0 + kLTile + tid - 32; p < min(W, t0 + 2 * kLTile); p += kLWalkThreads - 32) {
          const int32_t q = qidx(p);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(st.w_arrival + q));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(st.w_prefill + q));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(st.w_ttft + q));
        }
      }
      bar_sync(kBarWalk, kLWalkThreads);
#ifdef SL_LARGE_PROF
      SL_LCLK(pt1); pc[2] += pt1 - pt0; pt0 = pt1;
#endif
      bool keep[kLK], rj[kLK];
      int kr[kLK], rr[kLK];
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        rj[k] = rej0[k] || (sv[k] && sm.dec[0][slot[k]]);
        keep[k] = valid[k] && !rj[k];
        const unsigned mk = __ballot_sync(SL_FULL, keep[k]);
        const unsigned mr = __ballot_sync(SL_FULL, rj[k]);
        kr[k] = __popc(mk & lanemask_lt());
        rr[k] = __popc(mr & lanemask_lt());
        if (lane == 0) {
          sm.cnt[0][k * kLW + warp] = __popc(mk);
          sm.cnt[1][k * kLW + warp] = __popc(mr);
        }
      }
      bar_sync(kBarWalk, kLWalkThreads);
      if (warp == 0) {
        int tk, tr;
        chunk_scan(sm, 0, lane, &tk);
        chunk_scan(sm, 1, lane, &tr);
        if (lane == 0) {
          sm.kbase = sm.kept;
          sm.rbase = sm.nrej;
          sm.kept += tk;
          sm.nrej += tr;
        }
      }
      bar_sync(kBarWalk, kLWalkThreads);
      const int kbase = sm.kbase, rbase = sm.rbase;
#pragma unroll
      for (int k = 0; k < kLK; ++k) {
        if (keep[k]) kept_list[kbase + sm.off[0][k * kLW + warp] + kr[k]] = idx[k];
        if (rj[k]) {
          out.w_status[idx[k]] = SL_PLAN_REJECTED_TTFT;
          out.w_pos[idx[k]] = rbase + sm.off[1][k * kLW + warp] + rr[k];
        }
      }
      bar_sync(kBarWalk, kLWalkThreads);
#ifdef SL_LARGE_PROF
      SL_LCLK(pt1); pc[3] += pt1 - pt0; pt0 = pt1;
#endif
    }
  }
#ifdef SL_LARGE_PROF
  if (seg == 0 && tid == 0) {
    for (int q = 0; q < 4; ++q) sl_large_prof[8 + q] = pc[q];
    sl_large_prof[12] = n_sv_tot;
  }
#endif
  bar_sync(kBarWalk, kLWalkThreads);
  const int kept = sm.kept;
  int nrej = sm.nrej;
  if (warp == 0) SL_LSTAMP(1);
  if (guard_only) {
    for (int p = tid; p < kept; p += kLWalkThreads) {
      out.w_status[kept_list[p]] = SL_PLAN_WAITING;
      out.w_pos[kept_list[p]] = p;
    }
    if (tid == 0) {
      out.seg_counts[4 * seg + 0] = kept;
      out.seg_counts[4 * seg + 1] = 0;
      out.seg_counts[4 * seg + 2] = nrej;
    }
    return;
  }
  // Parallel first admission round (all walk warps): until the first admission
  // the state is the pre-admission one, so every chunk of the kept list is
  // tested against it at once; the failing items before the first passing one
  // (all of them if none passes) are settled here in queue order -- kept waiting
  // if feasible alone, else rejected (:279-291) -- and warp 0 runs the serial
  // rounds from the first passing item on.
  const int nch = (kept + 31) / 32;
  const bool apar = SL_ADM_PAR && tpot_guard && nch > 1 && nch <= kAdmChunks;
  int c_start = 0, f_start = 0, nwait0 = 0, nrej_add = 0;
  if (apar) {
    if (warp == 0) {
      if (split) {
        flag_acquire(&sm.agg_ready);
        flag_acquire(&sm.inv_ready);
      } else {
        bar_sync(kBarAgg, agg_cnt);
      }
      if (lane == 0) sm.adm_inv = need_inv ? ps_result(PySum{sm.inv_f, sm.inv_c, 1}) : 0.0;
    }
    bar_sync(kBarWalk, kLWalkThreads);
    {
      const double inv = sm.adm_inv, min_d = sm.min_pre;
      const int64_t lens = sm.lens;
      const bool has_min = R > 0;
      for (int c = warp; c < nch; c += kLW) {
        const int p = 32 * c + lane;
        const bool valid = p < kept;
        int32_t ln = 0, pred = 0;
        double tp = 1.0, ic = 0.0;
        if (valid) {
          const int32_t idx = kept_list[p];
          tp = st.w_tpot[idx];
          ln = st.w_prompt[idx];
          pred = st.w_pred[idx];
          ic = frcp_(tp);
        }
        const bool solo = solo_ok(C, tp, ic, ln, pred);
        const bool lt = !has_min || tp < min_d;
        const double minp = lt ? tp : min_d;
        const double V = fmul_(minp, fadd_(inv, ic));
        const double L = div_int(lens + ln, (int64_t)R + 1);
        const double est = tpot_estimate(C, V, L, pred);
        const double thr = (r_only && has_min) ? min_d : minp;
        const unsigned okm = __ballot_sync(SL_FULL, valid && est <= thr);
        const int f = okm ? __ffs(okm) - 1 : 32;
        const unsigned failm = __ballot_sync(SL_FULL, valid && lane < f);
        const unsigned keepm = __ballot_sync(SL_FULL, valid && lane < f && solo);
        if (lane == 0) {
          sm.a_first[c] = f;
          sm.a_keepm[c] = keepm;
          sm.a_rejm[c] = failm & ~keepm;
        }
      }
    }
    bar_sync(kBarWalk, kLWalkThreads);
    if (warp == 0) {  // the first chunk with a passing item; offsets of the settled part
      int cstar = nch, kacc = 0, racc = 0;
      for (int c0 = 0; c0 < nch && cstar == nch; c0 += 32) {
        const int c = c0 + lane;
        const bool v = c < nch;
        const unsigned pm = __ballot_sync(SL_FULL, v && sm.a_first[c] < 32);
        const int last = pm ? __ffs(pm) - 1 : 31;  // chunks c0 .. c0 + last settle (partly)
        const bool in = v && lane <= last;
        const int kc = in ? __popc(sm.a_keepm[c]) : 0, rc = in ? __popc(sm.a_rejm[c]) : 0;
        int ks = kc, rs = rc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(SL_FULL, ks, o), z = __shfl_up_sync(SL_FULL, rs, o);
          if (lane >= o) {
            ks += y;
            rs += z;
          }
        }
        if (in) {
          sm.a_kofs[c] = kacc + ks - kc;
          sm.a_rofs[c] = racc + rs - rc;
        }
        kacc += __shfl_sync(SL_FULL, ks, 31);
        racc += __shfl_sync(SL_FULL, rs, 31);
        if (pm) cstar = c0 + __ffs(pm) - 1;
      }
      if (lane == 0) {
        sm.a_cstar = cstar;
        sm.a_nwait = kacc;
        sm.a_nrej = racc;
      }
    }
    bar_sync(kBarWalk, kLWalkThreads);
    const int cstar = sm.a_cstar;
    for (int c = warp; c <= min(cstar, nch - 1); c += kLW) {
      const unsigned km = sm.a_keepm[c], rm = sm.a_rejm[c];
      if (((km | rm) >> lane) & 1u) {
        const int32_t idx = kept_list[32 * c + lane];
        if ((km >> lane) & 1u) {
          out.w_status[idx] = SL_PLAN_WAITING;
          out.w_pos[idx] = sm.a_kofs[c] + __popc(km & lanemask_lt());
        } else {
          out.w_status[idx] = SL_PLAN_REJECTED_ADMISSION;
          out.w_pos[idx] = nrej + sm.a_rofs[c] + __popc(rm & lanemask_lt());
        }
      }
    }
    c_start = cstar;
    f_start = cstar < nch ? sm.a_first[cstar] : 0;
    nwait0 = sm.a_nwait;
    nrej_add = sm.a_nrej;
  }
  if (warp != 0) return;

  // ---------------------------------------------------- admission (warp 0)
  if (!apar) {
    if (split) {
      flag_acquire(&sm.agg_ready);
      flag_acquire(&sm.inv_ready);
    } else {
      bar_sync(kBarAgg, agg_cnt);
    }
  }
  int64_t lens = sm.lens;
  double min_d = sm.min_pre;
  const double min_pre = min_d;
  bool has_min = R > 0;
  int nadm = 0, nwait = nwait0;
  nrej += nrej_add;
  int32_t* adm = out.adm_order + wb;
  if (tpot_guard) {
    double inv = 0.0;
    if (need_inv) {  // ps_result of the split fold (R > 0 operands)
      const PySum ps = {sm.inv_f, sm.inv_c, 1};
      inv = ps_result(ps);
    }
    int64_t n_run = R;
    // software pipelined over chunks: the next chunk's fields and the slot
    // after it are requested before this chunk's rounds (the kept list and the
    // fields are dependent global round trips)
    auto kslot = [&](int p) -> int32_t { return p < kept ? kept_list[p] : -1; };
    const int cb = 32 * c_start;  // chunks before c_start were settled in parallel
    int32_t idx_n = kslot(cb + lane), idx_nn = kslot(cb + 32 + lane);
    double tp_n = 1.0;
    int32_t ln_n = 0, pd_n = 0;
    if (idx_n >= 0) {
      tp_n = st.w_tpot[idx_n];
      ln_n = st.w_prompt[idx_n];
      pd_n = st.w_pred[idx_n];
    }
    for (int c0 = cb; c0 < kept; c0 += 32) {
      const int p = c0 + lane;
      const bool valid = p < kept;
      const int32_t idx = valid ? idx_n : 0;
      const int32_t ln = valid ? ln_n : 0, pred = valid ? pd_n : 0;
      const double tp = valid ? tp_n : 1.0;
      const double ic = valid ? frcp_(tp) : 0.0;
      idx_n = idx_nn;
      idx_nn = kslot(c0 + 64 + lane);
      if (idx_n >= 0) {
        tp_n = st.w_tpot[idx_n];
        ln_n = st.w_prompt[idx_n];
        pd_n = st.w_pred[idx_n];
      }
      const bool solo = solo_ok(C, tp, ic, ln, pred);  // feasible alone (:279-289)
      // (the first chunk's items before f_start were settled in parallel)
      const unsigned vmask =
          __ballot_sync(SL_FULL, valid) & (c0 == cb ? ~((1u << f_start) - 1u) : ~0u);
      unsigned pend = vmask, admm = 0;
      // one round per admission: every pending candidate against the same state
      while (pend) {
        const bool lt = !has_min || tp < min_d;
        const double minp = lt ? tp : min_d;
        const double V = fmul_(minp, fadd_(inv, ic));
        const double L = div_int(lens + ln, n_run + 1);
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
        pend &= ~((2u << g) - 1u);  // lanes before g failed against this state; g admitted
        const double tp_g = bcast(tp, g);
        n_run += 1;
        inv = fadd_(inv, bcast(ic, g));  // :275
        lens += bcast(ln, g);
        if (!has_min || tp_g < min_d) min_d = tp_g;
        has_min = true;
      }
      // bookkeeping once per chunk: admitted in lane order, the rest failed
      const unsigned fail = vmask & ~admm;
      const unsigned keepm = __ballot_sync(SL_FULL, ((fail >> lane) & 1u) && solo);
      const unsigned rejm = fail & ~keepm;
      if ((admm >> lane) & 1u) {
        const int q = nadm + __popc(admm & lanemask_lt());
        out.w_status[idx] = SL_PLAN_ADMITTED;
        out.w_pos[idx] = q;
        adm[q] = idx;
      } else if ((keepm >> lane) & 1u) {
        out.w_status[idx] = SL_PLAN_WAITING;
        out.w_pos[idx] = nwait + __popc(keepm & lanemask_lt());
      } else if ((rejm >> lane) & 1u) {
        out.w_status[idx] = SL_PLAN_REJECTED_ADMISSION;
        out.w_pos[idx] = nrej + __popc(rejm & lanemask_lt());
      }
      nadm += __popc(admm);
      nwait += __popc(keepm);
      nrej += __popc(rejm);
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
  SL_LSTAMP(5);

  // plan.min_slo / plan.vbs over running + admitted, in order (:312-315)
  double vbs = 0.0;
  if (has_min) {
    PySum vs;
    int j0 = 0;  // first entry (running then admitted) still to fold
    if (R > 0) {
      if (split)
        flag_acquire(&sm.vbs_ready);
      else
        bar_sync(kBarVbs, vbs_cnt);
    }
    const int tot = R + nadm;
    auto slo = [&](int j) {
      return j < tot ? (j < R ? st.r_tpot[rb + j] : st.w_tpot[adm[j - R]]) : 1.0;
    };
    bool done = false;
    if (R > 0 && min_d == min_pre && sm.vbs_cert) {
      // the running part as a certified double-double: add the admitted terms
      // and certify the total (dd_certify), else the sequential fold below
      DD a = {0.0, 0.0};
      bool pos = true;
      for (int j = R + lane; j < tot; j += 32) {
        const double x = fdiv_(min_d, slo(j));
        pos = pos && x > 0.0 && x < 1e300;
        dd_add(a, x);
      }
      pos = __all_sync(SL_FULL, pos);
      a = dd_warp(a);
      const DD run = {sm.vbs_s, sm.vbs_cc};
      done = pos && dd_certify(dd_merge(run, a), tot, &vbs);
    }
    if (done) {
      j0 = tot;
      ps_init(vs);
    } else if (R > 0 && min_d == min_pre && !sm.vbs_cert) {
      vs = {sm.vbs_f, sm.vbs_c, 1};  // the vbs pair folded the running part with this minimum
      j0 = R;
    } else {
      ps_init(vs);
    }
    double t_n = slo(j0 + lane);
    for (int c0 = j0; c0 < tot; c0 += 32) {
      const double x = fdiv_(min_d, t_n);
      t_n = slo(c0 + 32 + lane);
      ps_add_warp_smem(vs, x, min(32, tot - c0), sm.fbuf);
    }
    if (!done) vbs = ps_result(vs);
  }
  if (lane == 0) {
    out.seg_counts[4 * seg + 0] = nwait;
    out.seg_counts[4 * seg + 1] = nadm;
    out.seg_counts[4 * seg + 2] = nrej;
    out.seg_vbs[seg] = vbs;
    out.seg_min_slo[seg] = has_min ? min_d : __longlong_as_double(0x7ff8000000000000LL);
    out.seg_min_fixed[seg] = has_min ? slo_fixed<false>(min_d, E) : ~0ull;
  }
  SL_LSTAMP(6);
}

}  // namespace

#ifdef SL_LARGE_PROF
extern "C" int sl_sort_prof_read(unsigned long long* out) {  // and reset; out[32..95]: per CTA
  static const unsigned long long z[32] = {0};
  if (cudaMemcpyFromSymbol(out + 32, sl_sort_cta, sizeof(unsigned long long) * 64) != cudaSuccess)
    return SL_ERR_CUDA;
  if (cudaMemcpyFromSymbol(out, sl_sort_prof, sizeof(z)) != cudaSuccess) return SL_ERR_CUDA;
  return cudaMemcpyToSymbol(sl_sort_prof, z, sizeof(z)) == cudaSuccess ? 0 : SL_ERR_CUDA;
}
extern "C" int sl_large_prof_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, sl_large_prof, sizeof(unsigned long long) * 16) == cudaSuccess
             ? 0
             : SL_ERR_CUDA;
}
#endif

// ---- LDF sort of few, large segments (<= 32,768 waiting each): one thread-block
// cluster per segment (up to 16 CTAs of 2,048 input items, 1,024 threads each),
// radix sorting with 8-bit digits.
//  Key: the deadline's bit pattern (deadlines are positive doubles, which order
//  like their bits) with its low 15 bits replaced by the item's position; only
//  bits 15..63 are sorted on (the input is in position order and every pass is
//  stable), and only the bits in which some key differs from the first.
//  1. MSD distribution: every CTA ranks its keys on the top varying digit, the
//     CTAs' digit histograms are pushed into each other's shared memory
//     (distributed shared memory stores, one cluster barrier), and each key is
//     stored straight into the CTA that owns its digit bucket -- CTA c owns the
//     buckets that start in [2048 c, 2048 (c + 1)), so it holds a contiguous
//     range of final positions (<= 4,096 keys; one more barrier).
//  2. Each CTA LSD-sorts its range in shared memory (CTA barriers only).
//  3. Adjacent sorted keys with equal top 49 bits (equal or near-equal
//     deadlines) -- always inside one CTA's range, as equal deadline bits give
//     equal buckets -- make that CTA re-sort its range by id, then arrival,
//     then deadline (order-preserving 64-bit images, stable passes), i.e. by the
//     full sort key (deadline, arrival, id) and then position -- the stable
//     order of list.sort (sched_scorpio.py:193).  A bucket distribution that
//     would overflow a CTA falls back to cluster-wide LSD passes on the packed
//     keys, with a cluster-wide tie check and exact passes.
//  Exact for every input.
namespace {

constexpr int kSortLoc = 2048;       // input items per CTA
constexpr int kSortCap = 4096;       // items a CTA can own after the MSD distribution
constexpr int kBucketMax = 64;       // largest local bucket placed by counting
constexpr int kLocalBins = 2048;     // local buckets per CTA
constexpr int kSortMaxCluster = 16;  // non-portable cluster size (B200 allows 16)
constexpr int kSortCtaThreads = 1024;
constexpr int kSortWarps = kSortCtaThreads / 32;
constexpr int kPosBits = 15;         // positions < 32,768
constexpr uint64_t kPosMask = (1ull << kPosBits) - 1;

struct RadixSmem {
  uint64_t buf[2][kSortCap];           // items, double-buffered (DSMEM scatter target)
  uint32_t cnt[257 * kSortWarps];      // per (digit, warp): count, then CTA-local offset
  uint32_t hall[kSortMaxCluster][256];  // every CTA's digit totals (pushed by each CTA)
  uint32_t gbase[256];
  int32_t owner[256];                  // MSD: owning CTA of each digit bucket
  int32_t bidx[256];                   // MSD: index among this CTA's non-empty buckets
  int32_t nmine;
  int32_t start[kSortMaxCluster + 1];  // MSD: first final position owned by each CTA
  uint32_t wsum[kSortWarps];
  unsigned long long vall[kSortMaxCluster];  // every CTA's flag word (pushed)
  unsigned long long vmin[kSortMaxCluster], vmax[kSortMaxCluster];    // key range exchange
  uint32_t lh[kLocalBins];             // bucket counts, then offsets (MSD: 256, local: 2048)
  unsigned long long bmin[256], bmax[256];  // local: each owned bucket's key range
  double bscale[256];
  unsigned long long vary, kmin, kmax;
};

// Cluster-wide minimum and maximum of the valid items (pushed into every CTA,
// one cluster barrier).
template <int NS>
__device__ __forceinline__ void cluster_minmax(RadixSmem& sm, const uint64_t (&v)[NS],
                                               const bool (&ok)[NS], uint64_t& gmin,
                                               uint64_t& gmax) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  __syncthreads();  // every thread has read the sample's kmin / kmax (range) before
  if (threadIdx.x == 0) {
    sm.kmin = ~0ull;
    sm.kmax = 0;
  }
  __syncthreads();
  uint64_t mn = ~0ull, mx = 0;
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (ok[x]) {
      mn = min(mn, v[x]);
      mx = max(mx, v[x]);
    }
  if (mn != ~0ull) atomicMin(&sm.kmin, (unsigned long long)mn);
  if (mx != 0) atomicMax(&sm.kmax, (unsigned long long)mx);
  __syncthreads();
  if ((int)threadIdx.x < cs) {
    cl.map_shared_rank(sm.vmin, (int)threadIdx.x)[rank] = sm.kmin;
    cl.map_shared_rank(sm.vmax, (int)threadIdx.x)[rank] = sm.kmax;
  }
  if (cs > 1) cl.sync(); else __syncthreads();
  gmin = ~0ull;
  gmax = 0;
  for (int q = 0; q < cs; ++q) {
    gmin = min(gmin, (uint64_t)sm.vmin[q]);
    gmax = max(gmax, (uint64_t)sm.vmax[q]);
  }
}

// Push this CTA's word v into slot `rank` of every CTA's vall[] (DSMEM stores,
// no round trips), then a cluster barrier; returns the OR over the cluster.
__device__ __forceinline__ unsigned long long cluster_or(RadixSmem& sm, unsigned long long v) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  if ((int)threadIdx.x < cs) cl.map_shared_rank(sm.vall, (int)threadIdx.x)[rank] = v;
  if (cs > 1) cl.sync(); else __syncthreads();
  unsigned long long all = 0;
  for (int q = 0; q < cs; ++q) all |= sm.vall[q];
  return all;
}

__device__ __forceinline__ void cluster_bar() {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  if (cl.num_blocks() > 1) cl.sync(); else __syncthreads();
}

// Order-preserving unsigned image of a double (-0.0 == 0.0, as Python compares).
__device__ __forceinline__ uint64_t dbl_ord(double v) {
  uint64_t u = v == 0.0 ? 0ull : (uint64_t)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}

// Exclusive scan of one value per thread over the CTA (1024 threads); returns
// this thread's exclusive prefix.
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t v, uint32_t* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(SL_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(SL_FULL, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s - wsum[lane];  // exclusive over warps
  }
  __syncthreads();
  return wsum[w] + x - v;
}

// NS items per thread: slot x of warp w holds local position (NS w + x) 32 + lane.
template <int NS>
struct RadixItems {
  uint64_t v[NS];
  bool ok[NS];
};
template <int NS>
__device__ __forceinline__ int item_pos(int x) {
  return (NS * (threadIdx.x >> 5) + x) * 32 + (threadIdx.x & 31);
}

// Counter of (digit d, warp w): warp-major rows padded to 257 words, so the
// ranking (lanes of one warp, distinct digits) and the scan (8 consecutive warps
// of a digit per thread) hit distinct banks.
__device__ __forceinline__ int cidx(int d, int w) { return w * 257 + d; }

// Stable ranks of the items' digits d[] (valid items only): r[x] = number of
// the warp's earlier items with the same digit (ballot peers; slots in order),
// and sm.cnt = CTA-local exclusive offsets in (digit, warp) order, so an item's
// rank in the CTA is cnt[cidx(d, w)] + r.
template <int NS>
__device__ __forceinline__ void rank_digits(RadixSmem& sm, const int (&d)[NS],
                                            const bool (&ok)[NS], uint32_t (&r)[NS]) {
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 257 * kSortWarps; i += blockDim.x) sm.cnt[i] = 0;
  __syncthreads();
#pragma unroll
  for (int x = 0; x < NS; ++x) {
    unsigned peers = __ballot_sync(SL_FULL, ok[x]);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool bit = (d[x] >> b) & 1;
      const unsigned bb = __ballot_sync(SL_FULL, bit);
      peers &= bit ? bb : ~bb;
    }
    const unsigned lt = peers & lanemask_lt();
    r[x] = ok[x] ? sm.cnt[cidx(d[x], w)] + __popc(lt) : 0u;
    __syncwarp();
    if (ok[x] && lt == 0) sm.cnt[cidx(d[x], w)] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive offsets in (digit, warp) order: thread t owns digit t / 4,
  // warps 8 (t % 4) .. 8 (t % 4) + 7
  const int sd = threadIdx.x >> 2, sw = (threadIdx.x & 3) * 8;
  uint32_t c8[8], s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    c8[k] = sm.cnt[cidx(sd, sw + k)];
    s += c8[k];
  }
  uint32_t e = cta_excl_scan(s, sm.wsum);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sm.cnt[cidx(sd, sw + k)] = e;
    e += c8[k];
  }
  __syncthreads();
}

// This CTA's total for digit dd (offsets (dd, 0) .. (dd + 1, 0)); n = valid items.
__device__ __forceinline__ uint32_t digit_total(const RadixSmem& sm, int dd, int n) {
  const uint32_t hi = dd < 255 ? sm.cnt[cidx(dd + 1, 0)] : (uint32_t)n;
  return hi - sm.cnt[cidx(dd, 0)];
}

// Push every digit total into slot `rank` of every CTA's hall[] (thread t:
// digit t & 255, CTAs t >> 8, + 4, ...), then a cluster barrier; thread t < 256
// gets the total of digit t over the cluster and over the CTAs before this one.
__device__ __forceinline__ void exchange_hist(RadixSmem& sm, int n, uint32_t& tot, uint32_t& pre) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int dd = threadIdx.x & 255;
  const uint32_t h = digit_total(sm, dd, n);
  for (int q = threadIdx.x >> 8; q < cs; q += kSortCtaThreads / 256)
    cl.map_shared_rank(&sm.hall[rank][0], q)[dd] = h;
  cluster_bar();
  tot = 0;
  pre = 0;
  if (threadIdx.x < 256)
    for (int q = 0; q < cs; ++q) {
      const uint32_t x = sm.hall[q][threadIdx.x];
      tot += x;
      pre += q < rank ? x : 0u;
    }
}

// One stable LSD pass over the cluster on digit (IMG(item) >> shift) & 255,
// items in the input layout (2 per thread, kSortLoc per CTA).
template <class Img>
__device__ __forceinline__ void cluster_pass(RadixSmem& sm, RadixItems<2>& it, int& cur,
                                             int shift, const Img& img, int n_here) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int w = threadIdx.x >> 5;
  int d[2];
  uint32_t r[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) d[x] = it.ok[x] ? (int)((img(it.v[x]) >> shift) & 255u) : 0;
  rank_digits<2>(sm, d, it.ok, r);
  uint32_t tot, pre;
  exchange_hist(sm, n_here, tot, pre);
  // global base per digit: all CTAs' items of smaller digits + earlier CTAs' items
  const uint32_t ex = cta_excl_scan(threadIdx.x < 256 ? tot : 0u, sm.wsum);
  if (threadIdx.x < 256) sm.gbase[threadIdx.x] = ex + pre - sm.cnt[cidx(threadIdx.x, 0)];
  __syncthreads();
  uint64_t* dst = sm.buf[cur ^ 1];
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    if (!it.ok[x]) continue;
    const uint32_t pos = sm.gbase[d[x]] + sm.cnt[cidx(d[x], w)] + r[x];
    if (cs > 1)
      cl.map_shared_rank(dst, (int)(pos / kSortLoc))[pos % kSortLoc] = it.v[x];
    else
      dst[pos] = it.v[x];
  }
  cluster_bar();
  cur ^= 1;
#pragma unroll
  for (int x = 0; x < 2; ++x)
    if (it.ok[x]) it.v[x] = sm.buf[cur][item_pos<2>(x)];
}

// One stable LSD pass inside the CTA on digit (item >> shift) & 255.
template <int NS>
__device__ __forceinline__ void local_pass(RadixSmem& sm, RadixItems<NS>& it, int& cur,
                                           int shift) {
  const int w = threadIdx.x >> 5;
  int d[NS];
  uint32_t r[NS];
#pragma unroll
  for (int x = 0; x < NS; ++x) d[x] = it.ok[x] ? (int)((it.v[x] >> shift) & 255u) : 0;
  rank_digits<NS>(sm, d, it.ok, r);
  uint64_t* dst = sm.buf[cur ^ 1];
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (it.ok[x]) dst[sm.cnt[cidx(d[x], w)] + r[x]] = it.v[x];
  __syncthreads();
  cur ^= 1;
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (it.ok[x]) it.v[x] = sm.buf[cur][item_pos<NS>(x)];
}

// One stable LSD pass inside the CTA on digit (IMG(item) >> shift) & 255.
template <int NS, class Img>
__device__ __forceinline__ void local_pass_img(RadixSmem& sm, RadixItems<NS>& it, int& cur,
                                               int shift, const Img& img) {
  const int w = threadIdx.x >> 5;
  int d[NS];
  uint32_t r[NS];
#pragma unroll
  for (int x = 0; x < NS; ++x) d[x] = it.ok[x] ? (int)((img(it.v[x]) >> shift) & 255u) : 0;
  rank_digits<NS>(sm, d, it.ok, r);
  uint64_t* dst = sm.buf[cur ^ 1];
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (it.ok[x]) dst[sm.cnt[cidx(d[x], w)] + r[x]] = it.v[x];
  __syncthreads();
  cur ^= 1;
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (it.ok[x]) it.v[x] = sm.buf[cur][item_pos<NS>(x)];
}

// CTA-local LSD sort of the items on the bits of IMG in which some item differs
// from the first one (CTA barriers only).
template <int NS, class Img>
__device__ __forceinline__ void local_sort_on(RadixSmem& sm, RadixItems<NS>& it, int& cur, int n,
                                              const Img& img) {
  if (threadIdx.x == 0) sm.vary = 0;
  __syncthreads();
  const uint64_t ref = n > 0 ? img(sm.buf[cur][0]) : 0ull;
  uint64_t v = 0;
#pragma unroll
  for (int x = 0; x < NS; ++x)
    if (it.ok[x]) v |= img(it.v[x]) ^ ref;
  const unsigned hi = __reduce_or_sync(SL_FULL, (unsigned)(v >> 32));
  const unsigned lo = __reduce_or_sync(SL_FULL, (unsigned)v);
  if ((threadIdx.x & 31) == 0 && (hi | lo))
    atomicOr(&sm.vary, ((unsigned long long)hi << 32) | lo);
  __syncthreads();
  const uint64_t all = sm.vary;
  const int nbits = all ? 64 - __clzll((long long)all) : 0;
  for (int b = 0; b < nbits; b += 8) local_pass_img<NS>(sm, it, cur, b, img);
}

// Images of a packed key's position p (low 15 bits) for the exact order.
struct KeyId {
  const int64_t* id;
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const {
    return (uint64_t)id[k & kPosMask] ^ (1ull << 63);
  }
};
struct KeyArr {
  const double* arr;
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const {
    return dbl_ord(arr[k & kPosMask]);
  }
};
struct KeyDl {
  const double* arr;
  const double* ttft;
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const {
    return dbl_ord(fadd_(arr[k & kPosMask], ttft[k & kPosMask]));  // core.py:50-53
  }
};

// Varying bits of IMG over the cluster's items, relative to `ref` (cluster barrier).
template <class Img>
__device__ __forceinline__ uint64_t cluster_vary(RadixSmem& sm, const RadixItems<2>& it,
                                                 uint64_t ref, const Img& img) {
  uint64_t v = 0;
#pragma unroll
  for (int x = 0; x < 2; ++x)
    if (it.ok[x]) v |= img(it.v[x]) ^ ref;
  const unsigned hi = __reduce_or_sync(SL_FULL, (unsigned)(v >> 32));
  const unsigned lo = __reduce_or_sync(SL_FULL, (unsigned)v);
  if (threadIdx.x == 0) sm.vary = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && (hi | lo))
    atomicOr(&sm.vary, ((unsigned long long)hi << 32) | lo);
  __syncthreads();
  return cluster_or(sm, sm.vary);
}

// Cluster LSD sort on the varying bits [lo_bit, 64) of IMG (relative to ref).
template <class Img>
__device__ __forceinline__ void cluster_sort_on(RadixSmem& sm, RadixItems<2>& it, int& cur,
                                                int lo_bit, uint64_t ref, const Img& img,
                                                int n_here) {
  const uint64_t all = cluster_vary(sm, it, ref, img) >> lo_bit;
  const int nbits = all ? 64 - __clzll((long long)all) : 0;
  SL_SSTAMP();
  for (int b = 0; b < nbits; b += 8) {
    cluster_pass(sm, it, cur, lo_bit + b, img, n_here);
    SL_SSTAMP();
  }
  if (nbits == 0) cluster_bar();  // vall read everywhere before it is reused
}

struct ImgKey {  // fast pass: the packed key itself
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const { return k; }
};
struct ImgId {  // exact pass, items = positions: id as an unsigned image
  const int64_t* id;
  __device__ __forceinline__ uint64_t operator()(uint64_t p) const {
    return (uint64_t)id[p] ^ (1ull << 63);
  }
};
struct ImgArr {
  const double* arr;
  __device__ __forceinline__ uint64_t operator()(uint64_t p) const { return dbl_ord(arr[p]); }
};
struct ImgDl {
  const double* arr;
  const double* ttft;
  __device__ __forceinline__ uint64_t operator()(uint64_t p) const {
    return dbl_ord(fadd_(arr[p], ttft[p]));  // Request.deadline, core.py:50-53
  }
};

__device__ __forceinline__ uint64_t packed_key(const sl_plan_state& st, int64_t wb, int p) {
  const double d = fadd_(st.w_arrival[wb + p], st.w_ttft[wb + p]);  // > 0 (core.py:40-47)
  return ((uint64_t)__double_as_longlong(d) & ~kPosMask) | (uint64_t)p;
}

// Adjacent sorted keys (x, next) with equal top 49 bits?
__device__ __forceinline__ bool near_tie(uint64_t x, uint64_t nx) {
  return ((x ^ nx) >> kPosBits) == 0;
}

// MSD distribution + CTA-local bucket sort (see above).  Returns false (nothing
// written, no shared state pending) if some CTA would own more than kSortCap
// keys.  Otherwise writes the sorted positions to perm unless *tie (near-ties:
// the caller runs the exact path).  Neither step needs to be stable: keys are
// unique, and every key's final place is decided by the local sort.
__device__ __forceinline__ bool msd_sort(RadixSmem& sm, RadixItems<2>& in, int W, double dlo,
                                         double dhi, int64_t wb,
                                         const int64_t* sm_seg_id, const double* sm_seg_arr,
                                         const double* sm_seg_tt, int32_t* perm, bool* tie) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  // 1. bucket = floor(256 (d - dlo) / (dhi - dlo)), clamped to [0, 255]: monotone
  // in the key's deadline d (IEEE subtraction of, and multiplication by, a
  // constant are monotone); slot inside the CTA's part of the bucket from a
  // shared atomic
  const double sc = 256.0 / (dhi - dlo);  // dhi > dlo
  if (threadIdx.x < 256) sm.lh[threadIdx.x] = 0;
  __syncthreads();
  int d[2];
  uint32_t slot[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const double dk = __longlong_as_double((long long)(in.v[x] & ~kPosMask));
    d[x] = in.ok[x] ? min(255, max(0, (int)((dk - dlo) * sc))) : 0;
    if (in.ok[x]) slot[x] = atomicAdd(&sm.lh[d[x]], 1u);
  }
  __syncthreads();
  // push the CTA's bucket totals into slot `rank` of every CTA's hall[]
  {
    const int dd = threadIdx.x & 255;
    const uint32_t h = sm.lh[dd];
    for (int q = threadIdx.x >> 8; q < cs; q += kSortCtaThreads / 256)
      cl.map_shared_rank(&sm.hall[rank][0], q)[dd] = h;
  }
  cluster_bar();
  uint32_t tot = 0, pre = 0;
  if (threadIdx.x < 256)
    for (int q = 0; q < cs; ++q) {
      const uint32_t x = sm.hall[q][threadIdx.x];
      tot += x;
      pre += q < rank ? x : 0u;
    }
  const uint32_t base = cta_excl_scan(threadIdx.x < 256 ? tot : 0u, sm.wsum);
  if (threadIdx.x <= kSortMaxCluster) sm.start[threadIdx.x] = W;
  __syncthreads();
  int own = 0;
  if (threadIdx.x < 256) {
    own = (int)(base / kSortLoc);
    sm.owner[threadIdx.x] = own;
    if (tot) atomicMin(&sm.start[own], (int)base);
    sm.gbase[threadIdx.x] = base + pre;  // this CTA's first place in the bucket
  }
  // index of each non-empty bucket among the ones this CTA owns (local sub-bucketing)
  const bool mine = threadIdx.x < 256 && tot > 0 && own == rank;
  const uint32_t bix = cta_excl_scan(mine ? 1u : 0u, sm.wsum);
  if (threadIdx.x < 256) sm.bidx[threadIdx.x] = (int)bix;
  if (threadIdx.x == 255) sm.nmine = (int)bix + (mine ? 1 : 0);
  __syncthreads();
  // owned counts (every CTA computes the same table): start of the next owner
  bool over = false;
  int my_start = W, my_n = 0;
  {
    int nxt = W;
    for (int c = cs - 1; c >= 0; --c) {
      const int s0 = sm.start[c];
      if (s0 < W) {
        over |= nxt - s0 > kSortCap;
        if (c == rank) {
          my_start = s0;
          my_n = nxt - s0;
        }
        nxt = s0;
      }
    }
  }
  if (over) {
    cluster_bar();  // hall / start read everywhere before the fallback reuses them
    return false;
  }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    if (!in.ok[x]) continue;
    const int own = sm.owner[d[x]];
    const int pos = (int)(sm.gbase[d[x]] + slot[x]) - sm.start[own];
    if (cs > 1)
      cl.map_shared_rank(sm.buf[0], own)[pos] = in.v[x];
    else
      sm.buf[0][pos] = in.v[x];
  }
  cluster_bar();
  SL_SSTAMP();
  SL_CTASTAMP(0, sl_gtime());
  SL_CTASTAMP(3, my_n);
  // 2. CTA-local sort of the owned range: each owned non-empty MSD bucket is cut
  // into K = kLocalBins / (owned non-empty buckets) sub-buckets by linear
  // interpolation inside it -- local digit = (bucket index) K + sub-bucket, monotone
  // in the deadline like the MSD bucket -- with slots by shared atomics; then
  // each key's place inside its sub-bucket by counting the sub-bucket's smaller
  // keys.  A sub-bucket of more than kBucketMax keys (clustered deadlines) sends
  // the CTA to LSD passes on its varying bits instead.
  RadixItems<4> it;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    it.ok[x] = item_pos<4>(x) < my_n;
    it.v[x] = it.ok[x] ? sm.buf[0][item_pos<4>(x)] : 0ull;
  }
  for (int i = threadIdx.x; i < kLocalBins; i += blockDim.x) sm.lh[i] = 0;
  if (threadIdx.x < 256) {
    sm.bmin[threadIdx.x] = ~0ull;
    sm.bmax[threadIdx.x] = 0;
  }
  __syncthreads();
  const int K = kLocalBins / max(1, sm.nmine);
  // each owned bucket's own key range (deadline bits: positive doubles order
  // like their bits), so clamped edge buckets and gaps cost nothing
  int B[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint64_t kb = it.v[x] & ~kPosMask;
    const double xs = (__longlong_as_double((long long)kb) - dlo) * sc;  // the MSD bucket
    B[x] = it.ok[x] ? min(255, max(0, (int)xs)) : 0;
    if (it.ok[x]) {
      atomicMin(&sm.bmin[B[x]], (unsigned long long)kb);
      atomicMax(&sm.bmax[B[x]], (unsigned long long)kb);
    }
  }
  __syncthreads();
  if (threadIdx.x < 256 && sm.bmax[threadIdx.x] != 0) {
    const double lo = __longlong_as_double((long long)sm.bmin[threadIdx.x]);
    const double hi = __longlong_as_double((long long)sm.bmax[threadIdx.x]);
    sm.bscale[threadIdx.x] = hi > lo ? (double)K / (hi - lo) : 0.0;
  }
  __syncthreads();
  int ld[4];
  uint32_t ls[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint64_t kb = it.v[x] & ~kPosMask;
    const double lo = __longlong_as_double((long long)sm.bmin[B[x]]);
    const int sub = it.ok[x] ? min(K - 1, max(0, (int)((__longlong_as_double((long long)kb) - lo) *
                                                        sm.bscale[B[x]])))
                             : 0;
    ld[x] = sm.bidx[B[x]] * K + sub;
    if (it.ok[x]) ls[x] = atomicAdd(&sm.lh[ld[x]], 1u);
  }
  __syncthreads();
  // exclusive scan of the bucket counts (kLocalBins / blockDim per thread)
  constexpr int kPer = kLocalBins / kSortCtaThreads;
  uint32_t hc[kPer], hs = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hc[k] = sm.lh[kPer * threadIdx.x + k];
    hs += hc[k];
  }
  bool big = false;
#pragma unroll
  for (int k = 0; k < kPer; ++k) big |= hc[k] > (uint32_t)kBucketMax;
  uint32_t e = cta_excl_scan(hs, sm.wsum);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    sm.lh[kPer * threadIdx.x + k] = e;
    e += hc[k];
  }
  big = __syncthreads_or(big) != 0;
  int cur = 0;
  if (!big) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (it.ok[x]) sm.buf[1][sm.lh[ld[x]] + ls[x]] = it.v[x];
    __syncthreads();
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      if (!it.ok[x]) continue;
      const int b0 = (int)sm.lh[ld[x]];
      const int b1 = ld[x] + 1 < kLocalBins ? (int)sm.lh[ld[x] + 1] : my_n;
      int k = 0;
      for (int j = b0; j < b1; ++j) k += sm.buf[1][j] < it.v[x];
      sm.buf[0][b0 + k] = it.v[x];
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (it.ok[x]) it.v[x] = sm.buf[0][item_pos<4>(x)];
  } else {
    if (threadIdx.x == 0) {
      sm.kmin = ~0ull;
      sm.kmax = 0;
    }
    __syncthreads();
    uint64_t mn = ~0ull, mx = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (it.ok[x]) {
        mn = min(mn, it.v[x]);
        mx = max(mx, it.v[x]);
      }
    if (mn != ~0ull) atomicMin(&sm.kmin, (unsigned long long)mn);
    if (mx != 0) atomicMax(&sm.kmax, (unsigned long long)mx);
    __syncthreads();
    const uint64_t lv = (sm.kmin ^ sm.kmax) >> kPosBits;
    const int lhb = lv ? kPosBits + 63 - __clzll((long long)lv) : kPosBits - 1;
    for (int b = kPosBits; b <= lhb; b += 8) local_pass<4>(sm, it, cur, b);
  }
  SL_SSTAMP();
  SL_CTASTAMP(1, sl_gtime());
  SL_CTASTAMP(2, big);
  // 3. near-ties (equal top 49 bits) have equal bucket values, so they share an
  // owner: check adjacent keys inside the range only, and on a near-tie re-sort
  // the range with the full key -- id, then arrival, then deadline, stable
  // CTA-local passes (the packed order, i.e. position, breaks exact ties).
  // No cluster-wide decision: the CTAs finish independently.
  bool t = false;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int p = item_pos<4>(x);
    if (it.ok[x] && p + 1 < my_n) t |= near_tie(it.v[x], sm.buf[cur][p + 1]);
  }
  if (__syncthreads_or(t)) {
    const int64_t* idp = sm_seg_id;
    local_sort_on<4>(sm, it, cur, my_n, KeyId{idp});
    local_sort_on<4>(sm, it, cur, my_n, KeyArr{sm_seg_arr});
    local_sort_on<4>(sm, it, cur, my_n, KeyDl{sm_seg_arr, sm_seg_tt});
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
    if (it.ok[x]) perm[wb + my_start + item_pos<4>(x)] = (int32_t)(wb + (int64_t)(it.v[x] & kPosMask));
  *tie = false;
  return true;  // no DSMEM access is pending: CTAs may exit
}

__global__ void __launch_bounds__(kSortCtaThreads) sort_cluster_kernel(const sl_plan_state st,
                                                                       int32_t* perm) {
  namespace cg = cooperative_groups;
  extern __shared__ unsigned char sort_smem_raw[];
  RadixSmem& sm = *reinterpret_cast<RadixSmem*>(sort_smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int seg = blockIdx.x / cs;
  const int64_t wb = st.w_begin[seg];
  const int W = (int)(st.w_begin[seg + 1] - wb);
  const int g0 = rank * kSortLoc;  // this CTA's first input position
  const int n_here = max(0, min(kSortLoc, W - g0));
  SL_SSTAMP();
  // arrive now, wait before the first DSMEM access (cluster_minmax): the key
  // loads overlap the cluster's start-up
  if (cs > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  RadixItems<2> it;
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int p = item_pos<2>(x);
    it.ok[x] = p < n_here;
    it.v[x] = it.ok[x] ? packed_key(st, wb, g0 + p) : 0ull;
    if (it.ok[x]) sm.buf[0][p] = it.v[x];  // read by the tie check if no pass moves them
  }
  // bucket range from a fixed sample of 128 keys, read by every CTA from global
  // memory (no exchange needed: every CTA computes the same range)
  if (threadIdx.x == 0) {
    sm.kmin = ~0ull;
    sm.kmax = 0;
  }
  __syncthreads();
  if ((int)threadIdx.x < min(W, 128)) {
    const int p = W >= 128 ? (int)(((int64_t)threadIdx.x * W) >> 7) : (int)threadIdx.x;
    const uint64_t k = packed_key(st, wb, p) & ~kPosMask;
    atomicMin(&sm.kmin, (unsigned long long)k);
    atomicMax(&sm.kmax, (unsigned long long)k);
  }
  __syncthreads();
  const double slo = __longlong_as_double((long long)sm.kmin);
  const double shi = __longlong_as_double((long long)sm.kmax);
  // every CTA of the cluster has started (the arrive above) before the first
  // store into another CTA's shared memory
  if (cs > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  SL_SSTAMP();
  bool tie = false;
  bool done = false;
  if (cs > 1 && W > 1 && slo < shi)
    done = msd_sort(sm, it, W, slo, shi, wb, st.w_id + wb, st.w_arrival + wb, st.w_ttft + wb,
                    perm, &tie);
  uint64_t all = 0;  // bits 15.. in which two keys differ (the highest: that of max ^ min)
  if (!done) {  // one CTA, a sample without spread, or a skewed bucket distribution:
                // cluster LSD passes on the varying bits
    uint64_t gmin, gmax;
    cluster_minmax<2>(sm, it.v, it.ok, gmin, gmax);
    all = (gmin ^ gmax) >> kPosBits;
    tie = W > 1 && all == 0;  // every deadline shares its top 49 bits
  }
  if (!done && !tie) {
    int cur = 0;
    const int nbits = all ? 64 - __clzll((long long)all) : 0;
    for (int b = 0; b < nbits; b += 8) cluster_pass(sm, it, cur, kPosBits + b, ImgKey{}, n_here);
    bool t = false;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int p = item_pos<2>(x);
      if (!it.ok[x] || g0 + p + 1 >= W) continue;
      const uint64_t nx = p + 1 < kSortLoc ? sm.buf[cur][p + 1]
                                           : cl.map_shared_rank(sm.buf[cur], rank + 1)[0];
      t |= near_tie(it.v[x], nx);
    }
    t = __syncthreads_or(t) != 0;
    tie = cluster_or(sm, t) != 0;
    cluster_bar();  // vall read before it is reused
    if (!tie) {
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (it.ok[x])
          perm[wb + g0 + item_pos<2>(x)] = (int32_t)(wb + (int64_t)(it.v[x] & kPosMask));
    }
  }
  if (tie && W > 0) {
    // exact: positions sorted by id, then arrival, then deadline (stable passes)
    int cur = 0;
#pragma unroll
    for (int x = 0; x < 2; ++x) it.v[x] = (uint64_t)(g0 + item_pos<2>(x));
    const int64_t* id = st.w_id + wb;
    const double* arr = st.w_arrival + wb;
    const double* tt = st.w_ttft + wb;
    cluster_sort_on(sm, it, cur, 0, ImgId{id}(0), ImgId{id}, n_here);
    cluster_sort_on(sm, it, cur, 0, ImgArr{arr}(0), ImgArr{arr}, n_here);
    cluster_sort_on(sm, it, cur, 0, ImgDl{arr, tt}(0), ImgDl{arr, tt}, n_here);
#pragma unroll
    for (int x = 0; x < 2; ++x)
      if (it.ok[x]) perm[wb + g0 + item_pos<2>(x)] = (int32_t)(wb + (int64_t)it.v[x]);
  }
  SL_SSTAMP();
}

}  // namespace
