/* Native trace synthesis, stream-identical to workload.generate (reference
 * workload.py:107-137): numpy's PCG64 bit generator
 * restated here (pcg_setseq_128 XSL-RR, the state taken from
 * numpy.random.default_rng(seed)), and numpy's own distribution code
 * (libnpyrandom.a, shipped with numpy: ziggurat exponential / normal,
 * lognormal) drawing in the reference's per-request order:
 *   t += exponential(1/qps); stop if t > duration
 *   category = searchsorted(cdf, random(), side="right")
 *   prompt = max(1, round(lognormal(mu_p, sigma_p)))
 *   output = max(1, round(lognormal(mu_o, sigma_o)))
 * Host code (the reference generates traces on the host too); ~100x the
 * Python loop.  Only LogNormal length distributions take this path. */
#include <math.h>
#include <stdint.h>

#include "numpy/random/bitgen.h"

double random_exponential(bitgen_t* bitgen_state, double scale);
double random_lognormal(bitgen_t* bitgen_state, double mean, double sigma);

typedef struct {
  unsigned __int128 state, inc;
  int has_uint32;
  uint32_t uinteger;
} pcg64_t;

static const unsigned __int128 kMult =
    ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;

static uint64_t pcg64_next64(void* p) {
  pcg64_t* s = (pcg64_t*)p;
  s->state = s->state * kMult + s->inc;
  const uint64_t x = (uint64_t)(s->state >> 64) ^ (uint64_t)s->state;
  const unsigned r = (unsigned)(s->state >> 122);
  return (x >> r) | (x << ((-r) & 63));
}

static uint32_t pcg64_next32(void* p) {
  pcg64_t* s = (pcg64_t*)p;
  if (s->has_uint32) {
    s->has_uint32 = 0;
    return s->uinteger;
  }
  const uint64_t n = pcg64_next64(p);
  s->has_uint32 = 1;
  s->uinteger = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

static double pcg64_next_double(void* p) {
  return (double)(pcg64_next64(p) >> 11) * (1.0 / 9007199254740992.0);
}

/* Python round(): half to even (the default rounding mode). */
static int32_t round_len(double x) {
  const double r = nearbyint(x);
  return r < 1.0 ? 1 : (int32_t)r;
}

/* Returns the number of requests drawn (<= cap; stops at `limit` >= 0 or when
 * the arrival time passes `duration`), -1 on bad arguments. */
int64_t sl_gen_trace_lognormal(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                               uint64_t inc_lo, double qps, double duration, int64_t limit,
                               const double* cdf, int32_t n_cat, double p_mu, double p_sigma,
                               double o_mu, double o_sigma, double* arrival, int32_t* category,
                               int32_t* prompt, int32_t* output, int64_t cap) {
  if (!(qps > 0.0) || n_cat < 1 || !cdf || !arrival || !category || !prompt || !output || cap < 0)
    return -1;
  pcg64_t st = {((unsigned __int128)state_hi << 64) | state_lo,
                ((unsigned __int128)inc_hi << 64) | inc_lo, 0, 0};
  bitgen_t bg = {&st, pcg64_next64, pcg64_next32, pcg64_next_double, pcg64_next64};
  const double scale = 1.0 / qps;
  double t = 0.0;
  int64_t n = 0;
  while ((limit < 0 || n < limit) && n < cap) {
    t += random_exponential(&bg, scale);
    if (t > duration) break;
    const double u = pcg64_next_double(&st);
    int32_t c = 0;
    while (c < n_cat && cdf[c] <= u) ++c;  /* searchsorted(side="right") */
    arrival[n] = t;
    category[n] = c;
    prompt[n] = round_len(random_lognormal(&bg, p_mu, p_sigma));
    output[n] = round_len(random_lognormal(&bg, o_mu, o_sigma));
    ++n;
  }
  return n;
}
