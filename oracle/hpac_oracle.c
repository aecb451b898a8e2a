/*
 * hpac_oracle.c — TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT PATH.
 *
 * A plain-C, single-threaded CPU restatement of the reference's
 * approximate-region engine (simtac `run_region`) and the techniques it
 * dispatches to. It exists to check the CUDA path: tests/, the smoke()
 * entry and bench.py's cpu_baseline leg are the only callers. The product
 * library (libhpac_b200.so) never links or calls it.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/include/simtac/.
 *
 * Parity pinning: this restatement is checked (tests/test_oracle_*.py)
 * against (a) the known-answer vectors of the reference's own tests and
 * (b) the reference itself, compiled from its headers into
 * oracle/_ref/libsimtac_ref.so (oracle/ref_shim.cpp), on randomised
 * configurations, plus committed golden fixtures generated from (b).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (no FMA contraction, IEEE
 * sqrt/div), matching the reference's x86-64 build where RSD and iACT
 * distance sums must be bit-identical.
 */
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hpac_offload.h"

#define ORACLE_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* error plumbing: status + message (errors.hpp:12-62)                 */
/* ------------------------------------------------------------------ */
static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

/* splitmix64, bench/synthetic.hpp:26-31 (the public SplitMix64 mixer) */
ORACLE_API uint64_t oracle_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* ------------------------------------------------------------------ */
/* applications                                                        */
/* ------------------------------------------------------------------ */

/* synthetic_value, bench/synthetic.hpp:36-49 */
ORACLE_API double oracle_synthetic_value(int profile, int64_t i, uint64_t seed) {
  switch (profile) {
    case HPAC_SYNTH_CONSTANT: return 7.5;
    case HPAC_SYNTH_SLOW_DRIFT: return 50.0 * (1.0 + 1e-5 * (double)i);
    case HPAC_SYNTH_NOISE: {
      uint64_t h = oracle_splitmix64(seed ^ (uint64_t)i);
      return 1.0 + (double)(h >> 11) * 0x1.0p-53;
    }
  }
  return 0.0;
}

/* synthetic_eval, bench/synthetic.hpp:53 */
static double synthetic_eval(double x) { return 3.0 * x + 1.0; }

/* norm_cdf / black_scholes_call, bench/blackscholes.hpp:21-36.
   o = (spot, strike, rate, vol, maturity). Returns 0 or HPAC_ERR_CONFIG. */
ORACLE_API int oracle_black_scholes_call(const double* o, double* price) {
  double spot = o[0], strike = o[1], rate = o[2], vol = o[3], mat = o[4];
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol >= 0) || !isfinite(rate))
    return HPAC_ERR_CONFIG;
  double disc_strike = strike * exp(-rate * mat);
  double sst = vol * sqrt(mat);
  if (sst == 0.0) {
    double v = spot - disc_strike;
    *price = v < 0.0 ? 0.0 : v; /* std::max(v, 0.0) */
    return 0;
  }
  double d1 = (log(spot / strike) + (rate + 0.5 * vol * vol) * mat) / sst;
  double d2 = d1 - sst;
  double n1 = 0.5 * erfc(-d1 / sqrt(2.0));
  double n2 = 0.5 * erfc(-d2 / sqrt(2.0));
  *price = spot * n1 - disc_strike * n2;
  return 0;
}

/* binomial_price (CRR), bench/binomial.hpp:16-50 */
ORACLE_API int oracle_binomial_price(const double* o, int n_steps, int american, int is_put,
                                     double* price) {
  double spot = o[0], strike = o[1], rate = o[2], vol = o[3], mat = o[4];
  if (n_steps < 1) return HPAC_ERR_CONFIG;
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol > 0)) return HPAC_ERR_CONFIG;
  double dt = mat / n_steps;
  double up = exp(vol * sqrt(dt));
  double down = 1.0 / up;
  double growth = exp(rate * dt);
  double p_up = (growth - down) / (up - down);
  if (!(p_up > 0.0) || !(p_up < 1.0)) return HPAC_ERR_CONFIG;
  double disc = 1.0 / growth;
  double* v = (double*)malloc(sizeof(double) * (size_t)(n_steps + 1));
  if (!v) return HPAC_ERR_CONFIG;
  for (int j = 0; j <= n_steps; ++j) {
    double s = spot * pow(up, 2 * j - n_steps);
    double x = is_put ? strike - s : s - strike;
    v[j] = x < 0.0 ? 0.0 : x;
  }
  for (int level = n_steps - 1; level >= 0; --level) {
    for (int j = 0; j <= level; ++j) {
      double cont = disc * (p_up * v[j + 1] + (1.0 - p_up) * v[j]);
      if (american) {
        double s = spot * pow(up, 2 * j - level);
        double x = is_put ? strike - s : s - strike;
        double intr = x < 0.0 ? 0.0 : x;
        cont = cont < intr ? intr : cont; /* std::max(cont, intr) */
      }
      v[j] = cont;
    }
  }
  *price = v[0];
  free(v);
  return 0;
}

/* Whole portfolios (test convenience; options are independent). */
ORACLE_API int oracle_bs_prices(const double* opts, int64_t n, double* out) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i)
    if (oracle_black_scholes_call(opts + (size_t)i * 5, out + i)) {
      out[i] = NAN;
      ++bad;
    }
  return bad;
}

ORACLE_API int oracle_binomial_prices(const double* opts, int64_t n, int n_steps, int american,
                                      int is_put, double* out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i)
    if (oracle_binomial_price(opts + (size_t)i * 5, n_steps, american, is_put, out + i)) {
      out[i] = NAN;
      ++bad;
    }
  return bad;
}

/* ------------------------------------------------------------------ */
/* TAF, taf.hpp:29-163                                                 */
/* ------------------------------------------------------------------ */

/* rsd, taf.hpp:29-40: two-pass population sigma / |mu| in window order. */
ORACLE_API double oracle_rsd(const double* w, int len) {
  double mean = 0.0;
  for (int i = 0; i < len; ++i) mean += w[i];
  mean /= (double)len;
  double ssd = 0.0;
  for (int i = 0; i < len; ++i) ssd += (w[i] - mean) * (w[i] - mean);
  double sigma = sqrt(ssd / (double)len);
  if (mean == 0.0) return sigma == 0.0 ? 0.0 : INFINITY;
  return sigma / fabs(mean);
}

enum { TAF_FILLING = 0, TAF_CHECKING = 1, TAF_PREDICTING = 2 };

typedef struct {
  int h, p, dims;
  double thr;
  int mode, remaining, head, count;
  double* ring; /* dims * h, ring[d*h + slot] */
  double* last; /* dims */
} taf_state;

static void taf_init(taf_state* s, int h, int p, double thr, int dims, double* ring,
                     double* last) {
  s->h = h;
  s->p = p;
  s->thr = thr;
  s->dims = dims;
  s->mode = TAF_FILLING;
  s->remaining = s->head = s->count = 0;
  s->ring = ring;
  s->last = last;
  for (int i = 0; i < dims * h; ++i) ring[i] = 0.0;
  for (int d = 0; d < dims; ++d) last[d] = 0.0;
}

/* TafState::push, taf.hpp:123-132 */
static void taf_push(taf_state* s, const double* o) {
  if (s->count < s->h) {
    int slot = (s->head + s->count) % s->h;
    for (int d = 0; d < s->dims; ++d) s->ring[d * s->h + slot] = o[d];
    s->count++;
  } else {
    for (int d = 0; d < s->dims; ++d) s->ring[d * s->h + s->head] = o[d];
    s->head = (s->head + 1) % s->h;
  }
}

/* TafState::check_passes, taf.hpp:134-140 (conjunction over dims) */
static int taf_check(const taf_state* s) {
  double w[4096];
  for (int d = 0; d < s->dims; ++d) {
    int c = s->count;
    for (int j = 0; j < c; ++j) w[j] = s->ring[d * s->h + (s->head + j) % s->h];
    double r = oracle_rsd(w, c);
    if (!(r <= s->thr)) return 0;
  }
  return 1;
}

/* TafState::tick_regime, taf.hpp:147-153 */
static void taf_tick(taf_state* s) {
  if (--s->remaining == 0) {
    s->count = 0;
    s->head = 0;
    s->mode = TAF_FILLING;
  }
}

/* TafState::observe_accurate, taf.hpp:94-108 */
static void taf_observe(taf_state* s, const double* o) {
  taf_push(s, o);
  for (int d = 0; d < s->dims; ++d) s->last[d] = o[d];
  switch (s->mode) {
    case TAF_FILLING:
      if (s->count == s->h) {
        if (taf_check(s)) {
          s->remaining = s->p;
          s->mode = TAF_PREDICTING;
        } else {
          s->mode = TAF_CHECKING;
        }
      }
      break;
    case TAF_CHECKING:
      if (taf_check(s)) {
        s->remaining = s->p;
        s->mode = TAF_PREDICTING;
      }
      break;
    case TAF_PREDICTING: taf_tick(s); break;
  }
}

/* TafState::emit_approx, taf.hpp:114-117 */
static void taf_emit(taf_state* s, double* o) {
  for (int d = 0; d < s->dims; ++d) o[d] = s->last[d];
  if (s->mode == TAF_PREDICTING) taf_tick(s);
}

/* taf_step over a stream (taf.hpp:172-181): accurate invocations consume
   the stream; returns the number of invocations produced (stops where an
   accurate call would run past the stream end). */
ORACLE_API int64_t oracle_taf_drive(int h, int p, double thr, const double* stream,
                                    int64_t stream_len, int64_t invocations, uint8_t* approx,
                                    double* outputs) {
  double ring[4096], last[1];
  if (h > 4096) return -1;
  taf_state s;
  taf_init(&s, h, p, thr, 1, ring, last);
  int64_t pos = 0, k = 0;
  for (; k < invocations; ++k) {
    double out;
    if (s.mode == TAF_PREDICTING) {
      taf_emit(&s, &out);
      approx[k] = 1;
    } else {
      if (pos >= stream_len) break;
      out = stream[pos++];
      taf_observe(&s, &out);
      approx[k] = 0;
    }
    outputs[k] = out;
  }
  return k;
}

/* taf_state_bytes, taf.hpp:46-48 */
ORACLE_API uint64_t oracle_taf_state_bytes(int h, int dims) {
  return (uint64_t)dims * (uint64_t)h * 8u + 16u;
}

/* table_group_bytes, iact.hpp:149-154 */
ORACLE_API uint64_t oracle_table_group_bytes(int tpw, int tsize, int in_dims, int out_dims) {
  return (uint64_t)tpw * (uint64_t)tsize * (uint64_t)(in_dims + out_dims) * 8u +
         (uint64_t)tpw * 2u * 4u;
}

/* ------------------------------------------------------------------ */
/* iACT memo tables, iact.hpp:43-180                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  int cap, in_dims, out_dims;
  int rr, occ;
  double* in;  /* cap * in_dims */
  double* out; /* cap * out_dims */
} memo_table;

/* euclid_dist, iact.hpp:43-53 */
static double euclid(const double* a, const double* b, int dims) {
  double ssq = 0.0;
  for (int i = 0; i < dims; ++i) {
    double d = a[i] - b[i];
    ssq += d * d;
  }
  return sqrt(ssq);
}

/* MemoTable::lookup, iact.hpp:93-100: closest within threshold, ties to
   the lowest slot. Returns slot or -1. */
static int memo_lookup(const memo_table* t, const double* x, double thr) {
  int best = -1;
  double best_d = 0.0;
  for (int s = 0; s < t->occ; ++s) {
    double d = euclid(t->in + (size_t)s * t->in_dims, x, t->in_dims);
    if (d <= thr && (best < 0 || d < best_d)) {
      best = s;
      best_d = d;
    }
  }
  return best;
}

/* MemoTable::min_distance, iact.hpp:103-108 (std::min keeps the first on NaN) */
static double memo_min_distance(const memo_table* t, const double* x) {
  double best = INFINITY;
  for (int s = 0; s < t->occ; ++s) {
    double d = euclid(t->in + (size_t)s * t->in_dims, x, t->in_dims);
    best = (d < best) ? d : best;
  }
  return best;
}

/* MemoTable::nearest_slot, iact.hpp:111-122 */
static int memo_nearest(const memo_table* t, const double* x) {
  int best = -1;
  double best_d = INFINITY;
  for (int s = 0; s < t->occ; ++s) {
    double d = euclid(t->in + (size_t)s * t->in_dims, x, t->in_dims);
    if (d < best_d) {
      best_d = d;
      best = s;
    }
  }
  return best;
}

/* MemoTable::insert, iact.hpp:124-135 (round-robin) */
static void memo_insert(memo_table* t, const double* x, const double* y) {
  int s = t->rr;
  for (int d = 0; d < t->in_dims; ++d) t->in[(size_t)s * t->in_dims + d] = x[d];
  for (int d = 0; d < t->out_dims; ++d) t->out[(size_t)s * t->out_dims + d] = y[d];
  t->rr = (t->rr + 1) % t->cap;
  t->occ = t->occ + 1 < t->cap ? t->occ + 1 : t->cap;
}

/* ------------------------------------------------------------------ */
/* perforation, perfo.hpp:39-72 (+ RANDOM extension)                   */
/* ------------------------------------------------------------------ */
static int kind_uses_modulus(int k) {
  return k == HPAC_PERFO_SMALL || k == HPAC_PERFO_LARGE || k == HPAC_PERFO_HERDED_SMALL ||
         k == HPAC_PERFO_HERDED_LARGE;
}
static int kind_is_herded(int k) {
  return k == HPAC_PERFO_HERDED_SMALL || k == HPAC_PERFO_HERDED_LARGE;
}

/* RANDOM perforation (extension, parity unpinned in the reference,
   SPEC.md:345): skip iff splitmix64(seed ^ splitmix64(owner<<32 ^ counter))
   mod 100 < percent, owner = thread id (per-thread mapping) or team id
   (per-team mapping). Decisions are a pure function of (seed, owner,
   encounter counter); re-keying the seed per launch moves the skip set. */
ORACLE_API int oracle_random_skip(uint64_t seed, int64_t tid, int64_t counter, int percent) {
  uint64_t k = oracle_splitmix64(((uint64_t)tid << 32) ^ (uint64_t)counter);
  uint64_t h = oracle_splitmix64(seed ^ k);
  return (int)(h % 100u) < percent;
}

/* should_skip, perfo.hpp:52-72 */
static int should_skip(const hpac_spec_t* sp, int64_t key, int64_t trip, int64_t tid) {
  switch (sp->perfo_kind) {
    case HPAC_PERFO_SMALL:
    case HPAC_PERFO_HERDED_SMALL: return key % sp->perfo_modulus == sp->perfo_modulus - 1;
    case HPAC_PERFO_LARGE:
    case HPAC_PERFO_HERDED_LARGE: return key % sp->perfo_modulus != 0;
    case HPAC_PERFO_INI: return key < ((int64_t)sp->perfo_skip_percent * trip) / 100;
    case HPAC_PERFO_FINI: return key >= trip - ((int64_t)sp->perfo_skip_percent * trip) / 100;
    case HPAC_PERFO_RANDOM:
      return oracle_random_skip(sp->perfo_seed, tid, key, sp->perfo_skip_percent);
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* region adapters (engine.hpp:26-33 callbacks as app switch)          */
/* ------------------------------------------------------------------ */
typedef struct {
  const hpac_region_t* r;
  int in_dims, out_dims;
  int64_t n;
} region_view;

/* LavaMD (extension; the framework's restatement of Rodinia lavaMD, SURVEY
   Appendix C; Rodinia is not under /root/reference, so parity is unpinned):
   exp as the device's sequence (apps.cuh lava_exp): n = rint(64x/ln2),
   two-constant reduction r = x - n ln2/64, degree-5 Taylor e^r in fma()
   Horner form, times the correctly rounded 2^((n mod 64)/64), scaled by
   2^(n div 64) (fma() is exactly rounded on both sides). */
static const double lava_exp_t[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};
static double lava_exp(double x) {
  const double shift = 0x1.8p52;
  const double kd = fma(x, 0x1.71547652b82fep+6, shift) - shift;
  double r = fma(-kd, 0x1.62e42fefa39efp-7, x);
  r = fma(-kd, 0x1.abc9e3b39803fp-62, r);
  double s = 0x1.1111111111111p-7;
  s = fma(s, r, 0x1.5555555555555p-5);
  s = fma(s, r, 0x1.5555555555555p-3);
  s = fma(s, r, 0x1.0000000000000p-1);
  s = fma(s, r, 1.0);
  s = fma(s, r, 1.0);
  const int n = (int)kd;
  const double t = lava_exp_t[n & 63] * s;
  return ldexp(t, n >> 6);
}

/* self first, then the in-grid 26-neighbourhood in (dz, dy, dx) order */
static int lava_neighbours(int64_t box, int b1, int64_t* nb) {
  const int bx = (int)(box % b1), by = (int)((box / b1) % b1), bz = (int)(box / ((int64_t)b1 * b1));
  int c = 0;
  if (nb) nb[c] = box;
  ++c;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        int x = bx + dx, y = by + dy, z = bz + dz;
        if (x < 0 || y < 0 || z < 0 || x >= b1 || y >= b1 || z >= b1) continue;
        if (nb) nb[c] = ((int64_t)z * b1 + y) * b1 + x;
        ++c;
      }
  return c;
}

ORACLE_API double oracle_lava_exp(double x) { return lava_exp(x); }

/* LavaMD inputs (the framework's definition; hpac_make_lavamd): per particle
   rv = (v, x, y, z), qv, each (splitmix64(seed ^ (5 i + c)) % 10 + 1) / 10. */
ORACLE_API int oracle_make_lavamd(int b1, int particles, uint64_t seed, double* rv, double* qv) {
  if (b1 < 1 || particles < 1) return HPAC_ERR_CONFIG;
  const int64_t n = (int64_t)b1 * b1 * b1 * particles;
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < 5; ++c) {
      const double v = (double)(oracle_splitmix64(seed ^ (uint64_t)(5 * i + c)) % 10 + 1) / 10.0;
      if (c < 4)
        rv[i * 4 + c] = v;
      else
        qv[i] = v;
    }
  return 0;
}

static int region_encounters(const region_view* rv, int64_t idx) {
  if (rv->r->app == HPAC_APP_TABLE && rv->r->encounters) return rv->r->encounters[idx];
  if (rv->r->app == HPAC_APP_LAVAMD) return lava_neighbours(idx, rv->r->lavamd_boxes1d, NULL);
  return 1;
}

static void region_load(const region_view* rv, int64_t idx, double* in) {
  const hpac_region_t* r = rv->r;
  switch (r->app) {
    case HPAC_APP_SYNTHETIC: in[0] = oracle_synthetic_value(r->synthetic_profile, idx, r->seed); break;
    default:
      for (int d = 0; d < rv->in_dims; ++d) in[d] = r->in[(size_t)idx * rv->in_dims + d];
  }
}

/* evaluate; returns 0 or an error status (apps throw ConfigError) */
static int region_eval(const region_view* rv, int64_t idx, int lane, int round, double* out,
                       char* err, size_t el) {
  const hpac_region_t* r = rv->r;
  switch (r->app) {
    case HPAC_APP_LAVAMD: {
      const int P = r->lavamd_particles;
      const double na2 = -(2.0 * r->lavamd_alpha * r->lavamd_alpha);
      int64_t nb[27];
      lava_neighbours(idx, r->lavamd_boxes1d, nb);
      const int64_t b = nb[round];
      const double* me = r->in + (idx * P + lane) * 4;
      double fv = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
      for (int j = 0; j < P; ++j) {
        const double* o2 = r->in + (b * P + j) * 4;
        const double q = r->table_out[b * P + j];
        /* Rodinia lavaMD pair term: r2 = rA.v + rB.v - dot(rA, rB),
           vij = exp(-a2 r2), f += qB (vij, 2 vij (rA - rB)); FMA form with
           -a2 folded into rA (and into rB.v): x = -a2 vA + (-a2 vB + dot(a2 rA, rB)) */
        const double an = na2 * me[0], nax = -(na2 * me[1]), nay = -(na2 * me[2]), naz = -(na2 * me[3]);
        /* an + (-a2 vB + -a2 rA.rB) as three FMAs onto -a2 vB (apps.cuh) */
        const double sb = fma(naz, o2[3], fma(nay, o2[2], fma(nax, o2[1], na2 * o2[0])));
        const double vij = lava_exp(an + sb);
        const double qv = q * vij;
        const double t = qv + qv;
        fv = fv + qv;
        /* sum_j t (rA - rB) = rA sum_j t - sum_j t rB (apps.cuh
           lava_box_contribution): one FMA per component and pair */
        sx = fma(t, o2[1], sx);
        sy = fma(t, o2[2], sy);
        sz = fma(t, o2[3], sz);
      }
      const double f2 = fv + fv; /* sum_j t, exact */
      out[0] = fv;
      out[1] = fma(me[1], f2, -sx);
      out[2] = fma(me[2], f2, -sy);
      out[3] = fma(me[3], f2, -sz);
      return 0;
    }
    case HPAC_APP_TABLE:
      for (int d = 0; d < rv->out_dims; ++d) out[d] = r->table_out[(size_t)idx * rv->out_dims + d];
      return 0;
    case HPAC_APP_SYNTHETIC:
      out[0] = synthetic_eval(oracle_synthetic_value(r->synthetic_profile, idx, r->seed));
      return 0;
    case HPAC_APP_BLACKSCHOLES:
      if (oracle_black_scholes_call(r->in + (size_t)idx * 5, out))
        return fail(err, el, HPAC_ERR_CONFIG, "black_scholes_call: invalid option parameters");
      return 0;
    case HPAC_APP_BINOMIAL:
      if (oracle_binomial_price(r->in + (size_t)idx * 5, r->binomial_steps, r->binomial_american,
                                r->binomial_put, out))
        return fail(err, el, HPAC_ERR_CONFIG, "binomial_price: invalid option or lattice");
      return 0;
    case HPAC_APP_KMEANS: {
      /* bench/kmeans.hpp:85-95 */
      int dims = r->kmeans_dims, k = r->kmeans_k;
      if (r->table_out) { /* distances precomputed by kmeans_distances (same arithmetic) */
        for (int c = 0; c < k; ++c) out[c] = r->table_out[(size_t)idx * k + c];
        return 0;
      }
      const double* pt = r->in + (size_t)idx * dims;
      for (int c = 0; c < k; ++c) {
        double ssq = 0.0;
        for (int d = 0; d < dims; ++d) {
          double diff = pt[d] - r->centroids[c * dims + d];
          ssq += diff * diff;
        }
        out[c] = sqrt(ssq);
      }
      return 0;
    }
  }
  return fail(err, el, HPAC_ERR_UNSUPPORTED, "oracle: unsupported app %d", r->app);
}

static void region_store(const region_view* rv, int64_t idx, int lane, const double* out) {
  const hpac_region_t* r = rv->r;
  if (r->app == HPAC_APP_LAVAMD) {
    double* f = r->out + (idx * r->lavamd_particles + lane) * 4;
    for (int c = 0; c < 4; ++c) f[c] = f[c] + out[c];
    return;
  }
  if (r->app == HPAC_APP_KMEANS) {
    int k = r->kmeans_k;
    if (r->out)
      for (int c = 0; c < k; ++c) r->out[(size_t)idx * k + c] = out[c];
    /* host argmin, bench/kmeans.hpp:111-121 (strict <, lowest index) */
    int best = 0;
    double bd = out[0];
    for (int c = 1; c < k; ++c)
      if (out[c] < bd) {
        bd = out[c];
        best = c;
      }
    if (r->labels) r->labels[idx] = best;
    return;
  }
  if (!r->out) return;
  if (r->flags & HPAC_REGION_STORE_ACCUMULATE)
    for (int d = 0; d < rv->out_dims; ++d) r->out[(size_t)idx * rv->out_dims + d] += out[d];
  else
    for (int d = 0; d < rv->out_dims; ++d) r->out[(size_t)idx * rv->out_dims + d] = out[d];
}

static int region_bind(const hpac_region_t* r, region_view* rv, char* err, size_t el) {
  rv->r = r;
  switch (r->app) {
    case HPAC_APP_TABLE:
      rv->in_dims = r->input_dims;
      rv->out_dims = r->output_dims;
      if (!r->table_out) return fail(err, el, HPAC_ERR_CONFIG, "region has no evaluate function");
      if (rv->in_dims > 0 && !r->in)
        return fail(err, el, HPAC_ERR_CONFIG, "region declares inputs but has no load_input");
      if (rv->out_dims < 1) return fail(err, el, HPAC_ERR_CONFIG, "region output_dims must be >= 1");
      return 0;
    case HPAC_APP_SYNTHETIC: rv->in_dims = 1; rv->out_dims = 1; return 0;
    case HPAC_APP_BLACKSCHOLES:
    case HPAC_APP_BINOMIAL: rv->in_dims = 5; rv->out_dims = 1; return 0;
    case HPAC_APP_KMEANS:
      rv->in_dims = r->kmeans_dims;
      rv->out_dims = r->kmeans_k;
      return 0;
    case HPAC_APP_LAVAMD:
      rv->in_dims = 0;
      rv->out_dims = 4;
      return 0;
  }
  return fail(err, el, HPAC_ERR_UNSUPPORTED, "oracle: unsupported app %d", r->app);
}

/* ------------------------------------------------------------------ */
/* validation (grid.hpp:27-53, directive.hpp:72-84, taf/iact/perfo)    */
/* ------------------------------------------------------------------ */
static int validate_grid(const hpac_grid_t* g, char* err, size_t el) {
  if (g->num_teams < 1) return fail(err, el, HPAC_ERR_CONFIG, "num_teams must be positive");
  if (g->threads_per_team < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "threads_per_team must be positive");
  if (g->warp_size < 1 || g->warp_size > 64)
    return fail(err, el, HPAC_ERR_CONFIG, "warp_size must be in [1, 64]");
  if (g->threads_per_team % g->warp_size != 0)
    return fail(err, el, HPAC_ERR_CONFIG, "warp_size (%d) must divide threads_per_team (%d)",
                g->warp_size, g->threads_per_team);
  if (g->items_per_thread < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "items_per_thread must be positive");
  return 0;
}

static int validate_spec(const hpac_spec_t* s, char* err, size_t el) {
  switch (s->technique) {
    case HPAC_TECH_TAF:
      if (s->taf_h_size < 1) return fail(err, el, HPAC_ERR_CONFIG, "TAF history size must be >= 1");
      if (s->taf_p_size < 1) return fail(err, el, HPAC_ERR_CONFIG, "TAF prediction size must be >= 1");
      if (!(s->taf_threshold >= 0.0)) return fail(err, el, HPAC_ERR_CONFIG, "TAF threshold must be >= 0");
      break;
    case HPAC_TECH_IACT:
      if (s->iact_table_size < 1) return fail(err, el, HPAC_ERR_CONFIG, "iACT table size must be >= 1");
      if (!(s->iact_threshold >= 0.0))
        return fail(err, el, HPAC_ERR_CONFIG, "iACT threshold must be >= 0");
      if (s->iact_tables_per_warp < 0)
        return fail(err, el, HPAC_ERR_CONFIG, "tables_per_warp must be >= 1");
      break;
    case HPAC_TECH_PERFO:
      if (s->perfo_kind < 0 || s->perfo_kind > HPAC_PERFO_RANDOM)
        return fail(err, el, HPAC_ERR_CONFIG, "unknown perforation kind");
      if (kind_uses_modulus(s->perfo_kind)) {
        if (s->perfo_modulus < 2) return fail(err, el, HPAC_ERR_CONFIG, "perforation modulus must be >= 2");
      } else if (s->perfo_skip_percent < 1 || s->perfo_skip_percent > 99) {
        return fail(err, el, HPAC_ERR_CONFIG, "perforation skip percent must be in [1, 99]");
      }
      break;
    default: return fail(err, el, HPAC_ERR_CONFIG, "ApproxSpec must carry exactly one technique payload");
  }
  if (s->level < HPAC_LEVEL_THREAD || s->level > HPAC_LEVEL_TEAM)
    return fail(err, el, HPAC_ERR_CONFIG, "unknown decision level");
  if (s->technique == HPAC_TECH_IACT && s->n_input_sections < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "iACT requires at least one input section");
  if ((s->technique == HPAC_TECH_IACT || s->technique == HPAC_TECH_TAF) && s->n_output_sections < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "memoization requires at least one output section");
  return 0;
}

/* bind_technique arena charges, engine.hpp:83-116 + SharedArena::alloc_bytes
   (arena.hpp:37-38): the per-team bump allocator throws at the first
   allocation that crosses the budget with required = used + length. */
static int arena_account(const hpac_grid_t* g, const region_view* rv, const hpac_spec_t* s,
                         int tpw, uint64_t* required, uint64_t* available, char* err,
                         size_t el) {
  uint64_t cap = g->shared_mem_budget_bytes, used = 0;
  *available = cap;
  if (s->technique == HPAC_TECH_TAF) {
    uint64_t per = oracle_taf_state_bytes(s->taf_h_size, rv->out_dims);
    for (int t = 0; t < g->threads_per_team; ++t) {
      if (used + per > cap) goto overflow_taf;
      used += per;
      continue;
    overflow_taf:
      *required = used + per;
      return fail(err, el, HPAC_ERR_ARENA_OVERFLOW,
                  "shared arena overflow: required %llu bytes, available %llu bytes",
                  (unsigned long long)*required, (unsigned long long)cap);
    }
  } else if (s->technique == HPAC_TECH_IACT) {
    uint64_t per = oracle_table_group_bytes(tpw, s->iact_table_size, rv->in_dims, rv->out_dims);
    int wpt = g->threads_per_team / g->warp_size;
    for (int w = 0; w < wpt; ++w) {
      if (used + per > cap) {
        *required = used + per;
        return fail(err, el, HPAC_ERR_ARENA_OVERFLOW,
                    "shared arena overflow: required %llu bytes, available %llu bytes",
                    (unsigned long long)*required, (unsigned long long)cap);
      }
      used += per;
    }
  }
  if (s->level == HPAC_LEVEL_TEAM) {
    if (used + 8 > cap) {
      *required = used + 8;
      return fail(err, el, HPAC_ERR_ARENA_OVERFLOW,
                  "shared arena overflow: required %llu bytes, available %llu bytes",
                  (unsigned long long)*required, (unsigned long long)cap);
    }
    used += 8;
  }
  *required = used;
  return 0;
}

ORACLE_API int oracle_arena_required(const hpac_grid_t* g, const hpac_region_t* r,
                                     const hpac_spec_t* s, uint64_t* required,
                                     uint64_t* available, char* err, size_t el) {
  region_view rv;
  int rc = region_bind(r, &rv, err, el);
  if (rc) return rc;
  int tpw = s->iact_tables_per_warp > 0 ? s->iact_tables_per_warp : g->warp_size;
  return arena_account(g, &rv, s, tpw, required, available, err, el);
}

/* ------------------------------------------------------------------ */
/* the engine: run_region, engine.hpp:132-402                          */
/* ------------------------------------------------------------------ */
typedef struct {
  int in_round, predicate, hit;
  int64_t idx;
} lane_work;

/* Teams [team_begin, team_end) of the logical grid only (0, 0 = all): every
   thread keeps its global id and stride, so the executed teams make exactly
   the decisions they make in the whole-grid run (each team's technique state
   is its own); the C-ABI's hpac_launch_t.team_begin/team_end counterpart. */
static int run_region_range(const hpac_grid_t* g, int64_t n, int32_t mapping,
                            const hpac_region_t* reg, const hpac_spec_t* spec, hpac_stats_t* st,
                            uint8_t* paths, int32_t team_begin, int32_t team_end, char* err,
                            size_t el);

ORACLE_API int oracle_run_region(const hpac_grid_t* g, int64_t n, int32_t mapping,
                                 const hpac_region_t* reg, const hpac_spec_t* spec,
                                 hpac_stats_t* st, uint8_t* paths, char* err, size_t el) {
  return run_region_range(g, n, mapping, reg, spec, st, paths, 0, 0, err, el);
}

ORACLE_API int oracle_run_region_teams(const hpac_grid_t* g, int64_t n, int32_t mapping,
                                       const hpac_region_t* reg, const hpac_spec_t* spec,
                                       hpac_stats_t* st, uint8_t* paths, int32_t team_begin,
                                       int32_t team_end, char* err, size_t el) {
  return run_region_range(g, n, mapping, reg, spec, st, paths, team_begin, team_end, err, el);
}

static int run_region_range(const hpac_grid_t* g, int64_t n, int32_t mapping,
                            const hpac_region_t* reg, const hpac_spec_t* spec, hpac_stats_t* st,
                            uint8_t* paths, int32_t team_begin, int32_t team_end, char* err,
                            size_t el) {
  int rc;
  memset(st, 0, sizeof *st);
  if (err && el) err[0] = 0;
  /* grid.validate, check_coverage (engine.hpp:135-137) */
  if ((rc = validate_grid(g, err, el))) return rc;
  if (n < 0) return fail(err, el, HPAC_ERR_CONFIG, "problem size must be non-negative");
  int per_team = mapping == HPAC_MAP_PER_TEAM;
  int64_t cap = per_team ? (int64_t)g->num_teams * g->items_per_thread
                         : (int64_t)g->num_teams * g->threads_per_team * g->items_per_thread;
  if (n > cap)
    return fail(err, el, HPAC_ERR_CONFIG,
                "grid capacity %lld cannot cover problem size %lld (increase num_teams, "
                "threads_per_team, or items_per_thread)",
                (long long)cap, (long long)n);
  region_view rv;
  if ((rc = region_bind(reg, &rv, err, el))) return rc;
  rv.n = n;

  const int tpt = g->threads_per_team, ws = g->warp_size, nteams = g->num_teams;
  const int wpt = tpt / ws;
  const int total_threads = nteams * tpt;
  const int total_warps = nteams * wpt;
  const int64_t stride = per_team ? nteams : total_threads;
  const int64_t steps = n <= 0 ? 0 : (n + stride - 1) / stride;
  const int in_dims = rv.in_dims, out_dims = rv.out_dims;
  const int has_enc = (reg->app == HPAC_APP_TABLE && reg->encounters != NULL) || reg->app == HPAC_APP_LAVAMD;
  const int barrier_eval = (reg->flags & HPAC_REGION_BARRIER_IN_EVALUATE) != 0;

  /* bind_technique, engine.hpp:75-117 */
  int tech = spec ? spec->technique : -1;
  int level = HPAC_LEVEL_THREAD;
  int tpw = 0;
  if (spec) {
    if ((rc = validate_spec(spec, err, el))) return rc;
    level = spec->level;
    if (tech == HPAC_TECH_IACT) {
      if (in_dims < 1) return fail(err, el, HPAC_ERR_CONFIG, "iACT requires a region with inputs");
      tpw = spec->iact_tables_per_warp > 0 ? spec->iact_tables_per_warp : ws;
      if (tpw < 1 || ws % tpw != 0)
        return fail(err, el, HPAC_ERR_CONFIG, "tables_per_warp (%d) must divide warp_size (%d)",
                    tpw, ws);
    }
    uint64_t req = 0, avail = 0;
    rc = arena_account(g, &rv, spec, tpw, &req, &avail, err, el);
    st->arena_required = req;
    st->arena_available = avail;
    if (rc) return rc;
  }
  const int voting = spec && level != HPAC_LEVEL_THREAD;

  /* technique state */
  taf_state* taf = NULL;
  double *taf_ring = NULL, *taf_last = NULL;
  memo_table* tables = NULL;
  double *tab_in = NULL, *tab_out = NULL;
  int64_t *pcount = NULL, *hcount = NULL, *trips = NULL;
  if (tech == HPAC_TECH_TAF) {
    int h = spec->taf_h_size;
    taf = (taf_state*)malloc(sizeof(taf_state) * (size_t)total_threads);
    taf_ring = (double*)malloc(sizeof(double) * (size_t)total_threads * h * out_dims);
    taf_last = (double*)malloc(sizeof(double) * (size_t)total_threads * out_dims);
    for (int t = 0; t < total_threads; ++t)
      taf_init(&taf[t], h, spec->taf_p_size, spec->taf_threshold, out_dims,
               taf_ring + (size_t)t * h * out_dims, taf_last + (size_t)t * out_dims);
  } else if (tech == HPAC_TECH_IACT) {
    int ntab = total_warps * tpw, ts = spec->iact_table_size;
    tables = (memo_table*)malloc(sizeof(memo_table) * (size_t)ntab);
    tab_in = (double*)calloc((size_t)ntab * ts * in_dims, sizeof(double));
    tab_out = (double*)calloc((size_t)ntab * ts * out_dims, sizeof(double));
    for (int t = 0; t < ntab; ++t) {
      tables[t].cap = ts;
      tables[t].in_dims = in_dims;
      tables[t].out_dims = out_dims;
      tables[t].rr = tables[t].occ = 0;
      tables[t].in = tab_in + (size_t)t * ts * in_dims;
      tables[t].out = tab_out + (size_t)t * ts * out_dims;
    }
  } else if (tech == HPAC_TECH_PERFO) {
    pcount = (int64_t*)calloc((size_t)total_threads, sizeof(int64_t));
    hcount = (int64_t*)calloc((size_t)total_warps, sizeof(int64_t));
    if (spec->perfo_kind == HPAC_PERFO_INI || spec->perfo_kind == HPAC_PERFO_FINI) {
      /* engine.hpp:171-186 */
      if (has_enc) {
        free(pcount);
        free(hcount);
        return fail(err, el, HPAC_ERR_CONFIG,
                    "INI/FINI perforation requires a fixed trip count per thread");
      }
      trips = (int64_t*)calloc((size_t)total_threads, sizeof(int64_t));
      for (int tid = 0; tid < total_threads; ++tid) {
        int64_t owner = per_team ? tid / tpt : tid, cnt = 0;
        for (int64_t s = 0; s < steps; ++s)
          if (owner + s * stride < n) ++cnt;
        trips[tid] = cnt;
      }
    }
  }

  lane_work* lanes = (lane_work*)calloc((size_t)tpt, sizeof(lane_work));
  double* lin = (double*)calloc((size_t)tpt * (in_dims > 0 ? in_dims : 1), sizeof(double));
  double* lout = (double*)calloc((size_t)tpt * out_dims, sizeof(double));
  int* arrivals = (int*)calloc((size_t)tpt, sizeof(int));
  uint8_t* touched = (uint8_t*)calloc((size_t)total_warps, 1);
  int* miss = (int*)malloc(sizeof(int) * (size_t)ws);
  uint8_t* lpath = (uint8_t*)malloc((size_t)ws); /* 0 inactive, 1 accurate, 2 approx */
  rc = 0;

  const int tb = (team_begin || team_end) ? team_begin : 0;
  const int te = (team_begin || team_end) ? team_end : nteams;
  if (tb < 0 || te > nteams || tb > te) {
    rc = fail(err, el, HPAC_ERR_CONFIG, "team range [%d, %d) outside the grid's %d teams", tb, te,
              nteams);
  }
  for (int64_t step = 0; step < steps && !rc; ++step) {
    for (int team = tb; team < te && !rc; ++team) {
      int rounds = 0;
      for (int local = 0; local < tpt; ++local) {
        int tid = team * tpt + local;
        int64_t owner = per_team ? team : tid;
        int64_t idx = owner + step * stride;
        lanes[local].idx = idx < n ? idx : -1;
        lanes[local].in_round = 0;
        arrivals[local] = 0;
        if (lanes[local].idx >= 0) {
          int e = has_enc ? region_encounters(&rv, idx) : 1;
          if (e > rounds) rounds = e;
        }
      }

      for (int round = 0; round < rounds && !rc; ++round) {
        /* predicate phase, engine.hpp:221-251 */
        int team_active = 0;
        for (int local = 0; local < tpt; ++local) {
          lane_work* lw = &lanes[local];
          int tid = team * tpt + local, warp_id = team * wpt + local / ws, lane = local % ws;
          lw->in_round = lw->idx >= 0 && round < (has_enc ? region_encounters(&rv, lw->idx) : 1);
          lw->predicate = 0;
          lw->hit = -1;
          if (!lw->in_round) continue;
          ++team_active;
          double* in = lin + (size_t)local * (in_dims > 0 ? in_dims : 1);
          if (in_dims > 0) region_load(&rv, lw->idx, in);
          if (tech == HPAC_TECH_TAF) {
            lw->predicate = taf[tid].mode == TAF_PREDICTING;
          } else if (tech == HPAC_TECH_IACT) {
            memo_table* t = &tables[warp_id * tpw + lane / (ws / tpw)];
            lw->hit = memo_lookup(t, in, spec->iact_threshold);
            lw->predicate = lw->hit >= 0;
          } else if (tech == HPAC_TECH_PERFO) {
            int64_t key = kind_is_herded(spec->perfo_kind) ? hcount[warp_id] : pcount[tid];
            int64_t trip = trips ? trips[tid] : 0;
            /* RANDOM keys on the work owner: the thread, or the team under
               per-team mapping (keeps team-uniform decisions there) */
            lw->predicate = should_skip(spec, key, trip, per_team ? team : tid);
          }
        }
        if (team_active == 0) continue;

        /* team vote, engine.hpp:257-280 / decide_team hierarchy.hpp:56-70 */
        int have_team = 0, team_dec = 0;
        if (voting && level == HPAC_LEVEL_TEAM) {
          int yes = 0, act = 0;
          for (int local = 0; local < tpt; ++local)
            if (lanes[local].in_round) {
              ++act;
              if (lanes[local].predicate) ++yes;
            }
          team_dec = 2 * yes > act;
          have_team = 1;
          for (int local = 0; local < tpt; ++local)
            if (lanes[local].idx >= 0) arrivals[local] += 1;
        }

        for (int w = 0; w < wpt && !rc; ++w) {
          int warp_id = team * wpt + w;
          int any = 0;
          for (int lane = 0; lane < ws; ++lane) any |= lanes[w * ws + lane].in_round;
          if (!any) continue;
          touched[warp_id] = 1;
          int have_dec = have_team, dec = team_dec;
          if (voting && level == HPAC_LEVEL_WARP) {
            /* decide_warp, hierarchy.hpp:42-50 */
            int yes = 0, act = 0;
            for (int lane = 0; lane < ws; ++lane)
              if (lanes[w * ws + lane].in_round) {
                ++act;
                if (lanes[w * ws + lane].predicate) ++yes;
              }
            dec = 2 * yes > act;
            have_dec = 1;
          }
          int nmiss = 0, nacc = 0, napp = 0;
          /* lane execution, engine.hpp:303-347 */
          for (int lane = 0; lane < ws && !rc; ++lane) {
            int local = w * ws + lane, tid = team * tpt + local;
            lane_work* lw = &lanes[local];
            lpath[lane] = 0;
            if (!lw->in_round) continue;
            int approx = have_dec ? dec : lw->predicate;
            double* out = lout + (size_t)local * out_dims;
            double* in = lin + (size_t)local * (in_dims > 0 ? in_dims : 1);
            if (approx) {
              if (tech == HPAC_TECH_TAF) {
                taf_emit(&taf[tid], out);
                region_store(&rv, lw->idx, local, out);
              } else if (tech == HPAC_TECH_IACT) {
                memo_table* t = &tables[warp_id * tpw + lane / (ws / tpw)];
                if (lw->hit >= 0) {
                  region_store(&rv, lw->idx, local, t->out + (size_t)lw->hit * out_dims);
                } else if (t->occ > 0) {
                  int s = memo_nearest(t, in);
                  region_store(&rv, lw->idx, local, t->out + (size_t)s * out_dims);
                } else {
                  approx = 0; /* empty table: accurate fallback */
                }
              }
              /* perforation skip: output untouched */
            }
            if (!approx) {
              rc = region_eval(&rv, lw->idx, local, round, out, err, el);
              if (rc) break;
              if (barrier_eval) arrivals[local] += 1;
              region_store(&rv, lw->idx, local, out);
              if (tech == HPAC_TECH_TAF) taf_observe(&taf[tid], out);
              if (tech == HPAC_TECH_IACT && lw->hit < 0) miss[nmiss++] = lane;
            }
            lpath[lane] = approx ? 2 : 1;
            if (approx) ++napp; else ++nacc;
            st->total_invocations += 1;
            if (approx) st->approx_invocations += 1;
            if (paths && (!per_team || local == 0) && round < 8)
              paths[lw->idx] |= (uint8_t)((approx ? 1u : 0u) << round);
          }
          if (rc) break;

          /* iACT write phase, engine.hpp:351-366 / select_writer iact.hpp:166-180 */
          if (tech == HPAC_TECH_IACT && nmiss > 0) {
            int group = ws / tpw;
            for (int t = 0; t < tpw; ++t) {
              memo_table* tb = &tables[warp_id * tpw + t];
              int best_lane = -1;
              double best_d = -1.0;
              for (int m = 0; m < nmiss; ++m) {
                int lane = miss[m];
                if (lane / group != t) continue;
                double d = memo_min_distance(tb, lin + (size_t)(w * ws + lane) * in_dims);
                if (best_lane < 0 || d > best_d || (d == best_d && lane < best_lane)) {
                  best_lane = lane;
                  best_d = d;
                }
              }
              if (best_lane < 0) continue;
              int local = w * ws + best_lane;
              memo_insert(tb, lin + (size_t)local * in_dims, lout + (size_t)local * out_dims);
            }
          }

          /* perforation counters, engine.hpp:368-373 */
          if (tech == HPAC_TECH_PERFO) {
            for (int lane = 0; lane < ws; ++lane)
              if (lanes[w * ws + lane].in_round) pcount[team * tpt + w * ws + lane] += 1;
            hcount[warp_id] += 1;
          }

          /* accumulate_cost stats, cost.hpp:66-86 */
          if (nacc + napp > 0) {
            st->total_warp_steps += 1;
            if (nacc > 0 && napp > 0) st->divergent_warp_steps += 1;
          }
        }
      }
      if (rc) break;

      /* TeamState::end_step barrier check, machine.hpp:53-61; engine.hpp:382-386 */
      int maxa = 0, missing = 0;
      for (int local = 0; local < tpt; ++local)
        if (lanes[local].idx >= 0 && arrivals[local] > maxa) maxa = arrivals[local];
      for (int local = 0; local < tpt; ++local)
        if (lanes[local].idx >= 0 && arrivals[local] < maxa) ++missing;
      if (missing) {
        st->barrier_divergence_detected = 1;
        st->fail_team = team;
        st->fail_step = step;
        st->fail_missing = missing;
        rc = fail(err, el, HPAC_ERR_BARRIER_DIVERGENCE,
                  "barrier divergence in team %d at step %lld: %d thread(s) never arrived", team,
                  (long long)step, missing);
      }
    }
  }

  for (int w = 0; w < total_warps; ++w) st->resident_warps += touched[w];

  free(lanes);
  free(lin);
  free(lout);
  free(arrivals);
  free(touched);
  free(miss);
  free(lpath);
  free(taf);
  free(taf_ring);
  free(taf_last);
  free(tables);
  free(tab_in);
  free(tab_out);
  free(pcount);
  free(hcount);
  free(trips);
  return rc;
}

/* ------------------------------------------------------------------ */
/* K-Means Lloyd loop, bench/kmeans.hpp:62-144                         */
/* ------------------------------------------------------------------ */
/* All n*k distances of one iteration, the region's evaluate arithmetic
   (bench/kmeans.hpp:85-95: no-FMA sum in dimension order, IEEE sqrt) per
   point; points are independent, so the threads only change the speed. The
   engine then reads them instead of recomputing each evaluated point. */
static void kmeans_distances(const double* points, int64_t n, int dims, int k, const double* cent,
                             double* dcache) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* pt = points + (size_t)i * dims;
    for (int c = 0; c < k; ++c) {
      double ssq = 0.0;
      for (int d = 0; d < dims; ++d) {
        double diff = pt[d] - cent[c * dims + d];
        ssq += diff * diff;
      }
      dcache[(size_t)i * k + c] = sqrt(ssq);
    }
  }
}

ORACLE_API int oracle_kmeans_benchmark(const double* points, int64_t n, int dims, int k,
                                       const hpac_grid_t* g, const hpac_spec_t* spec,
                                       int max_iters, uint64_t perfo_seed_base,
                                       int32_t* assignments, double* centroids_out,
                                       int32_t* iterations, int32_t* converged,
                                       hpac_stats_t* total, char* err, size_t el) {
  double* cent = (double*)malloc(sizeof(double) * (size_t)k * dims);
  double* dist = (double*)calloc((size_t)n * k, sizeof(double));
  double* dcache = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * k);
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  double* sums = (double*)malloc(sizeof(double) * (size_t)k * dims);
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  int rc = 0;
  /* Forgy init on the first k points (kmeans.hpp:66-71) */
  for (int c = 0; c < k; ++c) {
    int64_t src = c < n - 1 ? c : n - 1;
    for (int d = 0; d < dims; ++d) cent[c * dims + d] = points[src * dims + d];
  }
  for (int64_t i = 0; i < n; ++i) assignments[i] = -1;
  memset(total, 0, sizeof *total);
  *iterations = 0;
  *converged = 0;
  hpac_region_t r;
  memset(&r, 0, sizeof r);
  r.app = HPAC_APP_KMEANS;
  r.kmeans_dims = dims;
  r.kmeans_k = k;
  r.in = points;
  r.centroids = cent;
  r.out = dist;
  r.table_out = dcache;
  r.labels = NULL;
  hpac_spec_t sp;
  if (spec) sp = *spec;
  for (int iter = 1; iter <= max_iters; ++iter) {
    hpac_stats_t st;
    if (spec && spec->technique == HPAC_TECH_PERFO && spec->perfo_kind == HPAC_PERFO_RANDOM)
      sp.perfo_seed = perfo_seed_base + (uint64_t)iter;
    /* RANDOM extension: the first iteration is exact (a skipped point must
       have a stale label to keep; the reference modes keep label 0) */
    const int exact_iter = spec && spec->technique == HPAC_TECH_PERFO &&
                           spec->perfo_kind == HPAC_PERFO_RANDOM && iter == 1;
    kmeans_distances(points, n, dims, k, cent, dcache);
    rc = oracle_run_region(g, n, HPAC_MAP_PER_THREAD, &r, (spec && !exact_iter) ? &sp : NULL, &st,
                           NULL, err, el);
    if (rc) break;
    total->total_invocations += st.total_invocations;
    total->approx_invocations += st.approx_invocations;
    total->divergent_warp_steps += st.divergent_warp_steps;
    total->total_warp_steps += st.total_warp_steps;
    *iterations = iter;
    int changed = 0;
    for (int64_t i = 0; i < n; ++i) {
      int best = 0;
      double bd = dist[i * k];
      for (int c = 1; c < k; ++c)
        if (dist[i * k + c] < bd) {
          bd = dist[i * k + c];
          best = c;
        }
      next[i] = best;
      if (best != assignments[i]) changed = 1;
    }
    memcpy(assignments, next, sizeof(int32_t) * (size_t)n);
    if (!changed) {
      *converged = 1;
      break;
    }
    for (int i = 0; i < k * dims; ++i) sums[i] = 0.0;
    for (int c = 0; c < k; ++c) counts[c] = 0;
    for (int64_t i = 0; i < n; ++i) {
      int c = assignments[i];
      counts[c] += 1;
      for (int d = 0; d < dims; ++d) sums[c * dims + d] += points[i * dims + d];
    }
    for (int c = 0; c < k; ++c) {
      if (counts[c] == 0) continue;
      for (int d = 0; d < dims; ++d) cent[c * dims + d] = sums[c * dims + d] / counts[c];
    }
  }
  if (centroids_out) memcpy(centroids_out, cent, sizeof(double) * (size_t)k * dims);
  free(cent);
  free(dist);
  free(dcache);
  free(next);
  free(sums);
  free(counts);
  return rc;
}

/* ------------------------------------------------------------------ */
/* metrics, metrics.hpp:17-45                                          */
/* ------------------------------------------------------------------ */
ORACLE_API double oracle_mape(const double* acc, const double* app, int64_t n) {
  if (n == 0) return 0.0;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = acc[i], b = app[i];
    if (a == 0.0) {
      if (b == 0.0) continue;
      return INFINITY;
    }
    sum += fabs(a - b) / fabs(a);
  }
  return sum / (double)n;
}

ORACLE_API double oracle_mcr(const int32_t* acc, const int32_t* app, int64_t n) {
  if (n == 0) return 0.0;
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) m += acc[i] != app[i];
  return (double)m / (double)n;
}
