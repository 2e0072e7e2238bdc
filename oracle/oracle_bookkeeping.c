/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h for the parity status).
 * Bookkeeping half: compiled with -ffp-contract=off so every double
 * expression rounds exactly like the reference build.
 *
 * Bookkeeping restates /root/reference/proj:
 *   Rng                      rng.hpp:13-39
 *   expected_accept_length   perf_model.cpp:159-169
 *   sample_accept_length     perf_model.cpp:171-177
 *   bisect_increasing        perf_model.cpp:30-41
 *   alpha_from_accept_length perf_model.cpp:213-224
 *   SignalGeometry / extract_signals byte accounting
 *   chronological 9:1 split
 * The neural step follows SURVEY.md Appendix A (no reference code exists).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ======================================================== mt19937_64 + Rng */
#define MT_N 312
#define MT_M 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MT_MATRIX_A;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:18 — 53 high bits scaled by 2^-53 */
double orc_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:21-26 — Box-Muller, cosine branch, u1 in (0, 1] */
double orc_normal(orc_rng* r, double mean, double sd) {
  double u1 = 1.0 - orc_uniform(r);
  double u2 = orc_uniform(r);
  return mean + sd * sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* rng.hpp:29-35 — inverse-CDF geometric on {1, 2, ...} */
int64_t orc_geometric(orc_rng* r, double mean) {
  if (mean <= 1.0) return 1;
  const double p = 1.0 / mean;
  const double u = orc_uniform(r);
  const double k = floor(log1p(-u) / log1p(-p));
  return 1 + (int64_t)(k > 0.0 ? k : 0.0);
}

/* ====================================================== accept-length math */
static int bad_alpha(double a) { return !(a >= 0.0 && a <= 1.0); }

int orc_expected_accept_length(double alpha, int gamma, double* out) {
  if (bad_alpha(alpha) || gamma < 1) return 1;
  double sum = 1.0, term = 1.0;
  for (int k = 1; k <= gamma; ++k) {
    term *= alpha;
    sum += term;
  }
  *out = sum;
  return 0;
}

int orc_sample_accept_length(orc_rng* r, double alpha, int gamma, int* out) {
  if (bad_alpha(alpha) || gamma < 1) return 1;
  int accepted = 0;
  while (accepted < gamma && orc_uniform(r) < alpha) ++accepted;
  *out = accepted + 1;
  return 0;
}

int orc_alpha_from_accept_length(double ell, int gamma, double* out) {
  if (gamma < 1) return 1;
  if (!(ell >= 1.0 && ell <= gamma + 1.0)) return 1;
  if (ell <= 1.0) {
    *out = 0.0;
    return 0;
  }
  if (ell >= gamma + 1.0) {
    *out = 1.0;
    return 0;
  }
  double lo = 0.0, hi = 1.0;
  while (hi - lo > 1e-6) { /* kBisectionTol, perf_model.hpp:83 */
    const double mid = 0.5 * (lo + hi);
    double f;
    orc_expected_accept_length(mid, gamma, &f);
    if (f < ell)
      lo = mid;
    else
      hi = mid;
  }
  *out = 0.5 * (lo + hi);
  return 0;
}

void orc_split_train_eval(int64_t n, int64_t* n_train, int64_t* n_eval) {
  const int64_t t = n > 0 ? (9 * n) / 10 : 0;
  *n_train = t;
  *n_eval = n > 0 ? n - t : 0;
}

int64_t orc_bytes_per_token(int hidden, int layers, int bytes_per_element) {
  return (int64_t)layers * hidden * bytes_per_element;
}

void orc_extract_signals(int64_t* st, int64_t n, int64_t bpt, int64_t flush_threshold) {
  if (n <= 0) return;
  st[0] += n;
  st[1] += n * bpt;
  if (st[1] > flush_threshold) {
    st[3] += st[1];
    st[1] = 0;
    st[2] += 1;
  }
}

/* ============================================================ bf16 helpers */
uint16_t orc_f32_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40); /* NaN */
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================= synthetic capture */
int orc_synth_capture(uint64_t seed, int64_t index, int length, int vocab, int hidden,
                      int layers, double alpha, int gamma, int32_t* ids, uint16_t* features,
                      int32_t* accept_lengths, int32_t* n_steps, double* alpha_s) {
  if (length < 1 || vocab < 1 || hidden < 1 || layers < 1) return 1;
  if (bad_alpha(alpha) || gamma < 1) return 1;
  orc_rng r;
  orc_rng_seed(&r, seed + (uint64_t)index);
  int total = 0, steps = 0;
  while (total < length) {
    int k;
    orc_sample_accept_length(&r, alpha, gamma, &k);
    if (k > length - total) k = length - total; /* SPEC.md:294 truncation */
    if (accept_lengths) accept_lengths[steps] = k;
    total += k;
    ++steps;
  }
  if (n_steps) *n_steps = steps;
  if (alpha_s) orc_alpha_from_accept_length((double)length / steps, gamma, alpha_s);
  for (int i = 0; i < length; ++i) {
    int32_t id = (int32_t)floor(orc_uniform(&r) * vocab);
    if (ids) ids[i] = id;
  }
  if (features) {
    const int64_t w = (int64_t)layers * hidden;
    for (int64_t i = 0; i < (int64_t)length * w; ++i)
      features[i] = orc_f32_to_bf16((float)orc_normal(&r, 0.0, 1.0));
  }
  return 0;
}

void orc_init_normal_block(uint64_t seed_base, int p, int64_t n, float* out) {
  const int64_t nblk = (n + (1 << 20) - 1) >> 20;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < nblk; ++j) {
    orc_rng r;
    orc_rng_seed(&r, seed_base + ((uint64_t)p << 32) + (uint64_t)j);
    const int64_t e0 = j << 20, e1 = (e0 + (1 << 20)) < n ? e0 + (1 << 20) : n;
    for (int64_t e = e0; e < e1; ++e) out[e] = (float)orc_normal(&r, 0.0, 0.02);
  }
}

