/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h for the parity status).
 * Model half: the draft-head step of SURVEY.md Appendix A (no reference code
 * exists for it; cross-checked against torch autograd in
 * tests/test_oracle_vs_torch.py).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline float rb(float x) { return orc_bf16_to_f32(orc_f32_to_bf16(x)); }

static void round_vec(float* x, int64_t n, int on) {
  if (!on) return;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) x[i] = rb(x[i]);
}

/* ========================================================== param layout */
int64_t orc_param_layout(const orc_shape* s, const char** names, int64_t* rows, int64_t* cols,
                         int64_t* offsets) {
  static const char* N[ORC_NPARAMS] = {"fc",     "w_in",    "w_hid", "qkv",   "o",
                                       "w_post", "gate_up", "down",  "w_fin", "lm_head"};
  const int64_t H = s->H, Q = (int64_t)s->nh * s->hd, KV = (int64_t)s->nkv * s->hd;
  const int64_t R[ORC_NPARAMS] = {H, 1, 1, Q + 2 * KV, H, 1, 2 * (int64_t)s->I, H, 1, s->V};
  const int64_t Cc[ORC_NPARAMS] = {(int64_t)s->layers * H, H, H, 2 * H, Q, H, H, s->I, H, H};
  int64_t off = 0;
  for (int p = 0; p < ORC_NPARAMS; ++p) {
    if (names) names[p] = N[p];
    if (rows) rows[p] = R[p];
    if (cols) cols[p] = Cc[p];
    if (offsets) offsets[p] = off;
    off += R[p] * Cc[p];
  }
  return off;
}

/* ========================================================= batch assembly */
void orc_gather_batch(const orc_shape* s, int nsamples, const int32_t* const* ids,
                      const uint16_t* const* feats, const int32_t* lens, uint16_t* F,
                      int32_t* u, int32_t* y, int32_t* m) {
  const int64_t w = (int64_t)s->layers * s->H;
  for (int b = 0; b < s->B; ++b) {
    const int L = b < nsamples ? lens[b] : 0;
    for (int t = 0; t < s->S; ++t) {
      const int64_t row = (int64_t)b * s->S + t;
      if (t < L)
        memcpy(F + row * w, feats[b] + (int64_t)t * w, (size_t)w * 2);
      else
        memset(F + row * w, 0, (size_t)w * 2);
      u[row] = (t + 1 < L) ? ids[b][t + 1] : 0;
      y[row] = (t + 2 < L) ? ids[b][t + 2] : 0;
      m[row] = (t + 2 < L) ? 1 : 0;
    }
  }
}

/* ============================================================== dense math */
/* C[M,N] (+)= A[M,K] . B[N,K]^T, fp32.  Packed, register-blocked GEMM:
 * B is packed per (128-column block, 256-deep K block) into 16-wide panels,
 * A into 6-row panels; a 6x16 AVX2/FMA micro-kernel keeps the C tile in 12
 * ymm registers (outer products: 2 B loads + 6 broadcasts per 12 FMAs).
 * Parallel over column blocks (each thread owns disjoint C columns). */
#include <immintrin.h>

enum { MR = 6, NR = 16, KC = 256, NB = 128, MB = 96 };

static void micro_6x16(int64_t kc, const float* Ap, const float* Bp, float* C, int64_t ldc,
                       int mr, int nr) {
  __m256 c[MR][2];
  for (int i = 0; i < MR; ++i) c[i][0] = c[i][1] = _mm256_setzero_ps();
  for (int64_t k = 0; k < kc; ++k) {
    const __m256 b0 = _mm256_loadu_ps(Bp + k * NR), b1 = _mm256_loadu_ps(Bp + k * NR + 8);
    const float* a = Ap + k * MR;
    for (int i = 0; i < MR; ++i) {
      const __m256 ai = _mm256_broadcast_ss(a + i);
      c[i][0] = _mm256_fmadd_ps(ai, b0, c[i][0]);
      c[i][1] = _mm256_fmadd_ps(ai, b1, c[i][1]);
    }
  }
  if (mr == MR && nr == NR) {
    for (int i = 0; i < MR; ++i) {
      float* cr = C + i * ldc;
      _mm256_storeu_ps(cr, _mm256_add_ps(_mm256_loadu_ps(cr), c[i][0]));
      _mm256_storeu_ps(cr + 8, _mm256_add_ps(_mm256_loadu_ps(cr + 8), c[i][1]));
    }
  } else {
    float t[MR][NR];
    for (int i = 0; i < MR; ++i) {
      _mm256_storeu_ps(t[i], c[i][0]);
      _mm256_storeu_ps(t[i] + 8, c[i][1]);
    }
    for (int i = 0; i < mr; ++i)
      for (int j = 0; j < nr; ++j) C[i * ldc + j] += t[i][j];
  }
}

/* C[M,N] (+)= op(A) op(B)^T with op(A)[i][k] = at ? A[k*lda+i] : A[i*lda+k] and
 * op(B)[j][k] = bt ? B[k*ldb+j] : B[j*ldb+k]: the transposes happen while
 * packing, never as separate passes. */
static void mm_gen(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int at,
                   const float* B, int64_t ldb, int bt, float* C, int64_t ldc, int accumulate) {
  const int64_t nblocks = (N + NB - 1) / NB;
#pragma omp parallel
  {
    float* Bp = (float*)aligned_alloc(64, sizeof(float) * NB * KC);
    float* Ap = (float*)aligned_alloc(64, sizeof(float) * (MB + MR) * KC);
#pragma omp for schedule(dynamic, 1)
    for (int64_t jb = 0; jb < nblocks; ++jb) {
      const int64_t j0 = jb * NB, nj = (j0 + NB < N ? NB : N - j0);
      if (!accumulate)
        for (int64_t i = 0; i < M; ++i) memset(C + i * ldc + j0, 0, sizeof(float) * nj);
      for (int64_t k0 = 0; k0 < K; k0 += KC) {
        const int64_t kc = (k0 + KC < K ? KC : K - k0);
        /* pack B[j0 .. j0+nj) x [k0 .. k0+kc) into 16-column panels, k-major */
        for (int64_t p = 0; p < (nj + NR - 1) / NR; ++p)
          for (int64_t k = 0; k < kc; ++k)
            for (int j = 0; j < NR; ++j) {
              const int64_t jj = p * NR + j;
              Bp[(p * KC + k) * NR + j] =
                  jj < nj ? (bt ? B[(k0 + k) * ldb + j0 + jj] : B[(j0 + jj) * ldb + k0 + k]) : 0.f;
            }
        for (int64_t i0 = 0; i0 < M; i0 += MB) {
          const int64_t mi = (i0 + MB < M ? MB : M - i0);
          /* pack A rows into 6-row panels, k-major */
          for (int64_t p = 0; p < (mi + MR - 1) / MR; ++p)
            for (int64_t k = 0; k < kc; ++k)
              for (int i = 0; i < MR; ++i) {
                const int64_t ii = p * MR + i;
                Ap[(p * KC + k) * MR + i] =
                    ii < mi ? (at ? A[(k0 + k) * lda + i0 + ii] : A[(i0 + ii) * lda + k0 + k]) : 0.f;
              }
          for (int64_t pi = 0; pi < (mi + MR - 1) / MR; ++pi)
            for (int64_t pj = 0; pj < (nj + NR - 1) / NR; ++pj) {
              const int mr = (int)((mi - pi * MR) < MR ? (mi - pi * MR) : MR);
              const int nr = (int)((nj - pj * NR) < NR ? (nj - pj * NR) : NR);
              micro_6x16(kc, Ap + pi * KC * MR, Bp + pj * KC * NR,
                         C + (i0 + pi * MR) * ldc + j0 + pj * NR, ldc, mr, nr);
            }
        }
      }
    }
    free(Bp);
    free(Ap);
  }
}

static void mm_nt(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, int accumulate) {
  mm_gen(M, N, K, A, lda, 0, B, ldb, 0, C, ldc, accumulate);
}

/* C[M,K'] (+)= A[M,N'] . B[N',K']  (data-gradient form) */
static void mm_nn(int64_t M, int64_t Kp, int64_t Np, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, int accumulate) {
  mm_gen(M, Kp, Np, A, lda, 0, B, ldb, 1, C, ldc, accumulate);
}

/* C[N,K] = A[T,N]^T . X[T,K]  (weight-gradient form) */
static void mm_tn(int64_t N, int64_t K, int64_t T, const float* A, int64_t lda, const float* X,
                  int64_t ldx, float* C, int64_t ldc) {
  mm_gen(N, K, T, A, lda, 1, X, ldx, 1, C, ldc, 0);
}

static float* falloc(int64_t n) { return (float*)calloc((size_t)n, sizeof(float)); }

/* optional section timing (ORACLE_PROFILE=1), printed to stderr */
static double prof_t0 = 0;
static int prof_on = -1;
static void prof(const char* what) {
  if (prof_on < 0) prof_on = getenv("ORACLE_PROFILE") != NULL;
  if (!prof_on) return;
#ifdef _OPENMP
  const double t = omp_get_wtime();
#else
  const double t = 0;
#endif
  if (what) fprintf(stderr, "[oracle] %-28s %8.3f s\n", what, t - prof_t0);
  prof_t0 = t;
}

/* y = x * rstd * w ; returns rstd per row */
static void rmsnorm_fwd(int64_t T, int64_t H, const float* x, int64_t ldx, const float* w,
                        float eps, float* y, int64_t ldy, float* rstd) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const float* xr = x + t * ldx;
    double ss = 0.0;
    for (int64_t i = 0; i < H; ++i) ss += (double)xr[i] * xr[i];
    const float r = 1.0f / sqrtf((float)(ss / (double)H) + eps);
    rstd[t] = r;
    for (int64_t i = 0; i < H; ++i) y[t * ldy + i] = xr[i] * r * w[i];
  }
}

/* dx (+)= rstd * (dy*w) - x * rstd^3 * mean((dy*w) * x) ; dw += sum_t dy * x * rstd */
static void rmsnorm_bwd(int64_t T, int64_t H, const float* dy, int64_t lddy, const float* x,
                        int64_t ldx, const float* w, const float* rstd, float* dx, int64_t lddx,
                        int accumulate_dx, float* dw) {
  if (dx) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      const float* g = dy + t * lddy;
      const float* xr = x + t * ldx;
      double dot = 0.0;
      for (int64_t i = 0; i < H; ++i) dot += (double)g[i] * w[i] * xr[i];
      const float r = rstd[t];
      const float c = (float)(dot / (double)H) * r * r * r;
      for (int64_t i = 0; i < H; ++i) {
        const float v = r * g[i] * w[i] - xr[i] * c;
        if (accumulate_dx)
          dx[t * lddx + i] += v;
        else
          dx[t * lddx + i] = v;
      }
    }
  }
  if (dw) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H; ++i) {
      double s = 0.0;
      for (int64_t t = 0; t < T; ++t) s += (double)dy[t * lddy + i] * x[t * ldx + i] * rstd[t];
      dw[i] = (float)s;
    }
  }
}

/* NeoX rotate-half tables: cos/sin[pos * half + i], angle = pos * theta^(-2i/hd) in double */
static void rope_tables(int S, int hd, double theta, float* cs, float* sn) {
  const int half = hd / 2;
  for (int p = 0; p < S; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = pow(theta, -2.0 * (double)i / (double)hd);
      const double a = (double)p * inv;
      cs[p * half + i] = (float)cos(a);
      sn[p * half + i] = (float)sin(a);
    }
}

/* in-place rotation of n_heads vectors of one row; inverse = transpose rotation */
static void rope_row(float* x, int n_heads, int hd, const float* cs, const float* sn, int inverse) {
  const int half = hd / 2;
  for (int h = 0; h < n_heads; ++h) {
    float* v = x + (int64_t)h * hd;
    for (int i = 0; i < half; ++i) {
      const float c = cs[i], s = sn[i];
      const float x1 = v[i], x2 = v[i + half];
      if (!inverse) {
        v[i] = x1 * c - x2 * s;
        v[i + half] = x2 * c + x1 * s;
      } else {
        v[i] = x1 * c + x2 * s;
        v[i + half] = x2 * c - x1 * s;
      }
    }
  }
}

static float silu(float x) { return x / (1.0f + expf(-x)); }

/* ============================================================ model state */
typedef struct acts {
  int64_t T, H, Q, KV, NQKV, I, V, W3;
  float *F, *E_rows, *g, *U, *rstd_a, *rstd_b, *qkv, *o, *lse_attn, *r, *z, *rstd_post, *gu,
      *act, *h, *nrm, *rstd_fin, *lse, *dlog;
  int32_t* argmax;
  float *cs, *sn;
} acts;

static void acts_free(acts* a) {
  float** ptrs[] = {&a->F,   &a->E_rows, &a->g,   &a->U,   &a->rstd_a,   &a->rstd_b, &a->qkv,
                    &a->o,   &a->lse_attn, &a->r, &a->z,   &a->rstd_post, &a->gu,    &a->act,
                    &a->h,   &a->nrm,    &a->rstd_fin, &a->lse, &a->dlog, &a->cs,     &a->sn};
  for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) {
    free(*ptrs[i]);
    *ptrs[i] = NULL;
  }
  free(a->argmax);
}

static float* wcopy(const float* p, int64_t n, int round) {
  float* w = (float*)malloc(sizeof(float) * n);
  memcpy(w, p, sizeof(float) * n);
  round_vec(w, n, round);
  return w;
}

/* Forward through the LM-head logits; fills dlog with logits [T, V]. */
static void forward_core(const orc_shape* s, const float* P, const int64_t* off,
                         const uint16_t* E, const uint16_t* F16, const int32_t* u, int rnd,
                         acts* a, float** Wb /* bf16-rounded GEMM weights by param index */) {
  const int64_t T = (int64_t)s->B * s->S, H = s->H, Q = (int64_t)s->nh * s->hd,
                KV = (int64_t)s->nkv * s->hd, I = s->I, V = s->V, W3 = (int64_t)s->layers * H;
  a->T = T; a->H = H; a->Q = Q; a->KV = KV; a->NQKV = Q + 2 * KV; a->I = I; a->V = V; a->W3 = W3;
  a->F = falloc(T * W3);
  for (int64_t i = 0; i < T * W3; ++i) a->F[i] = orc_bf16_to_f32(F16[i]);
  a->g = falloc(T * H);
  mm_nt(T, H, W3, a->F, W3, Wb[ORC_FC], W3, a->g, H, 0);
  round_vec(a->g, T * H, rnd);
  a->E_rows = falloc(T * H);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < H; ++i) a->E_rows[t * H + i] = orc_bf16_to_f32(E[(int64_t)u[t] * H + i]);
  a->U = falloc(T * 2 * H);
  a->rstd_a = falloc(T);
  a->rstd_b = falloc(T);
  rmsnorm_fwd(T, H, a->E_rows, H, P + off[ORC_W_IN], s->eps, a->U, 2 * H, a->rstd_a);
  rmsnorm_fwd(T, H, a->g, H, P + off[ORC_W_HID], s->eps, a->U + H, 2 * H, a->rstd_b);
  round_vec(a->U, T * 2 * H, rnd);
  const int64_t NQ = a->NQKV;
  a->qkv = falloc(T * NQ);
  mm_nt(T, NQ, 2 * H, a->U, 2 * H, Wb[ORC_QKV], 2 * H, a->qkv, NQ, 0);
  round_vec(a->qkv, T * NQ, rnd);
  a->cs = falloc((int64_t)s->S * s->hd / 2);
  a->sn = falloc((int64_t)s->S * s->hd / 2);
  rope_tables(s->S, s->hd, s->theta, a->cs, a->sn);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const int pos = (int)(t % s->S);
    float* row = a->qkv + t * NQ;
    rope_row(row, s->nh, s->hd, a->cs + (int64_t)pos * s->hd / 2, a->sn + (int64_t)pos * s->hd / 2, 0);
    rope_row(row + Q, s->nkv, s->hd, a->cs + (int64_t)pos * s->hd / 2,
             a->sn + (int64_t)pos * s->hd / 2, 0);
    if (rnd)
      for (int64_t i = 0; i < Q + KV; ++i) row[i] = rb(row[i]);
  }
  /* causal GQA attention within each sample */
  a->o = falloc(T * Q);
  a->lse_attn = falloc(T * s->nh);
  const float scale = 1.0f / sqrtf((float)s->hd);
  const int grp = s->nh / s->nkv;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < s->B; ++b)
    for (int h = 0; h < s->nh; ++h) {
      const int kvh = h / grp;
      float* p = (float*)malloc(sizeof(float) * s->S);
      for (int i = 0; i < s->S; ++i) {
        const int64_t ti = (int64_t)b * s->S + i;
        const float* q = a->qkv + ti * NQ + (int64_t)h * s->hd;
        float mx = -INFINITY;
        for (int j = 0; j <= i; ++j) {
          const float* k = a->qkv + ((int64_t)b * s->S + j) * NQ + Q + (int64_t)kvh * s->hd;
          float d = 0.f;
          for (int c = 0; c < s->hd; ++c) d += q[c] * k[c];
          p[j] = d * scale;
          if (p[j] > mx) mx = p[j];
        }
        double sum = 0.0;
        for (int j = 0; j <= i; ++j) {
          p[j] = expf(p[j] - mx);
          sum += p[j];
        }
        a->lse_attn[ti * s->nh + h] = mx + (float)log(sum);
        const float inv = (float)(1.0 / sum);
        float* out = a->o + ti * Q + (int64_t)h * s->hd;
        for (int c = 0; c < s->hd; ++c) out[c] = 0.f;
        for (int j = 0; j <= i; ++j) {
          const float* vv = a->qkv + ((int64_t)b * s->S + j) * NQ + Q + KV + (int64_t)kvh * s->hd;
          const float pj = p[j] * inv;
          for (int c = 0; c < s->hd; ++c) out[c] += pj * vv[c];
        }
      }
      free(p);
    }
  round_vec(a->o, T * Q, rnd);
  a->r = falloc(T * H);
  memcpy(a->r, a->g, sizeof(float) * T * H);
  mm_nt(T, H, Q, a->o, Q, Wb[ORC_O], Q, a->r, H, 1);
  round_vec(a->r, T * H, rnd);
  a->z = falloc(T * H);
  a->rstd_post = falloc(T);
  rmsnorm_fwd(T, H, a->r, H, P + off[ORC_W_POST], s->eps, a->z, H, a->rstd_post);
  round_vec(a->z, T * H, rnd);
  a->gu = falloc(T * 2 * I);
  mm_nt(T, 2 * I, H, a->z, H, Wb[ORC_GATE_UP], H, a->gu, 2 * I, 0);
  round_vec(a->gu, T * 2 * I, rnd);
  a->act = falloc(T * I);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < I; ++i) {
      const float gt = a->gu[t * 2 * I + i], up = a->gu[t * 2 * I + I + i];
      a->act[t * I + i] = silu(gt) * up;
    }
  round_vec(a->act, T * I, rnd);
  a->h = falloc(T * H);
  memcpy(a->h, a->r, sizeof(float) * T * H);
  mm_nt(T, H, I, a->act, I, Wb[ORC_DOWN], I, a->h, H, 1);
  round_vec(a->h, T * H, rnd);
  a->nrm = falloc(T * H);
  a->rstd_fin = falloc(T);
  rmsnorm_fwd(T, H, a->h, H, P + off[ORC_W_FIN], s->eps, a->nrm, H, a->rstd_fin);
  round_vec(a->nrm, T * H, rnd);
  a->dlog = falloc(T * V);
  mm_nt(T, V, H, a->nrm, H, Wb[ORC_LM], H, a->dlog, V, 0);
}

/* lse / loss / top-1 from the logits in a->dlog */
static void ce_stats(const orc_shape* s, acts* a, const int32_t* y, const int32_t* mask,
                     int64_t global_valid, orc_step_out* out) {
  const int64_t T = a->T, V = a->V;
  a->lse = falloc(T);
  a->argmax = (int32_t*)calloc((size_t)T, sizeof(int32_t));
  double loss = 0.0;
  int64_t valid = 0, top1 = 0;
#pragma omp parallel for schedule(static) reduction(+ : loss, valid, top1)
  for (int64_t t = 0; t < T; ++t) {
    const float* l = a->dlog + t * V;
    float mx = -INFINITY;
    int32_t am = 0;
    for (int64_t v = 0; v < V; ++v)
      if (l[v] > mx) {
        mx = l[v];
        am = (int32_t)v;
      }
    double sum = 0.0;
    for (int64_t v = 0; v < V; ++v) sum += exp((double)l[v] - mx);
    const float lse = mx + (float)log(sum);
    a->lse[t] = lse;
    a->argmax[t] = am;
    if (mask[t]) {
      loss += (double)lse - l[y[t]];
      valid += 1;
      top1 += (am == y[t]);
    }
  }
  const double denom = global_valid > 0 ? (double)global_valid : (double)(valid > 0 ? valid : 1);
  out->loss = loss / denom;
  out->valid = valid;
  out->top1 = top1;
  (void)s;
}

/* bf16-rounded GEMM weights: one persistent buffer (re-used across steps, so
 * its pages are touched once) filled by a single parallel rounding pass. */
static float* wb_cache = NULL;
static int64_t wb_cache_n = 0;

static void weights_bf16(const orc_shape* s, const float* P, const int64_t* off, int rnd,
                         float** Wb) {
  int64_t rows[ORC_NPARAMS], cols[ORC_NPARAMS];
  const int64_t total = orc_param_layout(s, NULL, rows, cols, NULL);
  if (wb_cache_n != total) {
    free(wb_cache);
    wb_cache = (float*)malloc(sizeof(float) * total);
    wb_cache_n = total;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < total; ++i) wb_cache[i] = rnd ? rb(P[i]) : P[i];
  for (int p = 0; p < ORC_NPARAMS; ++p) Wb[p] = wb_cache + off[p];
}

int orc_forward(const orc_shape* s, const float* params, const uint16_t* E, const uint16_t* F,
                const int32_t* u, const int32_t* y, const int32_t* mask, int64_t global_valid,
                int round_bf16, orc_step_out* out, float* lse_out, int32_t* argmax_out) {
  int64_t off[ORC_NPARAMS];
  orc_param_layout(s, NULL, NULL, NULL, off);
  float* Wb[ORC_NPARAMS];
  weights_bf16(s, params, off, round_bf16, Wb);
  acts a;
  memset(&a, 0, sizeof(a));
  forward_core(s, params, off, E, F, u, round_bf16, &a, Wb);
  ce_stats(s, &a, y, mask, global_valid, out);
  if (lse_out) memcpy(lse_out, a.lse, sizeof(float) * a.T);
  if (argmax_out) memcpy(argmax_out, a.argmax, sizeof(int32_t) * a.T);
  acts_free(&a);
  return 0;
}

void orc_adamw(int64_t n, float* p, float* m, float* v, const float* g, const float* hp,
               int64_t step_k) {
  const float lr = hp[0], b1 = hp[1], b2 = hp[2], eps = hp[3], wd = hp[4];
  const double bc1 = 1.0 - pow((double)b1, (double)step_k);
  const double bc2 = 1.0 - pow((double)b2, (double)step_k);
  const float step_size = (float)(lr / bc1);
  const float bc2_sqrt = (float)sqrt(bc2);
  const float decay = 1.0f - lr * wd;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const float gi = g[i];
    float pi = p[i] * decay;
    const float mi = m[i] + (gi - m[i]) * (1.0f - b1);
    const float vi = v[i] * b2 + (1.0f - b2) * gi * gi;
    const float denom = sqrtf(vi) / bc2_sqrt + eps;
    pi = pi - step_size * (mi / denom);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
  }
}

int orc_train_step(const orc_shape* s, const float* adamw5, int64_t step_k, float* params,
                   float* mst, float* vst, float* grads, const uint16_t* E, const uint16_t* F16,
                   const int32_t* u, const int32_t* y, const int32_t* mask, int64_t global_valid,
                   int rnd, int do_update, orc_step_out* out) {
  if (s->nh % s->nkv != 0 || s->hd % 2 != 0) return 1;
  int64_t off[ORC_NPARAMS], rows[ORC_NPARAMS], cols[ORC_NPARAMS];
  const int64_t total = orc_param_layout(s, NULL, rows, cols, off);
  float* Wb[ORC_NPARAMS];
  prof(NULL);
  weights_bf16(s, params, off, rnd, Wb);
  prof("bf16 weight copies");
  acts a;
  memset(&a, 0, sizeof(a));
  forward_core(s, params, off, E, F16, u, rnd, &a, Wb);
  prof("forward (incl. LM head)");
  ce_stats(s, &a, y, mask, global_valid, out);
  prof("CE stats");
  const int64_t T = a.T, H = a.H, Q = a.Q, KV = a.KV, NQ = a.NQKV, I = a.I, V = a.V, W3 = a.W3;
  int64_t nvalid = 0;
  for (int64_t t = 0; t < T; ++t) nvalid += mask[t] ? 1 : 0;
  const double denom = global_valid > 0 ? (double)global_valid : (double)(nvalid > 0 ? nvalid : 1);
  memset(grads, 0, sizeof(float) * total);

  /* ---- LM head + CE backward: dlogits = (softmax - onehot) * m / N */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    float* l = a.dlog + t * V;
    const float coef = mask[t] ? (float)(1.0 / denom) : 0.f;
    for (int64_t v = 0; v < V; ++v) {
      const float p = expf(l[v] - a.lse[t]);
      float gval = (p - (v == y[t] ? 1.f : 0.f)) * coef;
      l[v] = rnd ? rb(gval) : gval;
    }
  }
  prof("CE backward (softmax grad)");
  float* dn = falloc(T * H);
  mm_nn(T, H, V, a.dlog, V, Wb[ORC_LM], H, dn, H, 0);
  prof("LM head dX");
  mm_tn(V, H, T, a.dlog, V, a.nrm, H, grads + off[ORC_LM], H);
  prof("LM head dW");

  /* ---- final norm */
  float* dh = falloc(T * H);
  rmsnorm_bwd(T, H, dn, H, a.h, H, params + off[ORC_W_FIN], a.rstd_fin, dh, H, 0,
              grads + off[ORC_W_FIN]);
  float* dh_b = wcopy(dh, T * H, rnd);

  /* ---- MLP */
  float* dact = falloc(T * I);
  mm_nn(T, I, H, dh_b, H, Wb[ORC_DOWN], I, dact, I, 0);
  round_vec(dact, T * I, rnd);
  mm_tn(H, I, T, dh_b, H, a.act, I, grads + off[ORC_DOWN], I);
  float* dgu = falloc(T * 2 * I);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < I; ++i) {
      const float gt = a.gu[t * 2 * I + i], up = a.gu[t * 2 * I + I + i];
      const float sg = 1.0f / (1.0f + expf(-gt));
      const float d = dact[t * I + i];
      dgu[t * 2 * I + i] = d * up * sg * (1.0f + gt * (1.0f - sg));
      dgu[t * 2 * I + I + i] = d * gt * sg;
    }
  round_vec(dgu, T * 2 * I, rnd);
  float* dz = falloc(T * H);
  mm_nn(T, H, 2 * I, dgu, 2 * I, Wb[ORC_GATE_UP], H, dz, H, 0);
  mm_tn(2 * I, H, T, dgu, 2 * I, a.z, H, grads + off[ORC_GATE_UP], H);

  /* ---- post-attention norm; residual */
  float* dr = falloc(T * H);
  memcpy(dr, dh, sizeof(float) * T * H);
  rmsnorm_bwd(T, H, dz, H, a.r, H, params + off[ORC_W_POST], a.rstd_post, dr, H, 1,
              grads + off[ORC_W_POST]);
  float* dr_b = wcopy(dr, T * H, rnd);

  /* ---- o projection */
  float* dO = falloc(T * Q);
  mm_nn(T, Q, H, dr_b, H, Wb[ORC_O], Q, dO, Q, 0);
  round_vec(dO, T * Q, rnd);
  mm_tn(H, Q, T, dr_b, H, a.o, Q, grads + off[ORC_O], Q);

  /* ---- attention backward */
  float* dqkv = falloc(T * NQ);
  const float scale = 1.0f / sqrtf((float)s->hd);
  const int grp = s->nh / s->nkv;
  /* dq per (b, h) rows; dk/dv accumulated per (b, kv head) over the group */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < s->B; ++b)
    for (int kvh = 0; kvh < s->nkv; ++kvh) {
      float* p = (float*)malloc(sizeof(float) * s->S);
      float* dp = (float*)malloc(sizeof(float) * s->S);
      for (int hh = 0; hh < grp; ++hh) {
        const int h = kvh * grp + hh;
        for (int i = 0; i < s->S; ++i) {
          const int64_t ti = (int64_t)b * s->S + i;
          const float* q = a.qkv + ti * NQ + (int64_t)h * s->hd;
          const float* dout = dO + ti * Q + (int64_t)h * s->hd;
          const float* oo = a.o + ti * Q + (int64_t)h * s->hd;
          const float lse = a.lse_attn[ti * s->nh + h];
          float Di = 0.f;
          for (int c = 0; c < s->hd; ++c) Di += dout[c] * oo[c];
          for (int j = 0; j <= i; ++j) {
            const int64_t tj = (int64_t)b * s->S + j;
            const float* k = a.qkv + tj * NQ + Q + (int64_t)kvh * s->hd;
            const float* vv = a.qkv + tj * NQ + Q + KV + (int64_t)kvh * s->hd;
            float d = 0.f, e = 0.f;
            for (int c = 0; c < s->hd; ++c) {
              d += q[c] * k[c];
              e += dout[c] * vv[c];
            }
            p[j] = expf(d * scale - lse);
            dp[j] = e;
          }
          float* dq = dqkv + ti * NQ + (int64_t)h * s->hd;
          for (int j = 0; j <= i; ++j) {
            const int64_t tj = (int64_t)b * s->S + j;
            const float* k = a.qkv + tj * NQ + Q + (int64_t)kvh * s->hd;
            float* dk = dqkv + tj * NQ + Q + (int64_t)kvh * s->hd;
            float* dv = dqkv + tj * NQ + Q + KV + (int64_t)kvh * s->hd;
            const float ds = p[j] * (dp[j] - Di) * scale;
            for (int c = 0; c < s->hd; ++c) {
              dq[c] += ds * k[c];
              dk[c] += ds * q[c];
              dv[c] += p[j] * dout[c];
            }
          }
        }
      }
      free(p);
      free(dp);
    }
  /* RoPE backward on dq, dk; round to bf16 (GEMM operand) */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const int pos = (int)(t % s->S);
    float* row = dqkv + t * NQ;
    if (rnd)
      for (int64_t i = 0; i < NQ; ++i) row[i] = rb(row[i]);
    rope_row(row, s->nh, s->hd, a.cs + (int64_t)pos * s->hd / 2, a.sn + (int64_t)pos * s->hd / 2, 1);
    rope_row(row + Q, s->nkv, s->hd, a.cs + (int64_t)pos * s->hd / 2,
             a.sn + (int64_t)pos * s->hd / 2, 1);
    if (rnd)
      for (int64_t i = 0; i < Q + KV; ++i) row[i] = rb(row[i]);
  }
  float* dU = falloc(T * 2 * H);
  mm_nn(T, 2 * H, NQ, dqkv, NQ, Wb[ORC_QKV], 2 * H, dU, 2 * H, 0);
  mm_tn(NQ, 2 * H, T, dqkv, NQ, a.U, 2 * H, grads + off[ORC_QKV], 2 * H);

  /* ---- input norms (embedding frozen: only dw_in) */
  rmsnorm_bwd(T, H, dU, 2 * H, a.E_rows, H, params + off[ORC_W_IN], a.rstd_a, NULL, 0, 0,
              grads + off[ORC_W_IN]);
  float* dg = dr; /* residual path: dg = dr + d(hidden norm) */
  rmsnorm_bwd(T, H, dU + H, 2 * H, a.g, H, params + off[ORC_W_HID], a.rstd_b, dg, H, 1,
              grads + off[ORC_W_HID]);
  round_vec(dg, T * H, rnd);
  mm_tn(H, W3, T, dg, H, a.F, W3, grads + off[ORC_FC], W3);

  prof("decoder backward");
  if (do_update) orc_adamw(total, params, mst, vst, grads, adamw5, step_k);
  prof("AdamW");

  free(dn); free(dh); free(dh_b); free(dact); free(dgu); free(dz); free(dr); free(dr_b);
  free(dO); free(dqkv); free(dU);
  acts_free(&a);
  (void)rows; (void)cols;
  return 0;
}
