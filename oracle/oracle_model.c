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
static int ttt_of(const orc_shape* s) { return s->ttt > 0 ? s->ttt : 1; }
static float decay_of(const orc_shape* s) { return s->ttt_decay > 0.f ? s->ttt_decay : 0.8f; }

void orc_gather_batch(const orc_shape* s, int nsamples, const int32_t* const* ids,
                      const uint16_t* const* feats, const int32_t* lens, uint16_t* F,
                      int32_t* u, int32_t* y, int32_t* m) {
  const int64_t w = (int64_t)s->layers * s->H, T = (int64_t)s->B * s->S;
  const int K = ttt_of(s);
  for (int b = 0; b < s->B; ++b) {
    const int L = b < nsamples ? lens[b] : 0;
    for (int t = 0; t < s->S; ++t) {
      const int64_t row = (int64_t)b * s->S + t;
      if (t < L)
        memcpy(F + row * w, feats[b] + (int64_t)t * w, (size_t)w * 2);
      else
        memset(F + row * w, 0, (size_t)w * 2);
      for (int j = 0; j < K; ++j) {
        const int64_t r = (int64_t)j * T + row;
        u[r] = (t + 1 + j < L) ? ids[b][t + 1 + j] : 0;
        y[r] = (t + 2 + j < L) ? ids[b][t + 2 + j] : 0;
        m[r] = (t + 2 + j < L) ? 1 : 0;
      }
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

/* C[N,K] (+)= A[T,N]^T . X[T,K]  (weight-gradient form; accumulates over
 * the unroll steps of a training-time-test step) */
static void mm_tn(int64_t N, int64_t K, int64_t T, const float* A, int64_t lda, const float* X,
                  int64_t ldx, float* C, int64_t ldc, int accumulate) {
  mm_gen(N, K, T, A, lda, 1, X, ldx, 1, C, ldc, accumulate);
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

/* dx (+)= rstd * (dy*w) - x * rstd^3 * mean((dy*w) * x) ; dw (+)= sum_t dy * x * rstd */
static void rmsnorm_bwd(int64_t T, int64_t H, const float* dy, int64_t lddy, const float* x,
                        int64_t ldx, const float* w, const float* rstd, float* dx, int64_t lddx,
                        int accumulate_dx, float* dw, int accumulate_dw) {
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
      dw[i] = accumulate_dw ? dw[i] + (float)s : (float)s;
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
#define ORC_MAX_TTT 16

/* activations of one unroll step of the decoder layer (+ its LM head) */
typedef struct step_acts {
  float *E_rows, *U, *rstd_a, *rstd_b, *qkv, *o, *lse_attn, *r, *z, *rstd_post, *gu, *act, *h,
      *nrm, *rstd_fin, *lse, *dlog, *margin;
  int32_t* argmax;
} step_acts;

typedef struct model {
  const orc_shape* s;
  int K;
  float decay;
  int64_t T, H, Q, KV, NQ, I, V, W3;
  float *F, *g0;  /* step-0 features and fc output g = W_fc f */
  float *cs, *sn; /* RoPE tables, positions [0, S + K - 1) */
  step_acts st[ORC_MAX_TTT];
} model;

static void model_free(model* M) {
  free(M->F);
  free(M->g0);
  free(M->cs);
  free(M->sn);
  for (int j = 0; j < M->K; ++j) {
    step_acts* a = &M->st[j];
    float** ptrs[] = {&a->E_rows, &a->U,   &a->rstd_a,   &a->rstd_b, &a->qkv, &a->o,
                      &a->lse_attn, &a->r, &a->z,        &a->rstd_post, &a->gu, &a->act,
                      &a->h,      &a->nrm, &a->rstd_fin, &a->lse,    &a->dlog, &a->margin};
    for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) {
      free(*ptrs[i]);
      *ptrs[i] = NULL;
    }
    free(a->argmax);
  }
}

static float* wcopy(const float* p, int64_t n, int round) {
  float* w = (float*)malloc(sizeof(float) * n);
  memcpy(w, p, sizeof(float) * n);
  round_vec(w, n, round);
  return w;
}

/* input of unroll step j: g = W_fc f at step 0, the previous step's output h after */
static const float* step_input(const model* M, int j) { return j == 0 ? M->g0 : M->st[j - 1].h; }

/* RoPE (forward or inverse) on the q and k heads of a [T, NQ] buffer; row t
 * is position t % S + j (unroll step j) */
static void rope_rows(const model* M, float* qkv, int j, int inverse) {
  const orc_shape* s = M->s;
  const int64_t half = s->hd / 2;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < M->T; ++t) {
    const int64_t pos = t % s->S + j;
    float* row = qkv + t * M->NQ;
    rope_row(row, s->nh, s->hd, M->cs + pos * half, M->sn + pos * half, inverse);
    rope_row(row + M->Q, s->nkv, s->hd, M->cs + pos * half, M->sn + pos * half, inverse);
  }
}

/* Causal GQA attention of unroll step j: query row t of step j sees step 0's
 * keys s <= t of its sample plus, for i = 1..j, step i's key at row t
 * (EAGLE-3 training-time-test cache, SpecForge's shifted-diagonal mask). */
static void attention_fwd(model* M, int j) {
  const orc_shape* s = M->s;
  const int64_t NQ = M->NQ, Q = M->Q, KV = M->KV;
  step_acts* A = &M->st[j];
  const float scale = 1.0f / sqrtf((float)s->hd);
  const int grp = s->nh / s->nkv;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < s->B; ++b)
    for (int h = 0; h < s->nh; ++h) {
      const int kvh = h / grp;
      float* p = (float*)malloc(sizeof(float) * (s->S + ORC_MAX_TTT));
      for (int i = 0; i < s->S; ++i) {
        const int64_t ti = (int64_t)b * s->S + i;
        const float* q = A->qkv + ti * NQ + (int64_t)h * s->hd;
        float mx = -INFINITY;
        for (int c0 = 0; c0 <= i + j; ++c0) {
          /* c0 <= i: step-0 key c0; c0 = i + d (d = 1..j): step d's key at row i */
          const float* k = c0 <= i
                               ? M->st[0].qkv + ((int64_t)b * s->S + c0) * NQ + Q + (int64_t)kvh * s->hd
                               : M->st[c0 - i].qkv + ti * NQ + Q + (int64_t)kvh * s->hd;
          float d = 0.f;
          for (int c = 0; c < s->hd; ++c) d += q[c] * k[c];
          p[c0] = d * scale;
          if (p[c0] > mx) mx = p[c0];
        }
        double sum = 0.0;
        for (int c0 = 0; c0 <= i + j; ++c0) {
          p[c0] = expf(p[c0] - mx);
          sum += p[c0];
        }
        A->lse_attn[ti * s->nh + h] = mx + (float)log(sum);
        const float inv = (float)(1.0 / sum);
        float* out = A->o + ti * Q + (int64_t)h * s->hd;
        for (int c = 0; c < s->hd; ++c) out[c] = 0.f;
        for (int c0 = 0; c0 <= i + j; ++c0) {
          const float* vv = c0 <= i ? M->st[0].qkv + ((int64_t)b * s->S + c0) * NQ + Q + KV +
                                          (int64_t)kvh * s->hd
                                    : M->st[c0 - i].qkv + ti * NQ + Q + KV + (int64_t)kvh * s->hd;
          const float pj = p[c0] * inv;
          for (int c = 0; c < s->hd; ++c) out[c] += pj * vv[c];
        }
      }
      free(p);
    }
}

/* Decoder layer + final norm + LM-head logits (into dlog) of unroll step j. */
static void decoder_fwd(model* M, int j, const float* P, const int64_t* off, const uint16_t* E,
                        const int32_t* u, int rnd, float** Wb) {
  const orc_shape* s = M->s;
  const int64_t T = M->T, H = M->H, Q = M->Q, KV = M->KV, NQ = M->NQ, I = M->I, V = M->V;
  step_acts* a = &M->st[j];
  const float* g = step_input(M, j);
  a->E_rows = falloc(T * H);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < H; ++i) a->E_rows[t * H + i] = orc_bf16_to_f32(E[(int64_t)u[t] * H + i]);
  a->U = falloc(T * 2 * H);
  a->rstd_a = falloc(T);
  a->rstd_b = falloc(T);
  rmsnorm_fwd(T, H, a->E_rows, H, P + off[ORC_W_IN], s->eps, a->U, 2 * H, a->rstd_a);
  rmsnorm_fwd(T, H, g, H, P + off[ORC_W_HID], s->eps, a->U + H, 2 * H, a->rstd_b);
  round_vec(a->U, T * 2 * H, rnd);
  a->qkv = falloc(T * NQ);
  mm_nt(T, NQ, 2 * H, a->U, 2 * H, Wb[ORC_QKV], 2 * H, a->qkv, NQ, 0);
  round_vec(a->qkv, T * NQ, rnd);
  rope_rows(M, a->qkv, j, 0);
  if (rnd)
    for (int64_t t = 0; t < T; ++t)
      for (int64_t i = 0; i < Q + KV; ++i) a->qkv[t * NQ + i] = rb(a->qkv[t * NQ + i]);
  a->o = falloc(T * Q);
  a->lse_attn = falloc(T * s->nh);
  attention_fwd(M, j);
  round_vec(a->o, T * Q, rnd);
  a->r = falloc(T * H);
  memcpy(a->r, g, sizeof(float) * T * H);
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

/* Full forward: fc, then the K unroll steps (each feeding its output h to the
 * next), logits of every step in st[j].dlog. */
static void model_fwd(model* M, const orc_shape* s, const float* P, const int64_t* off,
                      const uint16_t* E, const uint16_t* F16, const int32_t* u, int rnd,
                      float** Wb) {
  memset(M, 0, sizeof(*M));
  M->s = s;
  M->K = ttt_of(s);
  M->decay = decay_of(s);
  M->T = (int64_t)s->B * s->S;
  M->H = s->H;
  M->Q = (int64_t)s->nh * s->hd;
  M->KV = (int64_t)s->nkv * s->hd;
  M->NQ = M->Q + 2 * M->KV;
  M->I = s->I;
  M->V = s->V;
  M->W3 = (int64_t)s->layers * s->H;
  const int64_t T = M->T, H = M->H, W3 = M->W3;
  M->F = falloc(T * W3);
  for (int64_t i = 0; i < T * W3; ++i) M->F[i] = orc_bf16_to_f32(F16[i]);
  M->g0 = falloc(T * H);
  mm_nt(T, H, W3, M->F, W3, Wb[ORC_FC], W3, M->g0, H, 0);
  round_vec(M->g0, T * H, rnd);
  const int npos = s->S + M->K - 1;
  M->cs = falloc((int64_t)npos * s->hd / 2);
  M->sn = falloc((int64_t)npos * s->hd / 2);
  rope_tables(npos, s->hd, s->theta, M->cs, M->sn);
  for (int j = 0; j < M->K; ++j) decoder_fwd(M, j, P, off, E, u + (int64_t)j * T, rnd, Wb);
}

/* loss weight of unroll step j: decay^j (fp32, as the library's table) */
static float step_weight(const model* M, int j) { return (float)pow((double)M->decay, (double)j); }

/* lse / loss / top-1 from the logits in st[j].dlog: loss = sum_j decay^j
 * sum_t m_j (lse - l_y) / denom; valid / top1 over unroll step 0. */
static void ce_stats(model* M, const int32_t* y, const int32_t* mask, int64_t global_valid,
                     orc_step_out* out) {
  const int64_t T = M->T, V = M->V;
  int64_t valid0 = 0;
  for (int64_t t = 0; t < T; ++t) valid0 += mask[t] ? 1 : 0;
  const double denom =
      global_valid > 0 ? (double)global_valid : (double)(valid0 > 0 ? valid0 : 1);
  double total = 0.0;
  out->valid = valid0;
  out->top1 = 0;
  for (int j = 0; j < M->K; ++j) {
    const float w = step_weight(M, j);
    step_acts* a = &M->st[j];
    const int32_t* yj = y + (int64_t)j * T;
    const int32_t* mj = mask + (int64_t)j * T;
    a->lse = falloc(T);
    a->argmax = (int32_t*)calloc((size_t)T, sizeof(int32_t));
    a->margin = falloc(T);
    double loss = 0.0;
    int64_t top1 = 0;
#pragma omp parallel for schedule(static) reduction(+ : loss, top1)
    for (int64_t t = 0; t < T; ++t) {
      const float* l = a->dlog + t * V;
      float mx = -INFINITY, mx2 = -INFINITY; /* top-1 / top-2 logits (ties: margin 0) */
      int32_t am = 0;
      for (int64_t v = 0; v < V; ++v)
        if (l[v] > mx) {
          mx2 = mx;
          mx = l[v];
          am = (int32_t)v;
        } else if (l[v] > mx2) {
          mx2 = l[v];
        }
      a->margin[t] = mx - mx2;
      double sum = 0.0;
      for (int64_t v = 0; v < V; ++v) sum += exp((double)l[v] - mx);
      const float lse = mx + (float)log(sum);
      a->lse[t] = lse;
      a->argmax[t] = am;
      if (mj[t]) {
        loss += (double)lse - l[yj[t]];
        top1 += (am == yj[t]);
      }
    }
    total += w * (loss / denom);
    if (j == 0) out->top1 = top1;
  }
  out->loss = total;
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

static int shape_ok(const orc_shape* s) {
  return s->nh % s->nkv == 0 && s->hd % 2 == 0 && ttt_of(s) <= ORC_MAX_TTT;
}

int orc_forward(const orc_shape* s, const float* params, const uint16_t* E, const uint16_t* F,
                const int32_t* u, const int32_t* y, const int32_t* mask, int64_t global_valid,
                int round_bf16, orc_step_out* out, float* lse_out, int32_t* argmax_out) {
  return orc_forward_ex(s, params, E, F, u, y, mask, global_valid, round_bf16, out, lse_out,
                        argmax_out, NULL, NULL, NULL);
}

int orc_forward_ex(const orc_shape* s, const float* params, const uint16_t* E, const uint16_t* F,
                   const int32_t* u, const int32_t* y, const int32_t* mask, int64_t global_valid,
                   int round_bf16, orc_step_out* out, float* lse_out, int32_t* argmax_out,
                   float* margin_out, const int32_t* probe_idx, float* probe_gap) {
  if (!shape_ok(s)) return 1;
  int64_t off[ORC_NPARAMS];
  orc_param_layout(s, NULL, NULL, NULL, off);
  float* Wb[ORC_NPARAMS];
  weights_bf16(s, params, off, round_bf16, Wb);
  model M;
  model_fwd(&M, s, params, off, E, F, u, round_bf16, Wb);
  ce_stats(&M, y, mask, global_valid, out);
  for (int j = 0; j < M.K; ++j) {
    if (lse_out) memcpy(lse_out + (int64_t)j * M.T, M.st[j].lse, sizeof(float) * M.T);
    if (argmax_out) memcpy(argmax_out + (int64_t)j * M.T, M.st[j].argmax, sizeof(int32_t) * M.T);
    if (margin_out) memcpy(margin_out + (int64_t)j * M.T, M.st[j].margin, sizeof(float) * M.T);
    if (probe_idx && probe_gap)
      for (int64_t t = 0; t < M.T; ++t) {
        const int64_t r = (int64_t)j * M.T + t;
        const int32_t v = probe_idx[r];
        const float* l = M.st[j].dlog + t * M.V;
        probe_gap[r] = (v >= 0 && v < M.V) ? l[M.st[j].argmax[t]] - l[v] : NAN;
      }
  }
  model_free(&M);
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

/* Attention backward of unroll step j.  dq [T, Q] receives step j's query
 * gradient; dK / dV [K][T, KV] accumulate the key / value gradients of every
 * step (rotated space): step 0's from the causal part of all steps, step i's
 * (i >= 1) from the diagonal entries of steps j >= i. */
static void attention_bwd(model* M, int j, const float* dO, float* dq, float** dK, float** dV) {
  const orc_shape* s = M->s;
  const int64_t NQ = M->NQ, Q = M->Q, KV = M->KV;
  const step_acts* A = &M->st[j];
  const float scale = 1.0f / sqrtf((float)s->hd);
  const int grp = s->nh / s->nkv;
  /* (b, kv head) partitions: every dK / dV row it touches belongs to it */
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < s->B; ++b)
    for (int kvh = 0; kvh < s->nkv; ++kvh) {
      float* p = (float*)malloc(sizeof(float) * (s->S + ORC_MAX_TTT));
      float* dp = (float*)malloc(sizeof(float) * (s->S + ORC_MAX_TTT));
      for (int hh = 0; hh < grp; ++hh) {
        const int h = kvh * grp + hh;
        for (int i = 0; i < s->S; ++i) {
          const int64_t ti = (int64_t)b * s->S + i;
          const float* q = A->qkv + ti * NQ + (int64_t)h * s->hd;
          const float* dout = dO + ti * Q + (int64_t)h * s->hd;
          const float* oo = A->o + ti * Q + (int64_t)h * s->hd;
          const float lse = A->lse_attn[ti * s->nh + h];
          float Di = 0.f;
          for (int c = 0; c < s->hd; ++c) Di += dout[c] * oo[c];
          for (int c0 = 0; c0 <= i + j; ++c0) {
            const int st = c0 <= i ? 0 : c0 - i;
            const int64_t row = c0 <= i ? (int64_t)b * s->S + c0 : ti;
            const float* k = M->st[st].qkv + row * NQ + Q + (int64_t)kvh * s->hd;
            const float* vv = k + KV;
            float d = 0.f, e = 0.f;
            for (int c = 0; c < s->hd; ++c) {
              d += q[c] * k[c];
              e += dout[c] * vv[c];
            }
            p[c0] = expf(d * scale - lse);
            dp[c0] = e;
          }
          float* dqr = dq + ti * Q + (int64_t)h * s->hd;
          for (int c0 = 0; c0 <= i + j; ++c0) {
            const int st = c0 <= i ? 0 : c0 - i;
            const int64_t row = c0 <= i ? (int64_t)b * s->S + c0 : ti;
            const float* k = M->st[st].qkv + row * NQ + Q + (int64_t)kvh * s->hd;
            float* dk = dK[st] + row * KV + (int64_t)kvh * s->hd;
            float* dv = dV[st] + row * KV + (int64_t)kvh * s->hd;
            const float ds = p[c0] * (dp[c0] - Di) * scale;
            for (int c = 0; c < s->hd; ++c) {
              dqr[c] += ds * k[c];
              dk[c] += ds * q[c];
              dv[c] += p[c0] * dout[c];
            }
          }
        }
      }
      free(p);
      free(dp);
    }
}

int orc_train_step(const orc_shape* s, const float* adamw5, int64_t step_k, float* params,
                   float* mst, float* vst, float* grads, const uint16_t* E, const uint16_t* F16,
                   const int32_t* u, const int32_t* y, const int32_t* mask, int64_t global_valid,
                   int rnd, int do_update, orc_step_out* out) {
  if (!shape_ok(s)) return 1;
  int64_t off[ORC_NPARAMS], rows[ORC_NPARAMS], cols[ORC_NPARAMS];
  const int64_t total = orc_param_layout(s, NULL, rows, cols, off);
  float* Wb[ORC_NPARAMS];
  prof(NULL);
  weights_bf16(s, params, off, rnd, Wb);
  prof("bf16 weight copies");
  model M;
  model_fwd(&M, s, params, off, E, F16, u, rnd, Wb);
  prof("forward (incl. LM head)");
  ce_stats(&M, y, mask, global_valid, out);
  prof("CE stats");
  const int64_t T = M.T, H = M.H, Q = M.Q, KV = M.KV, NQ = M.NQ, I = M.I, V = M.V, W3 = M.W3;
  const int K = M.K;
  const double denom = global_valid > 0 ? (double)global_valid
                                        : (double)(out->valid > 0 ? out->valid : 1);
  memset(grads, 0, sizeof(float) * total);
  float *dK[ORC_MAX_TTT], *dV[ORC_MAX_TTT];
  for (int j = 0; j < K; ++j) {
    dK[j] = falloc(T * KV);
    dV[j] = falloc(T * KV);
  }
  float* dn = falloc(T * H);
  float* dh = falloc(T * H);
  float* dact = falloc(T * I);
  float* dgu = falloc(T * 2 * I);
  float* dz = falloc(T * H);
  float* dr = falloc(T * H);
  float* dO = falloc(T * Q);
  float* dq = falloc(T * Q);
  float* dqkv = falloc(T * NQ);
  float* dU = falloc(T * 2 * H);
  float* dg_next = NULL; /* gradient w.r.t. h_j arriving from step j + 1's input */
  /* unroll steps in reverse: step j's input gradient feeds step j - 1's output */
  for (int j = K - 1; j >= 0; --j) {
    step_acts* a = &M.st[j];
    const int32_t* yj = y + (int64_t)j * T;
    const int32_t* mj = mask + (int64_t)j * T;
    const float* g = step_input(&M, j);
    const float wj = step_weight(&M, j);

    /* ---- LM head + CE backward: dlogits = (softmax - onehot) * m * decay^j / N */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      float* l = a->dlog + t * V;
      const float coef = mj[t] ? (float)(1.0 / denom) * wj : 0.f;
      for (int64_t v = 0; v < V; ++v) {
        const float p = expf(l[v] - a->lse[t]);
        float gval = (p - (v == yj[t] ? 1.f : 0.f)) * coef;
        l[v] = rnd ? rb(gval) : gval;
      }
    }
    mm_nn(T, H, V, a->dlog, V, Wb[ORC_LM], H, dn, H, 0);
    mm_tn(V, H, T, a->dlog, V, a->nrm, H, grads + off[ORC_LM], H, 1);
    prof("LM head backward");

    /* ---- final norm (+ the gradient arriving through the next step's input) */
    if (dg_next)
      memcpy(dh, dg_next, sizeof(float) * T * H);
    rmsnorm_bwd(T, H, dn, H, a->h, H, params + off[ORC_W_FIN], a->rstd_fin, dh, H,
                dg_next != NULL, grads + off[ORC_W_FIN], 1);
    float* dh_b = wcopy(dh, T * H, rnd);

    /* ---- MLP */
    mm_nn(T, I, H, dh_b, H, Wb[ORC_DOWN], I, dact, I, 0);
    round_vec(dact, T * I, rnd);
    mm_tn(H, I, T, dh_b, H, a->act, I, grads + off[ORC_DOWN], I, 1);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t)
      for (int64_t i = 0; i < I; ++i) {
        const float gt = a->gu[t * 2 * I + i], up = a->gu[t * 2 * I + I + i];
        const float sg = 1.0f / (1.0f + expf(-gt));
        const float d = dact[t * I + i];
        dgu[t * 2 * I + i] = d * up * sg * (1.0f + gt * (1.0f - sg));
        dgu[t * 2 * I + I + i] = d * gt * sg;
      }
    round_vec(dgu, T * 2 * I, rnd);
    mm_nn(T, H, 2 * I, dgu, 2 * I, Wb[ORC_GATE_UP], H, dz, H, 0);
    mm_tn(2 * I, H, T, dgu, 2 * I, a->z, H, grads + off[ORC_GATE_UP], H, 1);

    /* ---- post-attention norm; residual */
    memcpy(dr, dh, sizeof(float) * T * H);
    rmsnorm_bwd(T, H, dz, H, a->r, H, params + off[ORC_W_POST], a->rstd_post, dr, H, 1,
                grads + off[ORC_W_POST], 1);
    float* dr_b = wcopy(dr, T * H, rnd);

    /* ---- o projection */
    mm_nn(T, Q, H, dr_b, H, Wb[ORC_O], Q, dO, Q, 0);
    round_vec(dO, T * Q, rnd);
    mm_tn(H, Q, T, dr_b, H, a->o, Q, grads + off[ORC_O], Q, 1);

    /* ---- attention: dq of this step; dK / dV of this step are complete now
     * (every step >= j has contributed) */
    memset(dq, 0, sizeof(float) * T * Q);
    attention_bwd(&M, j, dO, dq, dK, dV);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      float* row = dqkv + t * NQ;
      memcpy(row, dq + t * Q, sizeof(float) * Q);
      memcpy(row + Q, dK[j] + t * KV, sizeof(float) * KV);
      memcpy(row + Q + KV, dV[j] + t * KV, sizeof(float) * KV);
    }
    /* round, RoPE backward on dq / dk (position t % S + j), round: GEMM operand */
    round_vec(dqkv, T * NQ, rnd);
    rope_rows(&M, dqkv, j, 1);
    if (rnd)
      for (int64_t t = 0; t < T; ++t)
        for (int64_t i = 0; i < Q + KV; ++i) dqkv[t * NQ + i] = rb(dqkv[t * NQ + i]);
    mm_nn(T, 2 * H, NQ, dqkv, NQ, Wb[ORC_QKV], 2 * H, dU, 2 * H, 0);
    mm_tn(NQ, 2 * H, T, dqkv, NQ, a->U, 2 * H, grads + off[ORC_QKV], 2 * H, 1);

    /* ---- input norms (embedding frozen: only dw_in) */
    rmsnorm_bwd(T, H, dU, 2 * H, a->E_rows, H, params + off[ORC_W_IN], a->rstd_a, NULL, 0, 0,
                grads + off[ORC_W_IN], 1);
    float* dg = dr; /* residual path: dg = dr + d(hidden norm) */
    rmsnorm_bwd(T, H, dU + H, 2 * H, g, H, params + off[ORC_W_HID], a->rstd_b, dg, H, 1,
                grads + off[ORC_W_HID], 1);
    if (j > 0) {
      /* fp32 gradient w.r.t. h_{j-1} (the previous step's output) */
      if (!dg_next) dg_next = falloc(T * H);
      memcpy(dg_next, dg, sizeof(float) * T * H);
    } else {
      round_vec(dg, T * H, rnd);
      mm_tn(H, W3, T, dg, H, M.F, W3, grads + off[ORC_FC], W3, 0);
    }
    free(dh_b);
    free(dr_b);
    prof("decoder backward");
  }
  if (do_update) orc_adamw(total, params, mst, vst, grads, adamw5, step_k);
  prof("AdamW");

  for (int j = 0; j < K; ++j) {
    free(dK[j]);
    free(dV[j]);
  }
  free(dg_next);
  free(dn); free(dh); free(dact); free(dgu); free(dz); free(dr); free(dO); free(dq); free(dqkv);
  free(dU);
  model_free(&M);
  (void)rows; (void)cols;
  return 0;
}
