// Causal GQA attention of the draft decoder layer, forward and backward.
//
// Flash-style (no S x S matrix in HBM): per 64-query block the forward keeps
// an online softmax in registers and writes O (bf16) and the row log-sum-exp
// (fp32, natural log).  The backward is split into a dK/dV kernel (one CTA per
// 64-key block and KV head; loops over the query heads of its GQA group and
// all later query blocks) and a dQ kernel (one CTA per 64-query block), so
// every gradient element is written exactly once — deterministic, no atomics.
//
// This file is the FALLBACK path: warp-level mma.sync m16n8k16 bf16 with
// ldmatrix from XOR-swizzled shared memory and cp.async double buffering,
// used when S % 128 != 0 (or SPECSIM_ATTN_MMA_SYNC=1).  Every benchmarked
// configuration (S % 128 == 0) runs the tcgen05 / TMEM / TMA kernels of
// attention_tc.cu; the dispatch is in forward() / backward() below.
//
// Layouts: qkv [T, NQ] bf16 (T = B*S token rows; q head h at column h*HD, k
// head g at Q + g*HD, v head g at Q + KV + g*HD); o / dO [T, Q]; lse / D
// [nh, T] fp32; dqkv [T, NQ] bf16.
#include <cuda_bf16.h>

#include <cstdlib>

#include "attention.h"
#include "common.h"
#include "gemm.h"

namespace specsim {
namespace attn {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled tile of ROWS x HD bf16: 16-byte chunk c of row r lives at chunk
// c ^ (r & 7) so ldmatrix row groups hit distinct banks.
template <int HD>
struct Tile {
  __device__ static __forceinline__ int off(int r, int c /*chunk*/) {
    return r * HD + ((c ^ (r & 7)) << 3);
  }
};

// Cooperative cp.async of `rows` rows (ld elements apart) into a swizzled tile.
template <int HD, int NT>
__device__ __forceinline__ void load_tile(__nv_bfloat16* dst, const __nv_bfloat16* src,
                                          long long ld, int rows, int tid) {
  constexpr int C = HD / 8;
  for (int i = tid; i < rows * C; i += NT) {
    const int r = i / C, c = i % C;
    cp_async16(dst + Tile<HD>::off(r, c), src + static_cast<long long>(r) * ld + c * 8);
  }
}

// A-operand fragment (16 rows x 16 cols at (r0, k0)) from a swizzled tile.
template <int HD>
__device__ __forceinline__ void lds_a(const __nv_bfloat16* t, int r0, int k0, int lane,
                                      uint32_t (&a)[4]) {
  const int r = r0 + (lane & 15);
  const int c = (k0 >> 3) + (lane >> 4);
  ldsm_x4(smem_addr(t + Tile<HD>::off(r, c)), a[0], a[1], a[2], a[3]);
}

// B-operand fragments for two n-tiles where the tile is stored [n, k]
// (rows = n): n in [n0, n0+16), k in [k0, k0+16).  b[0..1] ntile 0, b[2..3] ntile 1.
template <int HD>
__device__ __forceinline__ void lds_b_nk(const __nv_bfloat16* t, int n0, int k0, int lane,
                                         uint32_t (&b)[4]) {
  const int r = n0 + (lane & 7) + ((lane >> 4) << 3);
  const int c = (k0 >> 3) + ((lane >> 3) & 1);
  ldsm_x4(smem_addr(t + Tile<HD>::off(r, c)), b[0], b[1], b[2], b[3]);
}

// B-operand fragments for two n-tiles where the tile is stored [k, n]
// (rows = k): k in [k0, k0+16), n in [n0, n0+16) (ldmatrix.trans).
template <int HD>
__device__ __forceinline__ void lds_b_kn(const __nv_bfloat16* t, int k0, int n0, int lane,
                                         uint32_t (&b)[4]) {
  const int r = k0 + (lane & 7) + (((lane >> 3) & 1) << 3);
  const int c = (n0 >> 3) + (lane >> 4);
  ldsm_x4_t(smem_addr(t + Tile<HD>::off(r, c)), b[0], b[1], b[2], b[3]);
}

// ------------------------------------------------------------------ forward
template <int HD>
__global__ void __launch_bounds__(128) attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       __nv_bfloat16* __restrict__ out,
                                                       float* __restrict__ lse, Dims d) {
  constexpr int BQ = 64, BKV = 64, NT = 128;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + BQ * HD;       // [2][BKV][HD]
  __nv_bfloat16* sV = sK + 2 * BKV * HD;  // [2][BKV][HD]

  const int qb = gridDim.x - 1 - blockIdx.x;  // heaviest (most keys) first
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / (d.nh / d.nkv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long row0 = static_cast<long long>(b) * d.S;
  const __nv_bfloat16* qbase = qkv + (row0 + qb * BQ) * d.NQ + h * HD;
  const __nv_bfloat16* kbase = qkv + row0 * d.NQ + d.Q + g * HD;
  const __nv_bfloat16* vbase = qkv + row0 * d.NQ + d.Q + d.KV + g * HD;

  load_tile<HD, NT>(sQ, qbase, d.NQ, BQ, tid);
  load_tile<HD, NT>(sK, kbase, d.NQ, BKV, tid);
  load_tile<HD, NT>(sV, vbase, d.NQ, BKV, tid);
  cp_async_commit();

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];
  const float sl2 = d.scale * kLog2e;
  const int q_lo = qb * BQ + warp * 16 + (lane >> 2);  // this thread's rows: q_lo, q_lo + 8

  const int nkv = qb + 1;
  for (int j = 0; j < nkv; ++j) {
    if (j + 1 < nkv) {
      const int nb = (j + 1) & 1;
      load_tile<HD, NT>(sK + nb * BKV * HD, kbase + static_cast<long long>(j + 1) * BKV * d.NQ,
                        d.NQ, BKV, tid);
      load_tile<HD, NT>(sV + nb * BKV * HD, vbase + static_cast<long long>(j + 1) * BKV * d.NQ,
                        d.NQ, BKV, tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) lds_a<HD>(sQ, warp * 16, kk * 16, lane, qf[kk]);
    }
    const __nv_bfloat16* tK = sK + (j & 1) * BKV * HD;
    const __nv_bfloat16* tV = sV + (j & 1) * BKV * HD;

    float s[BKV / 8][4];
#pragma unroll
    for (int i = 0; i < BKV / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < BKV / 16; ++np) {
        uint32_t bb[4];
        lds_b_nk<HD>(tK, np * 16, kk * 16, lane, bb);
        mma16816(s[2 * np], qf[kk], bb[0], bb[1]);
        mma16816(s[2 * np + 1], qf[kk], bb[2], bb[3]);
      }
    }
    // scale into the log2 domain, causal mask on the diagonal block
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nt][e] * sl2;
        if (j == qb) {
          const int key = j * BKV + nt * 8 + 2 * (lane & 3) + (e & 1);
          const int q = q_lo + ((e >> 1) << 3);
          if (key > q) v = -INFINITY;
        }
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
      const float m_new = fmaxf(m_run[r], mx[r]);
      corr[r] = exp2f(m_run[r] - m_new);  // m_run=-inf first time -> 0
      m_run[r] = m_new;
      l_run[r] *= corr[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    uint32_t pf[BKV / 16][4];
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - m_run[0]), p1 = exp2f(s[nt][1] - m_run[0]);
      const float p2 = exp2f(s[nt][2] - m_run[1]), p3 = exp2f(s[nt][3] - m_run[1]);
      l_run[0] += p0 + p1;
      l_run[1] += p2 + p3;
      const int kk = nt >> 1, hi = nt & 1;
      pf[kk][hi * 2 + 0] = pack2(p0, p1);
      pf[kk][hi * 2 + 1] = pack2(p2, p3);
    }
    // pf[kk] = {a0: rows lo cols 0-7, a1: rows hi cols 0-7, a2: rows lo cols 8-15, a3: rows hi}
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      const uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {
        uint32_t bb[4];
        lds_b_kn<HD>(tV, kk * 16, dp * 16, lane, bb);
        mma16816(o[2 * dp], a, bb[0], bb[1]);
        mma16816(o[2 * dp + 1], a, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffff, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffff, l_run[r], 2);
  }
  const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
  const long long t0 = row0 + q_lo, t1 = t0 + 8;
  __nv_bfloat16* o0 = out + t0 * d.Q + h * HD;
  __nv_bfloat16* o1 = out + t1 * d.Q + h * HD;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(o0 + c) = pack2(o[nt][0] * inv0, o[nt][1] * inv0);
    *reinterpret_cast<uint32_t*>(o1 + c) = pack2(o[nt][2] * inv1, o[nt][3] * inv1);
  }
  if ((lane & 3) == 0) {
    const long long T = static_cast<long long>(d.B) * d.S;
    lse[h * T + t0] = (m_run[0] + log2f(l_run[0])) * kLn2;
    lse[h * T + t1] = (m_run[1] + log2f(l_run[1])) * kLn2;
  }
}

// ------------------------------------------------- backward: D = rowsum(dO*O)
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ dout,
                                    const __nv_bfloat16* __restrict__ out,
                                    float* __restrict__ D, Dims d, int hd) {
  // one warp per (token, head)
  const long long T = static_cast<long long>(d.B) * d.S;
  const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= T * d.nh) return;
  const long long t = w / d.nh;
  const int h = static_cast<int>(w % d.nh);
  const __nv_bfloat16* a = dout + t * d.Q + h * hd;
  const __nv_bfloat16* b = out + t * d.Q + h * hd;
  float s = 0.f;
  for (int i = lane * 2; i < hd; i += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + i));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(b + i));
    s += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (lane == 0) D[h * T + t] = s;
}

// ------------------------------------------------------- backward: dK, dV
template <int HD>
__global__ void __launch_bounds__(128) attn_bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ Dv, __nv_bfloat16* __restrict__ dqkv,
    Dims d) {
  constexpr int BKV = 64, BQ = 32, NT = 128;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + BKV * HD;
  __nv_bfloat16* sQ = sV + BKV * HD;      // [2][BQ][HD]
  __nv_bfloat16* sdO = sQ + 2 * BQ * HD;  // [2][BQ][HD]
  float* sL = reinterpret_cast<float*>(sdO + 2 * BQ * HD);  // [2][BQ] lse * log2e
  float* sD = sL + 2 * BQ;                                   // [2][BQ]

  const int kb = gridDim.x - 1 - blockIdx.x;  // early keys see the most queries
  const int g = blockIdx.y, b = blockIdx.z;
  const int rep = d.nh / d.nkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long T = static_cast<long long>(d.B) * d.S;
  const long long row0 = static_cast<long long>(b) * d.S;
  const int key0 = kb * BKV;

  load_tile<HD, NT>(sK, qkv + (row0 + key0) * d.NQ + d.Q + g * HD, d.NQ, BKV, tid);
  load_tile<HD, NT>(sV, qkv + (row0 + key0) * d.NQ + d.Q + d.KV + g * HD, d.NQ, BKV, tid);
  cp_async_commit();

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  const float sl2 = d.scale * kLog2e;
  const int qb0 = key0 / BQ, nqb = d.S / BQ;
  const int iters_per_head = nqb - qb0;
  const int total = rep * iters_per_head;
  const int key_lo = key0 + warp * 16 + (lane >> 2);  // rows (keys) of this thread: key_lo, +8

  auto issue = [&](int it, int buf) {
    const int hh = it / iters_per_head, qb = qb0 + it % iters_per_head;
    const int h = g * rep + hh;
    const long long r = row0 + qb * BQ;
    load_tile<HD, NT>(sQ + buf * BQ * HD, qkv + r * d.NQ + h * HD, d.NQ, BQ, tid);
    load_tile<HD, NT>(sdO + buf * BQ * HD, dout + r * d.Q + h * HD, d.Q, BQ, tid);
    if (tid < BQ) {
      sL[buf * BQ + tid] = lse[h * T + r + tid] * kLog2e;
      sD[buf * BQ + tid] = Dv[h * T + r + tid];
    }
    cp_async_commit();
  };
  issue(0, 0);

  for (int it = 0; it < total; ++it) {
    const int buf = it & 1;
    if (it + 1 < total) {
      // the other buffer was released by the trailing __syncthreads of it-1
      issue(it + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int qb = qb0 + it % iters_per_head;
    const __nv_bfloat16* tQ = sQ + buf * BQ * HD;
    const __nv_bfloat16* tdO = sdO + buf * BQ * HD;
    const float* tL = sL + buf * BQ;
    const float* tD = sD + buf * BQ;

    // S^T = K Q^T and dP^T = V dO^T : [16 keys x 32 queries] per warp
    float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
    for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ka[4], va[4];
      lds_a<HD>(sK, warp * 16, kk * 16, lane, ka);
      lds_a<HD>(sV, warp * 16, kk * 16, lane, va);
#pragma unroll
      for (int np = 0; np < BQ / 16; ++np) {
        uint32_t bq[4], bo[4];
        lds_b_nk<HD>(tQ, np * 16, kk * 16, lane, bq);
        lds_b_nk<HD>(tdO, np * 16, kk * 16, lane, bo);
        mma16816(st[2 * np], ka, bq[0], bq[1]);
        mma16816(st[2 * np + 1], ka, bq[2], bq[3]);
        mma16816(dpt[2 * np], va, bo[0], bo[1]);
        mma16816(dpt[2 * np + 1], va, bo[2], bo[3]);
      }
    }
    // P^T, dS^T  (column index = query)
    uint32_t pa[BQ / 16][4], dsa[BQ / 16][4];
#pragma unroll
    for (int nt = 0; nt < BQ / 8; ++nt) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = nt * 8 + 2 * (lane & 3) + (e & 1);  // query within block
        const int key = key_lo + ((e >> 1) << 3);
        float v = exp2f(st[nt][e] * sl2 - tL[qi]);
        if (qb * BQ + qi < key) v = 0.f;
        p[e] = v;
        ds[e] = v * (dpt[nt][e] - tD[qi]);
      }
      const int kk = nt >> 1, hi = nt & 1;
      pa[kk][hi * 2 + 0] = pack2(p[0], p[1]);
      pa[kk][hi * 2 + 1] = pack2(p[2], p[3]);
      dsa[kk][hi * 2 + 0] = pack2(ds[0], ds[1]);
      dsa[kk][hi * 2 + 1] = pack2(ds[2], ds[3]);
    }
    // dV += P^T dO ; dK += dS^T Q   (k dim = queries)
#pragma unroll
    for (int kk = 0; kk < BQ / 16; ++kk) {
      const uint32_t a1[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
      const uint32_t a2[4] = {dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]};
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {
        uint32_t bo[4], bq[4];
        lds_b_kn<HD>(tdO, kk * 16, dp * 16, lane, bo);
        lds_b_kn<HD>(tQ, kk * 16, dp * 16, lane, bq);
        mma16816(dv[2 * dp], a1, bo[0], bo[1]);
        mma16816(dv[2 * dp + 1], a1, bo[2], bo[3]);
        mma16816(dk[2 * dp], a2, bq[0], bq[1]);
        mma16816(dk[2 * dp + 1], a2, bq[2], bq[3]);
      }
    }
    __syncthreads();
  }
  const long long t0 = row0 + key_lo, t1 = t0 + 8;
  __nv_bfloat16* k0p = dqkv + t0 * d.NQ + d.Q + g * HD;
  __nv_bfloat16* k1p = dqkv + t1 * d.NQ + d.Q + g * HD;
  __nv_bfloat16* v0p = dqkv + t0 * d.NQ + d.Q + d.KV + g * HD;
  __nv_bfloat16* v1p = dqkv + t1 * d.NQ + d.Q + d.KV + g * HD;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(k0p + c) = pack2(dk[nt][0] * d.scale, dk[nt][1] * d.scale);
    *reinterpret_cast<uint32_t*>(k1p + c) = pack2(dk[nt][2] * d.scale, dk[nt][3] * d.scale);
    *reinterpret_cast<uint32_t*>(v0p + c) = pack2(dv[nt][0], dv[nt][1]);
    *reinterpret_cast<uint32_t*>(v1p + c) = pack2(dv[nt][2], dv[nt][3]);
  }
}

// ------------------------------------------------------------ backward: dQ
template <int HD>
__global__ void __launch_bounds__(128) attn_bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ Dv, __nv_bfloat16* __restrict__ dqkv,
    Dims d) {
  constexpr int BQ = 64, BKV = 64, NT = 128;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sdO = sQ + BQ * HD;
  __nv_bfloat16* sK = sdO + BQ * HD;      // [2][BKV][HD]
  __nv_bfloat16* sV = sK + 2 * BKV * HD;  // [2][BKV][HD]

  const int qb = gridDim.x - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / (d.nh / d.nkv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long T = static_cast<long long>(d.B) * d.S;
  const long long row0 = static_cast<long long>(b) * d.S;
  const __nv_bfloat16* kbase = qkv + row0 * d.NQ + d.Q + g * HD;
  const __nv_bfloat16* vbase = qkv + row0 * d.NQ + d.Q + d.KV + g * HD;

  load_tile<HD, NT>(sQ, qkv + (row0 + qb * BQ) * d.NQ + h * HD, d.NQ, BQ, tid);
  load_tile<HD, NT>(sdO, dout + (row0 + qb * BQ) * d.Q + h * HD, d.Q, BQ, tid);
  load_tile<HD, NT>(sK, kbase, d.NQ, BKV, tid);
  load_tile<HD, NT>(sV, vbase, d.NQ, BKV, tid);
  cp_async_commit();

  const int q_lo = qb * BQ + warp * 16 + (lane >> 2);
  const float l2[2] = {lse[h * T + row0 + q_lo] * kLog2e, lse[h * T + row0 + q_lo + 8] * kLog2e};
  const float Dr[2] = {Dv[h * T + row0 + q_lo], Dv[h * T + row0 + q_lo + 8]};
  const float sl2 = d.scale * kLog2e;

  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  const int nkv = qb + 1;
  for (int j = 0; j < nkv; ++j) {
    if (j + 1 < nkv) {
      const int nb = (j + 1) & 1;
      load_tile<HD, NT>(sK + nb * BKV * HD, kbase + static_cast<long long>(j + 1) * BKV * d.NQ,
                        d.NQ, BKV, tid);
      load_tile<HD, NT>(sV + nb * BKV * HD, vbase + static_cast<long long>(j + 1) * BKV * d.NQ,
                        d.NQ, BKV, tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* tK = sK + (j & 1) * BKV * HD;
    const __nv_bfloat16* tV = sV + (j & 1) * BKV * HD;
    float s[BKV / 8][4], dp[BKV / 8][4];
#pragma unroll
    for (int i = 0; i < BKV / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t qa[4], oa[4];
      lds_a<HD>(sQ, warp * 16, kk * 16, lane, qa);
      lds_a<HD>(sdO, warp * 16, kk * 16, lane, oa);
#pragma unroll
      for (int np = 0; np < BKV / 16; ++np) {
        uint32_t bk[4], bv[4];
        lds_b_nk<HD>(tK, np * 16, kk * 16, lane, bk);
        lds_b_nk<HD>(tV, np * 16, kk * 16, lane, bv);
        mma16816(s[2 * np], qa, bk[0], bk[1]);
        mma16816(s[2 * np + 1], qa, bk[2], bk[3]);
        mma16816(dp[2 * np], oa, bv[0], bv[1]);
        mma16816(dp[2 * np + 1], oa, bv[2], bv[3]);
      }
    }
    uint32_t dsa[BKV / 16][4];
#pragma unroll
    for (int nt = 0; nt < BKV / 8; ++nt) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const int key = j * BKV + nt * 8 + 2 * (lane & 3) + (e & 1);
        float p = exp2f(s[nt][e] * sl2 - l2[r]);
        if (key > q_lo + (r << 3)) p = 0.f;
        ds[e] = p * (dp[nt][e] - Dr[r]);
      }
      const int kk = nt >> 1, hi = nt & 1;
      dsa[kk][hi * 2 + 0] = pack2(ds[0], ds[1]);
      dsa[kk][hi * 2 + 1] = pack2(ds[2], ds[3]);
    }
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      const uint32_t a[4] = {dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]};
#pragma unroll
      for (int dp2 = 0; dp2 < HD / 16; ++dp2) {
        uint32_t bk[4];
        lds_b_kn<HD>(tK, kk * 16, dp2 * 16, lane, bk);
        mma16816(dq[2 * dp2], a, bk[0], bk[1]);
        mma16816(dq[2 * dp2 + 1], a, bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
  const long long t0 = row0 + q_lo, t1 = t0 + 8;
  __nv_bfloat16* p0 = dqkv + t0 * d.NQ + h * HD;
  __nv_bfloat16* p1 = dqkv + t1 * d.NQ + h * HD;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(p0 + c) = pack2(dq[nt][0] * d.scale, dq[nt][1] * d.scale);
    *reinterpret_cast<uint32_t*>(p1 + c) = pack2(dq[nt][2] * d.scale, dq[nt][3] * d.scale);
  }
}

template <int HD>
constexpr int fwd_smem() {
  return (64 + 4 * 64) * HD * 2;
}
template <int HD>
constexpr int bwd_kv_smem() {
  return (2 * 64 + 4 * 32) * HD * 2 + 4 * 32 * 4;
}
template <int HD>
constexpr int bwd_q_smem() {
  return (2 * 64 + 4 * 64) * HD * 2;
}

template <int HD>
void prepare_t() {
  SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<HD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem<HD>()));
  SPECSIM_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv_kernel<HD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, bwd_kv_smem<HD>()));
  SPECSIM_CUDA(cudaFuncSetAttribute(attn_bwd_dq_kernel<HD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, bwd_q_smem<HD>()));
}

template <int HD>
void fwd_t(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, cudaStream_t s) {
  const int smem = fwd_smem<HD>();
  dim3 grid(d.S / 64, d.nh, d.B);
  count_launches();
  attn_fwd_kernel<HD><<<grid, 128, smem, s>>>(qkv, o, lse, d);
}

template <int HD>
void bwd_t(const __nv_bfloat16* qkv, const __nv_bfloat16* o, const __nv_bfloat16* dout,
           const float* lse, float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, cudaStream_t s) {
  const long long T = static_cast<long long>(d.B) * d.S;
  const long long warps = T * d.nh;
  count_launches();
  attn_bwd_dot_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(dout, o,
                                                                                      Dbuf, d, HD);
  const int smem_kv = bwd_kv_smem<HD>();
  const int smem_q = bwd_q_smem<HD>();
  count_launches();
  attn_bwd_dkdv_kernel<HD><<<dim3(d.S / 64, d.nkv, d.B), 128, smem_kv, s>>>(qkv, dout, lse, Dbuf,
                                                                           dqkv, d);
  count_launches();
  attn_bwd_dq_kernel<HD><<<dim3(d.S / 64, d.nh, d.B), 128, smem_q, s>>>(qkv, dout, lse, Dbuf, dqkv,
                                                                       d);
}

}  // namespace

void check_dims(const Dims& d, int hd) {
  Problems p("attention shape");
  p.check(hd == 64 || hd == 128, "head_dim must be 64 or 128");
  p.check(d.S % 64 == 0, "seq_len must be a multiple of 64");
  p.check(d.nkv > 0 && d.nh % d.nkv == 0, "n_heads must be a multiple of n_kv_heads");
  p.throw_if_any();
}

void forward_tc(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, int hd,
                const CUtensorMap& tm, cudaStream_t s);
void prepare_tc(int hd);
void backward_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse,
                 const float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, int hd, cudaStream_t s);

namespace {
bool use_tc(const Dims& d) {
  static const bool off = [] {
    const char* e = std::getenv("SPECSIM_ATTN_MMA_SYNC");
    return e && e[0] == '1';
  }();
  return !off && d.S % 128 == 0;
}
}  // namespace

void prepare(int hd) {
  if (hd == 128)
    prepare_t<128>();
  else
    prepare_t<64>();
  prepare_tc(hd);
}

void forward(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, int hd,
             cudaStream_t s) {
  const bool ttt = d.q_row_off != 0 || d.n_diag != 0;
  if (ttt && d.S % 128 != 0)
    throw std::invalid_argument("training-time-test attention needs seq_len % 128 == 0");
  if (ttt && (d.n_diag < 0 || d.n_diag > kMaxDiag || (d.n_diag > 0 && !d.diag_qkv)))
    throw std::invalid_argument("training-time-test attention: bad n_diag / diag_qkv");
  if (ttt || use_tc(d)) {
    // tcgen05 / TMEM / TMA path (attention_tc.cu); the map spans every unroll
    // step's rows up to this one
    const CUtensorMap tm = gemm::make_tensor_map(
        qkv, d.q_row_off + static_cast<long long>(d.B) * d.S, d.NQ, d.NQ, 64, 128);
    forward_tc(qkv, o, lse, d, hd, tm, s);
    return;
  }
  if (hd == 128)
    fwd_t<128>(qkv, o, lse, d, s);
  else
    fwd_t<64>(qkv, o, lse, d, s);
}

void bwd_dot(const __nv_bfloat16* dout, const __nv_bfloat16* o, float* D, const Dims& d, int hd,
             cudaStream_t s) {
  const long long T = static_cast<long long>(d.B) * d.S;
  count_launches();
  attn_bwd_dot_kernel<<<static_cast<unsigned>((T * d.nh * 32 + 255) / 256), 256, 0, s>>>(
      dout, o, D, d, hd);
}

bool backward(const __nv_bfloat16* qkv, const __nv_bfloat16* o, const __nv_bfloat16* dout,
              const float* lse, float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, int hd,
              cudaStream_t s) {
  if (use_tc(d)) {
    const long long T = static_cast<long long>(d.B) * d.S;
    count_launches();
    attn_bwd_dot_kernel<<<static_cast<unsigned>((T * d.nh * 32 + 255) / 256), 256, 0, s>>>(
        dout, o, Dbuf, d, hd);
    backward_tc(qkv, dout, lse, Dbuf, dqkv, d, hd, s);
    return d.rope_cos != nullptr;
  }
  if (hd == 128)
    bwd_t<128>(qkv, o, dout, lse, Dbuf, dqkv, d, s);
  else
    bwd_t<64>(qkv, o, dout, lse, Dbuf, dqkv, d, s);
  return false;
}

}  // namespace attn
}  // namespace specsim
