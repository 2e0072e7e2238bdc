// HBM-bound kernels of the draft-training step.  See kernels.h.
#include "common.h"
#include <algorithm>
#include <cstdlib>
#include <cuda_fp16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace specsim {
namespace kern {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  return q;
}

unsigned blocks_for(long long n, int per_block) {
  return static_cast<unsigned>((n + per_block - 1) / per_block);
}

// ------------------------------------------------------------ batch gather
__global__ void gather_batch_kernel(const uint4* __restrict__ ring_feat,
                                    const int32_t* __restrict__ ring_ids, long long cap, int W8,
                                    const BatchSpec* __restrict__ specp, int S, int K,
                                    uint4* __restrict__ F, int32_t* __restrict__ u,
                                    int32_t* __restrict__ y, int32_t* __restrict__ m) {
  const long long row = blockIdx.x;
  const int b = static_cast<int>(row / S), t = static_cast<int>(row % S);
  const BatchSpec& spec = *specp;
  const int L = b < spec.n ? spec.len[b] : 0;
  uint4* dst = F + row * W8;
  if (t < L) {
    const long long r = (spec.start[b] + t) % cap;
    const uint4* src = ring_feat + r * W8;
    for (int i = threadIdx.x; i < W8; i += blockDim.x) dst[i] = src[i];
  } else {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < W8; i += blockDim.x) dst[i] = z;
  }
  if (threadIdx.x < K) {
    const int j = threadIdx.x;
    const long long base = b < spec.n ? spec.start[b] : 0;
    const long long r = static_cast<long long>(j) * gridDim.x + row;
    u[r] = (t + 1 + j < L) ? ring_ids[(base + t + 1 + j) % cap] : 0;
    y[r] = (t + 2 + j < L) ? ring_ids[(base + t + 2 + j) % cap] : 0;
    m[r] = (t + 2 + j < L) ? 1 : 0;
  }
}

// Token gather only (the fc GEMMs read the features straight from the ring):
// u / y / m of every unroll slice, one thread per (slice, row), and the ring
// row of every 64-row block of the micro-batch (block j of sample b starts at
// ring row (start_b + 64 j) % cap; padding samples read row 0).
__global__ void gather_tokens_kernel(const int32_t* __restrict__ ring_ids, long long cap,
                                     const BatchSpec* __restrict__ specp, int S, int K, long long T,
                                     int32_t* __restrict__ u, int32_t* __restrict__ y,
                                     int32_t* __restrict__ m, int32_t* __restrict__ blk_rows) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const BatchSpec& spec = *specp;
  if (i < K * T) {
    const int j = static_cast<int>(i / T);
    const long long row = i - j * T;
    const int b = static_cast<int>(row / S), t = static_cast<int>(row % S);
    const int L = b < spec.n ? spec.len[b] : 0;
    const long long base = b < spec.n ? spec.start[b] : 0;
    u[i] = (t + 1 + j < L) ? ring_ids[(base + t + 1 + j) % cap] : 0;
    y[i] = (t + 2 + j < L) ? ring_ids[(base + t + 2 + j) % cap] : 0;
    m[i] = (t + 2 + j < L) ? 1 : 0;
  }
  if (i < T / 64) {
    const long long row = i * 64;
    const int b = static_cast<int>(row / S), t = static_cast<int>(row % S);
    blk_rows[i] = b < spec.n ? static_cast<int32_t>((spec.start[b] + t) % cap) : 0;
  }
}

__global__ void mask_count_kernel(const int32_t* __restrict__ m, long long T, long long* out) {
  __shared__ long long part[32];
  long long c = 0;
  for (long long i = threadIdx.x; i < T; i += blockDim.x) c += m[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffff, c, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += part[i];
    *out = s;
  }
}

__global__ void select_count_kernel(const long long* __restrict__ o, const long long* __restrict__ c,
                                    long long* __restrict__ n) {
  *n = *o > 0 ? *o : *c;
}

__global__ void ce_coef_kernel(const int32_t* __restrict__ m, const long long* __restrict__ n,
                               float* __restrict__ coef, StepWeights sw) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= sw.K * sw.T) return;
  const long long N = *n > 0 ? *n : 1;
  coef[i] = m[i] ? static_cast<float>(1.0 / static_cast<double>(N)) * sw.w[i / sw.T] : 0.f;
}

// ------------------------------------------------------------ RMSNorm fwd
constexpr int kNormThreads = 128;
// Rows are cached in registers as kMaxChunks 16-byte chunks per thread
// (H <= 1024 * kMaxChunks); the kernels are instantiated for 1, 2, 4, 8 so
// register use (and occupancy) follows the actual hidden size.

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) s += red[i];
  return s;
}

template <int kMaxChunks>
__global__ void __launch_bounds__(kNormThreads) rmsnorm_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, long long ldx, const int32_t* __restrict__ gather,
    const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ y, long long ldy,
    float* __restrict__ rstd, int H) {
  __shared__ float red[kNormThreads / 32];
  const long long t = blockIdx.x;
  const long long src_row = gather ? gather[t] : t;
  const uint4* xr = reinterpret_cast<const uint4*>(x + src_row * ldx);
  const int H8 = H >> 3;
  float v[kMaxChunks][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k) {
    const int c = threadIdx.x + k * kNormThreads;
    if (c < H8) {
      unpack8(xr[c], v[k]);
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
    }
  }
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / static_cast<float>(H) + eps);
  if (threadIdx.x == 0) rstd[t] = r;
  uint4* yr = reinterpret_cast<uint4*>(y + t * ldy);
  const float4* w4 = reinterpret_cast<const float4*>(w);
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k) {
    const int c = threadIdx.x + k * kNormThreads;
    if (c < H8) {
      const float4 wa = w4[2 * c], wb = w4[2 * c + 1];
      const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = v[k][j] * r * wv[j];
      yr[c] = pack8(o);
    }
  }
}

// ------------------------------------------------------------ RMSNorm bwd
constexpr int kBwdRows = 16;  // rows per CTA (dw partial granularity)

template <int kMaxChunks>
__global__ void __launch_bounds__(kNormThreads) rmsnorm_bwd_kernel(
    const float* __restrict__ dy, long long lddy, const __nv_bfloat16* __restrict__ x,
    long long ldx, const int32_t* __restrict__ gather, const float* __restrict__ w,
    const float* __restrict__ rstd, const float* __restrict__ resid, float* __restrict__ out32,
    __nv_bfloat16* __restrict__ out16, long long ldo, float* __restrict__ dw_part, long long T,
    int H) {
  __shared__ float red[kNormThreads / 32];
  const int H8 = H >> 3;
  float dwacc[kMaxChunks][8];
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) dwacc[k][j] = 0.f;
  const float4* w4 = reinterpret_cast<const float4*>(w);
  const bool need_dx = out32 || out16;
  const long long t0 = static_cast<long long>(blockIdx.x) * kBwdRows;
  for (long long t = t0; t < t0 + kBwdRows && t < T; ++t) {
    const long long src_row = gather ? gather[t] : t;
    const uint4* xr = reinterpret_cast<const uint4*>(x + src_row * ldx);
    const float4* gr = reinterpret_cast<const float4*>(dy + t * lddy);
    const float r = rstd[t];
    float xv[kMaxChunks][8], gw[kMaxChunks][8];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k) {
      const int c = threadIdx.x + k * kNormThreads;
      if (c < H8) {
        unpack8(xr[c], xv[k]);
        const float4 ga = gr[2 * c], gb = gr[2 * c + 1];
        const float gv[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const float4 wa = w4[2 * c], wb = w4[2 * c + 1];
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          dwacc[k][j] += gv[j] * xv[k][j] * r;
          gw[k][j] = gv[j] * wv[j];
          dot += gw[k][j] * xv[k][j];
        }
      }
    }
    if (!need_dx) continue;
    dot = block_sum(dot, red);
    const float c3 = dot / static_cast<float>(H) * r * r * r;
#pragma unroll
    for (int k = 0; k < kMaxChunks; ++k) {
      const int c = threadIdx.x + k * kNormThreads;
      if (c < H8) {
        float o[8];
        float rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (resid) {
          const float4 ra = reinterpret_cast<const float4*>(resid + t * ldo)[2 * c];
          const float4 rb = reinterpret_cast<const float4*>(resid + t * ldo)[2 * c + 1];
          rv[0] = ra.x; rv[1] = ra.y; rv[2] = ra.z; rv[3] = ra.w;
          rv[4] = rb.x; rv[5] = rb.y; rv[6] = rb.z; rv[7] = rb.w;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rv[j] + (r * gw[k][j] - xv[k][j] * c3);
        if (out32) {
          float4* op = reinterpret_cast<float4*>(out32 + t * ldo);
          op[2 * c] = make_float4(o[0], o[1], o[2], o[3]);
          op[2 * c + 1] = make_float4(o[4], o[5], o[6], o[7]);
        }
        if (out16) reinterpret_cast<uint4*>(out16 + t * ldo)[c] = pack8(o);
      }
    }
  }
  if (!dw_part) return;
  float4* dp = reinterpret_cast<float4*>(dw_part + static_cast<long long>(blockIdx.x) * H);
#pragma unroll
  for (int k = 0; k < kMaxChunks; ++k) {
    const int c = threadIdx.x + k * kNormThreads;
    if (c < H8) {
      dp[2 * c] = make_float4(dwacc[k][0], dwacc[k][1], dwacc[k][2], dwacc[k][3]);
      dp[2 * c + 1] = make_float4(dwacc[k][4], dwacc[k][5], dwacc[k][6], dwacc[k][7]);
    }
  }
}

// dw[i] = sum over partial rows.  Block = 32 columns x 8 row-slices: each
// thread sums a strided slice (rows r, r+8, ...) for one column (coalesced 128-B
// row segments across the warp), then the 8 slices are added in fixed order
// (deterministic).
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ part,
                                                     long long rows, int H,
                                                     float* __restrict__ out) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, slice = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  // four independent accumulators (rows r, r+8, r+16, r+24 of the slice):
  // four loads in flight per thread, still a fixed summation order
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  if (col < H) {
    long long r = slice;
    for (; r + 24 < rows; r += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] += part[(r + 8 * u) * H + col];
    }
    for (int u = 0; r < rows; r += 8, ++u) a[u] += part[r * H + col];
  }
  red[slice][lane] = (a[0] + a[1]) + (a[2] + a[3]);
  __syncthreads();
  if (slice == 0 && col < H) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][lane];
    out[col] = t;
  }
}

// ------------------------------------------------------------------ RoPE
__global__ void rope_kernel(__nv_bfloat16* __restrict__ qkv, long long T, int S, int NQ,
                            int n_rot_heads, int hd, const float* __restrict__ cos_t,
                            const float* __restrict__ sin_t, int inverse) {
  const int half = hd >> 1;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long per_row = static_cast<long long>(n_rot_heads) * (half >> 1);  // pairs of i
  if (idx >= T * per_row) return;
  const long long t = idx / per_row;
  const int rem = static_cast<int>(idx % per_row);
  const int h = rem / (half >> 1);
  const int i = (rem % (half >> 1)) * 2;  // two consecutive rotation indices
  const int pos = static_cast<int>(t % S);
  __nv_bfloat16* v = qkv + t * NQ + static_cast<long long>(h) * hd;
  const float2 x1 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(v + i));
  const float2 x2 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(v + i + half));
  const float c0 = cos_t[pos * half + i], c1 = cos_t[pos * half + i + 1];
  const float s0 = sin_t[pos * half + i], s1 = sin_t[pos * half + i + 1];
  float a0, a1, b0, b1;
  if (!inverse) {
    a0 = x1.x * c0 - x2.x * s0;
    a1 = x1.y * c1 - x2.y * s1;
    b0 = x2.x * c0 + x1.x * s0;
    b1 = x2.y * c1 + x1.y * s1;
  } else {
    a0 = x1.x * c0 + x2.x * s0;
    a1 = x1.y * c1 + x2.y * s1;
    b0 = x2.x * c0 - x1.x * s0;
    b1 = x2.y * c1 - x1.y * s1;
  }
  *reinterpret_cast<__nv_bfloat162*>(v + i) = __floats2bfloat162_rn(a0, a1);
  *reinterpret_cast<__nv_bfloat162*>(v + i + half) = __floats2bfloat162_rn(b0, b1);
}

// ---------------------------------------------------------------- SwiGLU
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                  __nv_bfloat16* __restrict__ act, long long T, int I) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int I8 = I >> 3;
  if (idx >= T * I8) return;
  const long long t = idx / I8;
  const int c = static_cast<int>(idx % I8);
  float g[8], u[8], o[8];
  unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * I)[c], g);
  unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * I + I)[c], u);
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = g[j] / (1.f + __expf(-g[j])) * u[j];
  reinterpret_cast<uint4*>(act + t * I)[c] = pack8(o);
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                  const __nv_bfloat16* __restrict__ dact,
                                  __nv_bfloat16* __restrict__ dgu, long long T, int I) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int I8 = I >> 3;
  if (idx >= T * I8) return;
  const long long t = idx / I8;
  const int c = static_cast<int>(idx % I8);
  float g[8], u[8], d[8], dg[8], du[8];
  unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * I)[c], g);
  unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * I + I)[c], u);
  unpack8(reinterpret_cast<const uint4*>(dact + t * I)[c], d);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float sg = 1.f / (1.f + __expf(-g[j]));
    dg[j] = d[j] * u[j] * sg * (1.f + g[j] * (1.f - sg));
    du[j] = d[j] * g[j] * sg;
  }
  reinterpret_cast<uint4*>(dgu + t * 2 * I)[c] = pack8(dg);
  reinterpret_cast<uint4*>(dgu + t * 2 * I + I)[c] = pack8(du);
}

// ------------------------------------------------------------ CE reduce
// Block = 32 consecutive rows x 8 warps.  Warp w merges the partial columns
// nb = w, w+8, ... with lane = row, so every load is 32 consecutive rows x 16 B
// (coalesced); the 8 per-warp results are merged through shared memory in
// fixed order (deterministic).
struct CeAcc {
  float max, sum, tgt;
  int arg;
};

__device__ __forceinline__ void ce_merge(CeAcc& a, float pmax, float psum, float ptgt, int parg) {
  if (pmax > a.max || (pmax == a.max && parg < a.arg)) {
    if (psum > 0.f) a.sum = a.sum * exp2f((a.max - pmax) * 1.4426950408889634f) + psum;
    a.max = pmax;
    a.arg = parg;
  } else if (psum > 0.f) {
    a.sum += psum * exp2f((pmax - a.max) * 1.4426950408889634f);
  }
  a.tgt = fmaxf(a.tgt, ptgt);
}

__global__ void __launch_bounds__(256) ce_reduce_kernel(
    const gemm::CePartial* __restrict__ part, int num_nb, long long T,
    const int32_t* __restrict__ y, const int32_t* __restrict__ m, float* __restrict__ lse,
    float* __restrict__ row_loss, int32_t* __restrict__ argmax) {
  __shared__ CeAcc red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t = static_cast<long long>(blockIdx.x) * 32 + lane;
  CeAcc a{-INFINITY, 0.f, -INFINITY, 0x7fffffff};
  if (t < T) {
    // eight partials in flight per lane before merging (the merge chain is
    // serial; the loads are not)
    constexpr int U = 8;
    for (int nb0 = warp; nb0 < num_nb; nb0 += 8 * U) {
      gemm::CePartial p[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (nb0 + 8 * u < num_nb) p[u] = part[static_cast<long long>(nb0 + 8 * u) * T + t];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (nb0 + 8 * u < num_nb) ce_merge(a, p[u].max, p[u].sum, p[u].target, p[u].argmax);
    }
  }
  red[warp][lane] = a;
  __syncthreads();
  if (warp == 0 && t < T) {
    CeAcc r = red[0][lane];
    for (int w = 1; w < 8; ++w) {
      const CeAcc o = red[w][lane];
      ce_merge(r, o.max, o.sum, o.tgt, o.arg);
    }
    const float l = r.max + logf(r.sum);
    lse[t] = l;
    argmax[t] = r.arg;
    row_loss[t] = m[t] ? (l - r.tgt) : 0.f;
  }
}

__global__ void ce_finalize_kernel(const float* __restrict__ row_loss,
                                   const int32_t* __restrict__ argmax,
                                   const int32_t* __restrict__ y, const int32_t* __restrict__ m,
                                   const long long* __restrict__ n_global, StepWeights sw,
                                   double* __restrict__ stats) {
  __shared__ double sl[32], sv[32], sc[32];
  __shared__ double step_loss[kMaxTtt];
  const long long T = sw.T;
  for (int j = 0; j < sw.K; ++j) {
    double l = 0.0, v = 0.0, c = 0.0;
    const long long r0 = static_cast<long long>(j) * T;
    for (long long i = threadIdx.x; i < T; i += blockDim.x) {
      l += row_loss[r0 + i];
      if (j == 0 && m[i]) {
        v += 1.0;
        c += (argmax[i] == y[i]) ? 1.0 : 0.0;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      l += __shfl_xor_sync(0xffffffff, l, o);
      v += __shfl_xor_sync(0xffffffff, v, o);
      c += __shfl_xor_sync(0xffffffff, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
      sl[threadIdx.x >> 5] = l;
      sv[threadIdx.x >> 5] = v;
      sc[threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double L = 0, V = 0, Cc = 0;
      for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
        L += sl[i];
        V += sv[i];
        Cc += sc[i];
      }
      step_loss[j] = L;
      if (j == 0) {
        stats[1] = V;
        stats[2] = Cc;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double V = stats[1];
    const double N = *n_global > 0 ? static_cast<double>(*n_global) : (V > 0 ? V : 1.0);
    double total = 0.0;
    for (int j = 0; j < sw.K; ++j) total += static_cast<double>(sw.w[j]) * (step_loss[j] / N);
    stats[0] = total;
  }
}

// ----------------------------------------------------------------- AdamW
__global__ void adamw_kernel(long long n4, float4* __restrict__ p, float4* __restrict__ m,
                             float4* __restrict__ v, const float4* __restrict__ g,
                             uint2* __restrict__ p16, const gemm::AdamDev* __restrict__ hpp) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const gemm::AdamDev hp = *hpp;
  float4 pp = p[i], mm = m[i], vv = v[i];
  const float4 gg = g[i];
  float* pa = &pp.x;
  float* ma = &mm.x;
  float* va = &vv.x;
  const float* ga = &gg.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float pi = pa[j] * hp.decay;
    const float mi = ma[j] + (ga[j] - ma[j]) * (1.f - hp.beta1);
    const float vi = va[j] * hp.beta2 + (1.f - hp.beta2) * ga[j] * ga[j];
    const float denom = sqrtf(vi) / hp.bc2_sqrt + hp.eps;
    pi = pi - hp.step_size * (mi / denom);
    pa[j] = pi;
    ma[j] = mi;
    va[j] = vi;
  }
  p[i] = pp;
  m[i] = mm;
  v[i] = vv;
  __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y), hi = __floats2bfloat162_rn(pp.z, pp.w);
  p16[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

__global__ void f32_to_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ y,
                                   long long n4) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 a = x[i];
  __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
  y[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

// ------------------------------------------------------- signal packing
__global__ void pack_signals_kernel(LayerPtrs layers, int n_layers, long long ld, int H8,
                                    const int32_t* __restrict__ idx, int n,
                                    uint4* __restrict__ ring, long long cap, long long pos) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const long long src_row = idx ? idx[i] : i;
  uint4* dst = ring + ((pos + i) % cap) * static_cast<long long>(H8) * n_layers;
  for (int l = 0; l < n_layers; ++l) {
    const uint4* src = reinterpret_cast<const uint4*>(layers.p[l] + src_row * ld);
    for (int c = threadIdx.x; c < H8; c += blockDim.x) dst[l * H8 + c] = src[c];
  }
}

// TMA-staged pack: one warp per CTA, lane 0 drives the bulk-copy engine --
// every accepted row's layer segments are bulk-loaded (cp.async.bulk, no
// register staging) into shared memory at their packed offsets, then each
// assembled [layers*H] row is bulk-stored to its ring row.  The SMs issue a
// handful of instructions per row, so a capture on the serving GPU leaves its
// compute to verification.  Requires 16-byte aligned rows (H % 8, ld % 8).
constexpr int kPackRowsMax = 4;
__global__ void __launch_bounds__(32) pack_signals_tma_kernel(
    LayerPtrs layers, int n_layers, long long ld, int H, const int32_t* __restrict__ idx, int n,
    int rows_per_cta, __nv_bfloat16* __restrict__ ring, long long cap, long long pos) {
  extern __shared__ __align__(128) uint8_t pack_smem[];
  __shared__ __align__(8) uint64_t bar;
  const int i0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, n - i0);
  const uint32_t seg = static_cast<uint32_t>(H) * 2;  // bytes per layer segment
  const uint32_t row_bytes = seg * n_layers;
  if (threadIdx.x == 0 && nr > 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
    ptx::mbar_arrive_expect_tx(&bar, row_bytes * nr);
    for (int r = 0; r < nr; ++r) {
      const long long src_row = idx ? idx[i0 + r] : i0 + r;
      for (int l = 0; l < n_layers; ++l)
        ptx::bulk_load(pack_smem + r * row_bytes + l * seg, layers.p[l] + src_row * ld, seg, &bar);
    }
    ptx::mbar_wait(&bar, 0);
    for (int r = 0; r < nr; ++r) {
      const long long dst_row = (pos + i0 + r) % cap;
      ptx::bulk_store(reinterpret_cast<uint8_t*>(ring) + dst_row * row_bytes,
                      pack_smem + r * row_bytes, row_bytes);
    }
    ptx::bulk_commit();
    ptx::bulk_wait_all();
  }
}

__global__ void pack_packed_kernel(const uint4* __restrict__ src, int W8, int n,
                                   uint4* __restrict__ ring, long long cap, long long pos) {
  const int i = blockIdx.x;
  if (i >= n) return;
  uint4* dst = ring + ((pos + i) % cap) * W8;
  const uint4* s = src + static_cast<long long>(i) * W8;
  for (int c = threadIdx.x; c < W8; c += blockDim.x) dst[c] = s[c];
}

constexpr int kCeGradSeg = 4;  // 16-byte segments per thread, all loads issued first

__global__ void __launch_bounds__(256) ce_grad_kernel(
    const __half* __restrict__ logits, long long ldl, const gemm::CePartial* __restrict__ part,
    const float* __restrict__ lse, const float* __restrict__ coef,
    const int32_t* __restrict__ y, int v0, int vn, long long T, __nv_bfloat16* __restrict__ dlog,
    long long ldd) {
  // one row per blockIdx.x (T may exceed the 65535 limit of grid.y); each
  // thread owns kCeGradSeg 8-column segments
  // strided by the block width (coalesced), with every logit load in flight
  // before the first use; the stored value is l - m with m the row max of the
  // 128-column half tile (the forward's partial), so p = 2^((delta + m - lse) log2 e)
  const long long t = blockIdx.x;
  const int j0 = (blockIdx.y * kCeGradSeg * blockDim.x + threadIdx.x) * 8;
  const int stride = blockDim.x * 8;
  const float l2e = 1.4426950408889634f;
  uint4 raw[kCeGradSeg];
#pragma unroll
  for (int k = 0; k < kCeGradSeg; ++k) {
    const int j = j0 + k * stride;
    if (j < vn) raw[k] = __ldcs(reinterpret_cast<const uint4*>(logits + t * ldl + v0 + j));
  }
  const float lse_t = lse[t];
  const float coef_t = coef[t];
  const int tgt = y[t] - v0;
#pragma unroll
  for (int k = 0; k < kCeGradSeg; ++k) {
    const int j = j0 + k * stride;
    if (j >= vn) break;
    const float off = part[static_cast<long long>((v0 + j) >> 7) * T + t].max - lse_t;
    const uint32_t w[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
    float x[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float p = exp2f((x[i] + off) * l2e);
      x[i] = (p - (j + i == tgt ? 1.f : 0.f)) * coef_t;
    }
    *reinterpret_cast<uint4*>(dlog + t * ldd + j) = pack8(x);
  }
}

}  // namespace

// ============================================================== launchers
void gather_batch(const __nv_bfloat16* ring_feat, const int32_t* ring_ids, long long cap, int W,
                  const BatchSpec* spec, int B, int S, int K, __nv_bfloat16* F, int32_t* u,
                  int32_t* y, int32_t* m, cudaStream_t s) {
  const long long T = static_cast<long long>(B) * S;
  count_launches();
  gather_batch_kernel<<<static_cast<unsigned>(T), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(ring_feat), ring_ids, cap, W / 8, spec, S, K,
      reinterpret_cast<uint4*>(F), u, y, m);
}

void gather_tokens(const int32_t* ring_ids, long long cap, const BatchSpec* spec, int B, int S,
                   int K, int32_t* u, int32_t* y, int32_t* m, int32_t* blk_rows, cudaStream_t s) {
  const long long T = static_cast<long long>(B) * S;
  count_launches();
  gather_tokens_kernel<<<blocks_for(K * T, 256), 256, 0, s>>>(ring_ids, cap, spec, S, K, T, u, y,
                                                             m, blk_rows);
}

void mask_count(const int32_t* m, long long T, long long* out, cudaStream_t s) {
  count_launches();
  mask_count_kernel<<<1, 1024, 0, s>>>(m, T, out);
}

void select_count(const long long* override_n, const long long* counted, long long* n_global,
                  cudaStream_t s) {
  count_launches();
  select_count_kernel<<<1, 1, 0, s>>>(override_n, counted, n_global);
}

void ce_coef(const int32_t* m, const long long* n_global, float* coef, const StepWeights& sw,
             cudaStream_t s) {
  count_launches();
  ce_coef_kernel<<<blocks_for(sw.K * sw.T, 256), 256, 0, s>>>(m, n_global, coef, sw);
}

void rmsnorm_fwd(const __nv_bfloat16* x, long long ldx, const int32_t* gather, const float* w,
                 float eps, __nv_bfloat16* y, long long ldy, float* rstd, long long T, int H,
                 cudaStream_t s) {
  count_launches();
  const unsigned g = static_cast<unsigned>(T);
  if (H <= 1024)
    rmsnorm_fwd_kernel<1><<<g, kNormThreads, 0, s>>>(x, ldx, gather, w, eps, y, ldy, rstd, H);
  else if (H <= 2048)
    rmsnorm_fwd_kernel<2><<<g, kNormThreads, 0, s>>>(x, ldx, gather, w, eps, y, ldy, rstd, H);
  else if (H <= 4096)
    rmsnorm_fwd_kernel<4><<<g, kNormThreads, 0, s>>>(x, ldx, gather, w, eps, y, ldy, rstd, H);
  else
    rmsnorm_fwd_kernel<8><<<g, kNormThreads, 0, s>>>(x, ldx, gather, w, eps, y, ldy, rstd, H);
}

long long rmsnorm_bwd_partial_rows(long long T) { return (T + kBwdRows - 1) / kBwdRows; }

void rmsnorm_bwd(const float* dy, long long lddy, const __nv_bfloat16* x, long long ldx,
                 const int32_t* gather, const float* w, const float* rstd, const float* resid,
                 float* out_f32, __nv_bfloat16* out_bf16, long long ldo, float* dw,
                 float* dw_partial, long long T, int H, cudaStream_t s) {
  const long long nb = rmsnorm_bwd_partial_rows(T);
  count_launches();
  const unsigned g = static_cast<unsigned>(nb);
#define SPECSIM_RMS_BWD(C)                                                                     \
  rmsnorm_bwd_kernel<C><<<g, kNormThreads, 0, s>>>(dy, lddy, x, ldx, gather, w, rstd, resid, \
                                                   out_f32, out_bf16, ldo, dw_partial, T, H)
  if (H <= 1024)
    SPECSIM_RMS_BWD(1);
  else if (H <= 2048)
    SPECSIM_RMS_BWD(2);
  else if (H <= 4096)
    SPECSIM_RMS_BWD(4);
  else
    SPECSIM_RMS_BWD(8);
#undef SPECSIM_RMS_BWD
  if (!dw) return;
  colsum(dw_partial, nb, H, dw, s);
}

void colsum(const float* parts, long long rows, int H, float* out, cudaStream_t s) {
  count_launches();
  colsum_kernel<<<blocks_for(H, 32), 256, 0, s>>>(parts, rows, H, out);
}

void rope(__nv_bfloat16* qkv, long long T, int S, int NQ, int n_rot_heads, int hd,
          const float* cos_t, const float* sin_t, bool inverse, cudaStream_t s) {
  const long long n = T * n_rot_heads * (hd / 4);
  count_launches();
  rope_kernel<<<blocks_for(n, 256), 256, 0, s>>>(qkv, T, S, NQ, n_rot_heads, hd, cos_t, sin_t,
                                                 inverse ? 1 : 0);
}

void swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* act, long long T, int I, cudaStream_t s) {
  count_launches();
  swiglu_fwd_kernel<<<blocks_for(T * (I / 8), 256), 256, 0, s>>>(gu, act, T, I);
}

void swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* dact, __nv_bfloat16* dgu,
                long long T, int I, cudaStream_t s) {
  count_launches();
  swiglu_bwd_kernel<<<blocks_for(T * (I / 8), 256), 256, 0, s>>>(gu, dact, dgu, T, I);
}

void ce_grad(const __half* logits, long long ldl, const gemm::CePartial* partials,
             const float* lse, const float* coef, const int32_t* y, int v0, long long T, int vn,
             __nv_bfloat16* dlog, long long ldd, cudaStream_t s) {
  if (T == 0) return;
  count_launches();
  ce_grad_kernel<<<dim3(static_cast<unsigned>(T), blocks_for(vn / 8, 256 * kCeGradSeg)), 256, 0,
                   s>>>(
      logits, ldl, partials, lse, coef, y, v0, vn, T, dlog, ldd);
}

void ce_reduce(const gemm::CePartial* partials, int num_nb, long long T, const int32_t* y,
               const int32_t* m, float* lse, float* row_loss, int32_t* argmax, cudaStream_t s) {
  count_launches();
  ce_reduce_kernel<<<blocks_for(T, 32), 256, 0, s>>>(partials, num_nb, T, y, m, lse, row_loss,
                                                     argmax);
}

void ce_finalize(const float* row_loss, const int32_t* argmax, const int32_t* y, const int32_t* m,
                 const long long* n_global, const StepWeights& sw, double* stats, cudaStream_t s) {
  count_launches();
  ce_finalize_kernel<<<1, 1024, 0, s>>>(row_loss, argmax, y, m, n_global, sw, stats);
}

void adamw(long long n, float* p, float* m, float* v, const float* g, __nv_bfloat16* p16,
           const gemm::AdamDev* hp, cudaStream_t s) {
  const long long n4 = n / 4;  // n is a multiple of 8 (checked at trainer creation)
  count_launches();
  adamw_kernel<<<blocks_for(n4, 256), 256, 0, s>>>(
      n4, reinterpret_cast<float4*>(p), reinterpret_cast<float4*>(m),
      reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(g),
      reinterpret_cast<uint2*>(p16), hp);
}

void f32_to_bf16(const float* x, __nv_bfloat16* y, long long n, cudaStream_t s) {
  count_launches();
  f32_to_bf16_kernel<<<blocks_for(n / 4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x),
                                                            reinterpret_cast<uint2*>(y), n / 4);
}

void pack_signals(const LayerPtrs& layers, int n_layers, long long ld, int H, const int32_t* idx,
                  int n, __nv_bfloat16* ring_feat, long long cap, long long pos, cudaStream_t s) {
  if (n <= 0) return;
  count_launches();
  static const bool tma = [] {
    const char* e = std::getenv("SPECSIM_PACK_SM");  // A/B: SM-copy pack kernel
    return !(e && e[0] == '1');
  }();
  const long long row_bytes = 2ll * H * n_layers;
  bool aligned = (ld % 8) == 0 && (H % 8) == 0 && reinterpret_cast<uintptr_t>(ring_feat) % 16 == 0;
  for (int l = 0; l < n_layers; ++l)
    aligned = aligned && reinterpret_cast<uintptr_t>(layers.p[l]) % 16 == 0;
  if (tma && aligned && row_bytes <= 96 * 1024) {
    const int rows = static_cast<int>(std::max<long long>(
        1, std::min<long long>(kPackRowsMax, (96 * 1024) / row_bytes)));
    const int smem = static_cast<int>(rows * row_bytes);
    static int smem_set = 0;
    if (smem > smem_set) {
      SPECSIM_CUDA(cudaFuncSetAttribute(pack_signals_tma_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
      smem_set = 200 * 1024;
    }
    pack_signals_tma_kernel<<<(n + rows - 1) / rows, 32, smem, s>>>(
        layers, n_layers, ld, H, idx, n, rows, ring_feat, cap, pos);
    return;
  }
  pack_signals_kernel<<<n, 128, 0, s>>>(layers, n_layers, ld, H / 8, idx,
                                        n, reinterpret_cast<uint4*>(ring_feat), cap, pos);
}

__global__ void fetch_mapped_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                    int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = __ldcv(src + i);
}

void fetch_mapped(const uint32_t* src, uint32_t* dst, int n_words, cudaStream_t s) {
  count_launches();
  // one block per ~1k words (a whole train(job) table moves in one launch;
  // PCIe reads are latency-bound, so more lanes in flight)
  const int blocks = std::max(1, std::min(64, (n_words + 1023) / 1024));
  fetch_mapped_kernel<<<blocks, 128, 0, s>>>(src, dst, n_words);
}

void store_mapped(const uint32_t* src, uint32_t* dst, int n_words, cudaStream_t s) {
  count_launches();
  fetch_mapped_kernel<<<1, 128, 0, s>>>(src, dst, n_words);
}

void pack_packed(const __nv_bfloat16* src, int W, int n, __nv_bfloat16* ring_feat, long long cap,
                 long long pos, cudaStream_t s) {
  if (n <= 0) return;
  count_launches();
  pack_packed_kernel<<<n, 128, 0, s>>>(reinterpret_cast<const uint4*>(src), W / 8, n,
                                       reinterpret_cast<uint4*>(ring_feat), cap, pos);
}

}  // namespace kern
}  // namespace specsim
