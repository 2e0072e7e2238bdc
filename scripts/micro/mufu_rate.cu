// Microbenchmark: MUFU.EX2 and FFMA2 issue rates per SM sub-partition on sm_100a
// (cycles per warp instruction with W warps per SMSP, 16 independent chains).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t f2(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void sp(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
// degree-4 polynomial 2^x for two values (as attention_tc.cu exp2_poly2)
__device__ __forceinline__ uint64_t poly2(uint64_t x2) {
  float x0, x1; sp(x2, x0, x1);
  const uint64_t x = f2(fmaxf(x0, -120.f), fmaxf(x1, -120.f));
  const uint64_t t = fadd2(x, f2(12582912.f, 12582912.f));
  const uint64_t jf = fadd2(t, f2(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(jf, f2(-1.f, -1.f), x);
  uint64_t p = ffma2(f2(0.0095700687f, 0.0095700687f), f, f2(0.0559178069f, 0.0559178069f));
  p = ffma2(p, f, f2(0.2402474433f, 0.2402474433f));
  p = ffma2(p, f, f2(0.6931218505f, 0.6931218505f));
  p = ffma2(p, f, f2(0.9999992847f, 0.9999992847f));
  float p0, p1, t0, t1; sp(p, p0, p1); sp(t, t0, t1);
  return f2(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
            __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}
// softmax-like stream: 64 pairs of scores -> x = s*c - m (FFMA2) -> 2^x -> bf16 pack + row sum;
// POLY of every 4 pairs through the polynomial
template <int POLY>
__global__ void sm(float* out, long long* cyc, int iters) {
  float v[128];
  for (int i = 0; i < 128; ++i) v[i] = -0.01f * ((threadIdx.x * 7 + i) & 63);
  uint64_t acc[4] = {0, 0, 0, 0}; uint32_t pk = 0;
  const uint64_t c2 = f2(0.125f, 0.125f), m2 = f2(-1.f, -1.f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      const uint64_t x2 = ffma2(f2(v[i], v[i + 1]), c2, m2);
      uint64_t p2;
      if (((i >> 1) & 3) < POLY) p2 = poly2(x2);
      else { float a, b; sp(x2, a, b); p2 = f2(ex2(a), ex2(b)); }
      acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], p2);
      float a, b; sp(p2, a, b);
      __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
      pk ^= *reinterpret_cast<uint32_t*>(&h);
    }
    v[it & 127] += 1e-7f;
  }
  long long t1 = clock64();
  float s = pk; for (int i = 0; i < 4; ++i) { float a, b; sp(acc[i], a, b); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[16]; uint64_t b[16];
  for (int i = 0; i < 16; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = __float_as_uint(a[i]); }
  const uint64_t m = 0x3f0000003f000000ull, c = 0x3e0000003e000000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]);
      else if (MODE == 1) b[i] = ffma2(b[i], m, c);
      else { a[i] = ex2(a[i]); b[i] = ffma2(b[i], m, c); }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i] + __uint_as_float((uint32_t)b[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2048;
  for (int mode = 0; mode < 3; ++mode)
    for (int w = 1; w <= 4; w *= 2) {
      const int threads = 128 * w;  // w warps per SMSP
      if (mode == 0) k<0><<<148, threads>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, threads>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, threads>>>(out, cyc, iters);
      long long h[148]; cudaDeviceSynchronize(); cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      double per = (double)h[0] / (iters * 16.0);  // cycles per instruction-slot per warp
      printf("mode %s warps/SMSP %d: %.2f cycles per (warp, op); SMSP rate %.2f warp-ops/cycle\n",
             mode == 0 ? "ex2" : mode == 1 ? "ffma2" : "ex2+ffma2", w, per, w / per);
    }
  for (int poly = 0; poly < 3; ++poly)
    for (int w = 1; w <= 2; ++w) {
      const int threads = 128 * w;
      if (poly == 0) sm<0><<<148, threads>>>(out, cyc, 256);
      if (poly == 1) sm<1><<<148, threads>>>(out, cyc, 256);
      if (poly == 2) sm<2><<<148, threads>>>(out, cyc, 256);
      long long h[148]; cudaDeviceSynchronize(); cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      printf("softmax stream poly %d/4 pairs, warps/SMSP %d: %.0f cycles per 128-score row block per warp\n",
             poly, w, (double)h[0] / 256);
    }
  return 0;
}
