// Microbenchmark: MUFU.EX2 and FFMA2 issue rates per SM sub-partition on sm_100a
// (cycles per warp instruction with W warps per SMSP, 16 independent chains).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
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
  return 0;
}
