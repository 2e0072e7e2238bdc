// Does other shared-memory / L1 traffic slow tcgen05.mma operand reads?
// One CTA per SM; thread 0 issues back-to-back M=128 N=128 K=16 MMAs (smem
// operands: 128 B/clk of operand reads at the dense rate, see umma_rate.cu)
// while warps 1..3 generate side traffic for the same number of cycles:
//   0 none; 1 TMA-free bulk copies global->smem (cp.async.bulk, 16 KB each);
//   2 LDS/STS (ld/st.shared.v4); 3 global loads, default caching;
//   4 global loads, L1::no_allocate; 5 global stores (st.global.cs).
// Prints the MMA rate and the side traffic's bytes per cycle.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2602_05145_b200/csrc/ptx.cuh"
using namespace specsim;

__global__ void __launch_bounds__(128, 1) k(int mode, const float4* __restrict__ g, float4* gout,
                                             long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;            // 16 KB
  uint8_t* sB = smem + 16384;    // 16 KB
  uint8_t* sX = smem + 32768;    // 3 x 16 KB side buffers (one per side warp)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768 + 3 * 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
  volatile int* stop = reinterpret_cast<volatile int*>(bar + 9);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    for (int i = 1; i < 4; ++i) ptx::mbar_init(bar + i, 1);
    *stop = 0;
    ptx::fence_barrier_init();
  }
  if ((threadIdx.x >> 5) == 0) ptx::tmem_alloc<512>(slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long side_bytes = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = ptx::make_idesc_bf16(128, 128, false, false);
    const uint32_t a = ptx::smem_u32(sA), b = ptx::smem_u32(sB);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::umma_bf16(tmem, ptx::make_sw128_desc(a + kk * 32, 16, 1024),
                       ptx::make_sw128_desc(b + kk * 32, 16, 1024), id, 1u);
    ptx::umma_commit(bar);
    ptx::mbar_wait(bar, 0);
    long long t1 = clock64();
    *stop = 1;
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (warp >= 1 && mode != 0) {
    uint8_t* mine = sX + (warp - 1) * 16384;
    const float4* gsrc = g + (static_cast<long long>(blockIdx.x) * 3 + (warp - 1)) * (1 << 16);
    float4 acc = make_float4(0, 0, 0, 0);
    uint32_t ph = 0;
    long long it = 0;
    while (!*stop) {
      if (mode == 1) {
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(bar + warp, 16384);
          ptx::bulk_load(mine, gsrc + (it & 63) * 1024, 16384, bar + warp);
          ptx::mbar_wait(bar + warp, ph);
        }
        ph ^= 1;
        __syncwarp();
        side_bytes += 16384;
      } else if (mode == 2) {
        float4* s4 = reinterpret_cast<float4*>(mine);
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          float4 v = s4[(i * 32 + lane) & 1023];
          v.x += 1.f;
          s4[((i + 7) * 32 + lane) & 1023] = v;
        }
        side_bytes += 32 * 32 * 32;
      } else if (mode == 3 || mode == 4) {
        const float4* p = gsrc + (it & 255) * 256;
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (mode == 3) v[i] = __ldcs(p + i * 32 + lane);
          else asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[i].x), "=f"(v[i].y), "=f"(v[i].z), "=f"(v[i].w) : "l"(p + i * 32 + lane));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc.x += v[i].x + v[i].w;
        side_bytes += 8 * 32 * 16;
      } else if (mode == 5) {
        float4* p = gout + (static_cast<long long>(blockIdx.x) * 3 + (warp - 1)) * 8192 + (it & 31) * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) __stcs(p + i * 32 + lane, make_float4(it, 1, 2, 3));
        side_bytes += 8 * 32 * 16;
      }
      ++it;
    }
    if (acc.x == 12345.f) gout[0] = acc;
    if (lane == 0 && blockIdx.x == 0) out[warp] = side_bytes;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

int main() {
  long long *d; cudaMalloc(&d, 8 * 8);
  float4 *g, *go; cudaMalloc(&g, 148ll * 3 * (1 << 16) * 16); cudaMalloc(&go, 148ll * 3 * 8192 * 16 + 16);
  cudaMemset(g, 0, 148ll * 3 * (1 << 16) * 16);
  const int smem = 1024 + 32768 + 3 * 16384 + 256;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"none", "bulk copy global->smem", "LDS/STS", "LDG (cs)", "LDG (L1::no_allocate)", "STG (cs)"};
  for (int mode = 0; mode < 6; ++mode) {
    const int reps = 8192;
    k<<<148, 128, smem>>>(mode, g, go, d, reps);
    long long h[4] = {0, 0, 0, 0};
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / (reps * 4.0);
    printf("side traffic %-24s: %.1f cycles per N=128 MMA (ideal 64, %.0f%%), side %.1f B/clk per SM %s\n",
           names[mode], per, 6400.0 / per, (h[1] + h[2] + h[3]) / (double)h[0],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
