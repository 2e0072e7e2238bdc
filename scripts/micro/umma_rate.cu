// tcgen05.mma issue-rate microbenchmark (sm_100a, cta_group::1, kind::f16):
// one CTA per SM, one thread issues R back-to-back M=128 x N x K=16 MMAs from
// SW128 K-major smem operands (or A from TMEM), accumulating into TMEM; the
// cycles between the first issue and the commit's mbarrier completion give
// the per-SM throughput as a fraction of the dense bf16 rate (8192 FLOP/clk).
// Shapes are the attention kernels' (N = 64 score tiles, N = 128 / 256).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2602_05145_b200/csrc/ptx.cuh"
using namespace specsim;

template <int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 128 x 64 bf16 (16 KB), K-major SW128
  uint8_t* sB = smem + 16384;         // N x 64 bf16
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_barrier_init(); }
  if ((threadIdx.x >> 5) == 0) ptx::tmem_alloc<512>(slot);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = ptx::make_idesc_bf16(128, N, false, false);
    const uint32_t a = ptx::smem_u32(sA), b = ptx::smem_u32(sB);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = ptx::make_sw128_desc(b + kk * 32, 16, 1024);
        if constexpr (A_TMEM) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
                       "r"(tmem + kk * 8), "l"(bd), "r"(id), "r"(1u) : "memory");
        } else {
          ptx::umma_bf16(tmem + 256, ptx::make_sw128_desc(a + kk * 32, 16, 1024), bd, id, 1u);
        }
      }
    }
    ptx::umma_commit(bar);
    ptx::mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int N, bool AT>
void run(long long* d) {
  const int reps = 4096, smem = 1024 + 16384 + 256 * 128 + 64;
  cudaFuncSetAttribute(k<N, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, AT><<<148, 128, smem>>>(d, reps);
  long long h = 0;
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (reps * 4.0);
  const double ideal = 2.0 * 128 * N * 16 / 8192.0;
  printf("M=128 N=%3d K=16 A from %s: %.1f cycles per MMA (dense-rate ideal %.0f) -> %.0f%% %s\n", N,
         AT ? "TMEM" : "smem", per, ideal, 100.0 * ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<64, true>(d); run<128, true>(d); run<256, true>(d);
  return 0;
}
