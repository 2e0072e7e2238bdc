// Minimal repro for the racecheck reports of the cta_group::2 GEMM prologue:
// a 2-CTA cluster whose only shared-memory use is the TMEM-allocation slot.
// Warp 1 of each CTA runs tcgen05.alloc.cta_group::2 / relinquish / dealloc
// (exactly the ptx.cuh helpers the GEMM uses) -- no other shared accesses.
// Second kernel: the other reported pattern (attn_bwd_kv_tc_kernel's lse / D
// slices): one thread bulk-copies (cp.async.bulk, async proxy) a global array
// into smem with mbarrier complete_tx, every thread waits on the mbarrier
// phase and then reads the data -- the documented completion mechanism.
// Run: compute-sanitizer --tool racecheck --racecheck-report hazard ./racecheck_tmem_alloc
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2602_05145_b200/csrc/ptx.cuh"
using namespace specsim;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1) k(int* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) ptx::tmem_alloc<512, 2>(&slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = static_cast<int>(base);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512, 2>(base);
  }
}

__global__ void __launch_bounds__(128, 1) k2(const float* g, float* out) {
  __shared__ __align__(128) float buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, sizeof(buf));
    ptx::bulk_load(buf, g, sizeof(buf), &bar);
  }
  ptx::mbar_wait(&bar, 0);
  out[threadIdx.x] = buf[threadIdx.x] + buf[threadIdx.x + 128];
}

// Third kernel: the attn_bwd_kv_tc_kernel ring.  A 3-slot ring of 256-float
// slices: thread 0 (producer) waits `empty[s]`, then bulk-copies slice it into
// slot s with complete_tx on `full[s]`; warp 1 (consumers, 32 threads) waits
// `full[s]`, reads the slice, and releases the slot.  MODE 0: the consumers
// arrive on `empty[s]` themselves; MODE 1: they arrive on `used[s]` and a
// third thread (warp 2 lane 0, the MMA issuer's role) waits `used[s]` and
// releases the slot with tcgen05.commit -> `empty[s]`, as the kernel does
// (the slot is free once the MMAs that read it have completed); MODE 2: as 1,
// but the releasing thread issues a tcgen05.mma (a dummy smem tile into TMEM)
// before the commit, so the arrive is performed asynchronously by the tensor
// core; MODE 3: as 2, with one consumer arrival per warp (lane 0 after
// __syncwarp) -- the kernel's exact situation.
template <int MODE>
__global__ void __launch_bounds__(96, 1) k3(const float* g, float* out, int iters) {
  __shared__ __align__(128) float ring[3][256];
  // dummy MMA operands, K-major SW128 (128-byte rows): A 128 rows (16 KB), B 32 rows (4 KB)
  __shared__ __align__(128) uint8_t tile_raw[20480 + 1024];
  uint8_t* tile = tile_raw + ((1024u - (ptx::smem_u32(tile_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[3], empty[3], used[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], MODE == 0 ? 32 : 1);
      ptx::mbar_init(&used[i], MODE == 3 ? 1 : 32);
    }
    ptx::fence_barrier_init();
  }
  if (MODE >= 1 && warp == 2) ptx::tmem_alloc<32>(&slot);
  for (int i = threadIdx.x; i < 5120; i += blockDim.x) reinterpret_cast<uint32_t*>(tile)[i] = 0;
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  float acc = 0.f;
  if (warp == 0 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % 3;
      ptx::mbar_wait(&empty[s], ((it / 3) & 1) ^ 1);
      ptx::mbar_arrive_expect_tx(&full[s], 1024);
      ptx::bulk_load(ring[s], g + (it & 7) * 256, 1024, &full[s]);
    }
  } else if (warp == 1) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % 3;
      ptx::mbar_wait(&full[s], (it / 3) & 1);
      acc += ring[s][lane] + ring[s][lane + 128];
      __syncwarp();
      // MODE 3: one arrival per warp by lane 0 after __syncwarp, as the kernels do
      if (MODE != 3 || lane == 0) ptx::mbar_arrive(MODE == 0 ? &empty[s] : &used[s]);
    }
  } else if (MODE >= 1 && warp == 2 && lane == 0) {
    constexpr uint32_t id = ptx::make_idesc_bf16(128, 32, false, false);
    const uint32_t a = ptx::smem_u32(tile), b = a + 16384;
    for (int it = 0; it < iters; ++it) {
      const int s = it % 3;
      ptx::mbar_wait(&used[s], (it / 3) & 1);
      ptx::tc_fence_after();
      if (MODE >= 2)
        ptx::umma_bf16(slot, ptx::make_sw128_desc(a, 16, 1024), ptx::make_sw128_desc(b, 16, 1024),
                       id, it > 0 ? 1u : 0u);
      ptx::umma_commit(&empty[s]);
    }
  }
  out[threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (MODE >= 1 && warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<32>(slot);
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  k<<<2, 64>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h = -1;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("tmem base %d: %s\n", h, cudaGetErrorString(e));
  float *g, *o;
  cudaMalloc(&g, 1024);
  cudaMalloc(&o, 512);
  cudaMemset(g, 0, 1024);
  k2<<<1, 128>>>(g, o);
  e = cudaDeviceSynchronize();
  printf("bulk-copy kernel: %s\n", cudaGetErrorString(e));
  k3<0><<<1, 96>>>(g, o, 12);
  e = cudaDeviceSynchronize();
  printf("ring, consumer release: %s\n", cudaGetErrorString(e));
  k3<1><<<1, 96>>>(g, o, 12);
  e = cudaDeviceSynchronize();
  printf("ring, tcgen05.commit release: %s\n", cudaGetErrorString(e));
  k3<2><<<1, 96>>>(g, o, 12);
  e = cudaDeviceSynchronize();
  printf("ring, tcgen05.mma + commit release: %s\n", cudaGetErrorString(e));
  k3<3><<<1, 96>>>(g, o, 12);
  e = cudaDeviceSynchronize();
  printf("ring, lane-0 arrival after __syncwarp: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
