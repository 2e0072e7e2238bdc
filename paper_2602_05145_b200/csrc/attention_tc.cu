// Causal GQA attention forward on the 5th-generation tensor cores.
//
// One CTA = one (sample, query head, 128-query block).  Warp roles:
//   warp 0      TMA producer: Q once, then K_j / V_j (128-key blocks) into a
//               2-deep ring (SWIZZLE_128B tiles, one tensor map over qkv)
//   warp 1      MMA issuer (one lane): S_j = Q K_j^T into one of two TMEM
//               S buffers, then O += P_j V_j with P_j from shared memory
//   warps 2..5  softmax: one query row per thread (TMEM lane), so row max /
//               sum need no shuffles; P_j written to smem in the UMMA K-major
//               SW128 layout; lazy rescaling (only when the row max grows by
//               more than 2^8) keeps O read-modify-writes rare
// TMEM: S0 | S1 | O  (128 + 128 + HD fp32 columns).
#include <cuda_bf16.h>

#include "attention.h"
#include "common.h"
#include "ptx.cuh"

namespace specsim {
namespace attn {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int BQ = 128, BKV = 128;
constexpr int TILE = BQ * 64 * 2;  // one [128 x 64] bf16 SW128 tile = 16 KB

template <int HD>
struct FwdSmem {
  static constexpr int ATOMS = HD / 64;            // 64-wide column tiles per operand
  static constexpr int Q = ATOMS * TILE;           // [128 q x HD]
  static constexpr int KV = ATOMS * TILE;          // [128 keys x HD]
  static constexpr int P = 2 * TILE;               // [128 q x 128 keys]
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q;          // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * KV;     // 2 stages
  static constexpr int OFF_P = OFF_V + 2 * KV;
  static constexpr int OFF_BAR = OFF_P + P;
  static constexpr int BYTES = 1024 + OFF_BAR + 256;
};

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// K-major SW128 descriptor for a multi-tile operand: 16-wide K step kk lives in
// tile kk/4 at +32 B per step inside the 128-byte swizzle atom.
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  return ptx::make_sw128_desc(base + (kk >> 2) * TILE + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor: 64-wide N chunks 16 KB apart (128 K-rows each),
// K step of 16 rows = 2048 B.
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int kk) {
  return ptx::make_sw128_desc(base + kk * 2048, TILE, 1024);
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, Dims d) {
  using L = FwdSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* k_empty = bar + 3;   // [2]
  uint64_t* v_full = bar + 5;    // [2]
  uint64_t* v_empty = bar + 7;   // [2]
  uint64_t* s_full = bar + 9;    // [2]
  uint64_t* s_free = bar + 11;   // [2]
  uint64_t* p_full = bar + 13;
  uint64_t* pv_done = bar + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int qb = gridDim.x - 1 - blockIdx.x;  // most keys first
  const int h = blockIdx.y, b = blockIdx.z;
  const int g = h / (d.nh / d.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * d.S;
  const int nkv = qb + 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
    }
    ptx::mbar_init(p_full, 4);
    ptx::mbar_init(pv_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA
      constexpr int A = L::ATOMS;
      ptx::mbar_arrive_expect_tx(q_full, L::Q);
      for (int a = 0; a < A; ++a)
        ptx::tma_load_2d(&tm, q_full, sQ + a * TILE, h * HD + 64 * a, row0 + qb * BQ);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        ptx::mbar_wait(&k_empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&k_full[s], L::KV);
        for (int a = 0; a < A; ++a)
          ptx::tma_load_2d(&tm, &k_full[s], sK + s * L::KV + a * TILE, d.Q + g * HD + 64 * a,
                           row0 + j * BKV);
        ptx::mbar_wait(&v_empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&v_full[s], L::KV);
        for (int a = 0; a < A; ++a)
          ptx::tma_load_2d(&tm, &v_full[s], sV + s * L::KV + a * TILE,
                           d.Q + d.KV + g * HD + 64 * a, row0 + j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA
      constexpr uint32_t idS = ptx::make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idO = ptx::make_idesc_bf16(BQ, HD, false, true);
      const uint32_t aQ = ptx::smem_u32(sQ), aP = ptx::smem_u32(sP);
      auto issue_s = [&](int j) {
        const int s = j & 1;
        ptx::mbar_wait(&k_full[s], (j >> 1) & 1);
        ptx::mbar_wait(&s_free[s], ((j >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t aK = ptx::smem_u32(sK + s * L::KV);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::umma_bf16(tS[s], kdesc(aQ, kk), kdesc(aK, kk), idS, kk > 0 ? 1u : 0u);
        ptx::umma_commit(&s_full[s]);
        ptx::umma_commit(&k_empty[s]);
      };
      ptx::mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        const int s = j & 1;
        ptx::mbar_wait(p_full, j & 1);
        ptx::mbar_wait(&v_full[s], (j >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aV = ptx::smem_u32(sV + s * L::KV);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          ptx::umma_bf16(tO, kdesc(aP, kk), mndesc(aV, kk), idO, (j > 0 || kk > 0) ? 1u : 0u);
        ptx::umma_commit(pv_done);
        ptx::umma_commit(&v_empty[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // query row within the block (= TMEM lane)
    const int q = qb * BQ + r;       // position within the sample
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float sl2 = d.scale * kLog2e;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int s = j & 1;
      ptx::mbar_wait(&s_full[s], (j >> 1) & 1);
      ptx::tc_fence_after();
      // row max over this block's 128 scores
      float mx = -INFINITY;
      uint32_t v[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x32(tS[s] + lane_off + c * 32, v[c]);
      ptx::tmem_ld_wait();
      const bool diag = (j == qb);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = __uint_as_float(v[c][i]) * sl2;
          if (diag && (c * 32 + i) > r) x = -INFINITY;
          v[c][i] = __float_as_uint(x);
          mx = fmaxf(mx, x);
        }
      // S buffer consumed: the MMA may overwrite it with S_{j+2}
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&s_free[s]);
      // O and the P buffer are free once PV_{j-1} has completed
      if (j > 0) ptx::mbar_wait(pv_done, (j - 1) & 1);
      ptx::tc_fence_after();
      // lazy rescale: a row moves its reference max only when the max grows by
      // more than 2^8; the O read-modify-write is warp-collective (tcgen05.ld /
      // st are .sync.aligned), so the whole warp does it when any lane needs it
      const bool need = mx > m_run + 8.f;
      float corr = 1.f;
      if (need) {
        corr = exp2f(m_run - mx);  // 0 on the first block
        l_run *= corr;
        m_run = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(tO + lane_off + c * 32, o);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
          tmem_st_32x32b_x32(tO + lane_off + c * 32, o);
        }
        tmem_st_wait();
      }
      // P = exp2(s - m) -> bf16, K-major SW128: row r, 16-byte chunk cc of
      // tile t at t*TILE + r*128 + ((cc ^ (r & 7)) * 16)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p[e] = exp2f(__uint_as_float(v[c][i + e]) - m_run);
            l_run += p[e];
          }
          const int key = c * 32 + i;  // 8 keys = one 16-byte chunk
          const int t = key >> 6, cc = (key & 63) >> 3;
          uint4 pk;
          pk.x = ptx::pack_bf16x2(p[0], p[1]);
          pk.y = ptx::pack_bf16x2(p[2], p[3]);
          pk.z = ptx::pack_bf16x2(p[4], p[5]);
          pk.w = ptx::pack_bf16x2(p[6], p[7]);
          *reinterpret_cast<uint4*>(sP + t * TILE + r * 128 + ((cc ^ (r & 7)) << 4)) = pk;
        }
      }
      ptx::fence_proxy_async_smem();  // generic-proxy P writes -> tensor-core reads
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(p_full);
    }
    ptx::mbar_wait(pv_done, (nkv - 1) & 1);
    ptx::tc_fence_after();
    const float inv = 1.f / l_run;
    __nv_bfloat16* orow = out + static_cast<long long>(row0 + q) * d.Q + h * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t o[32];
      ptx::tmem_ld_32x32b_x32(tO + lane_off + c * 32, o);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        ptx::st_global_v4(orow + c * 32 + i,
                          ptx::pack_bf16x2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv));
    }
    const long long T = static_cast<long long>(d.B) * d.S;
    lse[h * T + row0 + q] = (m_run + log2f(l_run)) * kLn2;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

}  // namespace

template <int HD>
void forward_tc_t(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d,
                  const CUtensorMap& tm, cudaStream_t s) {
  constexpr int smem = FwdSmem<HD>::BYTES;
  static_assert(smem <= 232448, "attention smem budget");
  static bool init = false;
  if (!init) {
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    init = true;
  }
  dim3 grid(d.S / BQ, d.nh, d.B);
  count_launches();
  attn_fwd_tc_kernel<HD><<<grid, 192, smem, s>>>(tm, o, lse, d);
}

void forward_tc(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, int hd,
                const CUtensorMap& tm, cudaStream_t s) {
  if (hd == 128)
    forward_tc_t<128>(qkv, o, lse, d, tm, s);
  else
    forward_tc_t<64>(qkv, o, lse, d, tm, s);
}

void prepare_tc(int hd) {
  if (hd == 128)
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<128>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      FwdSmem<128>::BYTES));
  else
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<64>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      FwdSmem<64>::BYTES));
}

}  // namespace attn
}  // namespace specsim
