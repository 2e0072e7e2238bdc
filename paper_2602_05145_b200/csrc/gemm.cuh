// tcgen05 / TMEM / TMA warp-specialised persistent GEMM for sm_100a.
//
//   D[M,N] = sum_k A[m,k] * B[n,k]       (bf16 x bf16 -> fp32 in TMEM)
//
// Operands may each be K-major (K contiguous) or MN-major (M / N contiguous),
// which covers the three contractions of the draft-head step without any
// transposes in HBM:
//   forward   Y  = X  . W^T    A = X  K-major,  B = W  K-major
//   data grad dX = dY . W      A = dY K-major,  B = W  MN-major
//   weight gr dW = dY^T . X    A = dY MN-major, B = X  MN-major
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (one
// elected lane), warps 2..5 epilogue (one TMEM lane quadrant each).  Tile
// 128 x 256 x 64, 4-stage smem ring (48 KB / stage), two TMEM accumulators
// (2 x 256 fp32 columns) so the epilogue of tile i overlaps the MMAs of i+1.
// Grid = min(#tiles, #SMs), static round-robin persistent schedule with
// grouped rasterisation for L2 reuse.
//
// Epilogues (template EPI) fuse the elementwise consumer of every GEMM in the
// step: bf16 / fp32 stores, fp32 accumulate, residual add, and the two halves
// of the vocabulary-chunked cross-entropy (online softmax statistics in the
// forward; softmax-minus-onehot gradient in the backward), so full logits
// never reach HBM.
#pragma once

#include "gemm.h"
#include "ptx.cuh"

namespace specsim {
namespace gemm {

// Per-CTA-group configuration.  CG = 1: one CTA computes a 128 x 256 tile
// (tcgen05.mma.cta_group::1, M = 128).  CG = 2: a cluster of two CTAs on one
// TPC computes a 256 x 256 tile with tcgen05.mma.cta_group::2 (M = 256): each
// CTA stages 128 rows of A and 128 of the 256 B rows, so per-SM shared-memory
// and L2 operand traffic drop by a third.
template <int CG>
struct Cfg {
  static constexpr int BN_CTA = BN / CG;                 // B rows staged per CTA
  static constexpr int A_STAGE = BM * BK * 2;            // 16 KB
  static constexpr int B_STAGE = BN_CTA * BK * 2;        // 32 KB (CG1) / 16 KB (CG2)
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int STAGES = CG == 1 ? 4 : 6;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
  static constexpr int TILE_M = BM * CG;                 // rows per (pair) tile
};
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;

__device__ __forceinline__ void tile_coords(int tile, const Args& a, int& mb, int& nb) {
  // Grouped rasterisation: consecutive tiles walk group_m row blocks first so
  // the concurrently resident CTAs share B column panels in L2; group_m is
  // chosen on the host so the A panel of a group stays L2-resident and B
  // streams through DRAM about once.
  const int group_size = a.group_m * a.num_n_blocks;
  const int group = tile / group_size;
  const int first_m = group * a.group_m;
  const int gm = min(a.num_m_blocks - first_m, a.group_m);
  const int in_group = tile - group * group_size;
  mb = first_m + in_group % gm;
  nb = in_group / gm;
}

template <bool A_MN, bool B_MN, int EPI, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Args args) {
  using C_ = Cfg<CG>;
  constexpr int STAGES = C_::STAGES;
  constexpr int A_STAGE_BYTES = C_::A_STAGE;
  constexpr int B_STAGE_BYTES = C_::B_STAGE;
  constexpr int STAGE_BYTES = C_::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;  // CTA within the pair
  const int unit = CG == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int num_units = CG == 2 ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull_bar[s], 1);
      ptx::mbar_init(&tempty_bar[s], 4 * CG);  // every epilogue warp of the group
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS, CG>(tmem_slot);
  ptx::tc_fence_before();
  if constexpr (CG == 2)
    ptx::cluster_sync();  // peer barriers initialised before any remote arrive
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_kb = (args.K + BK - 1) / BK;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto load = [&](const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
        if constexpr (CG == 2)
          ptx::tma_load_2d_pair(m, bar, dst, c0, c1);
        else
          ptx::tma_load_2d(m, bar, dst, c0, c1);
      };
      for (int tile = unit; tile < args.num_tiles; tile += num_units) {
        int mb, nb;
        tile_coords(tile, args, mb, nb);
        const int m0 = mb * C_::TILE_M + static_cast<int>(rank) * BM;    // this CTA's A rows
        const int n0 = nb * BN + static_cast<int>(rank) * C_::BN_CTA;     // this CTA's B rows
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          // the leader's barrier counts both CTAs' bytes; the peer only issues TMA
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES * CG);
          uint8_t* a_dst = smA + stage * A_STAGE_BYTES;
          uint8_t* b_dst = smB + stage * B_STAGE_BYTES;
          const int k0 = kb * BK;
          if constexpr (!A_MN) {
            load(&tmA, &full_bar[stage], a_dst, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              load(&tmA, &full_bar[stage], a_dst + j * 8192, m0 + 64 * j, k0);
          }
          if constexpr (!B_MN) {
            load(&tmB, &full_bar[stage], b_dst, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < C_::BN_CTA / 64; ++j)
              load(&tmB, &full_bar[stage], b_dst + j * 8192, n0 + 64 * j, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = ptx::make_idesc_bf16(BM * CG, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = unit; tile < args.num_tiles; tile += num_units) {
        ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smA + stage * A_STAGE_BYTES);
          const uint32_t b_base = ptx::smem_u32(smB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major SW128: 8-row core groups 1024 B apart, +32 B per K=16 step
            // inside the swizzle atom.  MN-major SW128: 64-element MN chunks
            // 8 KB apart (LBO), 8-row K groups 1024 B apart (SBO), +2048 B per
            // K=16 step.
            const uint64_t adesc = A_MN ? ptx::make_sw128_desc(a_base + k * 2048, 8192, 1024)
                                        : ptx::make_sw128_desc(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? ptx::make_sw128_desc(b_base + k * 2048, 8192, 1024)
                                        : ptx::make_sw128_desc(b_base + k * 32, 16, 1024);
            if constexpr (CG == 2)
              ptx::umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
            else
              ptx::umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          if constexpr (CG == 2)
            ptx::umma_commit_pair(&empty_bar[stage], 0x3);  // free the slot in both CTAs
          else
            ptx::umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2)
          ptx::umma_commit_pair(&tfull_bar[acc], 0x3);
        else
          ptx::umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad+32)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = unit; tile < args.num_tiles; tile += num_units) {
      int mb, nb;
      tile_coords(tile, args, mb, nb);
      const int m0 = mb * C_::TILE_M + static_cast<int>(rank) * BM, n0 = nb * BN;
      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      const bool row_ok = row < args.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;

      // per-row state for the cross-entropy epilogues
      float run_max = -INFINITY, run_sum = 0.f, tgt_logit = -INFINITY;
      int run_arg = 0;
      int tgt = -1;
      float lse_r = 0.f, coef_r = 0.f;
      if constexpr (EPI == EPI_CE_FWD || EPI == EPI_CE_BWD) {
        if (row_ok) tgt = args.targets[row] - args.vocab_offset;
      }
      if constexpr (EPI == EPI_CE_BWD) {
        if (row_ok) {
          lse_r = args.lse[row];
          coef_r = args.coef[row];
        }
      }

#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after masked lanes
        ptx::tmem_ld_32x32b_x32(t_row + c, r);
        ptx::tmem_ld_wait();
        const int col0 = n0 + c;
        if (!row_ok || col0 >= args.N) continue;
        const bool full_chunk = col0 + 32 <= args.N;
        const int ncol = full_chunk ? 32 : args.N - col0;
        if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_RESID || EPI == EPI_CE_BWD) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if constexpr (EPI == EPI_BF16_RESID) {
            const __nv_bfloat16* rp = args.R + static_cast<long long>(row) * args.ldr + col0;
            if (full_chunk) {
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                uint4 q = *reinterpret_cast<const uint4*>(rp + i);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float2 f = __bfloat1622float2(h[j]);
                  v[i + 2 * j] += f.x;
                  v[i + 2 * j + 1] += f.y;
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < ncol) v[i] += __bfloat162float(rp[i]);
            }
          }
          if constexpr (EPI == EPI_CE_BWD) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float p = exp2f((v[i] - lse_r) * 1.4426950408889634f);
              v[i] = (p - ((c + i) == tgt - n0 ? 1.f : 0.f)) * coef_r;
            }
          }
          __nv_bfloat16* cp =
              static_cast<__nv_bfloat16*>(args.C) + static_cast<long long>(row) * args.ldc + col0;
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 8)
              ptx::st_global_v4(cp + i, ptx::pack_bf16x2(v[i], v[i + 1]),
                                ptx::pack_bf16x2(v[i + 2], v[i + 3]),
                                ptx::pack_bf16x2(v[i + 4], v[i + 5]),
                                ptx::pack_bf16x2(v[i + 6], v[i + 7]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < ncol) cp[i] = __float2bfloat16_rn(v[i]);
          }
        } else if constexpr (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
          float* cp = static_cast<float*>(args.C) + static_cast<long long>(row) * args.ldc + col0;
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 o = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                     __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
              if constexpr (EPI == EPI_F32_ACC) {
                const float4 prev = *reinterpret_cast<const float4*>(cp + i);
                o.x += prev.x;
                o.y += prev.y;
                o.z += prev.z;
                o.w += prev.w;
              }
              *reinterpret_cast<float4*>(cp + i) = o;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (i < ncol) {
                float o = __uint_as_float(r[i]);
                if constexpr (EPI == EPI_F32_ACC) o += cp[i];
                cp[i] = o;
              }
            }
          }
        } else if constexpr (EPI == EPI_CE_FWD) {
          float cmax = -INFINITY;
          int carg = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = i < ncol ? __uint_as_float(r[i]) : -INFINITY;
            if (x > cmax) {
              cmax = x;
              carg = i;
            }
          }
          const float new_max = fmaxf(run_max, cmax);
          const float nm2 = new_max * 1.4426950408889634f;
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < ncol) s += exp2f(fmaf(__uint_as_float(r[i]), 1.4426950408889634f, -nm2));
          run_sum = run_sum * exp2f((run_max - new_max) * 1.4426950408889634f) + s;
          if (cmax > run_max) run_arg = col0 + carg;
          run_max = new_max;
          const int t_local = tgt - col0;
          if (t_local >= 0 && t_local < ncol) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i == t_local) tgt_logit = __uint_as_float(r[i]);
          }
        }
      }
      if constexpr (EPI == EPI_CE_FWD) {
        if (row_ok) {
          CePartial p;
          p.max = run_max;
          p.sum = run_sum;
          p.target = tgt_logit;
          p.argmax = run_arg + args.vocab_offset;
          args.partials[static_cast<long long>(nb) * args.M + row] = p;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          ptx::mbar_arrive_cluster(&tempty_bar[acc], 0);  // the leader's MMA waits on it
        else
          ptx::mbar_arrive(&tempty_bar[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2)
    ptx::cluster_sync();  // no CTA frees TMEM / smem the peer's MMA may still touch
  else
    __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS, CG>(tmem_base);
  }
}

}  // namespace gemm
}  // namespace specsim
