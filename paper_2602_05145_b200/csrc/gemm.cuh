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
// CTA = 10 warps: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (one
// elected lane), warps 2..9 epilogue (two per TMEM lane quadrant, each owning
// a 128-column half).  Default CG = 2: a CTA pair on one TPC computes a
// 256 x 256 x 64 tile with tcgen05.mma.cta_group::2 from a 5-stage smem ring
// (32 KB / stage / CTA); CG = 1 computes 128 x 256 from a 3-stage ring.  Two
// TMEM accumulators (2 x 256 fp32 columns) so the epilogue of tile i overlaps
// the MMAs of i+1.  Persistent grid = min(#tiles, #SMs / CG) units, static
// round-robin schedule with L2-aware rasterisation (make_plan).
//
// Epilogues (template EPI) fuse the elementwise consumer of every GEMM in the
// step: bf16 / fp32 stores, fp32 accumulate, residual add, q / k RoPE, the
// SwiGLU backward, AdamW on weight gradients, and the vocabulary-chunked
// cross-entropy: online softmax statistics in the forward (the logits are
// additionally stored as fp16 offsets for the backward -- DESIGN.md §3 K6
// explains why this beats the logit-free recompute, EPI_CE_BWD, which stays
// selectable) and the softmax-minus-onehot gradient in the recompute path.
// Operand rows can be gathered by 64-row blocks (Args::a_rows / b_rows): the
// fc GEMMs read the micro-batch straight from the signal ring.
#pragma once

#include "gemm.h"
#include "ptx.cuh"

#ifndef SPECSIM_ADAMW_VARIANT
// 0: production fused-AdamW epilogue (256-bit accesses); 1..4: the 128-bit
// epilogue's probe variants, 5: the 128-bit epilogue (scripts/adamw_probe.sh)
#define SPECSIM_ADAMW_VARIANT 0
#endif
#ifndef SPECSIM_ADAMW_PREFETCH
// fused-AdamW epilogue: L2 prefetch of the optimizer state (p, m, v) of the
// thread's row.  0 none; 1 the whole half-tile row before waiting for the
// accumulator; 2 the first 32-column chunk before the wait, then chunk c+1
// while chunk c is processed
#define SPECSIM_ADAMW_PREFETCH 0
#endif
#ifndef SPECSIM_ADAMW_LDNA
// 1: optimizer-state loads of the 256-bit epilogue bypass L1 allocation
// (ld.global.L1::no_allocate) instead of the evict-first streaming hint;
// 2: the same plus an L2 evict-first cache-hint policy
#define SPECSIM_ADAMW_LDNA 1
#endif
#ifndef SPECSIM_ADAMW_WINDOW
// probe only (scripts/adamw_probe.sh): > 0 folds every optimizer-state access
// of the 256-bit epilogue into a window of this many elements (a power of 2),
// i.e. the same SM <-> L2 traffic with the state L2-resident instead of in HBM
#define SPECSIM_ADAMW_WINDOW 0
#endif

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
  static constexpr int STAGES = CG == 1 ? 3 : 5;
  static constexpr int EPI_STAGE = 8 * 32 * 36 * 4;     // per-warp 32x32 fp32 (+pad) staging
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256 + EPI_STAGE;
  static constexpr int TILE_M = BM * CG;                 // rows per (pair) tile
};
constexpr int NUM_EPI_WARPS = 8;  // two per TMEM lane quadrant, each half the columns
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;
constexpr int TMEM_COLS = 512;

__device__ __forceinline__ void tile_coords(int tile, const Args& a, int& mb, int& nb) {
  // Grouped rasterisation (group sizes chosen on the host, make_plan): the
  // smaller operand is walked in groups of panels that stay L2-resident
  // (loaded evict_last) while the other operand streams through DRAM once
  // per group.  keep_b: groups of group_n column blocks, row blocks inside;
  // else groups of group_m row blocks, column blocks inside (keep_b == 2:
  // the same walk for long-K GEMMs whose panels do not fit L2 -- group_m is
  // chosen so each wave of concurrent tiles is a compact block whose CTAs
  // share A / B k-slices in L2 while they advance through K together).
  if (a.keep_b == 1) {
    const int group_size = a.group_n * a.num_m_blocks;
    const int group = tile / group_size;
    const int first_n = group * a.group_n;
    const int gn = min(a.num_n_blocks - first_n, a.group_n);
    const int in_group = tile - group * group_size;
    nb = first_n + in_group % gn;
    mb = in_group / gn;
  } else {
    const int group_size = a.group_m * a.num_n_blocks;
    const int group = tile / group_size;
    const int first_m = group * a.group_m;
    const int gm = min(a.num_m_blocks - first_m, a.group_m);
    const int in_group = tile - group * group_size;
    mb = first_m + in_group % gm;
    nb = in_group / gm;
  }
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
  // 1024-byte alignment by offsetting the __shared__ array itself (not via an
  // integer round-trip), so the compiler keeps the shared address space and
  // the epilogue's staging accesses compile to LDS / STS, not generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

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
      ptx::mbar_init(&tempty_bar[s], NUM_EPI_WARPS * CG);  // every epilogue warp of the group
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
      // the operand the rasterisation reuses (see make_plan) is loaded
      // evict_last so streaming outputs / optimizer state do not flush it
      const uint64_t pol_a =
          args.keep_b == 0 ? ptx::policy_evict_last() : ptx::policy_evict_normal();
      const uint64_t pol_b =
          args.keep_b == 1 ? ptx::policy_evict_last() : ptx::policy_evict_normal();
      // operand row r of a gathered operand lives at rows[r / 64] + r % 64
      auto remap = [](const int32_t* rows, int r) {
        return rows ? __ldg(rows + (r >> 6)) + (r & 63) : r;
      };
      auto load = [&](const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1,
                      uint64_t pol) {
        if constexpr (CG == 2)
          ptx::tma_load_2d_pair(m, bar, dst, c0, c1, pol);
        else
          ptx::tma_load_2d_hint(m, bar, dst, c0, c1, pol);
      };
      for (int tile = unit; tile < args.num_tiles; tile += num_units) {
        int mb, nb;
        tile_coords(tile, args, mb, nb);
        const int m0 = mb * C_::TILE_M + static_cast<int>(rank) * BM;    // this CTA's A rows
        const int n0 = nb * BN + static_cast<int>(rank) * C_::BN_CTA;     // this CTA's B rows
        // gathered K-major rows: one remap per tile (a 128-row box is two
        // consecutive 64-row blocks of one sample)
        const int a_row0 = A_MN ? m0 : remap(args.a_rows, m0);
        const int b_row0 = B_MN ? n0 : remap(args.b_rows, n0);
        for (int kb = 0; kb < num_kb; ++kb) {
          // MN-major operands are gathered along K: one remap per k-block,
          // read before the slot wait so the load latency overlaps it
          const int k0 = kb * BK;
          const int a_k0 = A_MN ? remap(args.a_rows, k0) : k0;
          const int b_k0 = B_MN ? remap(args.b_rows, k0) : k0;
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          // the leader's barrier counts both CTAs' bytes; the peer only issues TMA
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES * CG);
          uint8_t* a_dst = smA + stage * A_STAGE_BYTES;
          uint8_t* b_dst = smB + stage * B_STAGE_BYTES;
          if constexpr (!A_MN) {
            load(&tmA, &full_bar[stage], a_dst, k0, a_row0, pol_a);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              load(&tmA, &full_bar[stage], a_dst + j * 8192, m0 + 64 * j, a_k0, pol_a);
          }
          if constexpr (!B_MN) {
            load(&tmB, &full_bar[stage], b_dst, k0, b_row0, pol_b);
          } else {
#pragma unroll
            for (int j = 0; j < C_::BN_CTA / 64; ++j)
              load(&tmB, &full_bar[stage], b_dst + j * 8192, n0 + 64 * j, b_k0, pol_b);
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
    // TMEM gives one accumulator row per thread (32x32b loads).  Row-wise
    // reductions (CE forward) consume it directly; every other epilogue stages
    // each 32x32 chunk through shared memory (row stride 36 floats: conflict-
    // free float4 writes and reads) and then walks it row-contiguously, 4 rows
    // x 8 lanes x float4 per warp instruction, so global loads / stores are
    // coalesced 128-byte row segments.
    const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad+32) (hardware rule: warp % 4)
    const int half = (warp - 2) >> 2;  // which 128 columns of the 256-wide tile
    float* stg = epi_stage + (warp - 2) * (32 * 36);
    const int c_begin = half * (BN / 2), c_end = c_begin + BN / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = unit; tile < args.num_tiles; tile += num_units) {
      int mb, nb;
      tile_coords(tile, args, mb, nb);
      const int m0 = mb * C_::TILE_M + static_cast<int>(rank) * BM, n0 = nb * BN;
      if constexpr (EPI == EPI_ADAMW && SPECSIM_ADAMW_PREFETCH > 0) {
        // the state of this thread's row streams into L2 while the tile's
        // mainloop runs (the epilogue would otherwise wait on DRAM latency)
        const int prow = m0 + quad * 32 + lane;
        const int pc = n0 + c_begin;
        if (prow < args.M && pc < args.N) {
          const int ncol = SPECSIM_ADAMW_PREFETCH == 1 ? min(BN / 2, args.N - pc)
                                                       : min(32, args.N - pc);
          const long long e = static_cast<long long>(prow) * args.ldc + pc;
          ptx::prefetch_l2_bulk(args.opt_p + e, 4u * ncol);
          ptx::prefetch_l2_bulk(args.opt_m + e, 4u * ncol);
          ptx::prefetch_l2_bulk(args.opt_v + e, 4u * ncol);
        }
      }
      // SwiGLU backward: the gate / up values of the first 32-column chunk are
      // loaded before the accumulator wait (their DRAM latency hides behind
      // the tile's mainloop); later chunks are loaded one chunk ahead
      uint2 sw_g[8], sw_u[8];
      auto sw_load = [&](int c, uint2 (&g)[8], uint2 (&u)[8]) {
        const int col = n0 + c + (lane & 7) * 4;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = m0 + quad * 32 + it * 4 + (lane >> 3);
          if (rr < args.M && col < args.N) {
            const __nv_bfloat16* gp = args.R + static_cast<long long>(rr) * args.ldr + col;
            g[it] = *reinterpret_cast<const uint2*>(gp);
            u[it] = *reinterpret_cast<const uint2*>(gp + args.N);
          }
        }
      };
      if constexpr (EPI == EPI_SWIGLU_BWD) sw_load(c_begin, sw_g, sw_u);
      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const int row_base = m0 + quad * 32;
      const int row = row_base + lane;  // the row this thread owns in TMEM
      const bool row_ok = row < args.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;

      if constexpr (EPI == EPI_CE_FWD) {
        float run_max = -INFINITY, run_sum = 0.f, tgt_logit = -INFINITY;
        int run_arg = 0;
        const int tgt = row_ok ? args.targets[row] - args.vocab_offset : -1;
        // pass 1: per-row online softmax statistics of this 128-column half tile
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 32) {
          uint32_t r[32];
          __syncwarp();
          ptx::tmem_ld_32x32b_x32(t_row + c, r);
          ptx::tmem_ld_wait();
          const int col0 = n0 + c;
          if (!row_ok || col0 >= args.N) continue;
          const int ncol = min(32, args.N - col0);
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
        // pass 2: logits kept for the backward (no recompute) as fp16 offsets
        // from this half tile's row max (the max the partial below records):
        // l - max <= 0 keeps fp32-grade resolution where softmax weights are
        // not negligible (|error| <= 2^-11 |l - max|) at half the bytes.
        // Staged through smem so each store writes full 64-byte row segments.
        if (args.C != nullptr) {
          const float ref = row_ok ? run_max : 0.f;
          uint32_t* stw = reinterpret_cast<uint32_t*>(stg);
#pragma unroll 1
          for (int c = c_begin; c < c_end; c += 32) {
            const int col0 = n0 + c;
            if (col0 >= args.N) break;  // warp-uniform
            uint32_t r[32];
            __syncwarp();
            ptx::tmem_ld_32x32b_x32(t_row + c, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 8)
              *reinterpret_cast<uint4*>(stw + lane * 36 + i / 2) =
                  make_uint4(ptx::pack_f16x2(__uint_as_float(r[i]) - ref,
                                             __uint_as_float(r[i + 1]) - ref),
                             ptx::pack_f16x2(__uint_as_float(r[i + 2]) - ref,
                                             __uint_as_float(r[i + 3]) - ref),
                             ptx::pack_f16x2(__uint_as_float(r[i + 4]) - ref,
                                             __uint_as_float(r[i + 5]) - ref),
                             ptx::pack_f16x2(__uint_as_float(r[i + 6]) - ref,
                                             __uint_as_float(r[i + 7]) - ref));
            __syncwarp();
            const int cw = (lane & 3) * 4;  // 4 lanes x 16 B per 64-byte row segment
            const int col = col0 + cw * 2;
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int rl = it * 8 + (lane >> 2);
              const int rw = row_base + rl;
              if (rw < args.M && col < args.N)
                __stcs(reinterpret_cast<uint4*>(static_cast<__half*>(args.C) +
                                                static_cast<long long>(rw) * args.ldc + col),
                       *reinterpret_cast<const uint4*>(stw + rl * 36 + cw));
            }
          }
        }
        if (row_ok) {
          CePartial p;
          p.max = run_max;
          p.sum = run_sum;
          p.target = tgt_logit;
          p.argmax = run_arg + args.vocab_offset;
          // one partial per (128-column half tile, row)
          args.partials[static_cast<long long>(2 * nb + half) * args.M + row] = p;
        }
      } else if constexpr (EPI == EPI_BF16_ROPE) {
        // qkv projection + RoPE: a 128-column half tile holds whole heads
        // (head_dim 64 or 128), so each rotation pair (i, i + hd/2) lives in
        // this thread's registers.  Values are rounded to bf16 before rotating
        // (the unfused path rotates the stored bf16 projection).
        uint32_t rr[4][32];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) ptx::tmem_ld_32x32b_x32(t_row + c_begin + 32 * q, rr[q]);
        ptx::tmem_ld_wait();
        const int colh = n0 + c_begin;  // first column of this half tile
        if (row_ok && colh < args.N) {
          const int pos = row % args.rope_S + args.rope_pos_off;
          auto rot = [&](float& a, float& b, float cs, float sn) {
            const float x1 = __bfloat162float(__float2bfloat16_rn(a));
            const float x2 = __bfloat162float(__float2bfloat16_rn(b));
            a = x1 * cs - x2 * sn;
            b = x2 * cs + x1 * sn;
          };
          const long long S = args.rope_ld;
          // tables [hd/2, rope_ld]: lanes hold consecutive rows, so each load is coalesced
          if (args.rope_hd == 128) {
            if (colh < args.rope_cols) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const long long ti = (q * 32 + i) * S + pos;
                  float a = __uint_as_float(rr[q][i]), b = __uint_as_float(rr[q + 2][i]);
                  rot(a, b, __ldg(args.rope_cos + ti), __ldg(args.rope_sin + ti));
                  rr[q][i] = __float_as_uint(a);
                  rr[q + 2][i] = __float_as_uint(b);
                }
            }
          } else {  // head_dim 64: two heads per half tile
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              if (colh + 64 * hh < args.rope_cols) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const long long ti = i * S + pos;
                  float a = __uint_as_float(rr[2 * hh][i]), b = __uint_as_float(rr[2 * hh + 1][i]);
                  rot(a, b, __ldg(args.rope_cos + ti), __ldg(args.rope_sin + ti));
                  rr[2 * hh][i] = __float_as_uint(a);
                  rr[2 * hh + 1][i] = __float_as_uint(b);
                }
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col0 = colh + 32 * q;
          if (col0 >= args.N) break;  // warp-uniform
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(stg + lane * 36 + i) =
                make_float4(__uint_as_float(rr[q][i]), __uint_as_float(rr[q][i + 1]),
                            __uint_as_float(rr[q][i + 2]), __uint_as_float(rr[q][i + 3]));
          __syncwarp();
          const int cl = (lane & 7) * 4;
          const int col = col0 + cl;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rl = it * 4 + (lane >> 3);
            const int rw = row_base + rl;
            const float4 w = *reinterpret_cast<const float4*>(stg + rl * 36 + cl);
            if (rw < args.M && col < args.N)
              *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.C) +
                                        static_cast<long long>(rw) * args.ldc + col) =
                  make_uint2(ptx::pack_bf16x2(w.x, w.y), ptx::pack_bf16x2(w.z, w.w));
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU_BWD) {
        // d act rounded to bf16 (the operand the unfused path stores), then
        // silu' with the stored bf16 gate / up, as swiglu_bwd_kernel; the
        // 32x32 chunk is staged through smem (4 columns x 8 rows per lane)
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 32) {
          uint32_t r[32];
          __syncwarp();
          ptx::tmem_ld_32x32b_x32(t_row + c, r);
          ptx::tmem_ld_wait();
          const int col0 = n0 + c;
          if (col0 >= args.N) continue;  // warp-uniform
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(stg + lane * 36 + i) =
                make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                            __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          __syncwarp();
          uint2 nx_g[8], nx_u[8];
          if (c + 32 < c_end) sw_load(c + 32, nx_g, nx_u);
          const int cl = (lane & 7) * 4;
          const int col = col0 + cl;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rl = it * 4 + (lane >> 3);
            const int rr = row_base + rl;
            if (rr >= args.M || col >= args.N) continue;
            const float4 w = *reinterpret_cast<const float4*>(stg + rl * 36 + cl);
            const float wa[4] = {w.x, w.y, w.z, w.w};
            const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sw_g[it].x));
            const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sw_g[it].y));
            const float2 u01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sw_u[it].x));
            const float2 u23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sw_u[it].y));
            const float gv[4] = {g01.x, g01.y, g23.x, g23.y};
            const float uv[4] = {u01.x, u01.y, u23.x, u23.y};
            float dg[4], du[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float dv = __bfloat162float(__float2bfloat16_rn(wa[j]));
              const float sg = 1.f / (1.f + __expf(-gv[j]));
              dg[j] = dv * uv[j] * sg * (1.f + gv[j] * (1.f - sg));
              du[j] = dv * gv[j] * sg;
            }
            __nv_bfloat16* cp = static_cast<__nv_bfloat16*>(args.C) +
                                static_cast<long long>(rr) * args.ldc + col;
            *reinterpret_cast<uint2*>(cp) =
                make_uint2(ptx::pack_bf16x2(dg[0], dg[1]), ptx::pack_bf16x2(dg[2], dg[3]));
            *reinterpret_cast<uint2*>(cp + args.N) =
                make_uint2(ptx::pack_bf16x2(du[0], du[1]), ptx::pack_bf16x2(du[2], du[3]));
          }
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            sw_g[it] = nx_g[it];
            sw_u[it] = nx_u[it];
          }
        }
      } else if constexpr (EPI == EPI_ADAMW && SPECSIM_ADAMW_VARIANT == 0) {
        // Fused AdamW on the gradient tile.  The 32x32 chunk is staged through
        // smem and walked 4 lanes x 8 columns per row (8 rows per warp
        // instruction) so every optimizer-state access is one 256-bit
        // LDG / STG (p, m, v, optional g) and the bf16 copy one 128-bit STG:
        // half the LSU instructions of 128-bit accesses.  Two row groups are
        // loaded before any store (their DRAM latencies overlap).
        const AdamDev hp = *args.opt_hp;
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 32) {
          if constexpr (SPECSIM_ADAMW_PREFETCH == 2) {
            const int pc = n0 + c + 32;
            if (row_ok && c + 32 < c_end && pc < args.N) {
              const long long e = static_cast<long long>(row) * args.ldc + pc;
              const uint32_t nb4 = 4u * min(32, args.N - pc);
              ptx::prefetch_l2_bulk(args.opt_p + e, nb4);
              ptx::prefetch_l2_bulk(args.opt_m + e, nb4);
              ptx::prefetch_l2_bulk(args.opt_v + e, nb4);
            }
          }
          uint32_t r[32];
          __syncwarp();
          ptx::tmem_ld_32x32b_x32(t_row + c, r);
          ptx::tmem_ld_wait();
          const int col0 = n0 + c;
          if (col0 >= args.N) continue;  // warp-uniform
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(stg + lane * 36 + i) =
                make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                            __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          __syncwarp();
          const int cl = (lane & 3) * 8;  // this lane's 8 columns
          const int col = col0 + cl;
          const bool col_ok = col < args.N;  // N % 8 == 0 (make_plan)
#pragma unroll
          for (int g0 = 0; g0 < 4; g0 += 2) {
            float gv[2][8], pv[2][8], mv[2][8], vv[2][8];
            bool ok[2];
            long long e[2];
#pragma unroll
            for (int it = 0; it < 2; ++it) {
              const int rl = (g0 + it) * 8 + (lane >> 2);
              const int rw = row_base + rl;
              ok[it] = col_ok && rw < args.M;
              e[it] = static_cast<long long>(rw) * args.ldc + col;
              if constexpr (SPECSIM_ADAMW_WINDOW > 0) e[it] &= SPECSIM_ADAMW_WINDOW - 1;
              const float4 a = *reinterpret_cast<const float4*>(stg + rl * 36 + cl);
              const float4 b = *reinterpret_cast<const float4*>(stg + rl * 36 + cl + 4);
              gv[it][0] = a.x; gv[it][1] = a.y; gv[it][2] = a.z; gv[it][3] = a.w;
              gv[it][4] = b.x; gv[it][5] = b.y; gv[it][6] = b.z; gv[it][7] = b.w;
              if (ok[it]) {
                if constexpr (SPECSIM_ADAMW_LDNA == 2) {
                  const uint64_t pol = ptx::policy_evict_first();
                  ptx::ld_na_hint_v8(args.opt_p + e[it], pv[it], pol);
                  ptx::ld_na_hint_v8(args.opt_m + e[it], mv[it], pol);
                  ptx::ld_na_hint_v8(args.opt_v + e[it], vv[it], pol);
                } else if constexpr (SPECSIM_ADAMW_LDNA == 1) {
                  ptx::ld_na_v8(args.opt_p + e[it], pv[it]);
                  ptx::ld_na_v8(args.opt_m + e[it], mv[it]);
                  ptx::ld_na_v8(args.opt_v + e[it], vv[it]);
                } else {
                  ptx::ld_cs_v8(args.opt_p + e[it], pv[it]);
                  ptx::ld_cs_v8(args.opt_m + e[it], mv[it]);
                  ptx::ld_cs_v8(args.opt_v + e[it], vv[it]);
                }
              }
            }
#pragma unroll
            for (int it = 0; it < 2; ++it) {
              if (!ok[it]) continue;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float g = gv[it][j];
                const float pi = pv[it][j] * hp.decay;
                mv[it][j] = mv[it][j] + (g - mv[it][j]) * (1.f - hp.beta1);
                vv[it][j] = vv[it][j] * hp.beta2 + (1.f - hp.beta2) * g * g;
                const float denom = sqrtf(vv[it][j]) / hp.bc2_sqrt + hp.eps;
                pv[it][j] = pi - hp.step_size * (mv[it][j] / denom);
              }
              ptx::st_cs_v8(args.opt_p + e[it], pv[it]);
              ptx::st_cs_v8(args.opt_m + e[it], mv[it]);
              ptx::st_cs_v8(args.opt_v + e[it], vv[it]);
              __stcs(reinterpret_cast<uint4*>(args.opt_p16 + e[it]),
                     make_uint4(ptx::pack_bf16x2(pv[it][0], pv[it][1]),
                                ptx::pack_bf16x2(pv[it][2], pv[it][3]),
                                ptx::pack_bf16x2(pv[it][4], pv[it][5]),
                                ptx::pack_bf16x2(pv[it][6], pv[it][7])));
              if (args.opt_g) ptx::st_cs_v8(args.opt_g + e[it], gv[it]);
            }
          }
        }
      } else {
        // per-row constants, owned by lane (row - row_base); shuffled below
        float lse_r = 0.f, coef_r = 0.f;
        int tgt_r = -1;
        if constexpr (EPI == EPI_CE_BWD) {
          if (row_ok) {
            lse_r = args.lse[row];
            coef_r = args.coef[row];
            tgt_r = args.targets[row] - args.vocab_offset;
          }
        }
        AdamDev hp{};
        if constexpr (EPI == EPI_ADAMW) hp = *args.opt_hp;
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 32) {
          uint32_t r[32];
          __syncwarp();
          ptx::tmem_ld_32x32b_x32(t_row + c, r);
          ptx::tmem_ld_wait();
          const int col0 = n0 + c;
          if (col0 >= args.N) continue;  // warp-uniform
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(stg + lane * 36 + i) =
                make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                            __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          __syncwarp();
          const int cl = (lane & 7) * 4;  // this lane's 4 columns
          const int col = col0 + cl;
          const bool col_ok = col < args.N;  // N % 4 == 0: all 4 valid
          // phase 1: every global load of the chunk is issued before any store
          // (loads and stores may alias as far as the compiler knows), so the
          // 8 row groups' DRAM latencies overlap
          // AdamW keeps three state vectors per row group in flight: hoist 4
          // row groups at a time so everything stays in registers
          constexpr int RG = EPI == EPI_ADAMW ? (SPECSIM_ADAMW_VARIANT == 4 ? 8 : 4) : 8;
#pragma unroll
          for (int g0 = 0; g0 < 8; g0 += RG) {
          float4 v[RG], x1[RG], x2[RG], x3[RG];
          uint32_t okm = 0;  // bit it: row group g0 + it in range
          // element offset of row group it (recomputed: fewer live registers)
          const long long e0 =
              static_cast<long long>(row_base + 4 * g0 + (lane >> 3)) * args.ldc + col;
          const long long estep = 4 * args.ldc;
#define SPECSIM_E(it) (e0 + (it) * estep)
#pragma unroll
          for (int it = 0; it < RG; ++it) {
            const int rl = (g0 + it) * 4 + (lane >> 3);
            const int rr = row_base + rl;
            if (col_ok && rr < args.M) okm |= 1u << it;
            const long long e_it = SPECSIM_E(it);
            v[it] = *reinterpret_cast<const float4*>(stg + rl * 36 + cl);
            if constexpr (EPI == EPI_BF16_RESID) {
              if (okm >> it & 1) {
                const uint2 q = *reinterpret_cast<const uint2*>(
                    args.R + static_cast<long long>(rr) * args.ldr + col);
                x1[it].x = __uint_as_float(q.x);
                x1[it].y = __uint_as_float(q.y);
              }
            } else if constexpr (EPI == EPI_F32_ACC) {
              if (okm >> it & 1)
                x1[it] = *reinterpret_cast<const float4*>(static_cast<const float*>(args.C) + e_it);
            } else if constexpr (EPI == EPI_ADAMW) {
              if (okm >> it & 1) {  // optimizer state streams once: evict-first
                if constexpr (SPECSIM_ADAMW_VARIANT == 1) {
                  x1[it] = make_float4(0.01f, 0.01f, 0.01f, 0.01f);
                  x2[it] = x3[it] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else if constexpr (SPECSIM_ADAMW_VARIANT == 3) {
                  x1[it] = *reinterpret_cast<const float4*>(args.opt_p + e_it);
                  x2[it] = *reinterpret_cast<const float4*>(args.opt_m + e_it);
                  x3[it] = *reinterpret_cast<const float4*>(args.opt_v + e_it);
                } else {
                  x1[it] = __ldcs(reinterpret_cast<const float4*>(args.opt_p + e_it));
                  x2[it] = __ldcs(reinterpret_cast<const float4*>(args.opt_m + e_it));
                  x3[it] = __ldcs(reinterpret_cast<const float4*>(args.opt_v + e_it));
                }
              }
            } else if constexpr (EPI == EPI_CE_BWD) {
              // row constants: x1 = {lse, coef, target (bits)}
              x1[it].x = __shfl_sync(0xffffffffu, lse_r, rl);
              x1[it].y = __shfl_sync(0xffffffffu, coef_r, rl);
              x1[it].z = __int_as_float(__shfl_sync(0xffffffffu, tgt_r, rl));
            }
          }
          // phase 2: compute and store
#pragma unroll
          for (int it = 0; it < RG; ++it) {
            if (!(okm >> it & 1)) continue;
            const long long e_it = SPECSIM_E(it);
            float4 w = v[it];
            float* wa = &w.x;
            if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_RESID || EPI == EPI_CE_BWD) {
              if constexpr (EPI == EPI_BF16_RESID) {
                uint32_t q0 = __float_as_uint(x1[it].x), q1 = __float_as_uint(x1[it].y);
                const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q0));
                const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q1));
                w.x += a.x;
                w.y += a.y;
                w.z += b.x;
                w.w += b.y;
              }
              if constexpr (EPI == EPI_CE_BWD) {
                const float lse_x = x1[it].x, coef_x = x1[it].y;
                const int tgt_x = __float_as_int(x1[it].z);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float p = exp2f((wa[j] - lse_x) * 1.4426950408889634f);
                  wa[j] = (p - ((c + cl + j) == tgt_x - n0 ? 1.f : 0.f)) * coef_x;
                }
              }
              *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.C) + e_it) =
                  make_uint2(ptx::pack_bf16x2(w.x, w.y), ptx::pack_bf16x2(w.z, w.w));
            } else if constexpr (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
              if constexpr (EPI == EPI_F32_ACC) {
                w.x += x1[it].x;
                w.y += x1[it].y;
                w.z += x1[it].z;
                w.w += x1[it].w;
              }
              *reinterpret_cast<float4*>(static_cast<float*>(args.C) + e_it) = w;
            } else if constexpr (EPI == EPI_ADAMW) {
              float4 p = x1[it], m = x2[it], s2 = x3[it];
              float* pa = &p.x;
              float* ma = &m.x;
              float* sa = &s2.x;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float g = wa[j];
                const float pi = pa[j] * hp.decay;
                ma[j] = ma[j] + (g - ma[j]) * (1.f - hp.beta1);
                sa[j] = sa[j] * hp.beta2 + (1.f - hp.beta2) * g * g;
                const float denom = sqrtf(sa[j]) / hp.bc2_sqrt + hp.eps;
                pa[j] = pi - hp.step_size * (ma[j] / denom);
              }
              if constexpr (SPECSIM_ADAMW_VARIANT == 2) {
                // probe: only the bf16 working copy is stored
                __stcs(reinterpret_cast<uint2*>(args.opt_p16 + e_it),
                       make_uint2(ptx::pack_bf16x2(p.x + m.x + s2.x, p.y + m.y + s2.y),
                                  ptx::pack_bf16x2(p.z + m.z + s2.z, p.w + m.w + s2.w)));
              } else if constexpr (SPECSIM_ADAMW_VARIANT == 3) {
                *reinterpret_cast<float4*>(args.opt_p + e_it) = p;
                *reinterpret_cast<float4*>(args.opt_m + e_it) = m;
                *reinterpret_cast<float4*>(args.opt_v + e_it) = s2;
                *reinterpret_cast<uint2*>(args.opt_p16 + e_it) =
                    make_uint2(ptx::pack_bf16x2(p.x, p.y), ptx::pack_bf16x2(p.z, p.w));
              } else {
                __stcs(reinterpret_cast<float4*>(args.opt_p + e_it), p);
                __stcs(reinterpret_cast<float4*>(args.opt_m + e_it), m);
                __stcs(reinterpret_cast<float4*>(args.opt_v + e_it), s2);
                __stcs(reinterpret_cast<uint2*>(args.opt_p16 + e_it),
                       make_uint2(ptx::pack_bf16x2(p.x, p.y), ptx::pack_bf16x2(p.z, p.w)));
              }
              if (args.opt_g) __stcs(reinterpret_cast<float4*>(args.opt_g + e_it), w);
            }
          }
          }  // g0
#undef SPECSIM_E
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
