// Host interface of the tcgen05 GEMM (kernel in gemm.cuh).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>

namespace specsim {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;

enum Epi : int {
  EPI_BF16 = 0,        // C(bf16) = acc
  EPI_F32 = 1,         // C(f32)  = acc
  EPI_F32_ACC = 2,     // C(f32) += acc
  EPI_BF16_RESID = 3,  // C(bf16) = acc + R(bf16)
  EPI_CE_FWD = 4,      // per-row partial (max, sum exp, target logit, argmax) per N tile;
                       // also C(f32) = acc when C is set (logits kept for the backward)
  EPI_CE_BWD = 5,      // C(bf16) = (exp(acc - lse[row]) - [col == y[row]]) * coef[row]
  EPI_ADAMW = 6,       // acc is a weight gradient: fused PyTorch-AdamW update of p/m/v (+ bf16 p)
  EPI_BF16_ROPE = 7,   // C(bf16) = acc with NeoX RoPE applied to columns < rope_cols (q | k heads)
  EPI_SWIGLU_BWD = 8,  // acc = d act (N = I columns): with gate | up = R[:, c] | R[:, I + c],
                       // C[:, c] = d gate, C[:, I + c] = d up (bf16; ldc = ldr = 2I)
};

// Device-resident AdamW hyper-parameters of the current step (updated per step
// by a tiny copy so GEMM plans stay fixed).
struct AdamDev {
  float lr, beta1, beta2, eps, decay /* 1 - lr*wd */, step_size /* lr / bc1 */, bc2_sqrt;
  float pad;
};

// Per-(row, N-tile) partial softmax statistics written by EPI_CE_FWD.
struct CePartial {
  float max;       // max logit over the tile's valid columns
  float sum;       // sum exp(logit - max)
  float target;    // logit of the target column if it lies in this tile, else -inf
  int32_t argmax;  // global vocabulary index of the (first) max
};

struct Args {
  int M, N, K;
  void* C;
  long long ldc;  // elements
  const __nv_bfloat16* R;
  long long ldr;
  // cross-entropy epilogues
  const int32_t* targets;  // [M] target vocabulary ids
  const float* lse;        // [M] log-sum-exp (bwd)
  const float* coef;       // [M] mask / global token count (bwd)
  CePartial* partials;     // [2 * num_n_blocks, M] (fwd): one per 128-column half tile
  int vocab_offset;        // vocabulary index of output column 0
  int num_m_blocks, num_n_blocks, num_tiles;
  int group_m;  // rasterisation group (row blocks), used when keep_b == 0
  int group_n;  // rasterisation group (column blocks), used when keep_b == 1
  int l2_budget_mb;  // host hint for make_plan: resident-panel budget (0: default)
  int keep_b;   // 1: B panels are the L2-resident operand, 0: A panels, 2: compact waves (long K)
  // fused AdamW epilogue: parameter tensors laid out like C (ldc)
  float *opt_p, *opt_m, *opt_v;
  __nv_bfloat16* opt_p16;
  float* opt_g;  // optional gradient store (nullable)
  const AdamDev* opt_hp;
  // RoPE epilogue: row r is position r % rope_S + rope_pos_off (training-time-test
  // unroll step); tables transposed [rope_hd / 2, rope_ld] (rope_ld 0 -> rope_S)
  const float* rope_cos;
  const float* rope_sin;
  int rope_S, rope_cols, rope_hd;
  int rope_pos_off, rope_ld;
  // Row gather by 64-row blocks (nullable): the operand's tensor-map row r
  // (M for a K-major operand, K for an MN-major one) is read from row
  // a_rows[r / 64] + r % 64 -- the fc GEMMs read the micro-batch's feature
  // rows straight from the signal ring (a sample's 64-row blocks are
  // contiguous ring rows; K-major boxes of 128 rows need two consecutive
  // blocks of one sample, i.e. S % 128 == 0).
  const int32_t* a_rows;
  const int32_t* b_rows;
};

// A matrix operand in HBM.  K-major: stored [MN, K] row-major (K contiguous).
// MN-major: stored [K, MN] row-major (MN contiguous).  ld in elements.
struct Operand {
  const void* ptr;
  long long ld;
  bool mn_major;
  long long rows = 0;  // tensor-map row extent when rows are gathered (Args::a_rows / b_rows)
};

struct GemmPlan {
  CUtensorMap map_a, map_b;
  Args args;
  int epi = 0;
  bool a_mn = false, b_mn = false;
  int cg = 2;  // CTAs per MMA tile (1 or 2)
  int grid = 0;
  double flops = 0;
  void launch(cudaStream_t s) const;
  void prepare() const;  // one-time kernel attributes (never inside a graph capture)
};

// 2-D bf16 TMA map (SWIZZLE_128B) over a row-major [rows, cols] matrix.
CUtensorMap make_tensor_map(const void* ptr, long long rows, long long cols, long long ld,
                            int box_cols, int box_rows);

// Throws std::invalid_argument on bad shapes / alignment.
GemmPlan make_plan(const Operand& A, const Operand& B, int M, int N, int K, int epi,
                   const Args& extra, int cg = 2);

}  // namespace gemm
}  // namespace specsim
