// Causal GQA attention (forward / backward) of the draft decoder layer.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace specsim {
namespace attn {

struct Dims {
  int B, S, nh, nkv;
  int NQ;  // row stride of qkv / dqkv (= Q + 2 KV)
  int Q, KV;
  float scale;  // 1 / sqrt(head_dim)
  // Optional NeoX RoPE tables, transposed [hd/2, S] (a warp's rows = consecutive
  // positions, so each table read is one coalesced line): when set, backward() writes dq / dk
  // already inverse-rotated (gradients w.r.t. the pre-RoPE projection).
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int rope_len = 0;  // rows (positions) of the transposed tables; 0 -> S
  // Training-time-test unroll (EAGLE-3 TTT): the rows of K unroll steps are
  // stacked [K][T] in one qkv buffer.  The step computed has its queries at
  // rows q_row_off + [0, T) and RoPE positions t % S + pos_off; the causal
  // keys / values are step 0's (rows [0, T)); n_diag = j > 0 adds, for query
  // row t, the keys / values of steps 1..j at row t (rows i*T + t of
  // diag_qkv), softmaxed together with the causal scores.
  long long q_row_off = 0;
  int pos_off = 0;
  int n_diag = 0;
  const __nv_bfloat16* diag_qkv = nullptr;
};

constexpr int kMaxDiag = 15;

void check_dims(const Dims& d, int hd);  // throws std::invalid_argument
void prepare(int hd);                    // one-time kernel attributes
void forward(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, int hd,
             cudaStream_t s);
// Dbuf: [nh, T] fp32 scratch.  Writes every element of dqkv.  Returns true
// when the inverse RoPE (d.rope_cos) was applied inside the kernels; the
// mma.sync fallback leaves it to the caller.
bool backward(const __nv_bfloat16* qkv, const __nv_bfloat16* o, const __nv_bfloat16* dout,
              const float* lse, float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, int hd,
              cudaStream_t s);

// ---- unroll-step pieces of the backward (tcgen05 path, S % 128 == 0) ----
// D[h * T + t] = rowsum(dO * O) of one step.
void bwd_dot(const __nv_bfloat16* dout, const __nv_bfloat16* o, float* D, const Dims& d, int hd,
             cudaStream_t s);
// Diagonal (cache) entries of unroll step j = d.n_diag >= 1: writes dq_add
// [T, Q] fp32 (rotated, scaled: added to the causal dQ before rounding),
// accumulates the k | v gradients of steps 1..j into dkv_acc [K][T, 2 KV]
// fp32 (zeroed before the last step), and stores step j's finished dk
// (inverse RoPE at t % S + j) / dv as bf16 into the k / v columns of
// dqkv_step.  qkv_all / dout / lse / D as in the forward of step j.
void bwd_diag(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout, const float* lse,
              const float* D, float* dq_add, float* dkv_acc, __nv_bfloat16* dqkv_step,
              const Dims& d, int hd, cudaStream_t s);
// dQ of one step (queries at d.q_row_off) against step 0's causal keys, plus
// dq_add (nullable); writes the q columns of dqkv_step (inverse RoPE when
// d.rope_cos, positions t % S + d.pos_off).
void bwd_dq(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout, const float* lse,
            const float* D, const float* dq_add, __nv_bfloat16* dqkv_step, const Dims& d, int hd,
            cudaStream_t s);
// dK / dV of step 0's keys from the causal scores of n_steps unroll steps:
// queries at rows [n_steps][T] of qkv_all, dout_all [n_steps * T, Q],
// lse_all / D_all [n_steps][nh][T]; writes the k / v columns of dqkv0 (step
// 0's rows).
void bwd_dkdv(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout_all, const float* lse_all,
              const float* D_all, __nv_bfloat16* dqkv0, const Dims& d, int hd, int n_steps,
              cudaStream_t s);

}  // namespace attn
}  // namespace specsim
