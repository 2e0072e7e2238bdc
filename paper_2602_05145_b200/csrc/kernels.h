// HBM-bound kernels of the draft-training step (norms, RoPE, SwiGLU, CE
// reduction, AdamW, batch gather, signal packing).  All use 16-byte vector
// accesses along the contiguous dimension; reductions are deterministic
// (fixed-order partials, no float atomics).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm.h"

namespace specsim {
namespace kern {

constexpr int kMaxBatch = 64;
constexpr int kMaxTtt = 16;  // training-time-test unroll steps

// Rows of K unroll steps are stacked [K][T]; step j's loss weight is w[j] = decay^j.
struct StepWeights {
  float w[kMaxTtt];
  int K;
  long long T;  // rows per step
};

// One micro-batch: sample b's tokens live at ring rows (start[b] + t) % cap.
struct BatchSpec {
  int n;                       // samples present (<= B); rows b >= n are padding
  long long start[kMaxBatch];  // ring row of token 0
  int len[kMaxBatch];          // L (tokens)
};

// F[T, W] bf16, u/y int32, mask int32 (SURVEY A.2 alignment).  u / y / m hold
// K slices of T rows: slice j is the rule shifted by j tokens (training-time
// test), u = x[t+1+j], y = x[t+2+j], m = [t+2+j < L].
// spec lives in device memory (so the launch can sit in a CUDA graph)
void gather_batch(const __nv_bfloat16* ring_feat, const int32_t* ring_ids, long long cap, int W,
                  const BatchSpec* spec, int B, int S, int K, __nv_bfloat16* F, int32_t* u,
                  int32_t* y, int32_t* m, cudaStream_t s);

// The same u / y / m without the feature copy, plus blk_rows[T / 64] = the
// ring row of every 64-row block of the micro-batch (S % 64 == 0): the fc
// GEMMs TMA-load F straight from the ring (HiddenStateBuffer::kMirrorRows
// keeps a block contiguous across the ring's end).  Rows past a sample's end
// read ring rows of other samples: their targets are masked, so every
// gradient contribution of those rows is exactly zero.
void gather_tokens(const int32_t* ring_ids, long long cap, const BatchSpec* spec, int B, int S,
                   int K, int32_t* u, int32_t* y, int32_t* m, int32_t* blk_rows, cudaStream_t s);

// coef[r] = m[r] / n_global * w[r / T] over K*T rows; n_global read from a
// device scalar (int64)
void ce_coef(const int32_t* m, const long long* n_global, float* coef, const StepWeights& sw,
             cudaStream_t s);
// count of mask (int64 device scalar)
void mask_count(const int32_t* m, long long T, long long* out, cudaStream_t s);
// n_global = override > 0 ? override : counted
void select_count(const long long* override_n, const long long* counted, long long* n_global,
                  cudaStream_t s);

// y[t, :H] = bf16(x_row * rstd * w); x_row = x[t] or x[gather[t]] (embedding).
void rmsnorm_fwd(const __nv_bfloat16* x, long long ldx, const int32_t* gather, const float* w,
                 float eps, __nv_bfloat16* y, long long ldy, float* rstd, long long T, int H,
                 cudaStream_t s);

// dx = rstd*(dy*w) - x*rstd^3*mean(dy*w*x);  out_f32 = resid + dx (resid nullable),
// out_bf16 = bf16(out_f32) (nullable); dx skipped entirely when both outputs null.
// dw[i] = sum_t dy*x*rstd (deterministic two-pass; dw_partial scratch
// [ceil(T/rows_per_block), H]).  dw null: the per-block partials are only
// written (when dw_partial is non-null) for a later colsum over several calls.
// x may be gathered (embedding rows).
void rmsnorm_bwd(const float* dy, long long lddy, const __nv_bfloat16* x, long long ldx,
                 const int32_t* gather, const float* w, const float* rstd, const float* resid,
                 float* out_f32, __nv_bfloat16* out_bf16, long long ldo, float* dw,
                 float* dw_partial, long long T, int H, cudaStream_t s);
long long rmsnorm_bwd_partial_rows(long long T);
// out[i] = sum over rows of parts[row, i] (fixed order: deterministic)
void colsum(const float* parts, long long rows, int H, float* out, cudaStream_t s);

// dst[0..n_words) = src[...] where src is MAPPED pinned host memory, read by
// the SMs over PCIe: stages the per-step inputs without a copy-engine H2D,
// which would queue behind bulk ingest DMA issued earlier on another stream.
void fetch_mapped(const uint32_t* src, uint32_t* dst, int n_words, cudaStream_t s);
// The reverse: dst (mapped pinned host memory) = src (device), stores over
// PCIe from the SMs; used for the per-step loss / counters so no D2H
// copy-engine transfer sits in the trainer stream behind ingest DMA.
void store_mapped(const uint32_t* src, uint32_t* dst, int n_words, cudaStream_t s);

// NeoX RoPE on the q and k heads of a [T, NQ] row-major buffer, in place.
void rope(__nv_bfloat16* qkv, long long T, int S, int NQ, int n_rot_heads, int hd,
          const float* cos_t, const float* sin_t, bool inverse, cudaStream_t s);

// act[t, i] = silu(gu[t, i]) * gu[t, I + i]
void swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* act, long long T, int I, cudaStream_t s);
// dgu[t, i] = dact*up*silu'(g), dgu[t, I+i] = dact*silu(g)
void swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* dact, __nv_bfloat16* dgu,
                long long T, int I, cudaStream_t s);

// Combine per-N-tile softmax partials into lse / per-row loss / argmax.
void ce_reduce(const gemm::CePartial* partials, int num_nb, long long T, const int32_t* y,
               const int32_t* m, float* lse, float* row_loss, int32_t* argmax, cudaStream_t s);
// CE gradient from the logits the forward GEMM stored as fp16 offsets from
// their 128-column half tile's row max (partials[(v / 128) * T + t].max):
// dlog[t, j] = bf16((exp(delta + max - lse[t]) - [v0 + j == y[t]]) * coef[t])
// for j < vn (same arithmetic as the EPI_CE_BWD recompute epilogue up to the
// fp16 rounding of the offset).  vn % 8 == 0, v0 % 128 == 0.
void ce_grad(const __half* logits, long long ldl, const gemm::CePartial* partials,
             const float* lse, const float* coef, const int32_t* y, int v0, long long T, int vn,
             __nv_bfloat16* dlog, long long ldd, cudaStream_t s);
// stats[0] = sum_j w[j] * (sum of step j's row_loss / n_global) (double),
// stats[1] = valid (as double), stats[2] = top-1 correct, both of step 0.
// Single block, fixed order.
void ce_finalize(const float* row_loss, const int32_t* argmax, const int32_t* y, const int32_t* m,
                 const long long* n_global, const StepWeights& sw, double* stats, cudaStream_t s);

// PyTorch AdamW on flat fp32 state; writes the bf16 working copy.
struct AdamHyper {
  float lr, beta1, beta2, eps, decay /* 1 - lr*wd */, step_size /* lr / bc1 */,
      bc2_sqrt;
};
void adamw(long long n, float* p, float* m, float* v, const float* g, __nv_bfloat16* p16,
           const gemm::AdamDev* hp, cudaStream_t s);

void f32_to_bf16(const float* x, __nv_bfloat16* y, long long n, cudaStream_t s);

// Signal packing: ring row (pos + i) % cap = [layer0[idx[i]] | layer1[idx[i]] | ...].
struct LayerPtrs {
  const __nv_bfloat16* p[8];
};
void pack_signals(const LayerPtrs& layers, int n_layers, long long ld, int H, const int32_t* idx,
                  int n, __nv_bfloat16* ring_feat, long long cap, long long pos, cudaStream_t s);
void pack_packed(const __nv_bfloat16* src, int W, int n, __nv_bfloat16* ring_feat, long long cap,
                 long long pos, cudaStream_t s);

}  // namespace kern
}  // namespace specsim
