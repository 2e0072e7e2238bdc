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
};

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

}  // namespace attn
}  // namespace specsim
