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
};

void check_dims(const Dims& d, int hd);  // throws std::invalid_argument
void prepare(int hd);                    // one-time kernel attributes
void forward(const __nv_bfloat16* qkv, __nv_bfloat16* o, float* lse, const Dims& d, int hd,
             cudaStream_t s);
// Dbuf: [nh, T] fp32 scratch.  Writes every element of dqkv.
void backward(const __nv_bfloat16* qkv, const __nv_bfloat16* o, const __nv_bfloat16* dout,
              const float* lse, float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, int hd,
              cudaStream_t s);

}  // namespace attn
}  // namespace specsim
