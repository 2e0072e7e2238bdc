// Kernel test hooks: host-buffer wrappers around single device kernels so the
// parity tests can exercise them through the C ABI (no framework types).
#include <cmath>
#include <cstring>
#include <vector>

#include "common.h"
#include "attention.h"
#include "gemm.h"

namespace specsim {
namespace {

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) SPECSIM_CUDA(cudaMalloc(&p, bytes));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace
}  // namespace specsim

extern "C" int specsim_debug_gemm(int a_mn, int b_mn, int epi_cg, int32_t M, int32_t N, int32_t K,
                                  const uint16_t* A, int64_t lda, const uint16_t* B, int64_t ldb,
                                  void* C, int64_t ldc, const uint16_t* R, int64_t ldr,
                                  int32_t iters, float* mean_ms) {
  using namespace specsim;
  return guard([&] {
    const int epi = epi_cg & 0xff;
    const int cg = (epi_cg >> 8) ? (epi_cg >> 8) : 2;
    Problems pr("specsim_debug_gemm");
    pr.check(M > 0 && N > 0 && K > 0, "M, N, K must be > 0");
    pr.check(A && B && C, "A, B, C must be non-null");
    pr.check((epi >= 0 && epi <= 3) || epi == 6, "epi must be 0..3 or 6 (fused AdamW)");
    pr.check(epi != 3 || R, "epi 3 needs R");
    pr.throw_if_any();
    const size_t a_elems = static_cast<size_t>(a_mn ? K : M) * lda;
    const size_t b_elems = static_cast<size_t>(b_mn ? K : N) * ldb;
    const size_t c_esz = (epi == 1 || epi == 2 || epi == 6) ? 4 : 2;
    const size_t c_bytes = static_cast<size_t>(M) * ldc * c_esz;
    DevBuf dA(a_elems * 2), dB(b_elems * 2), dC(c_bytes), dR(R ? static_cast<size_t>(M) * ldr * 2 : 0);
    SPECSIM_CUDA(cudaMemcpy(dA.p, A, a_elems * 2, cudaMemcpyHostToDevice));
    SPECSIM_CUDA(cudaMemcpy(dB.p, B, b_elems * 2, cudaMemcpyHostToDevice));
    SPECSIM_CUDA(cudaMemcpy(dC.p, C, c_bytes, cudaMemcpyHostToDevice));
    if (R) SPECSIM_CUDA(cudaMemcpy(dR.p, R, static_cast<size_t>(M) * ldr * 2, cudaMemcpyHostToDevice));
    gemm::Args args{};
    args.C = dC.p;
    args.ldc = ldc;
    args.R = static_cast<const __nv_bfloat16*>(dR.p);
    args.ldr = ldr;
    // epi 6: AdamW fused into the epilogue over device-resident state laid
    // out like C (p = C's fp32 contents, m = v = 0, step 1); C receives p
    const size_t n_state = static_cast<size_t>(M) * ldc;
    DevBuf dM(epi == 6 ? n_state * 4 : 0), dV(epi == 6 ? n_state * 4 : 0),
        dP16(epi == 6 ? n_state * 2 : 0), dHp(epi == 6 ? sizeof(gemm::AdamDev) : 0);
    if (epi == 6) {
      SPECSIM_CUDA(cudaMemset(dM.p, 0, n_state * 4));
      SPECSIM_CUDA(cudaMemset(dV.p, 0, n_state * 4));
      const gemm::AdamDev hp{1e-3f, 0.9f, 0.95f, 1e-8f, 1.f, 1e-3f / 0.1f, std::sqrt(0.05f), 0.f};
      SPECSIM_CUDA(cudaMemcpy(dHp.p, &hp, sizeof(hp), cudaMemcpyHostToDevice));
      args.opt_p = static_cast<float*>(dC.p);
      args.opt_m = static_cast<float*>(dM.p);
      args.opt_v = static_cast<float*>(dV.p);
      args.opt_p16 = static_cast<__nv_bfloat16*>(dP16.p);
      args.opt_hp = static_cast<const gemm::AdamDev*>(dHp.p);
    }
    gemm::GemmPlan plan = gemm::make_plan({dA.p, lda, a_mn != 0}, {dB.p, ldb, b_mn != 0}, M, N,
                                          K, epi, args, cg);
    cudaStream_t s;
    SPECSIM_CUDA(cudaStreamCreate(&s));
    plan.launch(s);
    SPECSIM_CHECK_LAUNCH();
    SPECSIM_CUDA(cudaStreamSynchronize(s));
    // Copy the single-launch result out before any timing re-launches
    // (accumulating epilogues would otherwise compound).
    SPECSIM_CUDA(cudaMemcpy(C, dC.p, c_bytes, cudaMemcpyDeviceToHost));
    if (iters > 1 && mean_ms) {
      cudaEvent_t e0, e1;
      SPECSIM_CUDA(cudaEventCreate(&e0));
      SPECSIM_CUDA(cudaEventCreate(&e1));
      for (int i = 0; i < 3; ++i) plan.launch(s);
      SPECSIM_CUDA(cudaEventRecord(e0, s));
      for (int i = 0; i < iters; ++i) plan.launch(s);
      SPECSIM_CUDA(cudaEventRecord(e1, s));
      SPECSIM_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      SPECSIM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      *mean_ms = ms / iters;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    SPECSIM_CUDA(cudaStreamDestroy(s));
  });
}

extern "C" int specsim_debug_attention(int32_t B, int32_t S, int32_t nh, int32_t nkv, int32_t hd,
                                       const uint16_t* qkv, const uint16_t* dout, uint16_t* o,
                                       float* lse, uint16_t* dqkv) {
  using namespace specsim;
  return guard([&] {
    attn::Dims d;
    d.B = B;
    d.S = S;
    d.nh = nh;
    d.nkv = nkv;
    d.Q = nh * hd;
    d.KV = nkv * hd;
    d.NQ = d.Q + 2 * d.KV;
    d.scale = 1.0f / std::sqrt(static_cast<float>(hd));
    attn::check_dims(d, hd);
    attn::prepare(hd);
    if (!qkv || !o || !lse) throw std::invalid_argument("null argument");
    const size_t T = static_cast<size_t>(B) * S;
    DevBuf dq(T * d.NQ * 2), dO(T * d.Q * 2), dl(T * nh * 4), ddo(T * d.Q * 2),
        ddq(T * d.NQ * 2), dD(T * nh * 4);
    SPECSIM_CUDA(cudaMemcpy(dq.p, qkv, T * d.NQ * 2, cudaMemcpyHostToDevice));
    attn::forward(static_cast<const __nv_bfloat16*>(dq.p), static_cast<__nv_bfloat16*>(dO.p),
                  static_cast<float*>(dl.p), d, hd, 0);
    SPECSIM_CHECK_LAUNCH();
    if (dout && dqkv) {
      SPECSIM_CUDA(cudaMemcpy(ddo.p, dout, T * d.Q * 2, cudaMemcpyHostToDevice));
      attn::backward(static_cast<const __nv_bfloat16*>(dq.p), static_cast<const __nv_bfloat16*>(dO.p),
                     static_cast<const __nv_bfloat16*>(ddo.p), static_cast<const float*>(dl.p),
                     static_cast<float*>(dD.p), static_cast<__nv_bfloat16*>(ddq.p), d, hd, 0);
      SPECSIM_CHECK_LAUNCH();
    }
    SPECSIM_CUDA(cudaDeviceSynchronize());
    SPECSIM_CUDA(cudaMemcpy(o, dO.p, T * d.Q * 2, cudaMemcpyDeviceToHost));
    SPECSIM_CUDA(cudaMemcpy(lse, dl.p, T * nh * 4, cudaMemcpyDeviceToHost));
    if (dout && dqkv) SPECSIM_CUDA(cudaMemcpy(dqkv, ddq.p, T * d.NQ * 2, cudaMemcpyDeviceToHost));
  });
}
