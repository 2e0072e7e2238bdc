// Host side of the tcgen05 GEMM: TMA tensor-map encoding, plan construction
// and launch.  A GemmPlan is built once per (operands, shape, epilogue) when a
// trainer is created; the training step only replays plan.launch().
#include "gemm.h"

#include <cudaTypedefs.h>

#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "common.h"
#include "gemm.cuh"

namespace specsim {
namespace gemm {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with leading
// dimension ld (elements), box = {box_cols (inner), box_rows}, 128-byte swizzle.
CUtensorMap make_map(const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows) {
  if ((ld * 2) % 16 != 0) throw std::invalid_argument("gemm: leading dimension not 16B aligned");
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    throw std::invalid_argument("gemm: operand pointer not 16B aligned");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// SMs the persistent GEMM grid may occupy.  SPECSIM_GEMM_SMS=n caps it (A/B
// knob for data-parallel runs: leaves SMs free for the NCCL kernels that
// overlap the backward).
int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    if (const char* e = std::getenv("SPECSIM_GEMM_SMS")) {
      const int cap = std::atoi(e);
      if (cap >= 2 && cap < n) n = cap & ~1;  // whole CTA pairs
    }
  }
  return n;
}

template <bool A_MN, bool B_MN, int EPI, int CG>
void launch_t(const GemmPlan& p, cudaStream_t s, bool attr_only = false) {
  auto k = gemm_kernel<A_MN, B_MN, EPI, CG>;
  constexpr int smem = Cfg<CG>::SMEM;
  static_assert(smem <= 232448, "shared memory budget");
  static bool attr_set = false;  // per instantiation; set at plan time (never mid-capture)
  if (!attr_set) {
    SPECSIM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  if (attr_only) return;
  count_launches();
  if constexpr (CG == 1) {
    k<<<p.grid, NUM_THREADS, smem, s>>>(p.map_a, p.map_b, p.args);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;  // CTA pair on one TPC
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SPECSIM_CUDA(cudaLaunchKernelEx(&cfg, k, p.map_a, p.map_b, p.args));
  }
}

template <bool A_MN, bool B_MN, int CG>
void dispatch_epi(const GemmPlan& p, cudaStream_t s, bool a = false) {
  switch (p.epi) {
    case EPI_BF16: launch_t<A_MN, B_MN, EPI_BF16, CG>(p, s, a); break;
    case EPI_F32: launch_t<A_MN, B_MN, EPI_F32, CG>(p, s, a); break;
    case EPI_F32_ACC: launch_t<A_MN, B_MN, EPI_F32_ACC, CG>(p, s, a); break;
    case EPI_BF16_RESID: launch_t<A_MN, B_MN, EPI_BF16_RESID, CG>(p, s, a); break;
    case EPI_CE_FWD: launch_t<A_MN, B_MN, EPI_CE_FWD, CG>(p, s, a); break;
    case EPI_CE_BWD: launch_t<A_MN, B_MN, EPI_CE_BWD, CG>(p, s, a); break;
    case EPI_ADAMW: launch_t<A_MN, B_MN, EPI_ADAMW, CG>(p, s, a); break;
    case EPI_BF16_ROPE: launch_t<A_MN, B_MN, EPI_BF16_ROPE, CG>(p, s, a); break;
    case EPI_SWIGLU_BWD: launch_t<A_MN, B_MN, EPI_SWIGLU_BWD, CG>(p, s, a); break;
    default: throw std::invalid_argument("gemm: bad epilogue");
  }
}

template <int CG>
void dispatch_major(const GemmPlan& p, cudaStream_t s, bool a = false) {
  if (!p.a_mn && !p.b_mn)
    dispatch_epi<false, false, CG>(p, s, a);
  else if (!p.a_mn && p.b_mn)
    dispatch_epi<false, true, CG>(p, s, a);
  else if (p.a_mn && p.b_mn)
    dispatch_epi<true, true, CG>(p, s, a);
  else
    dispatch_epi<true, false, CG>(p, s, a);
}

}  // namespace

CUtensorMap make_tensor_map(const void* ptr, long long rows, long long cols, long long ld,
                            int box_cols, int box_rows) {
  return make_map(ptr, rows, cols, ld, box_cols, box_rows);
}

GemmPlan make_plan(const Operand& A, const Operand& B, int M, int N, int K, int epi,
                   const Args& extra, int cg) {
  if (M <= 0 || N <= 0 || K <= 0) throw std::invalid_argument("gemm: empty shape");
  if (N % 4 != 0) throw std::invalid_argument("gemm: N must be a multiple of 4");
  if (cg != 1 && cg != 2) throw std::invalid_argument("gemm: cg must be 1 or 2");
  GemmPlan p;
  p.a_mn = A.mn_major;
  p.b_mn = B.mn_major;
  p.epi = epi;
  p.cg = cg;
  const int bn_cta = BN / cg;
  // A: K-major = [M, K] rows; MN-major = [K, M] rows.  Boxes are per CTA.
  // gathered operands (Args::a_rows / b_rows): the map spans the source's rows
  const long long a_rows = A.rows > 0 ? A.rows : (A.mn_major ? K : M);
  const long long b_rows = B.rows > 0 ? B.rows : (B.mn_major ? K : N);
  p.map_a = A.mn_major ? make_map(A.ptr, a_rows, M, A.ld, 64, 64)
                       : make_map(A.ptr, a_rows, K, A.ld, 64, BM);
  p.map_b = B.mn_major ? make_map(B.ptr, b_rows, N, B.ld, 64, 64)
                       : make_map(B.ptr, b_rows, K, B.ld, 64, bn_cta);
  if ((extra.a_rows && !A.mn_major && M % BM) || (extra.a_rows && A.mn_major && K % 64) ||
      (extra.b_rows && B.mn_major && K % 64) || (extra.b_rows && !B.mn_major && N % 64))
    throw std::invalid_argument("gemm: gathered operand rows must be whole blocks");
  p.args = extra;
  p.args.M = M;
  p.args.N = N;
  p.args.K = K;
  const int tile_m = BM * cg;
  p.args.num_m_blocks = (M + tile_m - 1) / tile_m;
  p.args.num_n_blocks = (N + BN - 1) / BN;
  p.args.num_tiles = p.args.num_m_blocks * p.args.num_n_blocks;
  // L2-aware rasterisation: the smaller operand is kept resident in groups of
  // panels totalling ~32 MB (loaded evict_last; measured: larger resident
  // sets do not survive in the two-die L2 next to streaming traffic) while the
  // larger operand streams from DRAM once per group.
  const long long a_bytes = static_cast<long long>(M) * K * 2;
  const long long b_bytes = static_cast<long long>(N) * K * 2;
  static const long long budget = [] {
    const char* e = std::getenv("SPECSIM_L2_BUDGET_MB");  // A/B experiments
    const long long mb = e ? std::atoll(e) : 32;
    return (mb > 0 ? mb : 32) << 20;
  }();
  p.args.keep_b = b_bytes < a_bytes ? 1 : 0;
  const long long a_panel = static_cast<long long>(tile_m) * K * 2;
  const long long b_panel = static_cast<long long>(BN) * K * 2;
  const long long bud = extra.l2_budget_mb > 0 ? static_cast<long long>(extra.l2_budget_mb) << 20
                                               : budget;
  long long gm = bud / (a_panel > 0 ? a_panel : 1);
  long long gn = bud / (b_panel > 0 ? b_panel : 1);
  gm = gm < 1 ? 1 : (gm > p.args.num_m_blocks ? p.args.num_m_blocks : gm);
  gn = gn < 1 ? 1 : (gn > p.args.num_n_blocks ? p.args.num_n_blocks : gn);
  p.args.group_m = static_cast<int>(gm);
  p.args.group_n = static_cast<int>(gn);
  const int units = num_sms() / cg;  // CTA pairs (or CTAs) resident at once
  // Long K: when at most two panels of the smaller operand fit the budget the
  // resident walk degenerates to streaming the larger operand once per one or
  // two blocks; walk compact waves instead (group_m ~ sqrt(units * b/a) rows).
  static const int raster = [] {
    const char* e = std::getenv("SPECSIM_RASTER");  // A/B: "resident" | "wave"
    if (!e) return 0;
    return std::string(e) == "resident" ? 1 : (std::string(e) == "wave" ? 2 : 0);
  }();
  static const long long wave_g = [] {
    const char* e = std::getenv("SPECSIM_RASTER_WAVE_G");  // A/B: resident-group threshold
    return e ? std::atoll(e) : 2;
  }();
  const long long g_res = p.args.keep_b ? gn : gm;
  if (raster == 2 || (raster == 0 && g_res <= wave_g)) {
    const double w = std::sqrt(static_cast<double>(units) * b_panel / static_cast<double>(a_panel));
    long long gw = static_cast<long long>(w + 0.5);
    gw = gw < 1 ? 1 : (gw > p.args.num_m_blocks ? p.args.num_m_blocks : gw);
    p.args.keep_b = 2;
    p.args.group_m = static_cast<int>(gw);
  }
  p.grid = (p.args.num_tiles < units ? p.args.num_tiles : units) * cg;
  p.flops = 2.0 * M * static_cast<double>(N) * K;
  p.prepare();
  if (epi == EPI_ADAMW) {
    if (!p.args.opt_p || !p.args.opt_m || !p.args.opt_v || !p.args.opt_p16 || !p.args.opt_hp)
      throw std::invalid_argument("gemm: AdamW epilogue needs p/m/v/p16/hp");
    if (p.args.ldc % 8 != 0 || N % 8 != 0)
      throw std::invalid_argument("gemm: AdamW epilogue needs ldc and N multiples of 8");
  }
  if (epi == EPI_BF16_ROPE) {
    if (!p.args.rope_cos || !p.args.rope_sin || p.args.rope_S <= 0 ||
        (p.args.rope_hd != 64 && p.args.rope_hd != 128) || p.args.rope_cols % p.args.rope_hd ||
        p.args.rope_pos_off < 0)
      throw std::invalid_argument("gemm: bad RoPE epilogue arguments");
    if (p.args.rope_ld == 0) p.args.rope_ld = p.args.rope_S;
    if (p.args.rope_ld < p.args.rope_S + p.args.rope_pos_off)
      throw std::invalid_argument("gemm: RoPE table shorter than rope_S + rope_pos_off");
  }
  if (epi == EPI_SWIGLU_BWD && (!p.args.R || p.args.ldr != p.args.ldc || p.args.ldc < 2ll * N))
    throw std::invalid_argument("gemm: SwiGLU-backward epilogue needs R = gu and ldc = ldr >= 2N");
  if (epi == EPI_BF16 || epi == EPI_BF16_RESID || epi == EPI_CE_BWD || epi == EPI_F32 ||
      epi == EPI_F32_ACC || epi == EPI_BF16_ROPE || epi == EPI_SWIGLU_BWD) {
    if (!p.args.C) throw std::invalid_argument("gemm: missing output");
    if ((p.args.ldc * (epi == EPI_F32 || epi == EPI_F32_ACC ? 4 : 2)) % 16 != 0)
      throw std::invalid_argument("gemm: ldc not 16B aligned");
  }
  return p;
}

void GemmPlan::launch(cudaStream_t s) const {
  if (cg == 2)
    dispatch_major<2>(*this, s);
  else
    dispatch_major<1>(*this, s);
}

void GemmPlan::prepare() const {
  if (cg == 2)
    dispatch_major<2>(*this, nullptr, true);
  else
    dispatch_major<1>(*this, nullptr, true);
}

}  // namespace gemm
}  // namespace specsim
