// Causal GQA attention (forward, and the dK/dV and dQ backward kernels
// below) on the 5th-generation tensor cores.
//
// Forward: persistent, one CTA per SM looping over work items (sample, query
// head, 128-query block), most keys first.  Warp roles:
//   warp 0      TMA producer: the item's Q, then K_j / V_j (128-key blocks)
//               into a 2-deep ring (SWIZZLE_128B tiles, one tensor map over qkv)
//   warp 1      MMA issuer (one lane): S_j = Q K_j^T into one of two TMEM
//               S buffers, then O += P_j V_j with P_j from shared memory
//   warps 2..5  softmax: one query row per thread (TMEM lane), so row max /
//               sum need no shuffles; P_j written to smem in the UMMA K-major
//               SW128 layout, double-buffered so the softmax of block j+1
//               overlaps the PV MMA of block j; lazy rescaling (only when the
//               row max grows by more than 2^8) keeps O read-modify-writes --
//               the one step that must wait for PV_j -- rare
// TMEM: S0 | S1 | O0 | O1 (128 columns each; O double-buffered across items).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "attention.h"
#include "common.h"
#include "gemm.h"
#include "ptx.cuh"

#ifndef SPECSIM_ATTN_PROBE
#define SPECSIM_ATTN_PROBE 0
#endif

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
  static constexpr int OFF_P = OFF_V + 2 * KV;     // 2 buffers
  static constexpr int OFF_BAR = OFF_P + 2 * P;  // 20 mbarriers + the TMEM slot
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
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
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

// Persistent: grid = min(#items, #SMs); CTA c processes work items c, c + grid,
// ... where item i = (query block, head, sample) in decreasing-work order
// (most keys first).  Block counters (K / V stages, S and P buffers, their
// mbarrier phases) run across items; the O accumulator is double-buffered in
// TMEM (S0 | S1 | O0 | O1) so item i's epilogue overlaps item i+1's first
// MMAs, and the single Q tile is reloaded as soon as item i's last S MMA ran.
// A grid of #items reproduces one-item-per-CTA launches (SPECSIM_ATTN_FWD_GRID=items).
template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, Dims d) {
  using L = FwdSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
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
  uint64_t* p_full = bar + 13;   // [2]
  uint64_t* pv_done = bar + 15;  // [2]
  uint64_t* q_empty = bar + 17;
  uint64_t* o_free = bar + 18;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);

  const int nqb = d.S / BQ;
  const int n_items = nqb * d.nh * d.B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nd = d.n_diag;
  // item -> (query block, head, sample); most keys first
  auto decode = [&](int idx, int& qb, int& h, int& b) {
    qb = nqb - 1 - idx / (d.nh * d.B);
    const int hb = idx % (d.nh * d.B);
    h = hb % d.nh;
    b = hb / d.nh;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm);
    ptx::mbar_init(q_full, 1);
    // Q is free after the item's last S MMA; with training-time-test cache
    // entries the softmax epilogue also reads it (4 more arrivals)
    ptx::mbar_init(q_empty, nd > 0 ? 5 : 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&pv_done[i], 1);
      ptx::mbar_init(&o_free[i], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO[2] = {tmem + 256, tmem + 384};

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA
      constexpr int A = L::ATOMS;
      int n = 0;  // block counter across items
      for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
        int qb, h, b;
        decode(idx, qb, h, b);
        const int g = h / (d.nh / d.nkv), row0 = b * d.S;
        ptx::mbar_wait(q_empty, (li & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, L::Q);
        for (int a = 0; a < A; ++a)
          ptx::tma_load_2d(&tm, q_full, sQ + a * TILE, h * HD + 64 * a,
                           static_cast<int>(d.q_row_off) + row0 + qb * BQ);
        for (int j = 0; j <= qb; ++j, ++n) {
          const int s = n & 1;
          const uint32_t ph = (n >> 1) & 1;
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
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA
      constexpr uint32_t idS = ptx::make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idO = ptx::make_idesc_bf16(BQ, HD, false, true);
      const uint32_t aQ = ptx::smem_u32(sQ);
      // S_n = Q K_n^T for block n (item li, its block j of nkv); the item's
      // last S releases Q
      auto issue_s = [&](int n, int li, int j, int nkv) {
        const int s = n & 1;
        if (j == 0) ptx::mbar_wait(q_full, li & 1);
        ptx::mbar_wait(&k_full[s], (n >> 1) & 1);
        ptx::mbar_wait(&s_free[s], ((n >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t aK = ptx::smem_u32(sK + s * L::KV);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::umma_bf16(tS[s], kdesc(aQ, kk), kdesc(aK, kk), idS, kk > 0 ? 1u : 0u);
        ptx::umma_commit(&s_full[s]);
        ptx::umma_commit(&k_empty[s]);
        if (j == nkv - 1) ptx::umma_commit(q_empty);
      };
      int n = 0;
      for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
        int qb, h, b;
        decode(idx, qb, h, b);
        const int nkv = qb + 1, ob = li & 1;
        const int nidx = idx + gridDim.x;
        if (li == 0) issue_s(0, 0, 0, nkv);
        for (int j = 0; j < nkv; ++j, ++n) {
          if (j + 1 < nkv) issue_s(n + 1, li, j + 1, nkv);
          const int s = n & 1;  // K / V stage, S buffer and P buffer of block n
          // O[ob] was last read by the epilogue of item li - 2
          if (j == 0) ptx::mbar_wait(&o_free[ob], ((li >> 1) & 1) ^ 1);
          ptx::mbar_wait(&p_full[s], (n >> 1) & 1);
          ptx::mbar_wait(&v_full[s], (n >> 1) & 1);
          ptx::tc_fence_after();
          const uint32_t aV = ptx::smem_u32(sV + s * L::KV);
          const uint32_t aP = ptx::smem_u32(sP + s * L::P);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            ptx::umma_bf16(tO[ob], kdesc(aP, kk), mndesc(aV, kk), idO,
                           (j > 0 || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&pv_done[s]);
          ptx::umma_commit(&v_empty[s]);
          // the next item's first S goes after this item's last PV (its Q
          // load is then hidden behind this PV and the epilogue)
          if (j == nkv - 1 && nidx < n_items) {
            int qb2, h2, b2;
            decode(nidx, qb2, h2, b2);
            issue_s(n + 1, li + 1, 0, qb2 + 1);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // query row within the block (= TMEM lane)
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float sl2 = d.scale * kLog2e;
    const long long T = static_cast<long long>(d.B) * d.S;
    int n = 0;
    for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
      int qb, h, b;
      decode(idx, qb, h, b);
      const int g = h / (d.nh / d.nkv), row0 = b * d.S;
      const int q = qb * BQ + r;  // position within the sample
      const int nkv = qb + 1, ob = li & 1;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nkv; ++j, ++n) {
        const int s = n & 1;
        ptx::mbar_wait(&s_full[s], (n >> 1) & 1);
        ptx::tc_fence_after();
        // Row max over this block's 128 raw scores.  One softmax warp per SM
        // sub-partition, so the softmax is issue-bound: 3-input max with 4
        // independent partials, the scale folded into the exponent's FFMA2
        // (max(s * c) = c * max(s), c > 0), MUFU ex2 without range fix-up, and
        // packed fp32x2 row sums -- ~3 instructions per score instead of ~10.
        uint32_t v[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x32(tS[s] + lane_off + c * 32, v[c]);
        ptx::tmem_ld_wait();
        if (j == qb) {  // diagonal block: keys after the query are masked
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i > r) v[c][i] = __float_as_uint(-INFINITY);
        }
        float mxp[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            mxp[0] = ptx::max3f(mxp[0], __uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1]));
            mxp[1] =
                ptx::max3f(mxp[1], __uint_as_float(v[c][i + 2]), __uint_as_float(v[c][i + 3]));
            mxp[2] =
                ptx::max3f(mxp[2], __uint_as_float(v[c][i + 4]), __uint_as_float(v[c][i + 5]));
            mxp[3] =
                ptx::max3f(mxp[3], __uint_as_float(v[c][i + 6]), __uint_as_float(v[c][i + 7]));
          }
        const float mx = ptx::max3f(mxp[0], mxp[1], fmaxf(mxp[2], mxp[3])) * sl2;
        // S buffer consumed: the MMA may overwrite it with S_{n+2}
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_free[s]);
        // lazy rescale: a row moves its reference max only when the max grows
        // by more than 2^8; the O read-modify-write is warp-collective
        // (tcgen05.ld / st are .sync.aligned), so the whole warp does it when
        // any lane needs it -- and only then waits for the previous PV
        const bool need = mx > m_run + 8.f;
        float corr = 1.f;
        if (need) {
          corr = exp2f(m_run - mx);  // 0 on the first block
          l_run *= corr;
          m_run = mx;
        }
        const bool rescale = j > 0 && __any_sync(0xffffffffu, need);
        if (rescale) {
          ptx::mbar_wait(&pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(tO[ob] + lane_off + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st_32x32b_x32(tO[ob] + lane_off + c * 32, o);
          }
          tmem_st_wait();
        }
        // P buffer s was last read by PV_{n-2}
        if (n >= 2) ptx::mbar_wait(&pv_done[s], ((n - 2) >> 1) & 1);
        uint8_t* sPb = sP + s * L::P;
        // P = 2^(s * scale * log2e - m) -> bf16, K-major SW128: row r, 16-byte
        // chunk cc of tile t at t*TILE + r*128 + ((cc ^ (r & 7)) * 16); row
        // sum in 4 packed fp32x2 partials
        const uint64_t scale2 = ptx::f32x2(sl2, sl2), negm2 = ptx::f32x2(-m_run, -m_run);
        uint64_t lp2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            float p[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const uint64_t x2 = ptx::ffma2(
                  ptx::f32x2(__uint_as_float(v[c][i + e]), __uint_as_float(v[c][i + e + 1])),
                  scale2, negm2);
              float x0, x1;
              ptx::f32x2_split(x2, x0, x1);
              p[e] = ptx::ex2_ftz(x0);
              p[e + 1] = ptx::ex2_ftz(x1);
              lp2[e >> 1] = ptx::fadd2(lp2[e >> 1], ptx::f32x2(p[e], p[e + 1]));
            }
            const int key = c * 32 + i;  // 8 keys = one 16-byte chunk
            const int t = key >> 6, cc = (key & 63) >> 3;
            uint4 pk;
            pk.x = ptx::pack_bf16x2(p[0], p[1]);
            pk.y = ptx::pack_bf16x2(p[2], p[3]);
            pk.z = ptx::pack_bf16x2(p[4], p[5]);
            pk.w = ptx::pack_bf16x2(p[6], p[7]);
            *reinterpret_cast<uint4*>(sPb + t * TILE + r * 128 + ((cc ^ (r & 7)) << 4)) = pk;
          }
        }
        {
          float a0, a1;
          ptx::f32x2_split(ptx::fadd2(ptx::fadd2(lp2[0], lp2[1]), ptx::fadd2(lp2[2], lp2[3])),
                           a0, a1);
          l_run += a0 + a1;
        }
        ptx::fence_proxy_async_smem();  // generic-proxy P writes -> tensor-core reads
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[s]);
      }
      // ---- epilogue of the item: O[ob] -> bf16 rows, lse
      ptx::mbar_wait(&pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
      ptx::tc_fence_after();
      // Training-time-test cache entries (unroll step n_diag >= 1): one extra
      // score per earlier step i at this row, q . k_i (q from the swizzled
      // smem tile, k_i from HBM), merged into the running max / sum; their
      // values are added to O row-wise in the store loop below.
      float pd[kMaxDiag];
      float corr = 1.f;
      if (nd > 0) {
        float mnew = m_run;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          const uint4* kr = reinterpret_cast<const uint4*>(
              d.diag_qkv + (static_cast<long long>(i + 1) * T + row0 + q) * d.NQ + d.Q + g * HD);
          float dot = 0.f;
#pragma unroll
          for (int c8 = 0; c8 < HD / 8; ++c8) {
            const uint4 qv = *reinterpret_cast<const uint4*>(
                sQ + (c8 >> 3) * TILE + r * 128 + (((c8 & 7) ^ (r & 7)) << 4));
            const uint4 kv = __ldg(kr + c8);
            dot += ptx::dot_bf16x8(qv, kv);
          }
          pd[i] = dot * sl2;
          mnew = fmaxf(mnew, pd[i]);
        }
        // sQ read: the producer may load the next item's Q
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_empty);
        corr = exp2f(m_run - mnew);
        l_run *= corr;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          pd[i] = exp2f(pd[i] - mnew);
          l_run += pd[i];
        }
        m_run = mnew;
      }
      const float inv = 1.f / l_run;
      __nv_bfloat16* orow = out + static_cast<long long>(row0 + q) * d.Q + h * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(tO[ob] + lane_off + c * 32, o);
        ptx::tmem_ld_wait();
        float acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(o[i]) * corr;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          const uint4* vr = reinterpret_cast<const uint4*>(
              d.diag_qkv + (static_cast<long long>(i + 1) * T + row0 + q) * d.NQ + d.Q + d.KV +
              g * HD + c * 32);
#pragma unroll
          for (int v8 = 0; v8 < 4; ++v8) {
            float vf[8];
            ptx::unpack_bf16x8(__ldg(vr + v8), vf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[v8 * 8 + e] += pd[i] * vf[e];
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          ptx::st_global_v4(orow + c * 32 + i, ptx::pack_bf16x2(acc[i] * inv, acc[i + 1] * inv),
                            ptx::pack_bf16x2(acc[i + 2] * inv, acc[i + 3] * inv),
                            ptx::pack_bf16x2(acc[i + 4] * inv, acc[i + 5] * inv),
                            ptx::pack_bf16x2(acc[i + 6] * inv, acc[i + 7] * inv));
      }
      // O[ob] read: the MMA may start item li + 2's accumulation in it
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_free[ob]);
      lse[h * T + row0 + q] = (m_run + log2f(l_run)) * kLn2;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ======================================================================
// Forward, two query tiles per CTA (default when the GQA group is even).
//
// A work item is (sample, query block, head pair): heads 2p and 2p + 1 of one
// KV group see the same K / V blocks under the same causal mask, so every
// K / V tile a CTA stages feeds two S MMAs and two PV MMAs, and two softmax
// warpgroups (one per head; two warps per SM sub-partition) ping-pong with
// the tensor pipe: while warpgroup 0 turns S0_n into P0_n, the MMA warp runs
// PV1_{n-1} and S1_n, and vice versa.
//   TMEM: S0 | S1 | O0 | O1 (128 columns each).  P_t is written back over the
//   first 64 columns of S_t as packed bf16 (tcgen05.st) and read from TMEM
//   by the PV MMA (A operand in tensor memory): no P traffic through shared
//   memory, no async-proxy fence.  The pipe executes one issuer's MMAs in
//   order, so S_{t,n+1} (issued after PV_{t,n}) overwrites P_{t,n} only after
//   PV_{t,n} read it; S_{t,n+1} completing also implies PV_{t,n} completed, so
//   the lazy O rescale needs no extra wait.
//   smem: Q0 | Q1, K and V rings (2 slots each at hd 128, 3 at hd 64).
// SPECSIM_ATTN_POLY_PAIRS of every four exponential pairs (off-diagonal
// blocks) can run as a degree-4 polynomial on the FMA pipe (relative error
// 2.6e-6, below the bf16 rounding of P) instead of MUFU.EX2, which issues one
// warp instruction per 8 cycles per SM sub-partition (scripts/micro/mufu_rate.cu).
#ifndef SPECSIM_ATTN_POLY_PAIRS
#define SPECSIM_ATTN_POLY_PAIRS 0
#endif

template <int HD>
struct Fwd2Smem {
  static constexpr int ATOMS = HD / 64;
  static constexpr int Q = ATOMS * TILE;              // one query tile [128 q x HD]
  static constexpr int KV = ATOMS * TILE;             // one K or V block [128 keys x HD]
  static constexpr int NSLOT = HD == 128 ? 2 : 3;     // slots per K / V ring
  static constexpr int OFF_Q = 0;                     // 2 tiles
  static constexpr int OFF_K = OFF_Q + 2 * Q;
  static constexpr int OFF_V = OFF_K + NSLOT * KV;
  static constexpr int OFF_BAR = OFF_V + NSLOT * KV;  // mbarriers + the TMEM slot
  static constexpr int BYTES = 1024 + OFF_BAR + 256;
};

// 2^x for two values on the FMA pipe: x = j + f, j = rint(x) (the 1.5 * 2^23
// shifter), 2^f by a degree-4 minimax polynomial on [-0.5, 0.5] (relative
// error 2.6e-6), 2^j added to the exponent field.  x is clamped at -120 so
// the exponent never underflows (2^-120 stands in for anything smaller).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1;
  ptx::f32x2_split(x2, x0, x1);
  const uint64_t x = ptx::f32x2(fmaxf(x0, -120.f), fmaxf(x1, -120.f));
  const uint64_t t = ptx::fadd2(x, ptx::f32x2(12582912.f, 12582912.f));
  const uint64_t jf = ptx::fadd2(t, ptx::f32x2(-12582912.f, -12582912.f));
  const uint64_t f = ptx::ffma2(jf, ptx::f32x2(-1.f, -1.f), x);
  uint64_t p = ptx::ffma2(ptx::f32x2(0.009570068679749966f, 0.009570068679749966f), f,
                          ptx::f32x2(0.055917806923389435f, 0.055917806923389435f));
  p = ptx::ffma2(p, f, ptx::f32x2(0.240247443318367f, 0.240247443318367f));
  p = ptx::ffma2(p, f, ptx::f32x2(0.6931218504905701f, 0.6931218504905701f));
  p = ptx::ffma2(p, f, ptx::f32x2(0.9999992847442627f, 0.9999992847442627f));
  float p0, p1, t0, t1;
  ptx::f32x2_split(p, p0, p1);
  ptx::f32x2_split(t, t0, t1);
  return ptx::f32x2(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
                    __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}

// D[tmem] (+)= A[tmem] * B[smem]: A (M x 16, bf16 packed two per 32-bit
// column, row m in TMEM lane m) read from tensor memory
__device__ __forceinline__ void umma_bf16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int HD>
__global__ void __launch_bounds__(320, 1)
    attn_fwd2_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                        float* __restrict__ lse, Dims d) {
  using L = Fwd2Smem<HD>;
  constexpr int NS = L::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;        // [NS]
  uint64_t* k_empty = k_full + NS;   // [NS]
  uint64_t* v_full = k_empty + NS;   // [NS]
  uint64_t* v_empty = v_full + NS;   // [NS]
  uint64_t* s_full = v_empty + NS;   // [2] per tile
  uint64_t* p_full = s_full + 2;     // [2]
  uint64_t* o_full = p_full + 2;     // [2]
  uint64_t* o_free = o_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int nqb = d.S / BQ;
  const int nhp = d.nh / 2;
  const int n_items = nqb * nhp * d.B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nd = d.n_diag;
  auto decode = [&](int idx, int& qb, int& hp, int& b) {
    qb = nqb - 1 - idx / (nhp * d.B);
    const int hb = idx % (nhp * d.B);
    hp = hb % nhp;
    b = hb / nhp;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm);
    ptx::mbar_init(q_full, 1);
    // Q is free after the item's last S MMAs; with training-time-test cache
    // entries the eight softmax warps' epilogues also read it
    ptx::mbar_init(q_empty, nd > 0 ? 9 : 1);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 4);
      ptx::mbar_init(&o_full[t], 1);
      ptx::mbar_init(&o_free[t], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA
      constexpr int A = L::ATOMS;
      int n = 0;  // key block counter across items (K / V ring position)
      for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
        int qb, hp, b;
        decode(idx, qb, hp, b);
        const int h0 = 2 * hp, g = h0 / (d.nh / d.nkv), row0 = b * d.S;
        ptx::mbar_wait(q_empty, (li & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, 2 * L::Q);
        for (int t = 0; t < 2; ++t)
          for (int a = 0; a < A; ++a)
            ptx::tma_load_2d(&tm, q_full, sQ + t * L::Q + a * TILE, (h0 + t) * HD + 64 * a,
                             static_cast<int>(d.q_row_off) + row0 + qb * BQ);
        for (int j = 0; j <= qb; ++j, ++n) {
          const int s = n % NS;
          const uint32_t ph = ((n / NS) & 1) ^ 1;
          ptx::mbar_wait(&k_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&k_full[s], L::KV);
          for (int a = 0; a < A; ++a)
            ptx::tma_load_2d(&tm, &k_full[s], sK + s * L::KV + a * TILE, d.Q + g * HD + 64 * a,
                             row0 + j * BKV);
          ptx::mbar_wait(&v_empty[s], ph);
          ptx::mbar_arrive_expect_tx(&v_full[s], L::KV);
          for (int a = 0; a < A; ++a)
            ptx::tma_load_2d(&tm, &v_full[s], sV + s * L::KV + a * TILE,
                             d.Q + d.KV + g * HD + 64 * a, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA
      constexpr uint32_t idS = ptx::make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idO = ptx::make_idesc_bf16(BQ, HD, false, true);
      // S_t = Q_t K_n^T into the S_t columns
      auto issue_s = [&](int t, int n) {
        if (t == 0) {
          ptx::mbar_wait(&k_full[n % NS], (n / NS) & 1);
          ptx::tc_fence_after();
        }
        const uint32_t aQ = ptx::smem_u32(sQ + t * L::Q);
        const uint32_t aK = ptx::smem_u32(sK + (n % NS) * L::KV);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::umma_bf16(tmem + t * 128, kdesc(aQ, kk), kdesc(aK, kk), idS, kk > 0 ? 1u : 0u);
        ptx::umma_commit(&s_full[t]);
        if (t == 1) ptx::umma_commit(&k_empty[n % NS]);
      };
      int n = 0;
      for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
        int qb, hp, b;
        decode(idx, qb, hp, b);
        const int nkv = qb + 1;
        ptx::mbar_wait(q_full, li & 1);
        issue_s(0, n);
        issue_s(1, n);
        if (nkv == 1) ptx::umma_commit(q_empty);
        for (int j = 0; j < nkv; ++j, ++n) {
          ptx::mbar_wait(&v_full[n % NS], (n / NS) & 1);
          const uint32_t aV = ptx::smem_u32(sV + (n % NS) * L::KV);
          for (int t = 0; t < 2; ++t) {
            // O_t was last read by the epilogue of the previous item
            if (j == 0) ptx::mbar_wait(&o_free[t], (li & 1) ^ 1);
            ptx::mbar_wait(&p_full[t], n & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)
              umma_bf16_ta(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mndesc(aV, kk), idO,
                           (j > 0 || kk > 0) ? 1u : 0u);
            if (t == 1) ptx::umma_commit(&v_empty[n % NS]);
            if (j == nkv - 1) {
              ptx::umma_commit(&o_full[t]);
            } else {
              // S_{t,n+1} overwrites P_{t,n}: issued after PV_{t,n} (in-order pipe)
              issue_s(t, n + 1);
              if (t == 1 && j + 1 == nkv - 1) ptx::umma_commit(q_empty);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int tile = (warp - 2) >> 2;  // warpgroup = head of the pair
    const int quad = warp & 3;
    const int r = quad * 32 + lane;    // query row within the block (= TMEM lane)
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + tile * 128 + lane_off;
    const uint32_t tO = tmem + 256 + tile * 128 + lane_off;
    const uint8_t* sQt = sQ + tile * L::Q;
    const float sl2 = d.scale * kLog2e;
    const long long T = static_cast<long long>(d.B) * d.S;
    int n = 0;
    for (int li = 0, idx = blockIdx.x; idx < n_items; ++li, idx += gridDim.x) {
      int qb, hp, b;
      decode(idx, qb, hp, b);
      const int h = 2 * hp + tile, g = h / (d.nh / d.nkv), row0 = b * d.S;
      const int q = qb * BQ + r;
      const int nkv = qb + 1;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nkv; ++j, ++n) {
        ptx::mbar_wait(&s_full[tile], n & 1);
        ptx::tc_fence_after();
        uint32_t v[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x32(tS + c * 32, v[c]);
        ptx::tmem_ld_wait();
        const bool diag = j == qb;
        if (diag) {  // keys after the query are masked
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i > r) v[c][i] = __float_as_uint(-INFINITY);
        }
        float mxp[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            mxp[0] = ptx::max3f(mxp[0], __uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1]));
            mxp[1] =
                ptx::max3f(mxp[1], __uint_as_float(v[c][i + 2]), __uint_as_float(v[c][i + 3]));
            mxp[2] =
                ptx::max3f(mxp[2], __uint_as_float(v[c][i + 4]), __uint_as_float(v[c][i + 5]));
            mxp[3] =
                ptx::max3f(mxp[3], __uint_as_float(v[c][i + 6]), __uint_as_float(v[c][i + 7]));
          }
        const float mx = ptx::max3f(mxp[0], mxp[1], fmaxf(mxp[2], mxp[3])) * sl2;
        // lazy rescale (see attn_fwd_tc_kernel): only when the row max grows
        // by more than 2^8.  S_{t,n} complete implies PV_{t,n-1} complete.
        const bool need = mx > m_run + 8.f;
        float corr = 1.f;
        if (need) {
          corr = exp2f(m_run - mx);  // 0 on the first block
          l_run *= corr;
          m_run = mx;
        }
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          // 16-column pieces: the 128 scores stay live in registers meanwhile
#pragma unroll 1
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t o[16];
            tmem_ld_32x32b_x16(tO + c * 16, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st_32x32b_x16(tO + c * 16, o);
          }
        }
        // P = 2^(s * scale * log2e - m) -> packed bf16, written over S_t
        // columns [0, 64) in two 64-key halves
        const uint64_t scale2 = ptx::f32x2(sl2, sl2), negm2 = ptx::f32x2(-m_run, -m_run);
        uint64_t lp2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t pk[32];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hf + cc;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const bool poly = !diag && ((i >> 1) & 3) < SPECSIM_ATTN_POLY_PAIRS;
              const uint64_t x2 = ptx::ffma2(
                  ptx::f32x2(__uint_as_float(v[c][i]), __uint_as_float(v[c][i + 1])), scale2,
                  negm2);
              uint64_t p2;
              if (poly) {
                p2 = exp2_poly2(x2);
              } else {
                float x0, x1;
                ptx::f32x2_split(x2, x0, x1);
                p2 = ptx::f32x2(ptx::ex2_ftz(x0), ptx::ex2_ftz(x1));
              }
              lp2[(i >> 1) & 3] = ptx::fadd2(lp2[(i >> 1) & 3], p2);
              pk[cc * 16 + (i >> 1)] = ptx::pack_bf16x2_2(p2);
            }
          }
          tmem_st_32x32b_x32(tS + hf * 32, pk);
        }
        {
          float a0, a1;
          ptx::f32x2_split(ptx::fadd2(ptx::fadd2(lp2[0], lp2[1]), ptx::fadd2(lp2[2], lp2[3])),
                           a0, a1);
          l_run += a0 + a1;
        }
        tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[tile]);
      }
      // ---- epilogue of the item: O_t -> bf16 rows, lse
      ptx::mbar_wait(&o_full[tile], li & 1);
      ptx::tc_fence_after();
      float pd[kMaxDiag];
      float corr = 1.f;
      if (nd > 0) {  // training-time-test cache entries (see attn_fwd_tc_kernel)
        float mnew = m_run;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          const uint4* kr = reinterpret_cast<const uint4*>(
              d.diag_qkv + (static_cast<long long>(i + 1) * T + row0 + q) * d.NQ + d.Q + g * HD);
          float dot = 0.f;
#pragma unroll
          for (int c8 = 0; c8 < HD / 8; ++c8) {
            const uint4 qv = *reinterpret_cast<const uint4*>(
                sQt + (c8 >> 3) * TILE + r * 128 + (((c8 & 7) ^ (r & 7)) << 4));
            const uint4 kv = __ldg(kr + c8);
            dot += ptx::dot_bf16x8(qv, kv);
          }
          pd[i] = dot * sl2;
          mnew = fmaxf(mnew, pd[i]);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_empty);
        corr = exp2f(m_run - mnew);
        l_run *= corr;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          pd[i] = exp2f(pd[i] - mnew);
          l_run += pd[i];
        }
        m_run = mnew;
      }
      const float inv = 1.f / l_run;
      __nv_bfloat16* orow = out + static_cast<long long>(row0 + q) * d.Q + h * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(tO + c * 32, o);
        ptx::tmem_ld_wait();
        float acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(o[i]) * corr;
#pragma unroll 1
        for (int i = 0; i < nd; ++i) {
          const uint4* vr = reinterpret_cast<const uint4*>(
              d.diag_qkv + (static_cast<long long>(i + 1) * T + row0 + q) * d.NQ + d.Q + d.KV +
              g * HD + c * 32);
#pragma unroll
          for (int v8 = 0; v8 < 4; ++v8) {
            float vf[8];
            ptx::unpack_bf16x8(__ldg(vr + v8), vf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[v8 * 8 + e] += pd[i] * vf[e];
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          ptx::st_global_v4(orow + c * 32 + i, ptx::pack_bf16x2(acc[i] * inv, acc[i + 1] * inv),
                            ptx::pack_bf16x2(acc[i + 2] * inv, acc[i + 3] * inv),
                            ptx::pack_bf16x2(acc[i + 4] * inv, acc[i + 5] * inv),
                            ptx::pack_bf16x2(acc[i + 6] * inv, acc[i + 7] * inv));
      }
      // O_t read: the next item's first PV may overwrite it
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_free[tile]);
      lse[h * T + row0 + q] = (m_run + log2f(l_run)) * kLn2;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}


// ======================================================================
// Backward.  D = rowsum(dO * O) comes from attn_bwd_dot_kernel (attention.cu).
//
// dK / dV kernel: one CTA = (sample, KV head, 128-key block); loops over the
// query heads of the GQA group and every 64-query block at or after the key
// block.  Per block: S^T = K Q^T and dP^T = V dO^T (M = 128 keys, N = 64 q)
// into double-buffered TMEM; the "softmax" warps (one key row per thread)
// form P^T = exp2(S^T*scale*log2e - lse2) and dS^T = P^T (dP^T - D) as bf16
// K-major tiles in smem; then dV += P^T dO and dK += dS^T Q accumulate in
// TMEM (the Q / dO tiles double as MN-major B operands).
// Stores one dq / dk row (TMEM lane = row, HD fp32 columns at tm) scaled by
// sc as bf16.  With RoPE tables the row is first rounded to bf16 (the value
// the unfused path stores) and then inverse-rotated in registers:
// x1' = x1 c + x2 s, x2' = x2 c - x1 s.
// add (nullable): an fp32 row in the same (rotated, scaled) units, added
// before rounding (the training-time-test cache part of dq).
template <int HD>
__device__ __forceinline__ void store_grad_row(uint32_t tm, __nv_bfloat16* dst, float sc,
                                               const Dims& d, int pos,
                                               const float* __restrict__ add = nullptr) {
  constexpr int HALF = HD / 2;
  const long long L = d.rope_len > 0 ? d.rope_len : d.S;
  // rotation partners (i, i + HD/2) sit in chunks p and p + HD/64: process one
  // such pair of 32-column chunks at a time (64 live registers)
#pragma unroll
  for (int p = 0; p < HD / 64; ++p) {
    uint32_t a[32], b[32];
    ptx::tmem_ld_32x32b_x32(tm + p * 32, a);
    ptx::tmem_ld_32x32b_x32(tm + HALF + p * 32, b);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      a[i] = __float_as_uint(__uint_as_float(a[i]) * sc);
      b[i] = __float_as_uint(__uint_as_float(b[i]) * sc);
    }
    if (add != nullptr) {
      // 16-byte loads: a thread walks its own row (128 B per chunk)
      const float4* a4 = reinterpret_cast<const float4*>(add + p * 32);
      const float4* b4 = reinterpret_cast<const float4*>(add + HALF + p * 32);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 x = __ldg(a4 + i), y = __ldg(b4 + i);
        a[4 * i] = __float_as_uint(__uint_as_float(a[4 * i]) + x.x);
        a[4 * i + 1] = __float_as_uint(__uint_as_float(a[4 * i + 1]) + x.y);
        a[4 * i + 2] = __float_as_uint(__uint_as_float(a[4 * i + 2]) + x.z);
        a[4 * i + 3] = __float_as_uint(__uint_as_float(a[4 * i + 3]) + x.w);
        b[4 * i] = __float_as_uint(__uint_as_float(b[4 * i]) + y.x);
        b[4 * i + 1] = __float_as_uint(__uint_as_float(b[4 * i + 1]) + y.y);
        b[4 * i + 2] = __float_as_uint(__uint_as_float(b[4 * i + 2]) + y.z);
        b[4 * i + 3] = __float_as_uint(__uint_as_float(b[4 * i + 3]) + y.w);
      }
    }
    if (d.rope_cos != nullptr) {
      const float* cs = d.rope_cos + static_cast<long long>(p * 32) * L + pos;
      const float* sn = d.rope_sin + static_cast<long long>(p * 32) * L + pos;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float cv = __ldg(cs + static_cast<long long>(i) * L);
        const float sv = __ldg(sn + static_cast<long long>(i) * L);
        const float x1 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(a[i])));
        const float x2 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(b[i])));
        a[i] = __float_as_uint(x1 * cv + x2 * sv);
        b[i] = __float_as_uint(x2 * cv - x1 * sv);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t* o = h ? b : a;
      __nv_bfloat16* out = dst + h * HALF + p * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        ptx::st_global_v4(
            out + i, ptx::pack_bf16x2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])),
            ptx::pack_bf16x2(__uint_as_float(o[i + 2]), __uint_as_float(o[i + 3])),
            ptx::pack_bf16x2(__uint_as_float(o[i + 4]), __uint_as_float(o[i + 5])),
            ptx::pack_bf16x2(__uint_as_float(o[i + 6]), __uint_as_float(o[i + 7])));
    }
  }
}

constexpr int BQB = 64;               // query block of the dK/dV kernel
constexpr int TILE64 = BQB * 64 * 2;  // [64 x 64] bf16 SW128 tile = 8 KB

// Q / dO / (lse, D) stream in a 3-deep ring: the stage of iteration it is
// refilled only after the dV / dK MMAs of it complete, and the S^T MMA of
// it + 2 is issued right after those -- with two stages that TMA latency
// sat on the critical path of every iteration.
constexpr int KV_QSTAGES = 3;
template <int HD>
struct KvSmem {
  static constexpr int ATOMS = HD / 64;
  static constexpr int KV = ATOMS * TILE;       // [128 keys x HD]
  static constexpr int QT = ATOMS * TILE64;     // [64 q x HD]
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV;
  static constexpr int OFF_Q = OFF_V + KV;                    // KV_QSTAGES stages
  static constexpr int OFF_DO = OFF_Q + KV_QSTAGES * QT;      // KV_QSTAGES stages
  static constexpr int OFF_P = OFF_DO + KV_QSTAGES * QT;      // 2 x [128 keys x 64 q]
  static constexpr int OFF_DS = OFF_P + 2 * TILE;
  static constexpr int OFF_LD = OFF_DS + 2 * TILE;  // stages x (lse[64], D[64]) fp32
  static constexpr int OFF_BAR = OFF_LD + KV_QSTAGES * 2 * BQB * 4;
  static constexpr int BYTES = 1024 + OFF_BAR + 256;
};

__device__ __forceinline__ uint64_t kdesc64(uint32_t base, int kk) {
  return ptx::make_sw128_desc(base + (kk >> 2) * TILE64 + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc64(uint32_t base, int kk) {
  return ptx::make_sw128_desc(base + kk * 2048, TILE64, 1024);
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_bwd_kv_tc_kernel(const __grid_constant__ CUtensorMap tm_kv,  // qkv, box {64,128}
                          const __grid_constant__ CUtensorMap tm_q,   // qkv, box {64,64}
                          const __grid_constant__ CUtensorMap tm_do,  // dO,  box {64,64}
                          const float* __restrict__ lse, const float* __restrict__ Dv,
                          __nv_bfloat16* __restrict__ dqkv, Dims d, int n_steps) {
  using L = KvSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  constexpr int QS = KV_QSTAGES;
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;        // [QS]
  uint64_t* qd_empty = bar + 1 + QS;  // [QS]
  uint64_t* s_full = bar + 1 + 2 * QS;   // [2]
  uint64_t* s_free = bar + 3 + 2 * QS;   // [2]
  uint64_t* p_full = bar + 5 + 2 * QS;   // [2]
  uint64_t* p_free = bar + 7 + 2 * QS;   // [2]
  uint64_t* all_done = bar + 9 + 2 * QS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10 + 2 * QS);
  float* sLD = reinterpret_cast<float*>(smem + L::OFF_LD);

  // key block on the slowest grid axis: CTAs are dispatched in launch order,
  // so every early key block (the most queries, up to 16x the work of the
  // last) starts in the first waves instead of some of them forming the tail
  const int kb = blockIdx.z;
  const int g = blockIdx.x, b = blockIdx.y;
  const int rep = d.nh / d.nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * d.S;
  const long long T = static_cast<long long>(d.B) * d.S;
  const int qb0 = kb * (BKV / BQB), nqb = d.S / BQB;
  const int per_head = nqb - qb0;
  const int per_step = rep * per_head;  // (query head, 64-query block) pairs of one unroll step
  const int n_it = n_steps * per_step;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_kv);
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < QS; ++i) {
      ptx::mbar_init(&qd_full[i], 1);
      ptx::mbar_init(&qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&p_free[i], 1);
    }
    ptx::mbar_init(all_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdV = tmem, tdK = tmem + HD;
  const uint32_t tSt[2] = {tmem + 2 * HD, tmem + 2 * HD + 64};
  const uint32_t tdPt[2] = {tmem + 2 * HD + 128, tmem + 2 * HD + 192};

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA
      constexpr int A = L::ATOMS;
      ptx::mbar_arrive_expect_tx(kv_full, 2 * L::KV);
      for (int a = 0; a < A; ++a) {
        ptx::tma_load_2d(&tm_kv, kv_full, smem + L::OFF_K + a * TILE, d.Q + g * HD + 64 * a,
                         row0 + kb * BKV);
        ptx::tma_load_2d(&tm_kv, kv_full, smem + L::OFF_V + a * TILE,
                         d.Q + d.KV + g * HD + 64 * a, row0 + kb * BKV);
      }
      for (int it = 0; it < n_it; ++it) {
        const int st = it % QS;
        const uint32_t ph = (it / QS) & 1;
        const int step = it / per_step, rem = it % per_step;
        const int h = g * rep + rem / per_head;
        const int q0 = (qb0 + rem % per_head) * BQB;
        const int qrow = static_cast<int>(step * T) + row0 + q0;
        const long long li = (static_cast<long long>(step) * d.nh + h) * T + row0 + q0;
        ptx::mbar_wait(&qd_empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&qd_full[st], 2 * L::QT + 2 * BQB * 4);
        for (int a = 0; a < A; ++a) {
          ptx::tma_load_2d(&tm_q, &qd_full[st], smem + L::OFF_Q + st * L::QT + a * TILE64,
                           h * HD + 64 * a, qrow);
          ptx::tma_load_2d(&tm_do, &qd_full[st], smem + L::OFF_DO + st * L::QT + a * TILE64,
                           h * HD + 64 * a, qrow);
        }
        ptx::bulk_load(sLD + st * 2 * BQB, lse + li, BQB * 4, &qd_full[st]);
        ptx::bulk_load(sLD + st * 2 * BQB + BQB, Dv + li, BQB * 4, &qd_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA
      constexpr uint32_t idS = ptx::make_idesc_bf16(BKV, BQB, false, false);
      constexpr uint32_t idG = ptx::make_idesc_bf16(BKV, HD, false, true);
      const uint32_t aK = ptx::smem_u32(smem + L::OFF_K), aV = ptx::smem_u32(smem + L::OFF_V);
      auto issue_s = [&](int it) {
        const int qs = it % QS, sb = it & 1;  // Q / dO stage, TMEM S^T / dP^T buffer
        ptx::mbar_wait(&qd_full[qs], (it / QS) & 1);
        ptx::mbar_wait(&s_free[sb], ((it >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t aQ = ptx::smem_u32(smem + L::OFF_Q + qs * L::QT);
        const uint32_t adO = ptx::smem_u32(smem + L::OFF_DO + qs * L::QT);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          ptx::umma_bf16(tSt[sb], kdesc(aK, kk), kdesc64(aQ, kk), idS, kk > 0 ? 1u : 0u);
          ptx::umma_bf16(tdPt[sb], kdesc(aV, kk), kdesc64(adO, kk), idS, kk > 0 ? 1u : 0u);
        }
        ptx::umma_commit(&s_full[sb]);
      };
      ptx::mbar_wait(kv_full, 0);
      issue_s(0);
      for (int it = 0; it < n_it; ++it) {
        if (it + 1 < n_it) issue_s(it + 1);
        const int st = it & 1, qs = it % QS;  // P / dS buffer, Q / dO stage
        ptx::mbar_wait(&p_full[st], (it >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aP = ptx::smem_u32(smem + L::OFF_P + st * TILE);
        const uint32_t aS = ptx::smem_u32(smem + L::OFF_DS + st * TILE);
        const uint32_t aQ = ptx::smem_u32(smem + L::OFF_Q + qs * L::QT);
        const uint32_t adO = ptx::smem_u32(smem + L::OFF_DO + qs * L::QT);
#pragma unroll
        for (int kk = 0; kk < BQB / 16; ++kk) {
          ptx::umma_bf16(tdV, kdesc(aP, kk), mndesc64(adO, kk), idG, (it > 0 || kk > 0) ? 1u : 0u);
          ptx::umma_bf16(tdK, kdesc(aS, kk), mndesc64(aQ, kk), idG, (it > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&p_free[st]);
        ptx::umma_commit(&qd_empty[qs]);
      }
      ptx::umma_commit(all_done);
    }
  } else {
    // ------------------------------------------------------------ P^T / dS^T
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // key row within the block (TMEM lane)
    const int key = kb * BKV + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float sl2 = d.scale * kLog2e;
    for (int it = 0; it < n_it; ++it) {
      const int st = it & 1;
      const int q0 = (qb0 + (it % per_step) % per_head) * BQB;
      ptx::mbar_wait(&s_full[st], (it >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t sv[2][32], pv[2][32];
#if SPECSIM_ATTN_PROBE == 2  // probe: no TMEM reads (timing experiments only)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c][i] = pv[c][i] = __float_as_uint(0.01f * i);
#else
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        ptx::tmem_ld_32x32b_x32(tSt[st] + lane_off + c * 32, sv[c]);
        ptx::tmem_ld_32x32b_x32(tdPt[st] + lane_off + c * 32, pv[c]);
      }
      ptx::tmem_ld_wait();
#endif
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&s_free[st]);
      // lse / D slices arrived with this stage's TMA bytes: observe that
      // barrier directly (cannot have advanced: the stage is only refilled
      // after the dV/dK MMAs that need this iteration's P / dS)
      const int qs = it % QS;
      ptx::mbar_wait(&qd_full[qs], (it / QS) & 1);
      const float* l2 = sLD + qs * 2 * BQB;
      const float* Dq = l2 + BQB;
      // the P / dS smem buffer of this stage is free once the MMAs of it-2 ran
      ptx::mbar_wait(&p_free[st], ((it >> 1) & 1) ^ 1);
      uint8_t* sP = smem + L::OFF_P + st * TILE;
      uint8_t* sS = smem + L::OFF_DS + st * TILE;
      // causal mask only where this 64-query block crosses the key block's
      // diagonal (warp-uniform test); packed fp32x2 arithmetic and ftz ex2:
      // P = 2^(s * scale * log2e - lse * log2e), dS = P (dP - D)
      const bool masked = q0 < kb * BKV + BKV;
      const uint64_t sl2x2 = ptx::f32x2(sl2, sl2), nlog2e = ptx::f32x2(-kLog2e, -kLog2e);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t pp[4], dd[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const int qi = c * 32 + i + e;
            const float2 lq = *reinterpret_cast<const float2*>(l2 + qi);
            const float2 dq = *reinterpret_cast<const float2*>(Dq + qi);
            const uint64_t x = ptx::ffma2(
                ptx::f32x2(__uint_as_float(sv[c][i + e]), __uint_as_float(sv[c][i + e + 1])),
                sl2x2, ptx::fmul2(ptx::f32x2(lq.x, lq.y), nlog2e));
            float x0, x1;
            ptx::f32x2_split(x, x0, x1);
#if SPECSIM_ATTN_PROBE == 1  // probe: no MUFU (timing experiments only)
            float p0 = x0, p1 = x1;
#else
            float p0 = ptx::ex2_ftz(x0), p1 = ptx::ex2_ftz(x1);
#endif
            if (masked) {  // causal: query before key
              if (q0 + qi < key) p0 = 0.f;
              if (q0 + qi + 1 < key) p1 = 0.f;
            }
            const uint64_t p2 = ptx::f32x2(p0, p1);
            const uint64_t ds2 = ptx::fmul2(
                p2, ptx::fadd2(ptx::f32x2(__uint_as_float(pv[c][i + e]),
                                          __uint_as_float(pv[c][i + e + 1])),
                               ptx::f32x2(-dq.x, -dq.y)));
            pp[e >> 1] = ptx::pack_bf16x2_2(p2);
            dd[e >> 1] = ptx::pack_bf16x2_2(ds2);
          }
          const int cc = (c * 32 + i) >> 3;  // 16-byte chunk within the 128-byte row
          const int off = r * 128 + ((cc ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(sP + off) = make_uint4(pp[0], pp[1], pp[2], pp[3]);
          *reinterpret_cast<uint4*>(sS + off) = make_uint4(dd[0], dd[1], dd[2], dd[3]);
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[st]);
    }
    // epilogue: dV, dK (x scale) rows -> dqkv
    ptx::mbar_wait(all_done, 0);
    ptx::tc_fence_after();
    __nv_bfloat16* kp = dqkv + static_cast<long long>(row0 + key) * d.NQ + d.Q + g * HD;
    __nv_bfloat16* vp = kp + d.KV;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t o[32];
      ptx::tmem_ld_32x32b_x32(tdV + lane_off + c * 32, o);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        ptx::st_global_v4(vp + c * 32 + i,
                          ptx::pack_bf16x2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 2]), __uint_as_float(o[i + 3])),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 4]), __uint_as_float(o[i + 5])),
                          ptx::pack_bf16x2(__uint_as_float(o[i + 6]), __uint_as_float(o[i + 7])));
    }
    store_grad_row<HD>(tdK + lane_off, kp, d.scale, d, (row0 + key) % d.S + d.pos_off);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// dQ kernel: one CTA = (sample, query head, 128-query block); loops over the
// key blocks up to the diagonal.  S = Q K^T and dP = dO V^T (M = 128 q,
// N = 128 keys) into TMEM; dS = P (dP - D) written back over S as packed bf16
// (tcgen05.st); then dQ += dS K with dS as the TMEM A operand and the K tile
// doubling as an MN-major B operand.
template <int HD>
struct QSmem {
  static constexpr int ATOMS = HD / 64;
  static constexpr int T128 = ATOMS * TILE;  // [128 x HD]
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = OFF_Q + T128;
  static constexpr int OFF_K = OFF_DO + T128;   // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * T128;  // 2 stages
  static constexpr int OFF_BAR = OFF_V + 2 * T128;
  static constexpr int BYTES = 1024 + OFF_BAR + 256;
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_bwd_q_tc_kernel(const __grid_constant__ CUtensorMap tm_kv,  // qkv, box {64,128}
                         const __grid_constant__ CUtensorMap tm_do,  // dO,  box {64,128}
                         const float* __restrict__ lse, const float* __restrict__ Dv,
                         const float* __restrict__ dq_add, __nv_bfloat16* __restrict__ dqkv,
                         Dims d) {
  using L = QSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* ds_full = bar + 7;  // (bar + 6, bar + 8 unused)
  uint64_t* all_done = bar + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

  // query block on the slowest grid axis, most keys first (see the dK/dV kernel)
  const int qb = gridDim.z - 1 - blockIdx.z;
  const int h = blockIdx.x, b = blockIdx.y;
  const int g = h / (d.nh / d.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * d.S;
  const int nkv = qb + 1;
  const long long T = static_cast<long long>(d.B) * d.S;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_kv);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(ds_full, 4);
    ptx::mbar_init(all_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S is double-buffered (columns 128 and 384): S_{j+1} is computed while the
  // softmax warps turn S_j / dP_j into dS_j, off the per-block critical path
  const uint32_t tdQ = tmem, tS = tmem + 128, tdP = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      constexpr int A = L::ATOMS;
      ptx::mbar_arrive_expect_tx(q_full, 2 * L::T128);
      for (int a = 0; a < A; ++a) {
        ptx::tma_load_2d(&tm_kv, q_full, smem + L::OFF_Q + a * TILE, h * HD + 64 * a,
                         static_cast<int>(d.q_row_off) + row0 + qb * BQ);
        ptx::tma_load_2d(&tm_do, q_full, smem + L::OFF_DO + a * TILE, h * HD + 64 * a,
                         row0 + qb * BQ);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        ptx::mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&k_full[st], 2 * L::T128);
        for (int a = 0; a < A; ++a) {
          ptx::tma_load_2d(&tm_kv, &k_full[st], smem + L::OFF_K + st * L::T128 + a * TILE,
                           d.Q + g * HD + 64 * a, row0 + j * BKV);
          ptx::tma_load_2d(&tm_kv, &k_full[st], smem + L::OFF_V + st * L::T128 + a * TILE,
                           d.Q + d.KV + g * HD + 64 * a, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = ptx::make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idQ = ptx::make_idesc_bf16(BQ, HD, false, true);
      const uint32_t aQ = ptx::smem_u32(smem + L::OFF_Q), adO = ptx::smem_u32(smem + L::OFF_DO);
      ptx::mbar_wait(q_full, 0);
      // S_j into buffer j & 1; that buffer last held S_{j-2}, released by the
      // s_free of block j-2, which issuing dP_{j-1} already waited for
      auto issue_s = [&](int j) {
        const int st = j & 1;
        ptx::mbar_wait(&k_full[st], (j >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t aK = ptx::smem_u32(smem + L::OFF_K + st * L::T128);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::umma_bf16(tS + (j & 1) * 256, kdesc(aQ, kk), kdesc(aK, kk), idS, kk > 0 ? 1u : 0u);
      };
      // dP_j into the single dP buffer (free once the softmax of j-1 is done:
      // the caller has waited ds_full of j-1), then the S_j / dP_j commit
      auto issue_dp = [&](int j) {
        const uint32_t aV = ptx::smem_u32(smem + L::OFF_V + (j & 1) * L::T128);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ptx::umma_bf16(tdP, kdesc(adO, kk), kdesc(aV, kk), idS, kk > 0 ? 1u : 0u);
        ptx::umma_commit(s_full);  // S_j and dP_j
      };
      issue_s(0);
      issue_dp(0);
      if (nkv > 1) issue_s(1);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        ptx::mbar_wait(ds_full, j & 1);  // softmax of j done: dP, S_j buffer, dS_j written
        ptx::tc_fence_after();
        // dP_{j+1} first, so the softmax of j+1 starts while dQ_j runs
        if (j + 1 < nkv) issue_dp(j + 1);
        const uint32_t aK = ptx::smem_u32(smem + L::OFF_K + st * L::T128);
        // dS_j (bf16, packed over the first 64 columns of S_j's TMEM buffer)
        // is the A operand; S_{j+2} overwrites it only after these MMAs (one
        // issuer's MMAs run in order)
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          umma_bf16_ta(tdQ, tS + (j & 1) * 256 + kk * 8, mndesc(aK, kk), idQ,
                       (j > 0 || kk > 0) ? 1u : 0u);
        ptx::umma_commit(&k_empty[st]);
        // S_{j+2} reuses S_j's buffer and K stage j & 1 (refilled once dQ_j is done)
        if (j + 2 < nkv) issue_s(j + 2);
      }
      ptx::umma_commit(all_done);
    }
  } else {
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int q = qb * BQ + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float sl2 = d.scale * kLog2e;
    const float l2 = lse[h * T + row0 + q] * kLog2e;
    const float Dr = Dv[h * T + row0 + q];
    const uint64_t sl2x2 = ptx::f32x2(sl2, sl2), nl2x2 = ptx::f32x2(-l2, -l2),
                   nD2 = ptx::f32x2(-Dr, -Dr);
    for (int j = 0; j < nkv; ++j) {
      ptx::mbar_wait(s_full, j & 1);
      ptx::tc_fence_after();
      const bool diag = (j == qb);
      const uint32_t tSj = tS + (j & 1) * 256 + lane_off;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32], pv[32];
        ptx::tmem_ld_32x32b_x32(tSj + c * 32, sv);
        ptx::tmem_ld_32x32b_x32(tdP + lane_off + c * 32, pv);
        ptx::tmem_ld_wait();
        uint32_t ddc[4][4];
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t* dd = ddc[i >> 3];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const int kcol = c * 32 + i + e;
            // P = 2^(s * scale * log2e - lse * log2e), dS = P (dP - D): packed fp32x2
            const uint64_t x = ptx::ffma2(
                ptx::f32x2(__uint_as_float(sv[i + e]), __uint_as_float(sv[i + e + 1])), sl2x2,
                nl2x2);
            float x0, x1;
            ptx::f32x2_split(x, x0, x1);
            float p0 = ptx::ex2_ftz(x0), p1 = ptx::ex2_ftz(x1);
            if (diag) {
              if (kcol > r) p0 = 0.f;
              if (kcol + 1 > r) p1 = 0.f;
            }
            dd[e >> 1] = ptx::pack_bf16x2_2(ptx::fmul2(
                ptx::f32x2(p0, p1),
                ptx::fadd2(ptx::f32x2(__uint_as_float(pv[i + e]), __uint_as_float(pv[i + e + 1])),
                           nD2)));
          }
        }
        // dS chunk c (32 keys -> 16 packed columns) over S_j's columns
        // [16 c, 16 c + 16): this chunk's S values are already in registers and
        // later chunks read columns >= 32 (c + 1) > 16 c + 16
        uint32_t dsw[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) dsw[i] = ddc[i >> 2][i & 3];
        tmem_st_32x32b_x16(tSj + c * 16, dsw);
      }
      tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ds_full);  // also frees dP for the MMA warp
    }
    ptx::mbar_wait(all_done, 0);
    ptx::tc_fence_after();
    __nv_bfloat16* qp = dqkv + static_cast<long long>(row0 + q) * d.NQ + h * HD;
    const float* addp =
        dq_add ? dq_add + static_cast<long long>(row0 + q) * d.Q + h * HD : nullptr;
    store_grad_row<HD>(tdQ + lane_off, qp, d.scale, d, (row0 + q) % d.S + d.pos_off, addp);
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
  // persistent: one CTA per SM (SPECSIM_ATTN_FWD_GRID=items: one per work item)
  static const bool per_item = [] {
    const char* e = std::getenv("SPECSIM_ATTN_FWD_GRID");
    return e && std::string(e) == "items";
  }();
  // two query tiles (a head pair of one KV group) per CTA unless the GQA
  // group is odd (SPECSIM_ATTN_FWD1=1: the one-tile kernel)
  static const bool one_tile = [] {
    const char* e = std::getenv("SPECSIM_ATTN_FWD1");
    return e && e[0] == '1';
  }();
  int dev = 0, sms = 0;
  SPECSIM_CUDA(cudaGetDevice(&dev));
  SPECSIM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (!one_tile && !per_item && (d.nh / d.nkv) % 2 == 0) {
    constexpr int smem2 = Fwd2Smem<HD>::BYTES;
    static_assert(smem2 <= 232448, "attention smem budget");
    static bool init2 = false;
    if (!init2) {
      SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd2_tc_kernel<HD>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      init2 = true;
    }
    const int n_items2 = (d.S / BQ) * (d.nh / 2) * d.B;
    count_launches();
    attn_fwd2_tc_kernel<HD><<<std::min(n_items2, sms), 320, smem2, s>>>(tm, o, lse, d);
    return;
  }
  const int n_items = (d.S / BQ) * d.nh * d.B;
  const int grid = per_item ? n_items : std::min(n_items, sms);
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

namespace {
// ---------------------------------------------------------------------------
// Training-time-test cache entries of the backward (unroll step j >= 1), on
// CUDA cores: one warp per (row t, KV head g), lanes hold HD/32 consecutive
// columns.  For each query head of the group and each earlier step i <= j:
// p = exp(q.k_i*scale - lse), ds = p (dO.v_i - D) scale; dq += ds k_i,
// dk_i += ds q, dv_i += p dO (fp32 accumulators, fixed order: deterministic).
template <int HD, int kMaxRep>
__global__ void __launch_bounds__(256) attn_bwd_diag_kernel(
    const __nv_bfloat16* __restrict__ qkv_all, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ Dv, float* __restrict__ dq_add,
    float* __restrict__ dkv_acc, __nv_bfloat16* __restrict__ dqkv_step, Dims d) {
  constexpr int E = HD / 32;
  const long long T = static_cast<long long>(d.B) * d.S;
  const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= T * d.nkv) return;
  const long long t = w / d.nkv;
  const int g = static_cast<int>(w % d.nkv);
  const int rep = d.nh / d.nkv, j = d.n_diag;
  const int c0 = lane * E;
  const long long KV2 = 2ll * d.KV;
  auto ld = [](const __nv_bfloat16* p, float (&f)[E]) {
#pragma unroll
    for (int e = 0; e < E; ++e) f[e] = __bfloat162float(p[e]);
  };
  auto wsum = [](float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  // the group's q / dO rows live in registers (rep * 2E floats); every cache
  // entry i is loaded once and its dk / dv accumulated over the group before
  // one read-modify-write of the fp32 accumulator (kMaxRep >= rep: the
  // smallest power of two, so register use follows the GQA group)
  float q[kMaxRep][E], dO[kMaxRep][E], dq[kMaxRep][E], l[kMaxRep], Dh[kMaxRep];
#pragma unroll
  for (int hh = 0; hh < kMaxRep; ++hh) {
    if (hh >= rep) break;
    const int h = g * rep + hh;
    ld(qkv_all + (static_cast<long long>(j) * T + t) * d.NQ + h * HD + c0, q[hh]);
    ld(dout + t * d.Q + h * HD + c0, dO[hh]);
    l[hh] = lse[h * T + t];
    Dh[hh] = Dv[h * T + t];
#pragma unroll
    for (int e = 0; e < E; ++e) dq[hh][e] = 0.f;
  }
  for (int i = 1; i <= j; ++i) {
    const __nv_bfloat16* kr = qkv_all + (static_cast<long long>(i) * T + t) * d.NQ + d.Q + g * HD;
    float k[E], v[E], dk[E], dv[E];
    ld(kr + c0, k);
    ld(kr + d.KV + c0, v);
#pragma unroll
    for (int e = 0; e < E; ++e) dk[e] = dv[e] = 0.f;
#pragma unroll
    for (int hh = 0; hh < kMaxRep; ++hh) {
      if (hh >= rep) break;
      float sd = 0.f, sp = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        sd += q[hh][e] * k[e];
        sp += dO[hh][e] * v[e];
      }
      sd = wsum(sd);
      sp = wsum(sp);
      const float p = __expf(sd * d.scale - l[hh]);
      const float ds = p * (sp - Dh[hh]) * d.scale;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        dq[hh][e] += ds * k[e];
        dk[e] += ds * q[hh][e];
        dv[e] += p * dO[hh][e];
      }
    }
    float* acc = dkv_acc + (static_cast<long long>(i) * T + t) * KV2 + g * HD + c0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      acc[e] += dk[e];
      acc[d.KV + e] += dv[e];
    }
  }
#pragma unroll
  for (int hh = 0; hh < kMaxRep; ++hh) {
    if (hh >= rep) break;
    float* dqa = dq_add + t * d.Q + (g * rep + hh) * HD + c0;
#pragma unroll
    for (int e = 0; e < E; ++e) dqa[e] = dq[hh][e];
  }
  // step j's k / v receive no further contributions: round, inverse-rotate
  // k (position t % S + j; partner column c +- HD/2 lives 16 lanes away),
  // round, store into the GEMM operand
  const float* acc = dkv_acc + (static_cast<long long>(j) * T + t) * KV2 + g * HD + c0;
  __nv_bfloat16* kd = dqkv_step + t * d.NQ + d.Q + g * HD + c0;
  const long long L = d.rope_len > 0 ? d.rope_len : d.S;
  const int pos = static_cast<int>(t % d.S) + j;
  const bool lo = lane < 16;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float x = __bfloat162float(__float2bfloat16_rn(acc[e]));
    const float y = __shfl_xor_sync(0xffffffffu, x, 16);
    float r = x;
    if (d.rope_cos != nullptr) {
      const int i = (lane & 15) * E + e;  // rotation index in [0, HD/2)
      const float cv = __ldg(d.rope_cos + i * L + pos), sv = __ldg(d.rope_sin + i * L + pos);
      r = lo ? x * cv + y * sv : x * cv - y * sv;  // lo: x1' = x1 c + x2 s; hi: x2' = x2 c - x1 s
    }
    kd[e] = __float2bfloat16_rn(r);
    kd[d.KV + e] = __float2bfloat16_rn(acc[d.KV + e]);
  }
}

}  // namespace

template <int HD>
void bwd_dq_t(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout, const float* lse,
              const float* D, const float* dq_add, __nv_bfloat16* dqkv_step, const Dims& d,
              cudaStream_t s) {
  const long long T = static_cast<long long>(d.B) * d.S;
  const CUtensorMap kv = gemm::make_tensor_map(qkv_all, d.q_row_off + T, d.NQ, d.NQ, 64, 128);
  const CUtensorMap do128 = gemm::make_tensor_map(dout, T, d.Q, d.Q, 64, 128);
  count_launches();
  attn_bwd_q_tc_kernel<HD><<<dim3(d.nh, d.B, d.S / BQ), 192, QSmem<HD>::BYTES, s>>>(
      kv, do128, lse, D, dq_add, dqkv_step, d);
}

template <int HD>
void bwd_dkdv_t(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout_all, const float* lse_all,
                const float* D_all, __nv_bfloat16* dqkv0, const Dims& d, int n_steps,
                cudaStream_t s) {
  const long long T = static_cast<long long>(d.B) * d.S;
  const CUtensorMap kv = gemm::make_tensor_map(qkv_all, T, d.NQ, d.NQ, 64, 128);
  const CUtensorMap q64 = gemm::make_tensor_map(qkv_all, n_steps * T, d.NQ, d.NQ, 64, 64);
  const CUtensorMap do64 = gemm::make_tensor_map(dout_all, n_steps * T, d.Q, d.Q, 64, 64);
  count_launches();
  attn_bwd_kv_tc_kernel<HD><<<dim3(d.nkv, d.B, d.S / BKV), 192, KvSmem<HD>::BYTES, s>>>(
      kv, q64, do64, lse_all, D_all, dqkv0, d, n_steps);
}

void backward_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse,
                 const float* Dbuf, __nv_bfloat16* dqkv, const Dims& d, int hd, cudaStream_t s) {
  if (hd == 128) {
    bwd_dkdv_t<128>(qkv, dout, lse, Dbuf, dqkv, d, 1, s);
    bwd_dq_t<128>(qkv, dout, lse, Dbuf, nullptr, dqkv, d, s);
  } else {
    bwd_dkdv_t<64>(qkv, dout, lse, Dbuf, dqkv, d, 1, s);
    bwd_dq_t<64>(qkv, dout, lse, Dbuf, nullptr, dqkv, d, s);
  }
}

void bwd_diag(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout, const float* lse,
              const float* D, float* dq_add, float* dkv_acc, __nv_bfloat16* dqkv_step,
              const Dims& d, int hd, cudaStream_t s) {
  if (d.n_diag < 1 || d.n_diag > kMaxDiag)
    throw std::invalid_argument("bwd_diag: n_diag must be in [1, 15]");
  if (d.nh / d.nkv > 16) throw std::invalid_argument("bwd_diag: GQA group must be <= 16");
  const long long warps = static_cast<long long>(d.B) * d.S * d.nkv;
  const unsigned blocks = static_cast<unsigned>((warps * 32 + 255) / 256);
  count_launches();
  const int rep = d.nh / d.nkv;
#define SPECSIM_DIAG(HD_, R_)                                                                  \
  attn_bwd_diag_kernel<HD_, R_><<<blocks, 256, 0, s>>>(qkv_all, dout, lse, D, dq_add, dkv_acc, \
                                                       dqkv_step, d)
#define SPECSIM_DIAG_HD(HD_)        \
  if (rep <= 1)                     \
    SPECSIM_DIAG(HD_, 1);           \
  else if (rep <= 2)                \
    SPECSIM_DIAG(HD_, 2);           \
  else if (rep <= 4)                \
    SPECSIM_DIAG(HD_, 4);           \
  else if (rep <= 8)                \
    SPECSIM_DIAG(HD_, 8);           \
  else                              \
    SPECSIM_DIAG(HD_, 16);
  if (hd == 128) {
    SPECSIM_DIAG_HD(128)
  } else {
    SPECSIM_DIAG_HD(64)
  }
#undef SPECSIM_DIAG_HD
#undef SPECSIM_DIAG
}

void bwd_dq(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout, const float* lse,
            const float* D, const float* dq_add, __nv_bfloat16* dqkv_step, const Dims& d, int hd,
            cudaStream_t s) {
  if (d.S % BQ) throw std::invalid_argument("bwd_dq: seq_len must be a multiple of 128");
  if (hd == 128)
    bwd_dq_t<128>(qkv_all, dout, lse, D, dq_add, dqkv_step, d, s);
  else
    bwd_dq_t<64>(qkv_all, dout, lse, D, dq_add, dqkv_step, d, s);
}

void bwd_dkdv(const __nv_bfloat16* qkv_all, const __nv_bfloat16* dout_all, const float* lse_all,
              const float* D_all, __nv_bfloat16* dqkv0, const Dims& d, int hd, int n_steps,
              cudaStream_t s) {
  if (d.S % BKV) throw std::invalid_argument("bwd_dkdv: seq_len must be a multiple of 128");
  if (hd == 128)
    bwd_dkdv_t<128>(qkv_all, dout_all, lse_all, D_all, dqkv0, d, n_steps, s);
  else
    bwd_dkdv_t<64>(qkv_all, dout_all, lse_all, D_all, dqkv0, d, n_steps, s);
}

template <int HD>
void prepare_bwd_t() {
  static_assert(KvSmem<HD>::BYTES <= 232448 && QSmem<HD>::BYTES <= 232448, "smem budget");
  SPECSIM_CUDA(cudaFuncSetAttribute(attn_bwd_kv_tc_kernel<HD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    KvSmem<HD>::BYTES));
  SPECSIM_CUDA(cudaFuncSetAttribute(attn_bwd_q_tc_kernel<HD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, QSmem<HD>::BYTES));
}

void prepare_tc(int hd) {
  if (hd == 128)
    prepare_bwd_t<128>();
  else
    prepare_bwd_t<64>();
  if (hd == 128) {
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<128>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      FwdSmem<128>::BYTES));
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd2_tc_kernel<128>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Fwd2Smem<128>::BYTES));
  } else {
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<64>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      FwdSmem<64>::BYTES));
    SPECSIM_CUDA(cudaFuncSetAttribute(attn_fwd2_tc_kernel<64>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Fwd2Smem<64>::BYTES));
  }
}

}  // namespace attn
}  // namespace specsim
