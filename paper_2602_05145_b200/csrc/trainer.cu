// DraftTrainer: the real body behind the reference's analytic train()
// (SPEC.md:380-405).  One optimiser step = gather the micro-batch from the
// signal ring, forward the EAGLE-3 style draft head, fused
// vocabulary-chunked LM-head cross-entropy, backward, optional NCCL gradient
// all-reduce across data-parallel ranks, fused AdamW.
//
// Every dense contraction runs on the tcgen05 GEMM (gemm.cuh); the plans
// (tensor maps, shapes, epilogues) are built once here, so a step is a fixed
// sequence of launches on one stream.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "attention.h"
#include "bookkeeping.h"
#include "common.h"
#include "handles.h"
#include "gemm.h"
#include "kernels.h"
#include "nccl_dyn.h"
#include "specsim/draft_trainer.hpp"

namespace specsim {

namespace {

#define SPECSIM_NCCL(call)                                                              \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess)                                                              \
      throw NcclError(std::string(#call) + ": " + nccl::api().GetErrorString(_r));      \
  } while (0)

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    SPECSIM_CUDA(cudaGetDevice(&prev));
    if (prev != dev) SPECSIM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// One cudaMalloc carved into 256-byte aligned buffers.
class Arena {
 public:
  template <class T>
  void reserve(T** slot, long long count) {
    reqs_.push_back({reinterpret_cast<void**>(slot), static_cast<size_t>(count) * sizeof(T)});
  }
  void commit() {
    size_t total = 0;
    for (auto& r : reqs_) total += (r.bytes + 255) & ~size_t(255);
    SPECSIM_CUDA(cudaMalloc(&base_, total));
    size_t off = 0;
    for (auto& r : reqs_) {
      *r.slot = static_cast<uint8_t*>(base_) + off;
      off += (r.bytes + 255) & ~size_t(255);
    }
    reqs_.clear();
  }
  ~Arena() {
    if (base_) cudaFree(base_);
  }
 private:
  struct Req {
    void** slot;
    size_t bytes;
  };
  std::vector<Req> reqs_;
  void* base_ = nullptr;
};

enum Phase { PH_INGEST = 0, PH_GEMM, PH_ATTN, PH_ELEM, PH_LM, PH_ADAM, PH_COMM, PH_N };

struct ParamDesc {
  std::string name;
  long long rows, cols, off;
  bool norm;
};

// Parameter registry: flat fp32 layout, same order / offsets as the oracle.
std::vector<ParamDesc> param_registry(const DraftShape& sh, long long* total) {
  const long long H = sh.hidden, Q = static_cast<long long>(sh.n_heads) * sh.head_dim,
                  KV = static_cast<long long>(sh.n_kv_heads) * sh.head_dim, I = sh.ffn,
                  V = sh.vocab, W3 = static_cast<long long>(sh.layers_tapped) * H;
  std::vector<ParamDesc> ps;
  long long off = 0;
  auto add = [&](const char* n, long long r, long long c, bool norm) {
    ps.push_back({n, r, c, off, norm});
    off += r * c;
  };
  add("fc", H, W3, false);
  add("w_in", 1, H, true);
  add("w_hid", 1, H, true);
  add("qkv", Q + 2 * KV, 2 * H, false);
  add("o", H, Q, false);
  add("w_post", 1, H, true);
  add("gate_up", 2 * I, H, false);
  add("down", H, I, false);
  add("w_fin", 1, H, true);
  add("lm_head", V, H, false);
  if (total) *total = off;
  return ps;
}

// vocabulary chunk of the LM-head backward: multiple of the GEMM N tile, ~32k
// (SPECSIM_VOCAB_CHUNK overrides, A/B experiments)
long long vocab_chunk(long long V) {
  static const long long target = [] {
    const char* e = std::getenv("SPECSIM_VOCAB_CHUNK");
    const long long v = e ? std::atoll(e) : 32768;
    return v > 0 ? v : 32768;
  }();
  long long vc = std::min<long long>(V, target);
  vc = (vc + gemm::BN - 1) / gemm::BN * gemm::BN;
  return vc > V ? V : vc;
}

}  // namespace

// Gradient buckets of the data-parallel exchange, in the order the backward
// finalises them: LM-head vocabulary chunks, then [down, w_fin], [gate_up],
// [o, w_post], [qkv], [fc, w_in, w_hid].  Together they tile [0, total).
std::vector<DpBucket> dp_buckets(const DraftShape& sh) {
  long long total = 0;
  const auto ps = param_registry(sh, &total);
  auto off = [&](const char* n) {
    for (const auto& p : ps)
      if (p.name == n) return p.off;
    throw std::logic_error("registry");
  };
  const long long H = sh.hidden, V = sh.vocab, Vc = vocab_chunk(V);
  std::vector<DpBucket> b;
  for (long long v0 = 0; v0 < V; v0 += Vc)
    b.push_back({off("lm_head") + v0 * H, std::min(Vc, V - v0) * H});
  b.push_back({off("down"), off("lm_head") - off("down")});
  b.push_back({off("gate_up"), off("down") - off("gate_up")});
  b.push_back({off("o"), off("gate_up") - off("o")});
  b.push_back({off("qkv"), off("o") - off("qkv")});
  b.push_back({0, off("qkv")});
  return b;
}

// ZeRO-1 needs every bucket to split into `world` equal shards of whole
// 8-element (32-byte fp32 / 16-byte bf16) groups.
bool zero_shardable(const std::vector<DpBucket>& b, int world) {
  for (const auto& x : b)
    if (x.n % (8ll * world) != 0) return false;
  return true;
}

HiddenStateBuffer* hsbuf_unwrap(struct specsim_hsbuf* b);

void DraftShape::validate() const {
  Problems p("invalid draft shape");
  p.check(hidden > 0 && hidden % 64 == 0, "hidden must be a positive multiple of 64");
  p.check(hidden <= 8192, "hidden must be <= 8192");
  p.check(vocab > 0 && vocab % 8 == 0, "vocab must be a positive multiple of 8");
  p.check(seq_len > 0 && seq_len % 64 == 0, "seq_len must be a positive multiple of 64");
  p.check(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
  p.check(n_heads > 0 && n_kv_heads > 0 && n_heads % n_kv_heads == 0,
          "n_heads must be a positive multiple of n_kv_heads");
  p.check(ffn > 0 && ffn % 64 == 0, "ffn must be a positive multiple of 64");
  p.check(layers_tapped >= 1 && layers_tapped <= 8, "layers_tapped must be in [1, 8]");
  p.check(micro_batch >= 1 && micro_batch <= kern::kMaxBatch, "micro_batch must be in [1, 64]");
  p.check(rms_eps > 0.f, "rms_eps must be > 0");
  p.check(rope_theta > 0.0, "rope_theta must be > 0");
  p.check(ttt_steps >= 1 && ttt_steps <= kern::kMaxTtt, "ttt_steps must be in [1, 16]");
  p.check(ttt_steps == 1 || seq_len % 128 == 0,
          "ttt_steps > 1 needs seq_len % 128 == 0 (tcgen05 attention)");
  p.check(ttt_decay > 0.f && ttt_decay <= 1.f, "ttt_decay must be in (0, 1]");
  p.throw_if_any();
}

class DraftTrainerImpl {
 public:
  using Param = ParamDesc;

  DraftShape sh;
  AdamWConfig opt;
  int rank, world, device;
  long long T, H, Q, KV, NQ, I, V, W3, Vc;
  int n_chunks;
  // training-time-test unroll: K decoder passes; per-pass buffers are stacked
  // [K][T]; sw = loss weights over the K*T logit rows, sw1 = pass 0 only (eval)
  int K = 1;
  long long KT = 0;
  kern::StepWeights sw{}, sw1{};
  std::vector<Param> params;
  long long total = 0;
  int64_t step_count = 0;
  int64_t version = 0;
  bool timing = false;
  // deploy gate: device copy of the model [P | Mst | Vst] fp32 + P16 bf16
  void* snap = nullptr;
  int64_t snap_step = -1, snap_version = 0;
  double phase_ms[PH_N] = {}, phase_flops[PH_N] = {};
  int phase_launches[PH_N] = {};

  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  bool use_nccl = false;              // world > 1, or SPECSIM_FORCE_NCCL=1 (1-rank comm, tests)
  cudaStream_t comm_stream = nullptr;  // gradient buckets exchanged behind the backward
  // ZeRO-1 (world > 1 default, SPECSIM_DP_MODE=allreduce to disable): each
  // bucket is reduce-scattered in place, this rank's shard updated by AdamW on
  // the comm stream, and the bf16 working weights all-gathered in place
  bool zero = false;
  std::vector<DpBucket> buckets;
  std::vector<cudaEvent_t> bucket_events;
  size_t bucket_next = 0;
  cudaEvent_t ev_comm_done = nullptr;
  Arena arena;

  // parameters / optimiser state (flat, registry order)
  float *P = nullptr, *Mst = nullptr, *Vst = nullptr, *G = nullptr;
  __nv_bfloat16* P16 = nullptr;
  __nv_bfloat16* E = nullptr;  // frozen embedding [V, H]
  float *cos_t = nullptr, *sin_t = nullptr;    // [S, hd/2] (standalone RoPE kernel)
  float *cos_tr = nullptr, *sin_tr = nullptr;  // [hd/2, S] (fused epilogues: lane = position)
  // activations ([K][T] stacked per unroll pass; g is [K+1][T, H]: g[0] =
  // W_fc f, g[j+1] = h_j = the input of pass j+1, so h = g + T*H)
  __nv_bfloat16 *F, *g, *U, *qkv, *o, *r, *z, *gu, *act, *h, *nrm;
  int32_t *u, *y, *m, *argmax;
  // The fc GEMMs (forward A operand, weight-gradient B operand) read the
  // micro-batch's feature rows straight from the signal ring through a
  // per-step table of 64-row block ring rows (no [T, 3H] copy; S % 128 == 0;
  // SPECSIM_F_GATHER=1 keeps the gather copy into F for A/B runs).  Their
  // plans hold a tensor map of one buffer's ring, so they are built per
  // buffer (before the step is captured).
  bool f_direct = false;
  int32_t* blk_rows = nullptr;  // [T / 64]
  struct RingPlans {
    gemm::GemmPlan fc, dw_fc, f_dw_fc;
  };
  std::map<uint64_t, RingPlans> ring_plans;
  const RingPlans* cur_ring = nullptr;
  const void* last_ring = nullptr;  // ring of the last step / eval (read_rows("F"))
  float *coef, *rstd_a, *rstd_b, *lse_attn, *rstd_post, *rstd_fin, *lse, *row_loss;
  gemm::CePartial* partials;
  long long* n_global;
  double* stats;
  // backward
  __half* logits = nullptr;  // [KT, V] fp16 offsets from the half-tile row max (keep_logits)
  bool keep_logits = false;
  __nv_bfloat16 *dlog, *dh_b, *dact, *dgu, *dr_b, *dO, *dqkv, *dg_b;
  float *dn, *dh, *dz, *dr, *dU, *Dattn, *dw_part;
  // K > 1: fp32 gradient w.r.t. the pass input (flows into the previous pass's
  // output), the cache part of dq, and the k | v accumulators of passes >= 1
  float *dg_in = nullptr, *dq_add = nullptr, *dkv_acc = nullptr;
  // K > 1: per-pass dw partials of the final / post / hidden norms ([K][nbT, H]
  // each), summed once at pass 0 -- no extra pass over the K*T rows
  float *dwp_fin = nullptr, *dwp_post = nullptr, *dwp_hid = nullptr;
  long long nbT = 0;
  // pinned host scalars
  long long* h_nglobal = nullptr;
  double* h_stats = nullptr;
  // Per-step inputs (batch spec, caller's global token count, AdamW
  // constants).  The captured step reads them from device memory; the host
  // fills one of two mapped pinned slots and a stream-ordered one-warp fetch
  // kernel (outside the graph) moves it, so train() can enqueue steps
  // back-to-back.
  struct StepInputs {
    kern::BatchSpec spec;
    long long nglobal;  // > 0: caller-provided global valid-token count
    long long pad;
    gemm::AdamDev hp;
  };
  StepInputs* d_in = nullptr;
  StepInputs* h_in = nullptr;  // pinned, 2 slots
  // train(job): every step's inputs are built up front into a mapped pinned
  // table, moved to the device ONCE (one SM fetch over PCIe), and each step's
  // slot is copied device-to-device into d_in -- no per-step PCIe read, which
  // would queue behind the ingest DMA a caller streams during the job
  StepInputs* h_job = nullptr;
  StepInputs* d_job = nullptr;
  size_t job_cap = 0;
  cudaEvent_t in_ev[2] = {nullptr, nullptr};
  int in_slot = 0;
  gemm::AdamDev* adam_dev = nullptr;  // = &d_in->hp
  bool keep_grads = false;            // materialise fp32 grads in the fused-AdamW path
  bool swiglu_fused = true;           // SwiGLU backward in the d act GEMM epilogue

  // GEMM plans (vectors: one per unroll pass; LM head and weight gradients
  // span all K*T rows)
  gemm::GemmPlan p_fc, p_ce_fwd, p_ce_fwd_eval;
  std::vector<gemm::GemmPlan> p_qkv, p_o, p_gu, p_down;
  std::vector<gemm::GemmPlan> p_ce_bwd, p_lm_dx, p_lm_dw;
  std::vector<gemm::GemmPlan> p_dact, p_dz, p_dO, p_dU;
  gemm::GemmPlan p_dw_down, p_dw_gu, p_dw_o, p_dw_qkv, p_dw_fc;
  // weight-gradient GEMMs with the AdamW update fused into the epilogue
  // (single-replica path: no all-reduce between gradient and update)
  std::vector<gemm::GemmPlan> f_lm_dw;
  gemm::GemmPlan f_dw_down, f_dw_gu, f_dw_o, f_dw_qkv, f_dw_fc;

  // One recorded launch sequence (eager step, or a captured CUDA graph): the
  // phase-timing events it contains and the algorithmic work per phase.
  struct Recording {
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    std::vector<cudaEvent_t> events;
    size_t next = 0;
    unsigned long long kernels = 0;  // device kernels one replay launches
    double flops[PH_N] = {};
    int launches[PH_N] = {};
    cudaGraphExec_t exec = nullptr;
    void reset() {
      marks.clear();
      next = 0;
      for (int i = 0; i < PH_N; ++i) flops[i] = 0, launches[i] = 0;
    }
    ~Recording() {
      for (auto e : events) cudaEventDestroy(e);
      if (exec) cudaGraphExecDestroy(exec);
    }
  };
  Recording eager_rec;
  Recording* rec = &eager_rec;
  std::map<std::tuple<bool, bool, bool, uint64_t>, std::unique_ptr<Recording>> graphs;
  bool use_graphs = true;
  bool capturing = false;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  float last_ms = 0.f;  // device time of the last step (step(), eval(), or a job's last)
  long long* n_counted = nullptr;
  cudaEvent_t ev_region[2] = {nullptr, nullptr};

  const Param& param(const std::string& name) const {
    for (const auto& p : params)
      if (p.name == name) return p;
    throw std::invalid_argument("unknown parameter '" + name + "'");
  }
  float* pf(const char* n) { return P + param(n).off; }
  __nv_bfloat16* pb(const char* n) { return P16 + param(n).off; }
  float* gf(const char* n) { return G + param(n).off; }

  DraftTrainerImpl(const DraftShape& s, const AdamWConfig& a, uint64_t seed, int rk, int ws,
                   const uint8_t* nccl_id, int dev)
      : sh(s), opt(a), rank(rk), world(ws), device(dev) {
    sh.validate();
    Problems p("invalid trainer configuration");
    p.check(world >= 1, "world must be >= 1");
    p.check(rank >= 0 && rank < world, "rank must be in [0, world)");
    p.check(world == 1 || nccl_id != nullptr, "nccl_id is required when world > 1");
    p.check(opt.lr > 0.f, "lr must be > 0");
    p.check(opt.beta1 >= 0.f && opt.beta1 < 1.f && opt.beta2 >= 0.f && opt.beta2 < 1.f,
            "betas must be in [0, 1)");
    p.check(opt.eps > 0.f, "eps must be > 0");
    p.throw_if_any();
    DeviceGuard dg(device);
    int major = 0, minor = 0;
    SPECSIM_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    SPECSIM_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      throw CudaError("this build targets sm_100a (B200); device has sm_" + std::to_string(major) +
                      std::to_string(minor));
    T = static_cast<long long>(sh.micro_batch) * sh.seq_len;
    H = sh.hidden;
    Q = static_cast<long long>(sh.n_heads) * sh.head_dim;
    KV = static_cast<long long>(sh.n_kv_heads) * sh.head_dim;
    NQ = Q + 2 * KV;
    I = sh.ffn;
    V = sh.vocab;
    W3 = static_cast<long long>(sh.layers_tapped) * H;
    K = sh.ttt_steps;
    KT = K * T;
    sw.K = K;
    sw.T = T;
    for (int j = 0; j < K; ++j)
      sw.w[j] = static_cast<float>(std::pow(static_cast<double>(sh.ttt_decay), j));
    sw1 = sw;
    sw1.K = 1;
    Vc = vocab_chunk(V);
    n_chunks = static_cast<int>((V + Vc - 1) / Vc);
    params = param_registry(sh, &total);
    buckets = dp_buckets(sh);

    SPECSIM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    const long long nb_ce = (V + gemm::BN - 1) / gemm::BN;
    arena.reserve(&P, total);
    arena.reserve(&Mst, total);
    arena.reserve(&Vst, total);
    arena.reserve(&G, total);
    arena.reserve(&P16, total);
    arena.reserve(&E, V * H);
    arena.reserve(&cos_t, static_cast<long long>(sh.seq_len) * sh.head_dim / 2);
    arena.reserve(&sin_t, static_cast<long long>(sh.seq_len) * sh.head_dim / 2);
    arena.reserve(&cos_tr, rope_len() * sh.head_dim / 2);
    arena.reserve(&sin_tr, rope_len() * sh.head_dim / 2);
    {
      const char* e = std::getenv("SPECSIM_F_GATHER");
      f_direct = sh.seq_len % 128 == 0 && !(e && e[0] == '1');
    }
    F = nullptr;
    if (!f_direct) arena.reserve(&F, T * W3);
    arena.reserve(&blk_rows, (T + 63) / 64);
    arena.reserve(&g, (K + 1) * T * H);
    arena.reserve(&U, KT * 2 * H);
    arena.reserve(&qkv, KT * NQ);
    arena.reserve(&o, KT * Q);
    arena.reserve(&r, KT * H);
    arena.reserve(&z, KT * H);
    arena.reserve(&gu, KT * 2 * I);
    arena.reserve(&act, KT * I);
    arena.reserve(&nrm, KT * H);
    arena.reserve(&u, KT);
    arena.reserve(&y, KT);
    arena.reserve(&m, KT);
    arena.reserve(&argmax, KT);
    arena.reserve(&coef, KT);
    arena.reserve(&rstd_a, KT);
    arena.reserve(&rstd_b, KT);
    arena.reserve(&lse_attn, KT * sh.n_heads);
    arena.reserve(&rstd_post, KT);
    arena.reserve(&rstd_fin, KT);
    arena.reserve(&lse, KT);
    arena.reserve(&row_loss, KT);
    arena.reserve(&partials, 2 * nb_ce * KT);
    arena.reserve(&n_global, 2);
    arena.reserve(&stats, 4);
    arena.reserve(&dlog, KT * Vc);
    // logits [KT, V] kept from the forward so the backward needs no logit
    // recompute, as fp16 offsets from the row max of each 128-column half tile
    // (2.1 GB at C2); SPECSIM_CE_RECOMPUTE=1 or a > 32 GB table
    // selects the recompute path instead
    {
      const char* e = std::getenv("SPECSIM_CE_RECOMPUTE");
      keep_logits = !(e && e[0] == '1') && KT * V * 2 <= (32ll << 30);
      if (keep_logits) arena.reserve(&logits, KT * V);
    }
    arena.reserve(&dh_b, KT * H);
    arena.reserve(&dact, T * I);
    arena.reserve(&dgu, KT * 2 * I);
    arena.reserve(&dr_b, KT * H);
    arena.reserve(&dO, KT * Q);
    arena.reserve(&dqkv, KT * NQ);
    arena.reserve(&dg_b, T * H);
    arena.reserve(&dn, KT * H);
    arena.reserve(&dh, T * H);
    arena.reserve(&dz, KT * H);
    arena.reserve(&dr, T * H);
    arena.reserve(&dU, KT * 2 * H);
    arena.reserve(&Dattn, KT * sh.n_heads);
    arena.reserve(&dw_part, kern::rmsnorm_bwd_partial_rows(KT) * H);
    nbT = kern::rmsnorm_bwd_partial_rows(T);
    if (K > 1) {
      arena.reserve(&dwp_fin, K * nbT * H);
      arena.reserve(&dwp_post, K * nbT * H);
      arena.reserve(&dwp_hid, K * nbT * H);
      arena.reserve(&dg_in, T * H);
      arena.reserve(&dq_add, T * Q);
      arena.reserve(&dkv_acc, KT * 2 * KV);
    }
    arena.reserve(&d_in, 1);
    arena.reserve(&n_counted, 1);
    arena.commit();
    h = g + T * H;
    adam_dev = &d_in->hp;
    SPECSIM_CUDA(cudaHostAlloc(&h_in, 2 * sizeof(StepInputs), cudaHostAllocMapped));
    std::memset(h_in, 0, 2 * sizeof(StepInputs));
    for (auto& e : in_ev) SPECSIM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const char* ng = std::getenv("SPECSIM_NO_GRAPH");
    use_graphs = !(ng && ng[0] == '1');
    SPECSIM_CUDA(cudaMallocHost(&h_nglobal, sizeof(long long)));
    SPECSIM_CUDA(cudaHostAlloc(&h_stats, 4 * sizeof(double), cudaHostAllocMapped));
    SPECSIM_CUDA(cudaMemsetAsync(Mst, 0, sizeof(float) * total, stream));
    SPECSIM_CUDA(cudaMemsetAsync(Vst, 0, sizeof(float) * total, stream));
    SPECSIM_CUDA(cudaMemsetAsync(G, 0, sizeof(float) * total, stream));

    init_params(seed);
    init_rope();
    {
      const char* e = std::getenv("SPECSIM_SWIGLU_UNFUSED");
      swiglu_fused = !(e && e[0] == '1');
    }
    build_plans();
    attn::prepare(sh.head_dim);
    SPECSIM_CUDA(cudaEventCreate(&ev_begin));
    SPECSIM_CUDA(cudaEventCreate(&ev_end));
    SPECSIM_CUDA(cudaEventCreate(&ev_region[0]));
    SPECSIM_CUDA(cudaEventCreate(&ev_region[1]));
    const char* force = std::getenv("SPECSIM_FORCE_NCCL");
    use_nccl = world > 1 || (force && force[0] == '1');
    if (use_nccl) {
      ncclUniqueId id;
      if (world > 1)
        std::memcpy(&id, nccl_id, sizeof(id));
      else
        SPECSIM_NCCL(nccl::api().GetUniqueId(&id));
      SPECSIM_NCCL(nccl::api().CommInitRank(&comm, world, id, rank));
      SPECSIM_CUDA(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
      SPECSIM_CUDA(cudaEventCreateWithFlags(&ev_comm_done, cudaEventDisableTiming));
      const char* mode = std::getenv("SPECSIM_DP_MODE");
      zero = !(mode && std::strcmp(mode, "allreduce") == 0) && zero_shardable(buckets, world);
    }
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
  }

  ~DraftTrainerImpl() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (snap) cudaFree(snap);
    if (comm_stream) cudaStreamSynchronize(comm_stream);
    if (comm) nccl::api().CommDestroy(comm);
    for (auto e : bucket_events) cudaEventDestroy(e);
    if (ev_comm_done) cudaEventDestroy(ev_comm_done);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (ev_begin) cudaEventDestroy(ev_begin);
    if (ev_end) cudaEventDestroy(ev_end);
    for (auto e : ev_region)
      if (e) cudaEventDestroy(e);
    if (h_nglobal) cudaFreeHost(h_nglobal);
    if (h_stats) cudaFreeHost(h_stats);
    if (h_in) cudaFreeHost(h_in);
    if (h_job) cudaFreeHost(h_job);
    if (d_job) cudaFree(d_job);
    if (hist_buf) cudaFreeHost(hist_buf);
    for (auto e : in_ev)
      if (e) cudaEventDestroy(e);
    graphs.clear();
    if (stream) cudaStreamDestroy(stream);
  }

  // ------------------------------------------------------------ init
  static void fill_normal_blocks(uint64_t seed_base, int pidx, long long n, float* out) {
    // element e: Rng(seed_base + (p << 32) + (e >> 20)) in element order
    const long long nblk = (n + (1 << 20) - 1) >> 20;
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([=] {
        for (long long j = w; j < nblk; j += nt) {
          bk::Rng rng(seed_base + (static_cast<uint64_t>(pidx) << 32) + static_cast<uint64_t>(j));
          const long long e0 = j << 20, e1 = std::min(n, e0 + (1ll << 20));
          for (long long e = e0; e < e1; ++e) out[e] = static_cast<float>(rng.normal(0.0, 0.02));
        }
      });
    for (auto& t : th) t.join();
  }

  void init_params(uint64_t seed) {
    const long long slab = 1ll << 26;  // 64M elements per host slab
    std::vector<float> buf;
    for (size_t pi = 0; pi < params.size(); ++pi) {
      const Param& pr = params[pi];
      const long long n = pr.rows * pr.cols;
      if (pr.norm) {
        buf.assign(n, 1.0f);
        SPECSIM_CUDA(cudaMemcpy(P + pr.off, buf.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
        continue;
      }
      buf.resize(n);
      fill_normal_blocks(seed + 1, static_cast<int>(pi), n, buf.data());
      for (long long e = 0; e < n; e += slab) {
        const long long c = std::min(slab, n - e);
        SPECSIM_CUDA(cudaMemcpy(P + pr.off + e, buf.data() + e, sizeof(float) * c,
                                cudaMemcpyHostToDevice));
      }
    }
    kern::f32_to_bf16(P, P16, total, stream);
    // frozen embedding (parameter index 15, seed + 2), bf16
    const long long ne = V * H;
    buf.resize(ne);
    fill_normal_blocks(seed + 2, 15, ne, buf.data());
    std::vector<uint16_t> eb(ne);
    for (long long i = 0; i < ne; ++i) {
      uint32_t bits;
      std::memcpy(&bits, &buf[i], 4);
      bits += 0x7FFFu + ((bits >> 16) & 1u);
      eb[i] = static_cast<uint16_t>(bits >> 16);
    }
    SPECSIM_CUDA(cudaMemcpy(E, eb.data(), 2 * ne, cudaMemcpyHostToDevice));
    SPECSIM_CHECK_LAUNCH();
  }

  // positions covered by the RoPE tables: pass j rotates row t at t % S + j
  long long rope_len() const { return static_cast<long long>(sh.seq_len) + K - 1; }

  void init_rope() {
    // NeoX rotate-half tables, angle = pos * theta^(-2i/hd) in double
    const int half = sh.head_dim / 2;
    const int npos = static_cast<int>(rope_len());
    std::vector<float> c(static_cast<size_t>(npos) * half), s(c.size());
    for (int pos = 0; pos < npos; ++pos)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow(sh.rope_theta, -2.0 * i / sh.head_dim);
        const double ang = static_cast<double>(pos) * inv;
        c[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::cos(ang));
        s[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::sin(ang));
      }
    // [S, hd/2] (standalone kernel, single pass only): the first S positions
    const size_t n_std = static_cast<size_t>(sh.seq_len) * half;
    SPECSIM_CUDA(cudaMemcpy(cos_t, c.data(), sizeof(float) * n_std, cudaMemcpyHostToDevice));
    SPECSIM_CUDA(cudaMemcpy(sin_t, s.data(), sizeof(float) * n_std, cudaMemcpyHostToDevice));
    std::vector<float> ct(c.size()), st(c.size());
    for (int pos = 0; pos < npos; ++pos)
      for (int i = 0; i < half; ++i) {
        ct[static_cast<size_t>(i) * npos + pos] = c[static_cast<size_t>(pos) * half + i];
        st[static_cast<size_t>(i) * npos + pos] = s[static_cast<size_t>(pos) * half + i];
      }
    SPECSIM_CUDA(cudaMemcpy(cos_tr, ct.data(), sizeof(float) * ct.size(), cudaMemcpyHostToDevice));
    SPECSIM_CUDA(cudaMemcpy(sin_tr, st.data(), sizeof(float) * st.size(), cudaMemcpyHostToDevice));
  }

  // ------------------------------------------------------------ plans
  static gemm::Args out_args(void* C, long long ldc, const __nv_bfloat16* R = nullptr,
                             long long ldr = 0) {
    gemm::Args a{};
    a.C = C;
    a.ldc = ldc;
    a.R = R;
    a.ldr = ldr;
    return a;
  }

  void build_plans() {
    using gemm::Operand;
    using namespace gemm;
    // forward: Y = X W^T (both K-major)
    if (!f_direct)
      p_fc = make_plan({F, W3, false}, {pb("fc"), W3, false}, T, H, W3, EPI_BF16, out_args(g, H));
    for (int j = 0; j < K; ++j) {
      const long long R = j * T;  // first row of pass j in the stacked buffers
      // q / k heads rotated in the epilogue (NeoX RoPE at t % S + j); v as is
      Args qa = out_args(qkv + R * NQ, NQ);
      qa.rope_cos = cos_tr;
      qa.rope_sin = sin_tr;
      qa.rope_S = sh.seq_len;
      qa.rope_cols = static_cast<int>(Q + KV);
      qa.rope_hd = sh.head_dim;
      qa.rope_pos_off = j;
      qa.rope_ld = static_cast<int>(rope_len());
      p_qkv.push_back(make_plan({U + R * 2 * H, 2 * H, false}, {pb("qkv"), 2 * H, false}, T, NQ,
                                2 * H, EPI_BF16_ROPE, qa));
      // r_j = g_j + o_j W_o^T ; h_j (= g_{j+1}) = r_j + act_j W_d^T
      p_o.push_back(make_plan({o + R * Q, Q, false}, {pb("o"), Q, false}, T, H, Q, EPI_BF16_RESID,
                              out_args(r + R * H, H, g + R * H, H)));
      p_gu.push_back(make_plan({z + R * H, H, false}, {pb("gate_up"), H, false}, T, 2 * I, H,
                               EPI_BF16, out_args(gu + R * 2 * I, 2 * I)));
      p_down.push_back(make_plan({act + R * I, I, false}, {pb("down"), I, false}, T, H, I,
                                 EPI_BF16_RESID, out_args(h + R * H, H, r + R * H, H)));
    }
    auto ce_fwd = [&](long long rows) {
      Args ce{};
      ce.targets = y;
      ce.partials = partials;
      if (keep_logits) {
        ce.C = logits;
        ce.ldc = V;
      }
      if (const char* e = std::getenv("SPECSIM_CE_L2_MB")) ce.l2_budget_mb = std::atoi(e);
      return make_plan({nrm, H, false}, {pb("lm_head"), H, false}, static_cast<int>(rows), V, H,
                       EPI_CE_FWD, ce);
    };
    // LM head + CE over every pass's rows at once; eval runs pass 0 only
    p_ce_fwd = ce_fwd(KT);
    if (K > 1) p_ce_fwd_eval = ce_fwd(T);
    // LM head backward, vocabulary chunks, all K*T rows
    for (int c = 0; c < n_chunks; ++c) {
      const long long v0 = c * Vc, vn = std::min(Vc, V - v0);
      Args cb = out_args(dlog, Vc);
      cb.targets = y;
      cb.lse = lse;
      cb.coef = coef;
      cb.vocab_offset = static_cast<int>(v0);
      p_ce_bwd.push_back(make_plan({nrm, H, false}, {pb("lm_head") + v0 * H, H, false}, KT, vn,
                                   H, EPI_CE_BWD, cb));
      // dn (+)= dlog_c . W_c     (B = W_c stored [vn, H] -> MN-major)
      p_lm_dx.push_back(make_plan({dlog, Vc, false}, {pb("lm_head") + v0 * H, H, true}, KT, H, vn,
                                  c == 0 ? EPI_F32 : EPI_F32_ACC, out_args(dn, H)));
      // dW_c = dlog_c^T . nrm    (A = dlog stored [KT, vn] -> MN-major)
      p_lm_dw.push_back(make_plan({dlog, Vc, true}, {nrm, H, true}, vn, H, KT, EPI_F32,
                                  out_args(gf("lm_head") + v0 * H, H)));
    }
    // data gradients, per pass
    for (int j = 0; j < K; ++j) {
      const long long R = j * T;
      // d act = dh W_down; the SwiGLU backward runs in its epilogue (reads the
      // stored gate | up, writes d gate | d up) unless SPECSIM_SWIGLU_UNFUSED=1
      if (swiglu_fused)
        p_dact.push_back(make_plan({dh_b + R * H, H, false}, {pb("down"), I, true}, T, I, H,
                                   EPI_SWIGLU_BWD,
                                   out_args(dgu + R * 2 * I, 2 * I, gu + R * 2 * I, 2 * I)));
      else
        p_dact.push_back(make_plan({dh_b + R * H, H, false}, {pb("down"), I, true}, T, I, H,
                                   EPI_BF16, out_args(dact, I)));
      p_dz.push_back(make_plan({dgu + R * 2 * I, 2 * I, false}, {pb("gate_up"), H, true}, T, H,
                               2 * I, EPI_F32, out_args(dz + R * H, H)));
      p_dO.push_back(make_plan({dr_b + R * H, H, false}, {pb("o"), Q, true}, T, Q, H, EPI_BF16,
                               out_args(dO + R * Q, Q)));
      p_dU.push_back(make_plan({dqkv + R * NQ, NQ, false}, {pb("qkv"), 2 * H, true}, T, 2 * H, NQ,
                               EPI_F32, out_args(dU + R * 2 * H, 2 * H)));
    }
    // weight gradients: one GEMM over every pass's rows (the sum over passes
    // is the reduction over K*T)
    p_dw_down = make_plan({dh_b, H, true}, {act, I, true}, H, I, KT, EPI_F32,
                          out_args(gf("down"), I));
    p_dw_gu = make_plan({dgu, 2 * I, true}, {z, H, true}, 2 * I, H, KT, EPI_F32,
                        out_args(gf("gate_up"), H));
    p_dw_o = make_plan({dr_b, H, true}, {o, Q, true}, H, Q, KT, EPI_F32, out_args(gf("o"), Q));
    p_dw_qkv = make_plan({dqkv, NQ, true}, {U, 2 * H, true}, NQ, 2 * H, KT, EPI_F32,
                         out_args(gf("qkv"), 2 * H));
    // fc (pass 0 only; no dF: captured features are inputs)
    if (!f_direct)
      p_dw_fc = make_plan({dg_b, H, true}, {F, W3, true}, H, W3, T, EPI_F32,
                          out_args(gf("fc"), W3));
    for (int c = 0; c < n_chunks; ++c) f_lm_dw.push_back(fused(p_lm_dw[c], "lm_head", c * Vc));
    f_dw_down = fused(p_dw_down, "down", 0);
    f_dw_gu = fused(p_dw_gu, "gate_up", 0);
    f_dw_o = fused(p_dw_o, "o", 0);
    f_dw_qkv = fused(p_dw_qkv, "qkv", 0);
    if (!f_direct) f_dw_fc = fused(p_dw_fc, "fc", 0);
  }

  // fused-AdamW twin of a weight-gradient GEMM (rows from row0 of `name`)
  gemm::GemmPlan fused(const gemm::GemmPlan& src, const char* name, long long row0) {
    gemm::GemmPlan f = src;
    const long long off = param(name).off + row0 * param(name).cols;
    f.epi = gemm::EPI_ADAMW;
    f.args.opt_p = P + off;
    f.args.opt_m = Mst + off;
    f.args.opt_v = Vst + off;
    f.args.opt_p16 = P16 + off;
    f.args.opt_g = G + off;  // cleared per launch unless keep_grads
    f.args.opt_hp = adam_dev;
    return f;
  }

  // fc GEMMs over this buffer's ring (the ring is [capacity + kMirrorRows, 3H])
  const RingPlans& ring_plans_for(HiddenStateBuffer& buf) {
    auto it = ring_plans.find(buf.serial());
    if (it != ring_plans.end()) return it->second;
    using namespace gemm;
    const long long rows = buf.capacity() + HiddenStateBuffer::kMirrorRows;
    RingPlans rp;
    Args fa = out_args(g, H);
    fa.a_rows = blk_rows;
    rp.fc = make_plan({buf.ring_features(), W3, false, rows}, {pb("fc"), W3, false}, T, H, W3,
                      EPI_BF16, fa);
    Args da = out_args(gf("fc"), W3);
    da.b_rows = blk_rows;
    rp.dw_fc = make_plan({dg_b, H, true}, {buf.ring_features(), W3, true, rows}, H, W3, T,
                         EPI_F32, da);
    rp.f_dw_fc = fused(rp.dw_fc, "fc", 0);
    return ring_plans.emplace(buf.serial(), rp).first->second;
  }

  // weight-gradient GEMM: fused AdamW on a single replica, plain fp32 grads
  // (then bucketed all-reduce) when data-parallel
  void run_dw(const gemm::GemmPlan& plain, const gemm::GemmPlan& fusedp, int phase = PH_GEMM) {
    if (!fused_adamw()) {
      run(plain, phase);
      return;
    }
    gemm::GemmPlan f = fusedp;
    if (!keep_grads) f.args.opt_g = nullptr;
    run(f, phase, plain.flops);
  }

  // ------------------------------------------------------------ timing
  cudaEvent_t next_event() {
    if (rec->next == rec->events.size()) {
      cudaEvent_t e;
      SPECSIM_CUDA(cudaEventCreate(&e));
      rec->events.push_back(e);
    }
    return rec->events[rec->next++];
  }
  template <class Fn>
  void timed(int phase, double flops, Fn&& fn) {
    rec->flops[phase] += flops;
    rec->launches[phase] += 1;
    if (!timing) {
      fn();
      return;
    }
    cudaEvent_t a = next_event(), b = next_event();
    // inside a capture, External makes these real timestamp nodes (a plain
    // record would only express a dependency)
    const unsigned flags = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    SPECSIM_CUDA(cudaEventRecordWithFlags(a, stream, flags));
    fn();
    SPECSIM_CUDA(cudaEventRecordWithFlags(b, stream, flags));
    rec->marks.push_back({phase, {a, b}});
  }
  void run(const gemm::GemmPlan& p, int phase = PH_GEMM, double alg_flops = -1) {
    timed(phase, alg_flops < 0 ? p.flops : alg_flops, [&] { p.launch(stream); });
  }

  // ------------------------------------------------------------ step
  kern::BatchSpec batch_spec(HiddenStateBuffer& buf, const int64_t* ids, int n) {
    if (n < 0 || n > sh.micro_batch)
      throw std::invalid_argument("n must be in [0, micro_batch]");
    if (buf.geometry().hidden_dim != sh.hidden || buf.geometry().layers_tapped != sh.layers_tapped)
      throw std::invalid_argument("signal geometry does not match the draft shape");
    if (buf.device() != device) throw std::invalid_argument("buffer lives on another device");
    kern::BatchSpec spec{};
    spec.n = n;
    wait_seq = 0;
    for (int b = 0; b < n; ++b) {
      const auto& s = buf.sample(ids[b]);
      spec.start[b] = s.start;
      spec.len[b] = s.length;
      wait_seq = std::max<int64_t>(wait_seq, s.last_seq);
    }
    return spec;
  }
  int64_t wait_seq = 0;  // latest append the current batch depends on
  double* hist_buf = nullptr;  // pinned per-step stats of train()
  size_t hist_cap = 0;

  // Device work of the forward over `passes` unroll passes (K for a training
  // step, 1 for eval).  Everything that varies per step is read from
  // d_in (filled by stage() before the launch), so the whole step can be
  // captured once into a CUDA graph and replayed.
  void forward(HiddenStateBuffer& buf, int passes) {
    const int S = sh.seq_len;
    const kern::StepWeights& w = passes == K ? sw : sw1;
    timed(PH_INGEST, 0, [&] {
      if (f_direct)
        kern::gather_tokens(buf.ring_ids(), buf.capacity(), &d_in->spec, sh.micro_batch, S,
                            passes, u, y, m, blk_rows, stream);
      else
        kern::gather_batch(static_cast<const __nv_bfloat16*>(buf.ring_features()),
                           buf.ring_ids(), buf.capacity(), static_cast<int>(W3), &d_in->spec,
                           sh.micro_batch, S, passes, F, u, y, m, stream);
      kern::mask_count(m, T, n_counted, stream);
    });
    if (use_nccl)
      timed(PH_COMM, 0, [&] {
        SPECSIM_NCCL(nccl::api().AllReduce(n_counted, n_counted, 1, ncclInt64, ncclSum, comm, stream));
      });
    timed(PH_ELEM, 0, [&] {
      // caller-provided global count wins over the counted one
      kern::select_count(&d_in->nglobal, n_counted, n_global, stream);
      kern::ce_coef(m, n_global, coef, w, stream);
    });
    run(f_direct ? cur_ring->fc : p_fc);
    for (int j = 0; j < passes; ++j) {
      const long long R = j * T;
      timed(PH_ELEM, 0, [&] {
        kern::rmsnorm_fwd(E, H, u + R, pf("w_in"), sh.rms_eps, U + R * 2 * H, 2 * H, rstd_a + R,
                          T, sh.hidden, stream);
        kern::rmsnorm_fwd(g + R * H, H, nullptr, pf("w_hid"), sh.rms_eps, U + R * 2 * H + H, 2 * H,
                          rstd_b + R, T, sh.hidden, stream);
      });
      run(p_qkv[j]);  // RoPE fused into the epilogue
      const attn::Dims ad = attn_dims(j);
      timed(PH_ATTN, attn_flops(j, false), [&] {
        attn::forward(qkv, o + R * Q, lse_attn + R * sh.n_heads, ad, sh.head_dim, stream);
      });
      run(p_o[j]);
      timed(PH_ELEM, 0, [&] {
        kern::rmsnorm_fwd(r + R * H, H, nullptr, pf("w_post"), sh.rms_eps, z + R * H, H,
                          rstd_post + R, T, sh.hidden, stream);
      });
      run(p_gu[j]);
      timed(PH_ELEM, 0, [&] { kern::swiglu_fwd(gu + R * 2 * I, act + R * I, T, sh.ffn, stream); });
      run(p_down[j]);
    }
    const long long rows = passes * T;
    timed(PH_ELEM, 0, [&] {
      kern::rmsnorm_fwd(h, H, nullptr, pf("w_fin"), sh.rms_eps, nrm, H, rstd_fin, rows, sh.hidden,
                        stream);
    });
    const gemm::GemmPlan& ce = passes == K ? p_ce_fwd : p_ce_fwd_eval;
    run(ce, PH_LM);
    timed(PH_ELEM, 0, [&] {
      kern::ce_reduce(partials, 2 * ce.args.num_n_blocks, rows, y, m, lse, row_loss, argmax,
                      stream);
      kern::ce_finalize(row_loss, argmax, y, m, n_global, w, stats, stream);
    });
  }

  // algorithmic attention FLOPs of pass j (causal 2Q(S+1) per token forward,
  // plus 4Q per cache entry; backward twice that)
  double attn_flops(int j, bool bwd) const {
    const double f = (2.0 * Q * (sh.seq_len + 1) + 4.0 * Q * j) * T;
    return bwd ? 2.0 * f : f;
  }

  attn::Dims attn_dims(int j = 0) const {
    attn::Dims d;
    d.B = sh.micro_batch;
    d.S = sh.seq_len;
    d.nh = sh.n_heads;
    d.nkv = sh.n_kv_heads;
    d.NQ = static_cast<int>(NQ);
    d.Q = static_cast<int>(Q);
    d.KV = static_cast<int>(KV);
    d.scale = 1.0f / std::sqrt(static_cast<float>(sh.head_dim));
    d.rope_len = static_cast<int>(rope_len());
    // pass j: queries at rows j*T of the stacked qkv, RoPE positions t % S + j,
    // cache entries of passes 1..j
    d.q_row_off = j * T;
    d.pos_off = j;
    d.n_diag = j;
    d.diag_qkv = j > 0 ? qkv : nullptr;
    return d;
  }

  // Data-parallel exchange of bucket i (dp_buckets order): its gradient range
  // is final.  All-reduce mode: sum it on the comm stream while the backward
  // continues (AdamW after the join).  ZeRO-1: reduce-scatter in place, AdamW
  // on this rank's shard and in-place all-gather of the bf16 working weights,
  // all on the comm stream -- the weights of a finished bucket are not read
  // again by this step's backward, and the next step joins on ev_comm_done.
  void bucket_ready(int i) {
    if (!use_nccl) return;
    const DpBucket& bk = buckets[i];
    if (bucket_next == bucket_events.size()) {
      cudaEvent_t e;
      SPECSIM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      bucket_events.push_back(e);
    }
    cudaEvent_t e = bucket_events[bucket_next++];
    SPECSIM_CUDA(cudaEventRecord(e, stream));
    SPECSIM_CUDA(cudaStreamWaitEvent(comm_stream, e, 0));
    if (!zero) {
      SPECSIM_NCCL(nccl::api().AllReduce(G + bk.off, G + bk.off, static_cast<size_t>(bk.n),
                                         ncclFloat, ncclSum, comm, comm_stream));
      return;
    }
    const long long c = bk.n / world, o = bk.off + rank * c;
    SPECSIM_NCCL(nccl::api().ReduceScatter(G + bk.off, G + o, static_cast<size_t>(c), ncclFloat,
                                           ncclSum, comm, comm_stream));
    kern::adamw(c, P + o, Mst + o, Vst + o, G + o, P16 + o, adam_dev, comm_stream);
    SPECSIM_NCCL(nccl::api().AllGather(P16 + o, P16 + bk.off, static_cast<size_t>(c),
                                       ncclBfloat16, comm, comm_stream));
  }

  // ZeRO-1 keeps each rank's fp32 master current on its own shards only:
  // all-gather them (collective: every rank must call it, same order).
  void sync_master() {
    if (!zero || world == 1) return;
    for (const auto& bk : buckets) {
      const long long c = bk.n / world, o = bk.off + rank * c;
      SPECSIM_NCCL(nccl::api().AllGather(P + o, P + bk.off, static_cast<size_t>(c), ncclFloat,
                                         comm, stream));
    }
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
  }

  // Attention backward of pass j (K > 1): D_j, the cache entries (j >= 1),
  // dQ_j against step 0's keys; dK / dV of pass 0's keys from every pass's
  // queries once the last pass (j == 0) is reached.
  void attn_backward_pass(int j) {
    const long long R = j * T;
    attn::Dims ad = attn_dims(j);
    ad.rope_cos = cos_tr;
    ad.rope_sin = sin_tr;
    float* D = Dattn + R * sh.n_heads;
    const float* l = lse_attn + R * sh.n_heads;
    timed(PH_ATTN, attn_flops(j, true), [&] {
      attn::bwd_dot(dO + R * Q, o + R * Q, D, ad, sh.head_dim, stream);
      if (j > 0)
        attn::bwd_diag(qkv, dO + R * Q, l, D, dq_add, dkv_acc, dqkv + R * NQ, ad, sh.head_dim,
                       stream);
      attn::bwd_dq(qkv, dO + R * Q, l, D, j > 0 ? dq_add : nullptr, dqkv + R * NQ, ad,
                   sh.head_dim, stream);
      if (j == 0)
        attn::bwd_dkdv(qkv, dO, lse_attn, Dattn, dqkv, ad, sh.head_dim, K, stream);
    });
  }

  void backward() {
    const int S = sh.seq_len;
    bucket_next = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const long long v0 = c * Vc, vn = std::min(Vc, V - v0);
      if (keep_logits)
        timed(PH_LM, 0, [&] {
          kern::ce_grad(logits, V, partials, lse, coef, y, static_cast<int>(v0), KT,
                        static_cast<int>(vn), dlog, Vc, stream);
        });
      else
        run(p_ce_bwd[c], PH_LM, 0.0);  // logit recompute: not algorithmic work
      run(p_lm_dx[c], PH_LM);
      run_dw(p_lm_dw[c], f_lm_dw[c], PH_LM);
      // LM-head rows of this chunk are final: their all-reduce overlaps the rest
      bucket_ready(c);
    }
    if (K > 1)
      timed(PH_ELEM, 0, [&] {
        SPECSIM_CUDA(cudaMemsetAsync(dkv_acc, 0, sizeof(float) * KT * 2 * KV, stream));
      });
    // One pass: each norm backward produces dx and its weight gradient in one
    // launch.  K passes: dx per pass (in reverse: pass j's input gradient dg
    // flows into pass j-1's output h), weight gradients once over all K*T rows.
    const bool one = K == 1;
    for (int j = K - 1; j >= 0; --j) {
      const long long R = j * T;
      timed(PH_ELEM, 0, [&] {
        kern::rmsnorm_bwd(dn + R * H, H, h + R * H, H, nullptr, pf("w_fin"), rstd_fin + R,
                          j < K - 1 ? dg_in : nullptr, dh, dh_b + R * H, H,
                          one ? gf("w_fin") : nullptr, one ? dw_part : dwp_fin + j * nbT * H, T,
                          sh.hidden, stream);
        if (j == 0 && !one) kern::colsum(dwp_fin, K * nbT, sh.hidden, gf("w_fin"), stream);
      });
      run(p_dact[j]);
      if (j == 0) {
        run_dw(p_dw_down, f_dw_down);
        bucket_ready(n_chunks);  // down, w_fin
      }
      if (!swiglu_fused)
        timed(PH_ELEM, 0, [&] {
          kern::swiglu_bwd(gu + R * 2 * I, dact, dgu + R * 2 * I, T, sh.ffn, stream);
        });
      run(p_dz[j]);
      if (j == 0) {
        run_dw(p_dw_gu, f_dw_gu);
        bucket_ready(n_chunks + 1);  // gate_up
      }
      timed(PH_ELEM, 0, [&] {
        kern::rmsnorm_bwd(dz + R * H, H, r + R * H, H, nullptr, pf("w_post"), rstd_post + R, dh,
                          dr, dr_b + R * H, H, one ? gf("w_post") : nullptr,
                          one ? dw_part : dwp_post + j * nbT * H, T, sh.hidden, stream);
      });
      run(p_dO[j]);
      if (j == 0) {
        if (!one)
          timed(PH_ELEM, 0, [&] {
            kern::colsum(dwp_post, K * nbT, sh.hidden, gf("w_post"), stream);
          });
        run_dw(p_dw_o, f_dw_o);
        bucket_ready(n_chunks + 2);  // o, w_post
      }
      if (one) {
        attn::Dims ad = attn_dims();
        ad.rope_cos = cos_tr;
        ad.rope_sin = sin_tr;
        bool rope_fused = false;
        timed(PH_ATTN, attn_flops(0, true), [&] {
          rope_fused = attn::backward(qkv, o, dO, lse_attn, Dattn, dqkv, ad, sh.head_dim, stream);
        });
        if (!rope_fused)
          timed(PH_ELEM, 0, [&] {
            kern::rope(dqkv, T, S, static_cast<int>(NQ), sh.n_heads + sh.n_kv_heads,
                       sh.head_dim, cos_t, sin_t, true, stream);
          });
      } else {
        attn_backward_pass(j);
      }
      run(p_dU[j]);
      if (j == 0) {
        run_dw(p_dw_qkv, f_dw_qkv);
        bucket_ready(n_chunks + 3);  // qkv
      }
      timed(PH_ELEM, 0, [&] {
        float* dUj = dU + R * 2 * H;
        if (one)  // w_in: embedding is frozen, only the weight gradient is needed
          kern::rmsnorm_bwd(dU, 2 * H, E, H, u, pf("w_in"), rstd_a, nullptr, nullptr, nullptr, H,
                            gf("w_in"), dw_part, T, sh.hidden, stream);
        // hidden norm: dg = dr + d/dg RMSNorm(g); pass 0's bf16 copy feeds dW_fc,
        // a later pass's fp32 dg flows into the previous pass's output
        kern::rmsnorm_bwd(dUj + H, 2 * H, g + R * H, H, nullptr, pf("w_hid"), rstd_b + R, dr,
                          j > 0 ? dg_in : nullptr, j > 0 ? nullptr : dg_b, H,
                          one ? gf("w_hid") : nullptr, one ? dw_part : dwp_hid + j * nbT * H, T,
                          sh.hidden, stream);
        if (j == 0 && !one) {
          // w_in has no dx (frozen embedding): one dw pass over every pass's rows
          kern::rmsnorm_bwd(dU, 2 * H, E, H, u, pf("w_in"), rstd_a, nullptr, nullptr, nullptr, H,
                            gf("w_in"), dw_part, KT, sh.hidden, stream);
          kern::colsum(dwp_hid, K * nbT, sh.hidden, gf("w_hid"), stream);
        }
      });
    }
    if (f_direct)
      run_dw(cur_ring->dw_fc, cur_ring->f_dw_fc);
    else
      run_dw(p_dw_fc, f_dw_fc);
    bucket_ready(n_chunks + 4);  // fc, w_in, w_hid
    if (use_nccl) {
      // join: AdamW waits for every bucket
      timed(PH_COMM, 0, [&] {
        SPECSIM_CUDA(cudaEventRecord(ev_comm_done, comm_stream));
        SPECSIM_CUDA(cudaStreamWaitEvent(stream, ev_comm_done, 0));
      });
    }
  }

  void snapshot() {
    SPECSIM_CUDA(cudaSetDevice(device));
    sync_master();
    const size_t f = sizeof(float) * static_cast<size_t>(total);
    if (!snap) SPECSIM_CUDA(cudaMalloc(&snap, 3 * f + sizeof(__nv_bfloat16) * total));
    char* s = static_cast<char*>(snap);
    SPECSIM_CUDA(cudaMemcpyAsync(s, P, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(s + f, Mst, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(s + 2 * f, Vst, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(s + 3 * f, P16, sizeof(__nv_bfloat16) * total,
                                 cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
    snap_step = step_count;
    snap_version = version;
  }
  void restore() {
    if (snap_step < 0) throw std::invalid_argument("restore: no snapshot taken");
    SPECSIM_CUDA(cudaSetDevice(device));
    const size_t f = sizeof(float) * static_cast<size_t>(total);
    const char* s = static_cast<const char*>(snap);
    SPECSIM_CUDA(cudaMemcpyAsync(P, s, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(Mst, s + f, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(Vst, s + 2 * f, f, cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaMemcpyAsync(P16, s + 3 * f, sizeof(__nv_bfloat16) * total,
                                 cudaMemcpyDeviceToDevice, stream));
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
    step_count = snap_step;
    version = snap_version;  // the restored model is the snapshot's version
  }

  kern::AdamHyper next_hyper() const { return hyper_for(step_count + 1); }
  kern::AdamHyper hyper_for(int64_t k) const {
    const double bc1 = 1.0 - std::pow(static_cast<double>(opt.beta1), static_cast<double>(k));
    const double bc2 = 1.0 - std::pow(static_cast<double>(opt.beta2), static_cast<double>(k));
    kern::AdamHyper hp;
    hp.lr = opt.lr;
    hp.beta1 = opt.beta1;
    hp.beta2 = opt.beta2;
    hp.eps = opt.eps;
    hp.decay = 1.0f - opt.lr * opt.weight_decay;
    hp.step_size = static_cast<float>(opt.lr / bc1);
    hp.bc2_sqrt = static_cast<float>(std::sqrt(bc2));
    return hp;
  }

  // Host: fill the next pinned slot and enqueue its fetch into d_in (stream
  // ordered before the step's launch, after the previous step).  A slot is
  // reused only once the fetch issued from it two steps ago has executed.
  StepInputs make_inputs(const kern::BatchSpec& spec, int64_t global_valid, bool train,
                         int64_t step_k) const {
    StepInputs s{};
    s.spec = spec;
    s.nglobal = global_valid > 0 ? global_valid : 0;
    if (train) {
      const kern::AdamHyper hp = hyper_for(step_k);
      s.hp = gemm::AdamDev{hp.lr, hp.beta1, hp.beta2, hp.eps, hp.decay, hp.step_size,
                           hp.bc2_sqrt, 0.f};
    }
    return s;
  }

  void stage(const kern::BatchSpec& spec, int64_t global_valid, bool train) {
    in_slot ^= 1;
    SPECSIM_CUDA(cudaEventSynchronize(in_ev[in_slot]));
    StepInputs& s = h_in[in_slot];
    s.spec = spec;
    s.nglobal = global_valid > 0 ? global_valid : 0;
    if (train) {
      const kern::AdamHyper hp = next_hyper();
      s.hp = gemm::AdamDev{hp.lr, hp.beta1, hp.beta2, hp.eps, hp.decay, hp.step_size,
                           hp.bc2_sqrt, 0.f};
    }
    // SM loads from mapped pinned memory, not a copy-engine H2D: the latter
    // would wait behind whatever ingest DMA the caller queued before this step
    static_assert(sizeof(StepInputs) % 4 == 0, "StepInputs is copied in words");
    kern::fetch_mapped(reinterpret_cast<const uint32_t*>(&s), reinterpret_cast<uint32_t*>(d_in),
                       static_cast<int>(sizeof(StepInputs) / 4), stream);
    SPECSIM_CUDA(cudaEventRecord(in_ev[in_slot], stream));
  }

  // AdamW fused into the weight-gradient epilogues: single replica only (the
  // data-parallel path needs the all-reduced gradient first).
  // SPECSIM_NO_FUSED_ADAMW=1 selects the standalone kernel (A/B experiments).
  bool fused_adamw() const {
    static const bool off = [] {
      const char* e = std::getenv("SPECSIM_NO_FUSED_ADAMW");
      return e && e[0] == '1';
    }();
    return !use_nccl && !off;
  }

  void optimizer_update() {
    if (zero) return;  // every shard was updated on the comm stream (bucket_ready)
    if (!fused_adamw()) {
      timed(PH_ADAM, 0, [&] { kern::adamw(total, P, Mst, Vst, G, P16, adam_dev, stream); });
      return;
    }
    // GEMM weights were updated in their dW epilogues; the norm weights remain
    timed(PH_ADAM, 0, [&] {
      const auto& a = param("w_in");  // w_in, w_hid contiguous
      const auto& b = param("w_post");
      const auto& c = param("w_fin");
      kern::adamw(2 * H, P + a.off, Mst + a.off, Vst + a.off, G + a.off, P16 + a.off, adam_dev,
                  stream);
      kern::adamw(H, P + b.off, Mst + b.off, Vst + b.off, G + b.off, P16 + b.off, adam_dev, stream);
      kern::adamw(H, P + c.off, Mst + c.off, Vst + c.off, G + c.off, P16 + c.off, adam_dev, stream);
    });
  }

  // the step's loss / valid / correct (3 doubles) into mapped pinned memory
  // by a one-warp kernel: a D2H copy-engine transfer here would queue behind
  // ingest DMA the caller issued earlier and stall every later step
  void stats_to_host(double* dst_mapped) {
    kern::store_mapped(reinterpret_cast<const uint32_t*>(stats),
                       reinterpret_cast<uint32_t*>(dst_mapped), 6, stream);
  }

  // per-phase device time of the last launch (its timestamp events are the
  // last replay's when the step ran as a graph); call after a stream sync
  void collect_phases() {
    for (int i = 0; i < PH_N; ++i) {
      phase_ms[i] = 0;
      phase_flops[i] = rec->flops[i];
      phase_launches[i] = rec->launches[i];
    }
    if (timing)
      for (auto& mk : rec->marks) {
        float tm = 0;
        SPECSIM_CUDA(cudaEventElapsedTime(&tm, mk.second.first, mk.second.second));
        phase_ms[mk.first] += tm;
      }
  }

  StepResult end_step() {
    SPECSIM_CUDA(cudaEventRecord(ev_end, stream));
    stats_to_host(h_stats);
    SPECSIM_CHECK_LAUNCH();
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
    float ms = 0;
    SPECSIM_CUDA(cudaEventElapsedTime(&ms, ev_begin, ev_end));
    last_ms = ms;
    collect_phases();
    StepResult res;
    res.loss = h_stats[0];
    res.valid_tokens = static_cast<int64_t>(h_stats[1]);
    res.top1_correct = static_cast<int64_t>(h_stats[2]);
    res.positions = T * world;
    res.ms = ms;
    return res;
  }

  void allreduce_stats() {
    if (!use_nccl) return;
    // loss is already normalised by the global count: sum over ranks
    timed(PH_COMM, 0, [&] {
      SPECSIM_NCCL(nccl::api().AllReduce(stats, stats, 3, ncclDouble, ncclSum, comm, stream));
    });
  }

  // The device work of one step (train) or one forward (eval).
  void enqueue(HiddenStateBuffer& buf, bool train) {
    forward(buf, train ? K : 1);
    if (train) {
      backward();  // includes the bucketed gradient all-reduce when data-parallel
      optimizer_update();
    }
    allreduce_stats();
  }

  // Runs enqueue() eagerly, or replays (capturing on first use) a CUDA graph of
  // it: one launch per step instead of ~60, no idle gaps while the host
  // enqueues.  Graphs are keyed by (train, timing, keep_grads, buffer).
  void launch(HiddenStateBuffer& buf, bool train) {
    if (!use_graphs) {
      eager_rec.reset();
      rec = &eager_rec;
      SPECSIM_CUDA(cudaEventRecord(ev_begin, stream));
      enqueue(buf, train);
      return;
    }
    auto key = std::make_tuple(train, timing, keep_grads, buf.serial());
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      auto r = std::make_unique<Recording>();
      rec = r.get();
      cudaGraph_t g = nullptr;
      SPECSIM_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      const unsigned long long k0 = g_kernel_launches.load();
      try {
        enqueue(buf, train);
      } catch (...) {
        capturing = false;
        cudaStreamEndCapture(stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      capturing = false;
      // captured launches are not executions: count them on every replay instead
      r->kernels = g_kernel_launches.load() - k0;
      g_kernel_launches.fetch_sub(r->kernels);
      SPECSIM_CUDA(cudaStreamEndCapture(stream, &g));
      SPECSIM_CUDA(cudaGraphInstantiate(&r->exec, g, 0));
      SPECSIM_CUDA(cudaGraphDestroy(g));
      it = graphs.emplace(key, std::move(r)).first;
    }
    rec = it->second.get();
    SPECSIM_CUDA(cudaEventRecord(ev_begin, stream));
    SPECSIM_CUDA(cudaGraphLaunch(rec->exec, stream));
    count_launches(static_cast<unsigned>(rec->kernels));
  }

  // Host-side preparation shared by step / eval: batch spec + inputs staged,
  // and the stream ordered after the appends that wrote this batch's samples
  // only (so copies issued for later steps keep overlapping: async ingest).
  void prepare(HiddenStateBuffer& buf, const int64_t* ids, int n, int64_t global_valid,
               bool train) {
    const kern::BatchSpec spec = batch_spec(buf, ids, n);
    if (f_direct) cur_ring = &ring_plans_for(buf);  // host-side plan, before any capture
    last_ring = buf.ring_features();
    if (void* ev = buf.event_for(wait_seq))
      SPECSIM_CUDA(cudaStreamWaitEvent(stream, static_cast<cudaEvent_t>(ev), 0));
    stage(spec, global_valid, train);
  }

  StepResult step(HiddenStateBuffer& buf, const int64_t* ids, int n, int64_t global_valid) {
    DeviceGuard dg(device);
    prepare(buf, ids, n, global_valid, true);
    launch(buf, true);
    step_count += 1;
    return end_step();
  }

  StepResult eval(HiddenStateBuffer& buf, const int64_t* ids, int n) {
    DeviceGuard dg(device);
    prepare(buf, ids, n, 0, false);
    launch(buf, false);
    return end_step();
  }

  // sample i of step k's slice -> rank i mod world (same rule as specsim_dp_shard)
  void shard(long long n, long long k, std::vector<int64_t>& mine,
             const std::vector<int64_t>& ids) const {
    mine.clear();
    int64_t idx[kern::kMaxBatch];
    int32_t cnt = 0;
    if (specsim_dp_shard(n, sh.micro_batch, world, rank, k, idx, &cnt) != SPECSIM_OK)
      throw std::invalid_argument(specsim_last_error());
    for (int i = 0; i < cnt; ++i) mine.push_back(ids[idx[i]]);
  }

  // Every sample this rank will read must be resident BEFORE the first launch:
  // a lazily discovered eviction would throw after earlier steps had already
  // updated the weights (and, data-parallel, leave the other ranks blocked in
  // a collective).  The verdict is combined over ranks, so all fail together.
  void check_resident(HiddenStateBuffer& buf, const TrainJob& job) {
    const long long per_step = static_cast<long long>(sh.micro_batch) * world;
    std::vector<int64_t> mine, missing;
    auto scan = [&](const std::vector<int64_t>& ids) {
      const long long n = static_cast<long long>(ids.size());
      for (long long s0 = 0, j = 0; s0 < n; s0 += per_step, ++j) {
        shard(n, j, mine, ids);
        for (int64_t id : mine) {
          try {
            buf.sample(id);
          } catch (const std::out_of_range&) {
            missing.push_back(id);
          }
        }
      }
    };
    scan(job.train_ids);
    scan(job.eval_ids);
    long long any = static_cast<long long>(missing.size());
    if (use_nccl) {
      *h_nglobal = any;
      SPECSIM_CUDA(cudaMemcpyAsync(n_counted, h_nglobal, sizeof(long long),
                                   cudaMemcpyHostToDevice, stream));
      SPECSIM_NCCL(nccl::api().AllReduce(n_counted, n_counted, 1, ncclInt64, ncclSum, comm, stream));
      SPECSIM_CUDA(cudaMemcpyAsync(h_nglobal, n_counted, sizeof(long long),
                                   cudaMemcpyDeviceToHost, stream));
      SPECSIM_CUDA(cudaStreamSynchronize(stream));
      any = *h_nglobal;
    }
    if (any == 0) return;
    std::string m = "train job: " + std::to_string(any) +
                    " sample(s) not resident in the signal buffer (evicted or unknown)";
    if (!missing.empty()) {
      m += "; on this rank:";
      for (size_t i = 0; i < missing.size() && i < 8; ++i) m += " " + std::to_string(missing[i]);
    }
    throw std::invalid_argument(m + "; nothing was trained");
  }

  // train(job): every step and eval forward is enqueued back-to-back (no host
  // synchronisation between steps); per-step loss / counters are copied into a
  // pinned history and read once at the end.
  TrainingOutcome train(HiddenStateBuffer& buf, const TrainJob& job) {
    Problems p("train job");
    p.check(!job.train_ids.empty(), "D_train must be non-empty (SPEC.md:398 requires n > 0)");
    p.check(job.epochs >= 1, "epochs must be >= 1");
    p.throw_if_any();
    DeviceGuard dg(device);
    const auto t0 = std::chrono::steady_clock::now();
    const long long per_step = static_cast<long long>(sh.micro_batch) * world;
    const long long n = static_cast<long long>(job.train_ids.size());
    const long long ne = static_cast<long long>(job.eval_ids.size());
    check_resident(buf, job);
    const long long train_steps = ((n + per_step - 1) / per_step) * job.epochs;
    const long long eval_steps = (ne + per_step - 1) / per_step;
    const long long total_launch = train_steps + eval_steps;
    // pinned per-step history, grown on demand and kept (pinning is slow)
    const size_t need = static_cast<size_t>(3 * (total_launch > 0 ? total_launch : 1));
    if (need > hist_cap) {
      if (hist_buf) cudaFreeHost(hist_buf);
      hist_buf = nullptr;
      SPECSIM_CUDA(cudaHostAlloc(&hist_buf, sizeof(double) * need * 2, cudaHostAllocMapped));
      hist_cap = need * 2;
    }
    double* hist = hist_buf;
    // every launch's inputs up front (mapped pinned table -> device once)
    if (static_cast<size_t>(total_launch) > job_cap) {
      SPECSIM_CUDA(cudaStreamSynchronize(stream));
      if (h_job) cudaFreeHost(h_job);
      if (d_job) cudaFree(d_job);
      h_job = nullptr;
      d_job = nullptr;
      job_cap = static_cast<size_t>(total_launch) * 2;
      SPECSIM_CUDA(cudaHostAlloc(&h_job, sizeof(StepInputs) * job_cap, cudaHostAllocMapped));
      SPECSIM_CUDA(cudaMalloc(&d_job, sizeof(StepInputs) * job_cap));
    }
    std::vector<int64_t> mine, waits(static_cast<size_t>(total_launch));
    std::vector<char> is_train(static_cast<size_t>(total_launch));
    {
      long long k = 0;
      int64_t sc = step_count;
      for (int ep = 0; ep < job.epochs; ++ep)
        for (long long s0 = 0, j = 0; s0 < n; s0 += per_step, ++j, ++k) {
          shard(n, j, mine, job.train_ids);
          const kern::BatchSpec spec = batch_spec(buf, mine.data(), static_cast<int>(mine.size()));
          waits[k] = wait_seq;
          is_train[k] = 1;
          h_job[k] = make_inputs(spec, 0, true, ++sc);
        }
      for (long long s0 = 0, j = 0; s0 < ne; s0 += per_step, ++j, ++k) {
        shard(ne, j, mine, job.eval_ids);
        const kern::BatchSpec spec = batch_spec(buf, mine.data(), static_cast<int>(mine.size()));
        waits[k] = wait_seq;
        is_train[k] = 0;
        h_job[k] = make_inputs(spec, 0, false, 0);
      }
    }
    if (f_direct) cur_ring = &ring_plans_for(buf);
    last_ring = buf.ring_features();
    static_assert(sizeof(StepInputs) % 4 == 0, "StepInputs is copied in words");
    const int words = static_cast<int>(sizeof(StepInputs) / 4);
    kern::fetch_mapped(reinterpret_cast<const uint32_t*>(h_job), reinterpret_cast<uint32_t*>(d_job),
                       words * static_cast<int>(total_launch), stream);
    for (long long k = 0; k < total_launch; ++k) {
      if (void* ev = buf.event_for(waits[k]))
        SPECSIM_CUDA(cudaStreamWaitEvent(stream, static_cast<cudaEvent_t>(ev), 0));
      kern::fetch_mapped(reinterpret_cast<const uint32_t*>(d_job + k),
                         reinterpret_cast<uint32_t*>(d_in), words, stream);  // device -> device
      launch(buf, is_train[k] != 0);  // records ev_begin right before the graph launch
      if (is_train[k]) step_count += 1;
      stats_to_host(hist + 3 * k);
    }
    SPECSIM_CUDA(cudaEventRecord(ev_end, stream));  // last launch: ev_begin .. ev_end
    SPECSIM_CHECK_LAUNCH();
    SPECSIM_CUDA(cudaStreamSynchronize(stream));
    if (total_launch > 0) SPECSIM_CUDA(cudaEventElapsedTime(&last_ms, ev_begin, ev_end));
    // phase times of the job's last step (back-to-back with the steps before
    // it, i.e. at the steady-state clock of a long job)
    if (total_launch > 0) collect_phases();
    double loss_sum = 0;
    for (long long i = 0; i < train_steps; ++i) loss_sum += hist[3 * i];
    double valid = 0, correct = 0;
    for (long long i = train_steps; i < total_launch; ++i) {
      valid += hist[3 * i + 1];
      correct += hist[3 * i + 2];
    }
    const auto t1 = std::chrono::steady_clock::now();
    TrainingOutcome out;
    out.duration_hours = std::chrono::duration<double>(t1 - t0).count() / 3600.0;
    out.alpha_eval = valid > 0 ? correct / valid : 0.0;
    out.new_version = ++version;
    out.steps = train_steps;
    out.mean_loss = train_steps ? loss_sum / static_cast<double>(train_steps) : 0.0;
    return out;
  }
};

DraftTrainer::DraftTrainer(const DraftShape& shape, const AdamWConfig& opt, uint64_t seed,
                           int rank, int world, const uint8_t* nccl_id, int device)
    : impl_(std::make_unique<DraftTrainerImpl>(shape, opt, seed, rank, world, nccl_id, device)) {}
DraftTrainer::~DraftTrainer() = default;
StepResult DraftTrainer::step(HiddenStateBuffer& buf, const int64_t* ids, int n,
                              int64_t global_valid) {
  return impl_->step(buf, ids, n, global_valid);
}
StepResult DraftTrainer::eval(HiddenStateBuffer& buf, const int64_t* ids, int n) {
  return impl_->eval(buf, ids, n);
}
TrainingOutcome DraftTrainer::train(HiddenStateBuffer& buf, const TrainJob& job) {
  return impl_->train(buf, job);
}
void DraftTrainer::snapshot() { impl_->snapshot(); }
void DraftTrainer::restore() { impl_->restore(); }

}  // namespace specsim

// ================================================================== C ABI
using namespace specsim;


namespace {
DraftTrainerImpl& impl_of(const specsim_trainer* t) {
  if (!t || !t->t) throw std::invalid_argument("null trainer");
  return const_cast<DraftTrainer*>(t->t)->impl();
}
DraftShape to_shape(const specsim_draft_shape* shape) {
  if (!shape) throw std::invalid_argument("null shape");
  DraftShape s;
  s.hidden = shape->hidden;
  s.vocab = shape->vocab;
  s.seq_len = shape->seq_len;
  s.n_heads = shape->n_heads;
  s.n_kv_heads = shape->n_kv_heads;
  s.head_dim = shape->head_dim;
  s.ffn = shape->ffn;
  s.layers_tapped = shape->layers_tapped;
  s.micro_batch = shape->micro_batch;
  s.rms_eps = shape->rms_eps;
  s.rope_theta = shape->rope_theta;
  s.ttt_steps = shape->ttt_steps > 0 ? shape->ttt_steps : 1;
  s.ttt_decay = shape->ttt_decay > 0.f ? shape->ttt_decay : 0.8f;
  return s;
}

void fill(specsim_step_result* out, const StepResult& r) {
  if (!out) return;
  out->loss = r.loss;
  out->valid_tokens = r.valid_tokens;
  out->top1_correct = r.top1_correct;
  out->positions = r.positions;
  out->ms = r.ms;
}
}  // namespace

extern "C" {

int specsim_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    if (!out128) throw std::invalid_argument("null output");
    ncclUniqueId id;
    SPECSIM_NCCL(nccl::api().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int specsim_trainer_create(const specsim_draft_shape* shape, const specsim_adamw* opt,
                           uint64_t seed, int rank, int world, const uint8_t* nccl_id, int device,
                           specsim_trainer** out) {
  return guard([&] {
    if (!shape || !out) throw std::invalid_argument("null argument");
    const DraftShape s = to_shape(shape);
    AdamWConfig a;
    if (opt) {
      a.lr = opt->lr;
      a.beta1 = opt->beta1;
      a.beta2 = opt->beta2;
      a.eps = opt->eps;
      a.weight_decay = opt->weight_decay;
    }
    *out = new specsim_trainer{new DraftTrainer(s, a, seed, rank, world, nccl_id, device)};
  });
}

int specsim_dp_buckets(const specsim_draft_shape* shape, int32_t world, int64_t* off, int64_t* n,
                       int32_t cap, int32_t* count, int32_t* zero_ok) {
  return guard([&] {
    const DraftShape s = to_shape(shape);
    // layout only: the kernel constraints of validate() do not apply here
    Problems p("invalid draft shape");
    p.check(s.hidden > 0 && s.vocab > 0 && s.ffn > 0 && s.n_heads > 0 && s.n_kv_heads > 0 &&
                s.head_dim > 0 && s.layers_tapped > 0,
            "dimensions must be positive");
    p.check(world >= 1, "world must be >= 1");
    p.throw_if_any();
    const auto b = dp_buckets(s);
    if (count) *count = static_cast<int32_t>(b.size());
    for (size_t i = 0; i < b.size() && static_cast<int32_t>(i) < cap; ++i) {
      if (off) off[i] = b[i].off;
      if (n) n[i] = b[i].n;
    }
    if (zero_ok) *zero_ok = zero_shardable(b, world) ? 1 : 0;
  });
}

int specsim_trainer_destroy(specsim_trainer* t) {
  return guard([&] {
    if (!t) return;
    delete t->t;
    delete t;
  });
}

int specsim_trainer_step(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* ids, int32_t n,
                         int64_t global_valid, specsim_step_result* out) {
  return guard([&] {
    auto& im = impl_of(t);
    if (n > 0 && !ids) throw std::invalid_argument("null sample ids");
    fill(out, im.step(*hsbuf_unwrap(buf), ids, n, global_valid));
  });
}

int specsim_trainer_eval(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* ids, int32_t n,
                         specsim_step_result* out) {
  return guard([&] {
    auto& im = impl_of(t);
    if (n > 0 && !ids) throw std::invalid_argument("null sample ids");
    fill(out, im.eval(*hsbuf_unwrap(buf), ids, n));
  });
}

int specsim_trainer_train(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* train_ids,
                          int64_t n_train, const int64_t* eval_ids, int64_t n_eval,
                          int32_t epochs, specsim_training_outcome* out) {
  return guard([&] {
    auto& im = impl_of(t);
    TrainJob job;
    if (n_train > 0) job.train_ids.assign(train_ids, train_ids + n_train);
    if (n_eval > 0) job.eval_ids.assign(eval_ids, eval_ids + n_eval);
    job.epochs = epochs;
    const TrainingOutcome o = im.train(*hsbuf_unwrap(buf), job);
    if (out) {
      out->duration_hours = o.duration_hours;
      out->alpha_eval = o.alpha_eval;
      out->new_version = o.new_version;
      out->mean_loss = o.mean_loss;
      out->steps = o.steps;
    }
  });
}

int specsim_trainer_num_params(const specsim_trainer* t, int32_t* count, int64_t* total_elems) {
  return guard([&] {
    auto& im = impl_of(t);
    if (count) *count = static_cast<int32_t>(im.params.size());
    if (total_elems) *total_elems = im.total;
  });
}

int specsim_trainer_param_info(const specsim_trainer* t, int32_t index, const char** name,
                               int64_t* rows, int64_t* cols) {
  return guard([&] {
    auto& im = impl_of(t);
    if (index < 0 || index >= static_cast<int32_t>(im.params.size()))
      throw std::invalid_argument("parameter index out of range");
    const auto& p = im.params[index];
    if (name) *name = p.name.c_str();
    if (rows) *rows = p.rows;
    if (cols) *cols = p.cols;
  });
}

int specsim_trainer_get_param(const specsim_trainer* t, const char* name, float* host_out) {
  return guard([&] {
    auto& im = impl_of(t);
    const auto& p = im.param(name ? name : "");
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    im.sync_master();
    SPECSIM_CUDA(cudaMemcpy(host_out, im.P + p.off, sizeof(float) * p.rows * p.cols,
                            cudaMemcpyDeviceToHost));
  });
}

int specsim_trainer_set_param(specsim_trainer* t, const char* name, const float* host_in) {
  return guard([&] {
    auto& im = impl_of(t);
    const auto& p = im.param(name ? name : "");
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    SPECSIM_CUDA(cudaMemcpy(im.P + p.off, host_in, sizeof(float) * p.rows * p.cols,
                            cudaMemcpyHostToDevice));
    kern::f32_to_bf16(im.P + p.off, im.P16 + p.off, p.rows * p.cols, im.stream);
    SPECSIM_CHECK_LAUNCH();
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
  });
}

int specsim_trainer_get_grad(const specsim_trainer* t, const char* name, float* host_out) {
  return guard([&] {
    auto& im = impl_of(t);
    const auto& p = im.param(name ? name : "");
    if (im.fused_adamw() && !im.keep_grads && !p.norm)
      throw std::invalid_argument(
          "gradients of GEMM weights are consumed by the fused AdamW epilogue; enable "
          "specsim_trainer_keep_grads before the step to materialise them");
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    SPECSIM_CUDA(cudaMemcpy(host_out, im.G + p.off, sizeof(float) * p.rows * p.cols,
                            cudaMemcpyDeviceToHost));
  });
}

int specsim_trainer_set_embedding(specsim_trainer* t, const uint16_t* host_bf16) {
  return guard([&] {
    auto& im = impl_of(t);
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    SPECSIM_CUDA(cudaMemcpy(im.E, host_bf16, 2 * im.V * im.H, cudaMemcpyHostToDevice));
  });
}

int specsim_trainer_get_embedding(const specsim_trainer* t, uint16_t* host_bf16) {
  return guard([&] {
    auto& im = impl_of(t);
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    SPECSIM_CUDA(cudaMemcpy(host_bf16, im.E, 2 * im.V * im.H, cudaMemcpyDeviceToHost));
  });
}

int specsim_trainer_snapshot(specsim_trainer* t) {
  return guard([&] { t->t->snapshot(); });
}
int specsim_trainer_restore(specsim_trainer* t) {
  return guard([&] { t->t->restore(); });
}
int specsim_trainer_set_step_count(specsim_trainer* t, int64_t step) {
  return guard([&] {
    if (step < 0) throw std::invalid_argument("step must be >= 0");
    impl_of(t).step_count = step;
  });
}

int specsim_trainer_region(specsim_trainer* t, int end, double* ms) {
  return guard([&] {
    auto& im = impl_of(t);
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaEventRecord(im.ev_region[end ? 1 : 0], im.stream));
    if (end) {
      SPECSIM_CUDA(cudaEventSynchronize(im.ev_region[1]));
      float v = 0;
      SPECSIM_CUDA(cudaEventElapsedTime(&v, im.ev_region[0], im.ev_region[1]));
      if (ms) *ms = v;
    }
  });
}

int specsim_trainer_read_rows(const specsim_trainer* t, const char* name, void* host_out,
                              int64_t cap_elems, int64_t* n_elems) {
  return guard([&] {
    auto& im = impl_of(t);
    const std::string nm = name ? name : "";
    const void* src = nullptr;
    size_t esz = 4;
    long long n = im.KT;
    if (nm == "u") src = im.u;
    else if (nm == "y") src = im.y;
    else if (nm == "m") src = im.m;
    else if (nm == "argmax") src = im.argmax;
    else if (nm == "lse") src = im.lse;
    else if (nm == "F") {
      // the rows the fc GEMM read: the gathered copy, or (direct path) the
      // ring's 64-row blocks named by the step's block table
      n = im.T * im.W3;
      if (n_elems) *n_elems = n;
      if (!host_out) return;
      if (cap_elems < n) throw std::invalid_argument("host buffer too small");
      DeviceGuard dg(im.device);
      SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
      const size_t row = static_cast<size_t>(im.W3) * 2;
      if (!im.f_direct) {
        SPECSIM_CUDA(cudaMemcpy(host_out, im.F, row * im.T, cudaMemcpyDeviceToHost));
        return;
      }
      if (!im.last_ring) throw std::invalid_argument("no step has run yet");
      std::vector<int32_t> blk(static_cast<size_t>(im.T / 64));
      SPECSIM_CUDA(cudaMemcpy(blk.data(), im.blk_rows, sizeof(int32_t) * blk.size(),
                              cudaMemcpyDeviceToHost));
      for (size_t b = 0; b < blk.size(); ++b)
        SPECSIM_CUDA(cudaMemcpy(static_cast<uint8_t*>(host_out) + b * 64 * row,
                                static_cast<const uint8_t*>(im.last_ring) + blk[b] * row,
                                64 * row, cudaMemcpyDeviceToHost));
      return;
    } else
      throw std::invalid_argument("unknown row buffer '" + nm + "'");
    if (n_elems) *n_elems = n;
    if (!host_out) return;
    if (cap_elems < n) throw std::invalid_argument("host buffer too small");
    DeviceGuard dg(im.device);
    SPECSIM_CUDA(cudaStreamSynchronize(im.stream));
    SPECSIM_CUDA(cudaMemcpy(host_out, src, esz * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
  });
}

int specsim_trainer_keep_grads(specsim_trainer* t, int enabled) {
  return guard([&] { impl_of(t).keep_grads = enabled != 0; });
}

int specsim_trainer_set_timing(specsim_trainer* t, int enabled) {
  return guard([&] { impl_of(t).timing = enabled != 0; });
}

int specsim_trainer_last_step_ms(const specsim_trainer* t, double* ms) {
  return guard([&] {
    if (!ms) throw std::invalid_argument("null output");
    *ms = impl_of(t).last_ms;
  });
}

int specsim_trainer_phase_times(const specsim_trainer* t, double* ms7, double* flops7,
                                int32_t* launches7) {
  return guard([&] {
    auto& im = impl_of(t);
    for (int i = 0; i < PH_N; ++i) {
      if (ms7) ms7[i] = im.phase_ms[i];
      if (flops7) flops7[i] = im.phase_flops[i];
      if (launches7) launches7[i] = im.phase_launches[i];
    }
  });
}

}  // extern "C"
