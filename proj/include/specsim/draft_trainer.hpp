// C++ API of the B200-native TIDE draft-training hot path.
//
// Lives where the reference keeps its public headers (proj/include/specsim/)
// so it drops in next to errors.hpp / rng.hpp / perf_model.hpp /
// workload.hpp: it defines no name those headers define.  ConfigError is the
// reference's own class (errors.hpp:10) whenever that header is reachable;
// the reference's Rng and perf_model functions (rng.hpp:13,
// perf_model.hpp:54-80) are neither declared nor exported here (the library
// keeps its bit-exact restatement internal, behind hidden visibility, and
// exposes it only through the C ABI's specsim_rng_* / specsim_*accept*
// functions).  The classes implement the seams SPEC.md describes but the
// reference never implemented: the signal buffer (SPEC.md:237-241, 267-275,
// 341-344) and the trainer actor train(job) -> TrainingOutcome
// (SPEC.md:380-405).  The C ABI in include/specsim_draft_trainer.h wraps them.
#pragma once

#include <cstdint>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#if defined(__GNUC__)
#define SPECSIM_CXX_API __attribute__((visibility("default")))
#else
#define SPECSIM_CXX_API
#endif

// ---------------------------------------------------------------- errors
// The reference's split (errors.hpp:8-13): std::invalid_argument = domain
// error (CLI exit 1), ConfigError = configuration error (CLI exit 2).  The
// reference's header is used when it is on the include path (installed next
// to this file, or proj/include of the reference on -I); otherwise the same
// single-class definition stands in, token for token, so both spellings are
// one type (one typeinfo name) across the library boundary.
#if __has_include(<specsim/errors.hpp>)
#pragma GCC visibility push(default)
#include <specsim/errors.hpp>
#pragma GCC visibility pop
#else
#pragma GCC visibility push(default)
namespace specsim {
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
}  // namespace specsim
#pragma GCC visibility pop
#endif

namespace specsim {

// Device failures have their own types (C ABI status 3 / 4).
class SPECSIM_CXX_API CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class SPECSIM_CXX_API NcclError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// oldest floor(9n/10) samples train, the rest evaluate.
SPECSIM_CXX_API void split_train_eval(int64_t n, int64_t* n_train, int64_t* n_eval);

struct SPECSIM_CXX_API SignalGeometry {
  int hidden_dim = 0;
  int layers_tapped = 3;
  int bytes_per_element = 2;
  int64_t bytes_per_token() const;
  void validate() const;  // throws std::invalid_argument
};

// Synthetic captured request; stream Rng(seed + index).
struct SynthCapture {
  std::vector<int32_t> ids;
  std::vector<uint16_t> features;  // [length, layers * hidden] bf16 bits
  std::vector<int32_t> accept_lengths;
  double alpha_s = 0;
};
SPECSIM_CXX_API void synth_capture(uint64_t seed, int64_t index, int length, int vocab,
                                   int hidden, int layers, double alpha, int gamma, int32_t* ids,
                                   uint16_t* features, int32_t* accept_lengths, int32_t* n_steps,
                                   double* alpha_s);

// ---------------------------------------------------- hidden-state buffer
class SPECSIM_CXX_API HiddenStateBuffer {
 public:
  struct Stats {
    int64_t records = 0, bytes = 0, flushes = 0, cumulative_bytes = 0, samples = 0,
            resident_tokens = 0;
  };
  struct Sample {
    int64_t start = 0;  // ring row of token 0
    int32_t length = 0;
    double alpha = 0;
    int64_t last_seq = 0;  // append sequence number of the sample's last records
  };

  HiddenStateBuffer(const SignalGeometry& g, int64_t capacity_tokens, int64_t flush_threshold,
                    int device);
  ~HiddenStateBuffer();
  HiddenStateBuffer(const HiddenStateBuffer&) = delete;
  HiddenStateBuffer& operator=(const HiddenStateBuffer&) = delete;

  // extract_signals + record_sample (one verify step of one request).
  void append(int64_t sample_id, double alpha, const void* const* layer_ptrs, int64_t rows,
              int64_t ld, const int32_t* token_ids, const int32_t* accepted_idx, int n,
              bool on_device);
  // mode 0: host (copied before return); 1: device; 2: page-locked host,
  // asynchronous (the buffer must stay unmodified until the next step / eval
  // on this buffer returns or sync() is called).
  void append_packed(int64_t sample_id, double alpha, const uint16_t* features,
                     const int32_t* token_ids, int n, int mode);
  void sync() const;

  Stats stats() const { return stats_; }
  const Sample& sample(int64_t id) const;  // throws std::out_of_range if evicted/unknown
  void read_sample(int64_t id, uint16_t* features, int32_t* ids) const;

  const SignalGeometry& geometry() const { return geom_; }
  int64_t capacity() const { return cap_; }
  // Ring rows [capacity, capacity + kMirrorRows) repeat rows [0, kMirrorRows)
  // (kept in sync by every append), so a block of <= kMirrorRows consecutive
  // rows starting anywhere in the ring is contiguous in memory: the trainer's
  // GEMMs TMA-load a sample's 64 / 128-row blocks straight from the ring.
  static constexpr int kMirrorRows = 128;
  const void* ring_features() const { return ring_feat_; }
  const int32_t* ring_ids() const { return ring_ids_; }
  int device() const { return device_; }
  uint64_t serial() const { return serial_; }  // unique per buffer in the process
  void* stream() const { return stream_; }
  // Event recorded after append number `seq` (or a later one, when the event
  // ring has wrapped — waiting on it is then conservative but still correct).
  void* event_for(int64_t seq) const;

 private:
  void open_sample(int64_t sample_id, double alpha);
  void reserve(int n);  // evict oldest samples so n more tokens fit
  void account(int n);  // extract_signals byte accounting
  void record_append(void* stream);  // event + sequence number of this append
  void mirror(int64_t pos, int64_t n, void* stream);  // refresh mirrored rows written

  SignalGeometry geom_;
  uint64_t serial_ = 0;
  int64_t cap_, flush_threshold_;
  int device_;
  void* stream_ = nullptr;
  static constexpr int kEventRing = 256;
  std::vector<void*> events_;  // cudaEvent_t ring, one record per append
  int64_t append_seq_ = 0;
  void* ring_feat_ = nullptr;
  int32_t* ring_ids_ = nullptr;
  void* staging_dev_ = nullptr;   // device staging for host appends
  void* staging_host_ = nullptr;  // pinned staging
  size_t staging_bytes_ = 0;
  int64_t head_ = 0;  // next free ring row (monotonic; row = head % cap)
  int64_t tail_ = 0;  // oldest resident row (monotonic)
  int64_t open_id_ = -1;
  std::unordered_map<int64_t, Sample> samples_;  // resident samples by id
  std::deque<int64_t> order_;                   // resident sample ids, oldest first
  Stats stats_;
};

// ------------------------------------------------------------- trainer
struct SPECSIM_CXX_API DraftShape {
  int hidden = 0, vocab = 0, seq_len = 0, n_heads = 0, n_kv_heads = 0, head_dim = 0, ffn = 0,
      layers_tapped = 3, micro_batch = 1;
  float rms_eps = 1e-5f;
  double rope_theta = 10000.0;
  // EAGLE-3 training-time-test unroll: K decoder passes per step, step j's
  // loss weighted ttt_decay^j (see specsim_draft_shape)
  int ttt_steps = 1;
  float ttt_decay = 0.8f;
  void validate() const;  // collects every problem, throws std::invalid_argument
};

struct AdamWConfig {
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.f;
};

// One contiguous range [off, off + n) of the flat gradient vector exchanged as
// a unit by the data-parallel path (see dp_buckets).
struct DpBucket {
  long long off, n;
};
// Buckets in the order the backward finalises them (they tile the registry).
SPECSIM_CXX_API std::vector<DpBucket> dp_buckets(const DraftShape& shape);
// True when every bucket splits into `world` shards of whole 8-element groups
// (the ZeRO-1 path; otherwise the trainer all-reduces).
SPECSIM_CXX_API bool zero_shardable(const std::vector<DpBucket>& buckets, int world);

struct StepResult {
  double loss = 0;
  int64_t valid_tokens = 0, top1_correct = 0, positions = 0;
  double ms = 0;
};

struct TrainJob {
  std::vector<int64_t> train_ids, eval_ids;
  int epochs = 1;
};

struct TrainingOutcome {
  double duration_hours = 0;
  double alpha_eval = 0;
  int64_t new_version = 0;
  double mean_loss = 0;
  int64_t steps = 0;
};

// ------------------------------------------------------- capture side
// Serving-GPU side of the signal path (PAPER.md:130,
// SPEC.md:267-275, 293): each verify step's accepted-token hidden states of
// the tapped layers are packed on the device (on the serving stream: one
// small kernel) and copied D2H on the capture's own stream into a pinned
// host segment, so the copy overlaps the next verification step.  When the
// buffered bytes exceed the flush threshold (64 MiB default; SPEC
// accounting: n x bytes_per_token, ids not counted) the segment is handed to
// a writer thread that persists it as one shard file while capture continues
// into the other segment.  Shard format ("TIDESIG1"):
//   header  : char magic[8] = "TIDESIG1"; u32 version = 1; u32 layers;
//             u32 hidden; u32 bytes_per_element = 2; u64 n_records;
//             u64 payload_bytes                                  (40 B)
//   record  : i64 sample_id; f64 alpha; i32 n; i32 width (= layers*hidden);
//             i64 flags (1 = sample complete); bf16 features[n][width];
//             i32 ids[n]; zero padding to 16 B
//   batch record (flags 2, capture_batch): sample_id = -1, alpha = n_req,
//             n = total rows; i64 sample_ids[n_req]; i32 counts[n_req];
//             zero padding to 16 B; bf16 features[n][width]; i32 ids[n];
//             zero padding to 16 B
// A request's rows may be split over several records (one per verify step,
// interleaved with other requests of the batch); end_sample() writes its
// final alpha label.  load_shards() regroups records per sample.
class SPECSIM_CXX_API SignalCapture {
 public:
  struct Stats {
    int64_t records = 0, bytes = 0, flushes = 0, cumulative_bytes = 0;  // SPEC accounting
    int64_t samples = 0, files = 0, file_bytes = 0;
  };
  SignalCapture(const SignalGeometry& g, const std::string& directory, int64_t flush_threshold,
                int device);
  ~SignalCapture();  // close()
  SignalCapture(const SignalCapture&) = delete;
  SignalCapture& operator=(const SignalCapture&) = delete;

  // layer_ptrs[l]: device [rows, ld] bf16 hidden states of tapped layer l,
  // valid on `stream` (the serving stream) at the time of the call; host
  // token_ids[n] and accepted_idx[n] (NULL = rows 0..n).  Returns without
  // waiting for the copy.
  void capture(int64_t sample_id, const void* const* layer_ptrs, int64_t rows, int64_t ld,
               const int32_t* token_ids, const int32_t* accepted_idx, int n, void* stream);
  // One serving iteration for the whole batch (one pack kernel, one D2H):
  // request r's accepted rows are accepted_rows[offsets[r] .. offsets[r+1])
  // of the [rows, ld] layer matrices, token_ids likewise.
  void capture_batch(const int64_t* sample_ids, int n_req, const int32_t* offsets,
                     const int32_t* accepted_rows, const void* const* layer_ptrs, int64_t rows,
                     int64_t ld, const int32_t* token_ids, void* stream);
  void end_sample(int64_t sample_id, double alpha);  // record_sample: final alpha label
  void flush();  // persist the buffered records now (extra shard, not a SPEC flush)
  void close();  // flush + join the writer; idempotent
  Stats stats() const;
  std::vector<std::string> files() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// Loads shard files (in order) into the device ring: records are regrouped
// per sample_id (first-appearance order) and each sample is appended
// contiguously once its completion record (end_sample) has been read.  Rows
// of samples whose completion record has not appeared yet are carried over to
// the next load_shards call on the same buffer, so shards may be loaded one at
// a time as the writer produces them.  Returns the number of samples appended.
SPECSIM_CXX_API int64_t load_shards(HiddenStateBuffer& buf,
                                    const std::vector<std::string>& paths);

class DraftTrainerImpl;

class SPECSIM_CXX_API DraftTrainer {
 public:
  DraftTrainer(const DraftShape& shape, const AdamWConfig& opt, uint64_t seed, int rank,
               int world, const uint8_t* nccl_id, int device);
  ~DraftTrainer();
  StepResult step(HiddenStateBuffer& buf, const int64_t* ids, int n, int64_t global_valid);
  StepResult eval(HiddenStateBuffer& buf, const int64_t* ids, int n);
  TrainingOutcome train(HiddenStateBuffer& buf, const TrainJob& job);
  // Deploy gate support: device copy of the model (fp32 master, bf16 copy,
  // AdamW m / v, step count) and its restore (M_draft kept when M_new is not
  // deployed).
  void snapshot();
  void restore();
  DraftTrainerImpl& impl() { return *impl_; }
  const DraftTrainerImpl& impl() const { return *impl_; }

 private:
  std::unique_ptr<DraftTrainerImpl> impl_;
};

// ------------------------------------------------------------ controller
// Algorithm 1 (SPEC.md adapt_control): dual-EMA collection
// gate, sample store, and maybe_trigger_training -- the caller of train(job)
// -- with the deploy-if-improved gate.  Host logic in double precision, same
// operation order as the SPEC recurrences (bit-reproducible).
struct SPECSIM_CXX_API ControllerConfig {
  double lambda_short = 0.9;  // SPEC adapt_control DESIGN DECISIONS defaults
  double lambda_long = 0.99;
  double epsilon = 0.05;
  int32_t n_init = 32;
  int64_t n_threshold = 2048;
  void validate() const;  // throws ConfigError (every problem in one message)
};

enum class ControllerEventKind : int32_t {
  COLLECT_ON = 0,
  COLLECT_OFF = 1,
  TRAIN_TRIGGER = 2,
  DEPLOY = 3,
  REJECT = 4,
};
struct ControllerEvent {
  ControllerEventKind kind;
  int64_t observation;  // observations seen when it happened (the clock of this API)
};

struct TriggerDecision {
  bool triggered = false;
  TrainingOutcome outcome;
  double alpha_train = 0;  // mean alpha label of D_train, sequential order
  int64_t n_train = 0, n_eval = 0;
  int32_t action = -1;     // 1 deploy, 0 tie (neither), -1 reject / not triggered
};

class SPECSIM_CXX_API AdaptiveController {
 public:
  explicit AdaptiveController(const ControllerConfig& cfg);
  // Warm-up: the first n_init observations initialise both EMAs to their mean
  // (init_from_warmup); afterwards Eq. 6 plus the epsilon-gap gate.
  void observe(double alpha);
  // Store (h, alpha) when collection is enabled; returns whether it was stored.
  bool record_sample(int64_t sample_id, double alpha);
  // At >= n_threshold stored samples: chronological 9:1 split, train, deploy
  // if alpha_eval > alpha_train, disable collection if <, neither on a tie;
  // pending set cleared.  A throwing trainer leaves state, pending set and the
  // model unchanged (the exception propagates).
  TriggerDecision maybe_trigger_training(DraftTrainer& trainer, HiddenStateBuffer& buf,
                                         int epochs = 1);

  const ControllerConfig& config() const { return cfg_; }
  bool initialized() const { return initialized_; }
  double ema_short() const { return ema_short_; }
  double ema_long() const { return ema_long_; }
  bool collection_enabled() const { return collection_enabled_; }
  int64_t stored_samples() const { return static_cast<int64_t>(pending_ids_.size()); }
  int64_t draft_version() const { return draft_version_; }
  int64_t observations() const { return observations_; }
  const std::vector<ControllerEvent>& events() const { return events_; }
  const std::vector<int64_t>& pending_ids() const { return pending_ids_; }

 private:
  ControllerConfig cfg_;
  bool initialized_ = false;
  std::vector<double> warmup_;
  double ema_short_ = 0, ema_long_ = 0;
  bool collection_enabled_ = false;
  std::vector<int64_t> pending_ids_;
  std::vector<double> pending_alpha_;
  int64_t draft_version_ = 0;
  int64_t observations_ = 0;
  std::vector<ControllerEvent> events_;
};

}  // namespace specsim
