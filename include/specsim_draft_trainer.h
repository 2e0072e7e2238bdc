/*
 * specsim draft trainer — C ABI of the B200-native TIDE draft-training hot path.
 *
 * The reference (arxiv 2602.05145, /root/reference/proj) ships no trainer:
 * its `train_sim` module is SPEC prose with an analytic body
 * (SPEC.md:380-446), and `proj/include/specsim/` holds only errors.hpp,
 * rng.hpp, perf_model.hpp and workload.hpp.  This header is the drop-in for
 * the seams SPEC names:
 *
 *   - SignalGeometry / extract_signals / record_sample (SPEC.md:237-241,
 *     SPEC.md:267-275)        -> specsim_hsbuf_*
 *   - train(job) -> TrainingOutcome, called by
 *     maybe_trigger_training -> specsim_trainer_train
 *   - the step inside train(): forward / backward / AdamW / DP all-reduce of
 *     the EAGLE-3 style draft head
 *                                              -> specsim_trainer_step
 *   - accept-length bookkeeping (perf_model.hpp:52-80, rng.hpp:13-39)
 *                                              -> specsim_rng_*, specsim_*accept*
 *
 * Conventions (mirroring the reference):
 *   - Status codes: SPECSIM_EDOMAIN is the reference's std::invalid_argument
 *     (domain error, CLI exit 1), SPECSIM_ECONFIG is specsim::ConfigError
 *     (errors.hpp:8-13, CLI exit 2).  Every function returns a
 *     status; the message of the last failure on the calling thread is
 *     available from specsim_last_error().
 *   - Validation collects every problem into one message, like
 *     LatencyProfile's constructor (perf_model.cpp:57-82).
 *   - Handles are single-owner and not thread-safe (workload.hpp:60,
 *     SPEC.md:296).  One trainer per GPU; at most one job in flight
 *     (SPEC.md:367).
 *   - Plain pointers and sizes only; no framework types cross this boundary.
 *   - There is no CPU fallback: on a machine without a usable sm_100 GPU the
 *     GPU entry points fail with SPECSIM_ECUDA.
 */
#ifndef SPECSIM_DRAFT_TRAINER_H
#define SPECSIM_DRAFT_TRAINER_H

#include <stddef.h>
#include <stdint.h>

/* The library is built with hidden default visibility; every entry point
 * declared here is exported (and nothing else of the C++ internals). */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef enum specsim_status {
  SPECSIM_OK = 0,
  SPECSIM_EDOMAIN = 1, /* std::invalid_argument in the reference (exit 1)  */
  SPECSIM_ECONFIG = 2, /* specsim::ConfigError, errors.hpp:10-13 (exit 2)  */
  SPECSIM_ECUDA = 3,   /* CUDA runtime / kernel failure, or no GPU         */
  SPECSIM_ENCCL = 4    /* NCCL failure in the data-parallel exchange       */
} specsim_status;

/* Message of the last failing call on this thread ("" if none). */
const char* specsim_last_error(void);
const char* specsim_version(void);
/* Device kernels launched by this library so far (all handles, all streams). */
int specsim_kernel_launches(uint64_t* out);

/* ------------------------------------------------- bookkeeping (host only) */
/* Seeded mt19937_64 with the reference's hand-rolled conversions
 * (rng.hpp:13-39): uniform = (x >> 11) * 2^-53, Box-Muller cosine branch,
 * inverse-CDF geometric. */
typedef struct specsim_rng specsim_rng;
int specsim_rng_create(uint64_t seed, specsim_rng** out);
int specsim_rng_destroy(specsim_rng* rng);
int specsim_rng_uniform(specsim_rng* rng, double* out);
int specsim_rng_normal(specsim_rng* rng, double mean, double sd, double* out);
int specsim_rng_geometric(specsim_rng* rng, double mean, int64_t* out);
int specsim_rng_next_u64(specsim_rng* rng, uint64_t* out);

/* perf_model.cpp:159-169 */
int specsim_expected_accept_length(double alpha, int32_t gamma, double* out);
/* perf_model.cpp:171-177: k in [1, gamma+1] (accepted drafts + bonus token) */
int specsim_sample_accept_length(specsim_rng* rng, double alpha, int32_t gamma, int32_t* out);
/* perf_model.cpp:213-224 (bisection to kBisectionTol = 1e-6) */
int specsim_alpha_from_accept_length(double ell, int32_t gamma, double* out);
/* workload.cpp:41-47: the reference's analytic draft-quality law (the value its
 * train() returns as alpha_eval; the real trainer measures top-1 instead):
 * ceiling - (ceiling - start) exp(-max(n, 0) / tau), clamped to [0, 1].
 * Phase checks as workload.cpp:25-36 (SPECSIM_ECONFIG). */
int specsim_current_alpha(double alpha_start, double alpha_ceiling, double tau_samples,
                          double trained_samples, double* out);
/* SPEC.md:348 chronological 9:1 split: the oldest floor(9n/10) samples train. */
int specsim_split_train_eval(int64_t n, int64_t* n_train, int64_t* n_eval);

/* Data-parallel sharding of a job: optimiser step `step` takes
 * items [step*per_rank*world, (step+1)*per_rank*world); item i of that slice
 * goes to rank i mod world.  Writes this rank's item indices (<= per_rank). */
int specsim_dp_shard(int64_t n_items, int32_t per_rank, int32_t world, int32_t rank,
                     int64_t step, int64_t* out_idx, int32_t* out_n);

/* ------------------------------------------------------ signal geometry */
/* bytes per token = layers_tapped * hidden_dim * bytes_per_element */
typedef struct specsim_signal_geometry {
  int32_t hidden_dim;
  int32_t layers_tapped;     /* default 3 (low / mid / high) */
  int32_t bytes_per_element; /* default 2 (bf16); only 2 is trainable */
} specsim_signal_geometry;

int specsim_bytes_per_token(const specsim_signal_geometry* g, int64_t* out);

/* Synthetic captured request; stream = Rng(seed + index):
 *   accept lengths k = sample_accept_length(alpha, gamma), the last one
 *   truncated so that sum k == length;
 *   ids[i] = floor(uniform() * vocab);
 *   features[i, j] = bf16_rne(normal(0, 1)), j in [0, layers*hidden) in
 *   low | mid | high order;
 *   alpha_s = alpha_from_accept_length(length / steps, gamma).
 * Any output pointer may be NULL.  Host-only, multithreaded over samples. */
int specsim_synth_capture(uint64_t seed, int64_t index, int32_t length, int32_t vocab,
                          int32_t hidden, int32_t layers, double alpha, int32_t gamma,
                          int32_t* ids, uint16_t* features, int32_t* accept_lengths,
                          int32_t* n_steps, double* alpha_s);

/* --------------------------------------------------- hidden-state buffer */
/* Device-resident ring of captured samples: per token one packed
 * [layers * hidden] bf16 record plus its int32 token id.  Byte accounting
 * follows extract_signals: bytes grow by
 * records * bytes_per_token (ids are not counted) and move to the
 * cumulative total when they exceed the flush threshold (default 64 MiB,
 * SPEC.md:293). */
typedef struct specsim_hsbuf specsim_hsbuf;

typedef struct specsim_hsbuf_stats {
  int64_t records;          /* tokens appended since creation           */
  int64_t bytes;            /* bytes currently buffered (not flushed)   */
  int64_t flushes;          /* flush events                             */
  int64_t cumulative_bytes; /* bytes moved to storage by flushes        */
  int64_t samples;          /* samples recorded (record_sample calls)   */
  int64_t resident_tokens;  /* tokens currently held in the device ring */
} specsim_hsbuf_stats;

/* flush_threshold_bytes <= 0 selects 64 MiB. */
int specsim_hsbuf_create(const specsim_signal_geometry* geometry, int64_t capacity_tokens,
                         int64_t flush_threshold_bytes, int device, specsim_hsbuf** out);
int specsim_hsbuf_destroy(specsim_hsbuf* buf);

/* extract_signals for one verify step of one request + record_sample.
 * layer_ptrs[l] points at a [rows, ld] bf16 matrix of layer l's hidden
 * states (host memory unless on_device != 0); the n accepted positions are
 * rows accepted_idx[0..n) (or rows 0..n if accepted_idx is NULL).
 * token_ids[i] is the id at accepted position i.  Appending to a sample_id
 * different from the open one closes the open sample (its records stay
 * contiguous in the ring, which the fc GEMM's row gather relies on); a
 * closed sample cannot be reopened (SPECSIM_EDOMAIN).  So calls for one
 * request must not interleave with another request's: a single-request
 * serving loop appends per verify step, a BATCHED loop (requests verified
 * together, appends interleaved) captures through specsim_capture_* and
 * loads the shards with specsim_hsbuf_load_shards, which regroups each
 * request's rows.  alpha is the per-sample alpha label
 * (SPEC.md:365); the last value given for a sample wins.
 * Host pointers are only read during the call. */
int specsim_hsbuf_append(specsim_hsbuf* buf, int64_t sample_id, double alpha,
                         const void* const* layer_ptrs, int64_t rows, int64_t ld,
                         const int32_t* token_ids, const int32_t* accepted_idx, int32_t n,
                         int on_device);

/* Same, with records already packed [n, layers*hidden].  mode 0: host memory,
 * copied before return; 1: device memory; 2: page-locked host memory, copied
 * ASYNCHRONOUSLY on the buffer's stream so the DMA overlaps a running step —
 * the caller keeps the buffers unmodified until the next trainer step / eval
 * on this buffer returns or specsim_hsbuf_sync() is called.  Trainer steps
 * are ordered after every append by an event (no host synchronisation).
 * Keep at most ~2 GiB of mode-2 appends queued ahead of the steps that
 * consume them: beyond a few GB the driver's per-stream work queue is full,
 * the call blocks until earlier DMA drains and the overlap is lost
 * (DESIGN.md §10). */
int specsim_hsbuf_append_packed(specsim_hsbuf* buf, int64_t sample_id, double alpha,
                                const uint16_t* features, const int32_t* token_ids, int32_t n,
                                int mode);
/* Waits for every append issued on the buffer. */
int specsim_hsbuf_sync(specsim_hsbuf* buf);

int specsim_hsbuf_stats_get(const specsim_hsbuf* buf, specsim_hsbuf_stats* out);
int specsim_hsbuf_sample_info(const specsim_hsbuf* buf, int64_t sample_id, int32_t* length,
                              double* alpha);
/* Copies a sample's packed records / ids back to host (tests). */
int specsim_hsbuf_read_sample(const specsim_hsbuf* buf, int64_t sample_id, uint16_t* features,
                              int32_t* token_ids);

/* ------------------------------------------------------- capture side
 * Serving-GPU capture (PAPER.md:130, SPEC.md:267-275,
 * 293): pack accepted-token states on the serving stream, D2H on a side
 * stream into pinned segments, flush to "TIDESIG1" shard files in
 * `directory` on a writer thread at the flush threshold (<= 0: 64 MiB).
 * See include/specsim/draft_trainer.hpp for the file format. */
typedef struct specsim_capture specsim_capture;
typedef struct specsim_capture_stats {
  int64_t records, bytes, flushes, cumulative_bytes; /* SPEC extract_signals accounting */
  int64_t samples, files, file_bytes;
} specsim_capture_stats;
int specsim_capture_create(const specsim_signal_geometry* geometry, const char* directory,
                           int64_t flush_threshold_bytes, int device, specsim_capture** out);
/* closes (flushes, joins the writer) and frees */
int specsim_capture_destroy(specsim_capture* c);
/* layer_ptrs: device pointers valid on `stream` (cudaStream_t, NULL = legacy
 * default stream); token_ids / accepted_idx: host arrays read during the call. */
int specsim_capture_append(specsim_capture* c, int64_t sample_id, const void* const* layer_ptrs,
                           int64_t rows, int64_t ld, const int32_t* token_ids,
                           const int32_t* accepted_idx, int32_t n, void* stream);
/* one serving iteration for a batch: request r's accepted rows are
 * accepted_rows[offsets[r] .. offsets[r+1]) (offsets has n_req + 1 entries) */
int specsim_capture_append_batch(specsim_capture* c, const int64_t* sample_ids, int32_t n_req,
                                 const int32_t* offsets, const int32_t* accepted_rows,
                                 const void* const* layer_ptrs, int64_t rows, int64_t ld,
                                 const int32_t* token_ids, void* stream);
int specsim_capture_end_sample(specsim_capture* c, int64_t sample_id, double alpha);
int specsim_capture_flush(specsim_capture* c);
int specsim_capture_close(specsim_capture* c);
int specsim_capture_stats_get(const specsim_capture* c, specsim_capture_stats* out);
/* path of shard i (i < files) into buf (cap bytes, NUL-terminated) */
int specsim_capture_file(const specsim_capture* c, int64_t i, char* buf, int64_t cap);
/* load shard files into a device ring; *samples = samples appended */
int specsim_hsbuf_load_shards(specsim_hsbuf* buf, const char* const* paths, int32_t n_paths,
                              int64_t* samples);

/* ---------------------------------------------------------- draft trainer */
/* EAGLE-3 style draft head:
 *   g = W_fc f, u = [RMSNorm(E[x_{t+1}]); RMSNorm(g)], one decoder layer
 *   (GQA attention with NeoX RoPE, SwiGLU MLP, residual from g), final norm,
 *   LM head over the full target vocabulary. */
typedef struct specsim_draft_shape {
  int32_t hidden;        /* H                                       */
  int32_t vocab;         /* V                                       */
  int32_t seq_len;       /* S training positions per sample         */
  int32_t n_heads;       /* query heads                             */
  int32_t n_kv_heads;    /* key/value heads                         */
  int32_t head_dim;      /* 64 or 128                               */
  int32_t ffn;           /* I                                       */
  int32_t layers_tapped; /* 3                                       */
  int32_t micro_batch;   /* B samples per rank per step             */
  float rms_eps;
  double rope_theta;
  /* EAGLE-3 training-time-test unroll (SpecForge
   * convention, not in the reference): K = ttt_steps decoder passes per step
   * (0 reads as 1, max 16; K > 1 needs seq_len % 128 == 0).  Pass j >= 1
   * takes the previous pass's output h in place of g, tokens shifted by j
   * (u = x[t+1+j], y = x[t+2+j], m = [t+2+j < L]), RoPE positions t + j, and
   * its attention row t also sees the keys / values of passes 1..j at row t.
   * loss = sum_j ttt_decay^j CE_j / N (N = valid count of pass 0; decay 0
   * reads as 0.8); valid_tokens / top1_correct / alpha_eval are pass 0's;
   * eval runs pass 0 only. */
  int32_t ttt_steps;
  float ttt_decay;
} specsim_draft_shape;

/* Gradient buckets of the data-parallel exchange for a draft shape, in the
 * order the backward finalises them (LM-head vocabulary chunks, then
 * [down, w_fin], [gate_up], [o, w_post], [qkv], [fc, w_in, w_hid]); they tile
 * the flat parameter vector.  Writes up to cap (off, n) pairs; *count = total
 * buckets; *zero_ok = 1 when every bucket splits into `world` shards of whole
 * 8-element groups, i.e. when world > 1 runs ZeRO-1: each bucket is
 * reduce-scattered in place (rank r owns [off + r*n/world, off + (r+1)*n/world)),
 * AdamW updates the owned shard and the bf16 working weights are all-gathered,
 * all overlapped with the rest of the backward (SPECSIM_DP_MODE=allreduce
 * selects the replicated all-reduce + AdamW path instead).  Host only. */
int specsim_dp_buckets(const specsim_draft_shape* shape, int32_t world, int64_t* off, int64_t* n,
                       int32_t cap, int32_t* count, int32_t* zero_ok);

/* PyTorch AdamW semantics. */
typedef struct specsim_adamw {
  float lr, beta1, beta2, eps, weight_decay;
} specsim_adamw;

typedef struct specsim_trainer specsim_trainer;

typedef struct specsim_step_result {
  double loss;          /* sum_t m_t (lse_t - logit_t[y_t]) / global valid */
  int64_t valid_tokens; /* sum_t m_t on this rank                          */
  int64_t top1_correct; /* sum_t m_t [argmax_t == y_t] on this rank        */
  int64_t positions;    /* B * S processed positions on this rank          */
  double ms;            /* device time of the step (CUDA events)           */
} specsim_step_result;

typedef struct specsim_training_outcome {
  double duration_hours; /* measured wall time of the job     */
  double alpha_eval;     /* top-1 accuracy on D_eval (replaces current_alpha) */
  int64_t new_version;   /* draft version produced by this job            */
  double mean_loss;      /* mean training loss over the job's steps       */
  int64_t steps;
} specsim_training_outcome;

/* 128-byte NCCL unique id for world > 1 (rank 0 creates, caller broadcasts). */
int specsim_nccl_unique_id(uint8_t* out128);

/* Parameters are initialised from Rng(seed + 1) normal(0, 0.02) (norm
 * weights 1.0); the frozen embedding E from Rng(seed + 2) normal(0, 0.02).
 * nccl_id may be NULL when world == 1. */
int specsim_trainer_create(const specsim_draft_shape* shape, const specsim_adamw* opt,
                           uint64_t seed, int rank, int world, const uint8_t* nccl_id,
                           int device, specsim_trainer** out);
int specsim_trainer_destroy(specsim_trainer* t);

/* One optimiser step over n <= micro_batch samples of buf (missing rows are
 * padding with zero mask).  global_valid_tokens is sum m_t over all ranks'
 * samples of this step (0 = use this rank's own count).  Synchronous. */
int specsim_trainer_step(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* sample_ids,
                         int32_t n, int64_t global_valid_tokens, specsim_step_result* out);

/* Forward only: loss and top-1 over n <= micro_batch samples. */
int specsim_trainer_eval(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* sample_ids,
                         int32_t n, specsim_step_result* out);

/* train(job) -> TrainingOutcome with the real step as its
 * body: `epochs` passes over train_ids (sample i -> rank i mod world), then
 * top-1 accuracy on eval_ids.  The draft is trained in place; callers keep
 * get_param copies when they need the deploy/reject gate. */
int specsim_trainer_train(specsim_trainer* t, specsim_hsbuf* buf, const int64_t* train_ids,
                          int64_t n_train, const int64_t* eval_ids, int64_t n_eval,
                          int32_t epochs, specsim_training_outcome* out);

/* ---------------------------------------------------------- deploy gate
 * Device snapshot / restore of the model (fp32 master, bf16 working copy,
 * AdamW m / v, step count): M_draft is kept when M_new is not deployed
 * (PAPER.md:209-213).  restore without a snapshot -> SPECSIM_EDOMAIN. */
int specsim_trainer_snapshot(specsim_trainer* t);
int specsim_trainer_restore(specsim_trainer* t);

/* ------------------------------------------------- adaptive controller
 * Algorithm 1 (SPEC.md adapt_control): the caller of
 * train(job).  observe() = Eq. 6 dual EMA + epsilon-gap collection gate
 * (first n_init observations initialise both EMAs to their mean);
 * record_sample() = "Store (h, alpha)" (no-op when collection is off);
 * maybe_trigger_training() = SPEC.md:345-353: at >= n_threshold stored
 * samples, chronological 9:1 split, alpha_train = mean alpha of D_train,
 * train, deploy iff alpha_eval > alpha_train (version + 1), disable
 * collection iff alpha_eval < alpha_train, neither on a tie; the model is
 * restored unless deployed; pending set cleared.  A failing trainer leaves
 * controller state, pending set and model unchanged. */
typedef struct specsim_controller specsim_controller;
typedef struct specsim_controller_config {
  double lambda_short, lambda_long, epsilon;
  int32_t n_init;
  int64_t n_threshold;
} specsim_controller_config;
typedef struct specsim_controller_state {
  int32_t initialized, collection_enabled;
  double ema_short, ema_long;
  int64_t stored_samples, draft_version, observations, n_events;
} specsim_controller_state;
typedef struct specsim_trigger_decision {
  int32_t triggered, action; /* action: 1 deploy, 0 tie, -1 reject / not triggered */
  double alpha_train;
  int64_t n_train, n_eval;
  specsim_training_outcome outcome;
} specsim_trigger_decision;
/* event kinds: 0 COLLECT_ON, 1 COLLECT_OFF, 2 TRAIN_TRIGGER, 3 DEPLOY, 4 REJECT */
int specsim_controller_create(const specsim_controller_config* cfg, specsim_controller** out);
void specsim_controller_destroy(specsim_controller* c);
int specsim_controller_observe(specsim_controller* c, double alpha);
int specsim_controller_record_sample(specsim_controller* c, int64_t sample_id, double alpha,
                                     int32_t* stored);
int specsim_controller_maybe_trigger_training(specsim_controller* c, specsim_trainer* t,
                                              specsim_hsbuf* buf, int32_t epochs,
                                              specsim_trigger_decision* out);
int specsim_controller_state_get(const specsim_controller* c, specsim_controller_state* out);
/* copies up to cap events (kind, observation index); *n = total events */
int specsim_controller_events(const specsim_controller* c, int32_t* kinds, int64_t* at,
                              int64_t cap, int64_t* n);

/* Parameter registry (fp32 master copies; names: fc, w_in, w_hid, qkv, o,
 * w_post, gate_up, down, w_fin, lm_head).  Frozen embedding: "embed".
 * Under ZeRO-1 (world > 1) each rank's fp32 master is current on its own
 * shards only: get_param and snapshot first all-gather it, so they are
 * collective (every rank calls them, in the same order), and get_grad is
 * the reduced gradient on the rank's own shards only. */
int specsim_trainer_num_params(const specsim_trainer* t, int32_t* count, int64_t* total_elems);
int specsim_trainer_param_info(const specsim_trainer* t, int32_t index, const char** name,
                               int64_t* rows, int64_t* cols);
int specsim_trainer_get_param(const specsim_trainer* t, const char* name, float* host_out);
int specsim_trainer_set_param(specsim_trainer* t, const char* name, const float* host_in);
/* Gradient of the last step (after the DP all-reduce).  On a single replica the
 * GEMM-weight gradients are consumed by the AdamW update fused into the
 * weight-gradient GEMM epilogue and are only materialised after
 * specsim_trainer_keep_grads(t, 1) (an extra 4 B/param store); otherwise
 * get_grad fails with SPECSIM_EDOMAIN for them. */
int specsim_trainer_get_grad(const specsim_trainer* t, const char* name, float* host_out);
int specsim_trainer_keep_grads(specsim_trainer* t, int enabled);
int specsim_trainer_set_embedding(specsim_trainer* t, const uint16_t* host_bf16);
int specsim_trainer_get_embedding(const specsim_trainer* t, uint16_t* host_bf16);
int specsim_trainer_set_step_count(specsim_trainer* t, int64_t step);

/* Per-phase device timing of the last step (CUDA events on the step stream) --
 * after specsim_trainer_train, of the job's last step, which ran back to back
 * with the steps before it.
 * Phases: 0 ingest/gather, 1 GEMMs (sum over all tcgen05 GEMM launches),
 * 2 attention, 3 norms/elementwise, 4 LM-head+CE GEMMs, 5 AdamW,
 * 6 all-reduce.  flops[i] = algorithmic FLOPs of the phase (GEMM phases). */
int specsim_trainer_set_timing(specsim_trainer* t, int enabled);
/* Device-timed region on the trainer's stream: end == 0 records the start
 * event, end != 0 records the stop event, waits, and returns the elapsed ms
 * (idle gaps between steps included). */
int specsim_trainer_region(specsim_trainer* t, int end, double* ms);
int specsim_trainer_phase_times(const specsim_trainer* t, double* ms7, double* flops7,
                                int32_t* launches7);
/* Device time (ms) of the last step: the last step()/eval(), or the last step
 * of the last specsim_trainer_train job (from its graph launch to its end). */
int specsim_trainer_last_step_ms(const specsim_trainer* t, double* ms);

/* Per-row device state of the last step / eval, copied to the host (parity
 * tests: the target gather and top-1 are checked bit-exact against the
 * oracle).  name: "u", "y", "m", "argmax" (int32, K*B*S rows:
 * unroll slice j at rows j*B*S; eval fills slice 0 only), "lse" (fp32, K*B*S
 * rows), "F" (bf16 bits, [B*S, layers*hidden]: the micro-batch features the
 * fc GEMM read).  *n_elems (nullable) receives the element count; host_out
 * may be NULL to query it, otherwise it must hold cap_elems >= that count. */
int specsim_trainer_read_rows(const specsim_trainer* t, const char* name, void* host_out,
                              int64_t cap_elems, int64_t* n_elems);

/* ------------------------------------------------------ kernel test hooks */
/* Host-buffer wrappers around single kernels, used by the parity tests.
 * GEMM: epi 0 bf16 out, 1 f32 out, 2 f32 accumulate (C in/out), 3 bf16 out
 * plus residual R; bits 8..15 of epi select the CTA group (0 = default pair
 * kernel cta_group::2, 1 = single-CTA cta_group::1).  A is [M, lda] (K-major) or [K, lda] (MN-major); B is
 * [N, ldb] or [K, ldb].  iters > 1 re-launches and reports mean kernel ms. */
int specsim_debug_gemm(int a_mn, int b_mn, int epi_cg, int32_t M, int32_t N, int32_t K,
                       const uint16_t* A, int64_t lda, const uint16_t* B, int64_t ldb, void* C,
                       int64_t ldc, const uint16_t* R, int64_t ldr, int32_t iters,
                       float* mean_ms);
/* Attention forward (+ backward when dout/dqkv are non-null) on host
 * buffers: qkv [B*S, (nh+2*nkv)*hd] bf16 with RoPE already applied, o
 * [B*S, nh*hd], lse [nh, B*S] (natural log), dqkv like qkv. */
int specsim_debug_attention(int32_t B, int32_t S, int32_t nh, int32_t nkv, int32_t hd,
                            const uint16_t* qkv, const uint16_t* dout, uint16_t* o, float* lse,
                            uint16_t* dqkv);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif /* SPECSIM_DRAFT_TRAINER_H */
